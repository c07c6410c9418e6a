// int_peaks.cu -- integer-pipe microbenchmarks on the B200:
// POPC, LOP3, IMAD and the fused AND+POPC+IMAD inner loop of the tick
// kernel, plus red.global.or throughput.  The numbers are the denominators of
// the "alu" roofline of the popcount path.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o int_peaks int_peaks.cu
// Run:   ./int_peaks > gpurun_out/int_peaks.json
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                                       \
  do {                                                                                              \
    cudaError_t e = (x);                                                                            \
    if (e != cudaSuccess) {                                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                     \
      return 1;                                                                                     \
    }                                                                                               \
  } while (0)

constexpr int CH = 8;  // independent chains per thread

__global__ void k_popc(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = seed ^ (threadIdx.x * 0x9E3779B9u + i * 0x85EBCA6Bu);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) a[i] = __popc(a[i]) ^ (a[i] >> 1);
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[CH];
  uint32_t b = seed * 3u, c = seed * 7u;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = seed ^ (threadIdx.x * 0x9E3779B9u + i * 0x85EBCA6Bu);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) a[i] = (a[i] & b) ^ c ^ (a[i] | r);
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_imad(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[CH];
  const uint32_t m = seed | 1u, k = seed * 5u;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = seed ^ (threadIdx.x * 0x9E3779B9u + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) a[i] = a[i] * m + k;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

// the tick kernel's inner loop: acc += w[e] * popc(x[e] & s[e]), s from smem
template <int E>
__global__ void k_fused(uint32_t* out, uint32_t seed, int iters) {
  __shared__ uint32_t sp[64 * E];
  for (int i = threadIdx.x; i < 64 * E; i += blockDim.x) sp[i] = seed * (i + 1) * 0x9E3779B9u;
  __syncthreads();
  uint32_t x[E];
  int w[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    x[e] = seed ^ (threadIdx.x * 0x85EBCA6Bu + e * 0xC2B2AE35u);
    w[e] = (int)((seed >> e) & 15) - 8;
  }
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t* s = sp + (it & 63) * E;
#pragma unroll
    for (int e = 0; e < E; ++e) acc += w[e] * __popc(x[e] & s[e]);
  }
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void k_red(uint32_t* buf, size_t words, int iters) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  uint32_t h = (uint32_t)tid * 0x9E3779B9u;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    atomicOr(buf + (h % words), 1u << (h >> 27));
  }
}

template <class K>
float timeit(K kernel, int blocks, int threads, uint32_t* out, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kernel<<<blocks, threads>>>(out, 1234567u, iters / 8);
  cudaEventRecord(a);
  kernel<<<blocks, threads>>>(out, 1234567u, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int dev = 0;
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, dev));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  uint32_t* out;
  CK(cudaMalloc(&out, 16));
  const int SM = pr.multiProcessorCount;
  const int blocks = SM * 8, threads = 256, iters = 4096;
  const double thr = (double)blocks * threads;
  float ms;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", pr.name, SM, clk_khz);
  ms = timeit(k_popc, blocks, threads, out, iters);
  double popc = thr * iters * 16 * CH / (ms * 1e-3);
  printf(", \"popc_per_s\": %.4e, \"popc_per_clk_sm_at_1965\": %.2f", popc, popc / SM / 1.965e9);
  ms = timeit(k_lop3, blocks, threads, out, iters);
  double lop = thr * iters * 16 * CH / (ms * 1e-3);
  printf(", \"lop3_per_s\": %.4e, \"lop3_per_clk_sm_at_1965\": %.2f", lop, lop / SM / 1.965e9);
  ms = timeit(k_imad, blocks, threads, out, iters);
  double imad = thr * iters * 16 * CH / (ms * 1e-3);
  printf(", \"imad_per_s\": %.4e, \"imad_per_clk_sm_at_1965\": %.2f", imad, imad / SM / 1.965e9);
  ms = timeit(k_fused<12>, blocks, threads, out, iters * 8);
  double fused = thr * iters * 8 * 12 / (ms * 1e-3);
  printf(", \"fused_piece_per_s\": %.4e, \"fused_piece_per_clk_sm_at_1965\": %.2f", fused, fused / SM / 1.965e9);
  // red.global.or over a 64 MB buffer
  size_t words = 16u << 20;
  uint32_t* buf;
  CK(cudaMalloc(&buf, words * 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_red<<<blocks, threads>>>(buf, words, 64);
  cudaEventRecord(a);
  k_red<<<blocks, threads>>>(buf, words, 512);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf(", \"red_or_per_s\": %.4e", thr * 512 / (ms * 1e-3));
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
