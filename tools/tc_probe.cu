// tc_probe.cu -- standalone check of the tcgen05 kind::i8 mechanics used by the
// tensor-core tick kernel (descriptors, MMA, commit, TMEM ld): D[M x N] =
// A[M x K] (s8) * B[N x K]^T (u8) for two M=128 halves, compared with a CPU
// product.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// -I paper_2404_16208_b200/csrc -o tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tc.h"

using namespace ranc;

constexpr int K = 256, MH = 2;  // two 128-row halves

template <int N>
__global__ void probe(const int8_t* A, const uint8_t* B, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;                       // [256 rows][K] canonical
  uint8_t* Bs = sm + MH * 128 * K;        // [N rows][K] canonical
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < MH * 128 * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    As[tc::operand_offset(r, k, MH * 128)] = (uint8_t)A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    Bs[tc::operand_offset(r, k, N)] = B[i];
  }
  if (warp == 0) tc::alloc(&tbase, 512);
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t t0 = tbase;
  if (tid == 0) {
    const uint32_t id = tc::idesc_i8(128, N);
    for (int h = 0; h < MH; ++h)
      for (int kk = 0; kk < K / 32; ++kk) {
        uint64_t ad = tc::smem_desc(ptx::smem_u32(As + h * 2048 + kk * 2 * (MH * 128 * 16)), MH * 128 * 16, 128);
        uint64_t bd = tc::smem_desc(ptx::smem_u32(Bs + kk * 2 * (N * 16)), N * 16, 128);
        tc::mma_i8(t0 + h * N, ad, bd, id, kk > 0);
      }
    tc::commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  tc::fence_after();
  // 8 warps: warp w reads half w/4, lanes 32*(w%4)..
  const int h = warp / 4, q = warp % 4;
  for (int j = 0; j < N / 32; ++j) {
    uint32_t v[32];
    tc::ld32(t0 + ((uint32_t)(q * 32) << 16) + h * N + j * 32, v);
    tc::wait_ld();
    const int row = h * 128 + q * 32 + lane;
    for (int i = 0; i < 32; ++i) D[row * N + j * 32 + i] = (int32_t)v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(t0, 512);
}

template <int N>
int run() {
  const int M = MH * 128;
  int8_t* hA = (int8_t*)malloc(M * K);
  uint8_t* hB = (uint8_t*)malloc(N * K);
  int32_t* hD = (int32_t*)malloc(M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (int8_t)((rand() % 255) - 127);
  for (int i = 0; i < N * K; ++i) hB[i] = (uint8_t)(rand() & 1);
  int8_t* dA;
  uint8_t* dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  size_t smem = (size_t)M * K + (size_t)N * K;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<N><<<1, 256, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)hA[m * K + k] * (int32_t)hB[n * K + k];
      if (ref != hD[m * N + n]) {
        if (bad < 5) printf("N=%d mismatch (%d,%d): got %d want %d\n", N, m, n, hD[m * N + n], ref);
        ++bad;
      }
    }
  printf("N=%d: %s (%d mismatches of %d)\n", N, bad ? "FAIL" : "OK", bad, M * N);
  return bad != 0;
}

int rate_main();

int main() {
  rate_main();
  int f = 0;
  f |= run<64>();
  f |= run<128>();
  f |= run<256>();
  return f;
}

// ---- throughput of back-to-back MMAs for two operand layouts ---------------
__global__ void mma_rate(int iters, uint32_t lbo_a, uint32_t sbo_a, uint32_t stepA, uint32_t lbo_b, uint32_t sbo_b,
                         uint32_t stepB, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x == 0) {
    const uint32_t id = tc::idesc_i8(128, 64);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t ad = tc::smem_desc(ptx::smem_u32(sm + kk * stepA), lbo_a, sbo_a);
        uint64_t bd = tc::smem_desc(ptx::smem_u32(sm + 65536 + kk * stepB), lbo_b, sbo_b);
        tc::mma_i8(tbase, ad, bd, id, kk > 0);
      }
    tc::commit(&bar);
    ptx::mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tbase, 512);
}

int rate_main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  // old: rows of a K chunk spread (LBO=128, SBO=K*8); new: chunk-contiguous (LBO=R*16, SBO=128)
  const uint32_t cfg[2][6] = {{128, 256 * 8, 256, 128, 256 * 8, 256}, {256 * 16, 128, 2 * 256 * 16, 64 * 16, 128, 2 * 64 * 16}};
  for (int v = 0; v < 2; ++v) {
    mma_rate<<<1, 128, 100 * 1024>>>(iters, cfg[v][0], cfg[v][1], cfg[v][2], cfg[v][3], cfg[v][4], cfg[v][5], d);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("layout %s: %.1f cycles per MMA (M=128,N=64,K=32 i8)\n", v ? "chunk-contiguous" : "row-spread",
           (double)h / (iters * 8));
  }
  return 0;
}
