// tc_probe_mn.cu -- does tcgen05.mma kind::i8 take an MN-major B operand
// (instruction descriptor bit 16), and which descriptor field strides which
// direction?  B element (k, n) at (k/8)*KG + (n/16)*NG + (k%8)*16 + n%16
// (a 128-byte core matrix = 8 K rows of 16 contiguous N bytes).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2404_16208_b200/csrc -o /tmp/mn tools/tc_probe_mn.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tc.h"

using namespace ranc;

constexpr int K = 256, M = 128, N = 64;
constexpr uint32_t NG = 128, KG = (N / 16) * 128;   // N core matrices adjacent, then the next 8 K rows

__global__ void probe(const int8_t* A, const uint8_t* B, int32_t* D, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;
  uint8_t* Bs = sm + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) As[tc::operand_offset(i / K, i % K, M)] = (uint8_t)A[i];
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    Bs[(k / 8) * KG + (n / 16) * NG + (k % 8) * 16 + n % 16] = B[i];
  }
  if (warp == 0) tc::alloc(&tbase, 64);
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
    const uint32_t id = tc::idesc_i8(128, N) | (1u << 16);   // B MN-major
    for (int kk = 0; kk < K / 32; ++kk) {
      uint64_t ad = tc::smem_desc(ptx::smem_u32(As + kk * 2 * (M * 16)), M * 16, 128);
      uint64_t bd = tc::smem_desc(ptx::smem_u32(Bs + kk * 4 * KG), lbo, sbo);
      tc::mma_i8(t0, ad, bd, id, kk > 0);
    }
    tc::commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  tc::fence_after();
  for (int j = 0; j < N / 32; ++j) {
    uint32_t v[32];
    tc::ld32(t0 + ((uint32_t)(warp * 32) << 16) + j * 32, v);
    tc::wait_ld();
    const int row = warp * 32 + lane;
    for (int i = 0; i < 32; ++i) D[row * N + j * 32 + i] = (int32_t)v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(t0, 64);
}

int main() {
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
  const size_t smem = (size_t)M * K + (size_t)N * K;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const uint32_t cfg[2][2] = {{NG, KG}, {KG, NG}};
  for (int v = 0; v < 2; ++v) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, cfg[v][0], cfg[v][1]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("lbo=%u sbo=%u: CUDA error %s\n", cfg[v][0], cfg[v][1], cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        int32_t ref = 0;
        for (int k = 0; k < K; ++k) ref += (int32_t)hA[m * K + k] * (int32_t)hB[n * K + k];
        bad += ref != hD[m * N + n];
      }
    printf("MN-major B, lbo=%u sbo=%u: %s (%d mismatches of %d)\n", cfg[v][0], cfg[v][1], bad ? "FAIL" : "OK", bad, M * N);
  }
  return 0;
}
