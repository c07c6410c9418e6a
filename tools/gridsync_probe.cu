// gridsync_probe.cu -- cost of a grid-wide barrier on B200 for the streaming
// kernel's tick barrier: cooperative_groups grid.sync() vs a two-level
// counter barrier, for several grid sizes.  nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o gridsync_probe tools/gridsync_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}

// two-level barrier: CTAs arrive on one of 16 group counters; the last
// arriver of a group arrives on the top counter; the last top arriver bumps
// the generation that everybody polls.
__device__ unsigned int g_cnt[17 * 32];
__device__ volatile unsigned int g_gen;

__global__ void k_tree(int iters) {
  __shared__ unsigned int gen0;
  const int nb = gridDim.x, ng = 16;
  const int grp = blockIdx.x % ng;
  const int in_grp = nb / ng + (grp < nb % ng ? 1 : 0);
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      gen0 = g_gen;
      __threadfence();
      const unsigned int a = atomicAdd(&g_cnt[grp * 32], 1u);
      if (a == (unsigned)in_grp - 1) {
        g_cnt[grp * 32] = 0;
        const unsigned int b = atomicAdd(&g_cnt[16 * 32], 1u);
        if (b == (unsigned)ng - 1) {
          g_cnt[16 * 32] = 0;
          __threadfence();
          g_gen = gen0 + 1;
        }
      }
      while (g_gen == gen0) {
      }
      __threadfence();
    }
    __syncthreads();
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  int grids[] = {sms, 2 * sms, 512, 4 * sms};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int gsz : grids) {
    for (int kind = 0; kind < 2; ++kind) {
      void* args[] = {(void*)&iters};
      int it = iters;
      args[0] = &it;
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(kind ? (const void*)k_tree : (const void*)k_cg, dim3(gsz),
                                                  dim3(256), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d %-8s: %s %.3f us per barrier\n", gsz, kind ? "2-level" : "cg::sync",
             e == cudaSuccess ? "" : cudaGetErrorString(e), ms * 1e3 / iters);
    }
  }
  return 0;
}
