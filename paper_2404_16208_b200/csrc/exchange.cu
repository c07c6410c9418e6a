// exchange.cu -- core-sharded mode: per-tick delivery of the
// spikes whose route crosses a rank boundary.
//
// After the tick kernel of tick t has written the fired bits of every
// exporting core into `fired` [G_loc][Sr][Wn], `pack` gathers the rows of the
// cores each peer needs into one send buffer (rows [S][Wn] per core, peers
// concatenated).  The transport (grouped ncclSend/ncclRecv over NVLink, or
// device copies in the loopback mode) moves them; `unpack` then applies, on
// the receiving rank, the routes of the remote source neurons: exactly the
// scheduler write of Alg. 1 l.15-20 ("a spike bit is written
// directly into the scheduler SRAM array") for destinations it owns.  Delays
// are >= 1 so every such write lands in a row read at tick t+1 or later, and
// the next tick kernel is stream-ordered after the unpack.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace ranc {

namespace {

__global__ void pack_kernel(const uint32_t* __restrict__ fired, uint32_t* __restrict__ send,
                            const int32_t* __restrict__ send_list, int64_t rows, int S, int Sr, int Wn) {
  const int64_t total = rows * S * Wn;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % Wn);
    const int64_t rs = i / Wn;
    const int s = (int)(rs % S);
    const int64_t r = rs / S;
    send[i] = fired[((size_t)send_list[r] * Sr + s) * Wn + w];
  }
}

__global__ void unpack_kernel(const uint32_t* __restrict__ recv, const int32_t* __restrict__ recv_list, int64_t rows,
                              int S, int Wn, const uint2* __restrict__ route, int Npad, int N, int c_lo, int G_loc,
                              uint32_t* __restrict__ ring, int Sr, int W, int64_t t, int rp_mask, int wmajor) {
  const int64_t total = rows * S * Wn;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t word = recv[i];
    if (!word) continue;
    const int w = (int)(i % Wn);
    const int64_t rs = i / Wn;
    const int s = (int)(rs % S);
    const int cs = recv_list[rs / S];
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      const int n = w * 32 + b;
      if (n >= N) continue;
      const uint2 rt = route[(size_t)cs * Npad + n];
      if (route_kind(rt.x) != RK_ROUTE) continue;
      const uint32_t dl = rt.y - (uint32_t)c_lo;
      if (dl >= (uint32_t)G_loc) continue;
      const uint32_t ax = route_axon(rt.x);
      const int slot = (int)((t + route_delay(rt.x)) & rp_mask);
      // ring layout of the active kernel: [Rp][G][Sr][W] (popcount) or word-major [Rp][G][W][Sr] (tensor core)
      const size_t row = (size_t)slot * G_loc + dl;
      const size_t wi = wmajor ? (row * W + (ax >> 5)) * Sr + s : (row * Sr + s) * W + (ax >> 5);
      atomicOr(ring + wi, 1u << (ax & 31));
    }
  }
}

int blocks_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
}

}  // namespace

cudaError_t launch_pack(ranc_ctx* ctx) {
  const int64_t rows = ctx->n_send_words / std::max<int64_t>(1, ctx->S * ctx->net.Wn);
  if (!rows) return cudaSuccess;
  pack_kernel<<<blocks_for(ctx->n_send_words), 256, 0, ctx->stream>>>(
      (const uint32_t*)ctx->d_fired.p, (uint32_t*)ctx->d_send.p, (const int32_t*)ctx->d_send_list.p, rows,
      (int)ctx->S, (int)ctx->Sr, ctx->net.Wn);
  ctx->launches++;
  return cudaGetLastError();
}

cudaError_t launch_unpack(ranc_ctx* ctx, int64_t t) {
  const int64_t rows = ctx->n_recv_rows;
  if (!rows) return cudaSuccess;
  const Compiled& n = ctx->net;
  const uint2* route = (const uint2*)(ctx->kernel_active == RANC_KERNEL_TC ? ctx->d_route_tc.p : ctx->d_route.p);
  unpack_kernel<<<blocks_for(ctx->n_recv_words), 256, 0, ctx->stream>>>(
      (const uint32_t*)ctx->d_recv.p, (const int32_t*)ctx->d_recv_list.p, rows, (int)ctx->S, n.Wn, route, n.Npad, n.N,
      ctx->c_lo, ctx->G_loc, (uint32_t*)ctx->d_ring.p, (int)ctx->Sr, n.W, t, n.Rp - 1,
      ctx->ring_wmajor ? 1 : 0);
  ctx->launches++;
  return cudaGetLastError();
}

}  // namespace ranc
