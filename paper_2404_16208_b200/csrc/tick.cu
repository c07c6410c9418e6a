// tick.cu -- the fused per-tick kernel (popcount path) and state kernels.
//
// One launch = one tick of Alg. 1 for every core of every sample:
//   a1 scheduler read + clear  (Alg. 1 l.3-5; section III-E)
//   a2 input injection          (Alg. 1 l.6-9)
//   a3 synaptic integration     (Alg. 1 l.10-13)
//   a4 leak / threshold / reset (Alg. 1 l.14)
//   a5 route + scheduler write  (Alg. 1 l.15-20; section III-D)
//   a6 output bus
//   a7 tick barrier: the kernel boundary.
//
// Mapping (B200-first, not the paper's V100 mapping): CTA = (core c, tile of
// ST samples); thread = neuron.  Each thread keeps its neuron's crossbar
// pieces and weights in registers for the whole sample tile, so the
// (L2-resident) network is read once per tile while potentials stream from
// HBM once per tick.  Integration is sum_e w_e * popc(xbar_e & spikes_e) over
// the <= ceil(A/32)+K-1 type-sorted pieces (compile.cpp).
//
// Why no intra-tick barrier is needed: every route delay is in [1, D] and the
// ring has Rp >= D+1 physical rows, so no spike written during tick t lands in
// row t & (Rp-1), which is the only row read (and cleared) during tick t.
// Spike writes are idempotent ORs (G11), so their order is irrelevant.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace ranc {

namespace {

constexpr int kThreads = 256;

template <int E>
__global__ void __launch_bounds__(kThreads) tick_popc_kernel(const TickParams p) {
  extern __shared__ uint32_t smem[];
  const int c = blockIdx.x;
  const int s0 = blockIdx.y * p.ST;
  const int ns = min(p.ST, p.S - s0);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int W = p.W;
  uint32_t* raw = smem;                       // [ST][W]   ring rows of this tile
  uint32_t* pk = smem + p.ST * W;             // [ST][E]   spike word of each piece
  const int cur = (int)(p.t & p.rp_mask);

  // a1: stage the current scheduler rows of (core c, samples s0..) and clear
  // them (the row is free again for spikes due at t + Rp).
  uint32_t* row = p.ring + (((size_t)cur * p.G + c) * p.S + s0) * W;
  for (int i = tid; i < ns * W; i += blockDim.x) {
    raw[i] = row[i];
    row[i] = 0u;
  }
  __syncthreads();
  // a2: external input lines arriving at tick t (G8): one ballot per 32-axon word.
  if (p.t < p.T_in && p.has_in[c]) {
    const int32_t* inl = p.inl + (size_t)c * p.A;
    for (int idx = warp; idx < ns * W; idx += nwarps) {
      const int s = idx / W, w = idx - s * W;
      const int ap = w * 32 + lane;
      bool bit = false;
      if (ap < p.A) {
        const int32_t ln = inl[ap];
        if (ln >= 0) {
          const uint32_t* lb = p.lines + ((size_t)(s0 + s) * p.T_in + p.t) * p.WI;
          bit = (lb[ln >> 5] >> (ln & 31)) & 1u;
        }
      }
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
      if (lane == 0) raw[idx] |= m;
    }
    __syncthreads();
  }
  // expand to one spike word per piece
  const uint8_t* pword = p.pword + (size_t)c * E;
  for (int i = tid; i < ns * E; i += blockDim.x) {
    const int s = i / E, e = i - s * E;
    pk[i] = raw[s * W + pword[e]];
  }
  __syncthreads();

  for (int n = tid; n < p.Npad; n += blockDim.x) {
    uint32_t xp[E];
    int wp[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      xp[e] = __ldg(p.xp + ((size_t)c * E + e) * p.Npad + n);
      wp[e] = __ldg(p.wp + ((size_t)c * E + e) * p.Npad + n);
    }
    const short4 prm = p.prm[(size_t)c * p.Npad + n];
    const uint2 rt = p.route[(size_t)c * p.Npad + n];
    const uint32_t kind = route_kind(rt.x);
    const bool lin = route_lin(rt.x);
    const bool valid = n < p.N;
    int16_t* pot = p.pot + ((size_t)c * p.S + s0) * p.Npad + n;
    for (int s = 0; s < ns; ++s) {
      // a3: integration
      const uint32_t* sw = pk + s * E;
      int acc = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) acc += wp[e] * __popc(xp[e] & sw[e]);
      // a4: leak, thresholds, reset, saturate once (G1-G5)
      const int v = (int)pot[(size_t)s * p.Npad] + acc + prm.x;
      const bool fire = v >= prm.y;
      int nv;
      if (fire) nv = lin ? v - prm.y : prm.w;
      else if (v < prm.z) nv = lin ? v - prm.z : -prm.w;
      else nv = v;
      nv = min(max(nv, p.pot_lo), p.pot_hi);
      pot[(size_t)s * p.Npad] = (int16_t)nv;
      // a5 / a6: route into the destination ring row of tick t+delay, or count
      if (fire && valid) {
        if (kind == RK_ROUTE) {
          const uint32_t ax = route_axon(rt.x);
          const int slot = (int)((p.t + route_delay(rt.x)) & p.rp_mask);
          atomicOr(p.ring + (((size_t)slot * p.G + rt.y) * p.S + s0 + s) * W + (ax >> 5), 1u << (ax & 31));
        } else if (kind == RK_OUTPUT) {
          atomicAdd(p.counts + (size_t)(s0 + s) * p.C + rt.y, 1);
        }
      }
      if (p.raster) {
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, fire && valid);
        if (lane == 0)
          p.raster[(((size_t)(p.t - p.raster_t0) * p.S + s0 + s) * p.G + c) * p.Wn + (n >> 5)] = m;
      }
    }
  }
}

__global__ void reset_pot_kernel(int16_t* __restrict__ pot, const int16_t* __restrict__ init, int G, int S,
                                 int Npad) {
  const size_t total = (size_t)G * S * Npad;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t n = i % Npad;
    const size_t c = i / ((size_t)S * Npad);
    pot[i] = init[c * Npad + n];
  }
}

template <int E>
cudaError_t launch_one(const TickParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  tick_popc_kernel<E><<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

int pieces_template(int E) {
  const int opts[] = {4, 8, 12, 16, 24, 36};
  for (int o : opts)
    if (E <= o) return o;
  return 36;
}

int choose_sample_tile(const Compiled& n, int64_t S) {
  // enough CTAs to fill 148 SMs several times over, at most 64 samples per CTA
  int64_t want = (int64_t)n.G * S / (4 * 148);
  if (want < 1) want = 1;
  if (want > 64) want = 64;
  if (want > S) want = S;
  return (int)want;
}

cudaError_t launch_reset(ranc_ctx* ctx) {
  const Compiled& n = ctx->net;
  cudaError_t e;
  const size_t total = (size_t)n.G * ctx->S * n.Npad;
  int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
  if (blocks < 1) blocks = 1;
  reset_pot_kernel<<<blocks, 256, 0, ctx->stream>>>((int16_t*)ctx->d_pot.p, (const int16_t*)ctx->d_init.p, n.G,
                                                    (int)ctx->S, n.Npad);
  ctx->launches++;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ctx->d_ring.p, 0, ctx->d_ring.bytes, ctx->stream)) != cudaSuccess) return e;
  if (ctx->d_counts.bytes)
    if ((e = cudaMemsetAsync(ctx->d_counts.p, 0, ctx->d_counts.bytes, ctx->stream)) != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t launch_ticks(ranc_ctx* ctx, int64_t num_ticks) {
  const Compiled& n = ctx->net;
  TickParams p{};
  p.G = n.G; p.S = (int)ctx->S; p.N = n.N; p.Npad = n.Npad; p.A = n.A; p.W = n.W; p.E = n.E;
  p.Wn = n.Wn; p.C = n.C; p.T_in = ctx->T_in; p.WI = n.WI; p.ST = ctx->sample_tile;
  p.rp_mask = n.Rp - 1;
  p.pot_lo = -(1 << (n.pb - 1));
  p.pot_hi = (1 << (n.pb - 1)) - 1;
  p.xp = (const uint32_t*)ctx->d_xp.p;
  p.wp = (const int16_t*)ctx->d_wp.p;
  p.pword = (const uint8_t*)ctx->d_pword.p;
  p.prm = (const short4*)ctx->d_prm.p;
  p.route = (const uint2*)ctx->d_route.p;
  p.inl = (const int32_t*)ctx->d_inl.p;
  p.has_in = (const uint8_t*)ctx->d_has_in.p;
  p.lines = (const uint32_t*)ctx->d_lines.p;
  p.pot = (int16_t*)ctx->d_pot.p;
  p.ring = (uint32_t*)ctx->d_ring.p;
  p.counts = (int32_t*)ctx->d_counts.p;
  p.raster = (uint32_t*)ctx->d_raster.p;
  p.raster_t0 = ctx->raster_t0;
  const dim3 grid(n.G, (unsigned)((ctx->S + p.ST - 1) / p.ST));
  const size_t smem = (size_t)p.ST * (n.W + n.E) * sizeof(uint32_t);
  for (int64_t i = 0; i < num_ticks; ++i) {
    p.t = ctx->now + i;
    cudaError_t e;
    switch (n.E) {
      case 4: e = launch_one<4>(p, grid, smem, ctx->stream); break;
      case 8: e = launch_one<8>(p, grid, smem, ctx->stream); break;
      case 12: e = launch_one<12>(p, grid, smem, ctx->stream); break;
      case 16: e = launch_one<16>(p, grid, smem, ctx->stream); break;
      case 24: e = launch_one<24>(p, grid, smem, ctx->stream); break;
      default: e = launch_one<36>(p, grid, smem, ctx->stream); break;
    }
    ctx->launches++;
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ranc
