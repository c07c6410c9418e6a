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
// ST samples); thread = neuron.  The tile's potentials ([ST][Npad] int16,
// contiguous in the [G][S][Npad] layout) move HBM <-> shared memory with one
// TMA bulk copy each way (cp.async.bulk, UBLKCP); each thread keeps its
// neuron's crossbar pieces and weights in registers for the whole tile, so
// the (L2-resident) network is read once per tile.  Integration is
// sum_e w_e * popc(xbar_e & spikes_e) over the <= ceil(A/32)+K-1 type-sorted
// pieces (compile.cpp).
//
// Why no intra-tick barrier is needed: every route delay is in [1, D] and the
// ring has Rp >= D+1 physical rows, so no spike written during tick t lands in
// row t & (Rp-1), which is the only row read (and cleared) during tick t.
// Spike writes are idempotent ORs (G11), so their order is irrelevant.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "ptx.h"

namespace cg = cooperative_groups;

namespace ranc {

namespace {

constexpr int kThreads = 256;
constexpr int kPotTileBytes = 48 * 1024;  // shared-memory budget for the potential tile

struct SmemLayout {
  uint32_t pot, raw, pk, lines, total;
};

__host__ __device__ inline SmemLayout smem_layout(int ST, int Npad, int W, int E, int WI) {
  SmemLayout L;
  uint32_t o = 16;                                // mbarrier
  L.pot = o;   o += (uint32_t)ST * Npad * 2;      // int16 [ST][Npad]
  o = (o + 15) & ~15u;
  L.pk = o;    o += (uint32_t)ST * E * 4;         // u32 [ST][E]
  L.raw = o;   o += (uint32_t)ST * W * 4;         // u32 [ST][W]
  o = (o + 15) & ~15u;
  L.lines = o; o += (uint32_t)ST * WI * 4;        // u32 [ST][WI]
  L.total = (o + 15) & ~15u;
  return L;
}

// One (core, sample tile) of one tick, executed by a whole CTA.  `phase` is
// the parity of the CTA's potential-tile mbarrier (toggled per use, so that a
// persistent CTA can process many tiles).
// kResident (streaming kernel): the tile's potentials live in shared memory
// at pot_res for the whole run (no HBM round trip per tick).
template <int E, bool kResident>
__device__ __forceinline__ void popc_tile(const TickParams& p, int cl, int tile, uint8_t* smem, uint32_t& phase,
                                          int16_t* pot_res) {
  const int c = p.c_lo + cl;             // global core (network index); cl = local core (state index)
  const int s0 = tile * p.ST;
  const int ns = min(p.ST, p.S - s0);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int W = p.W;
  const SmemLayout L = smem_layout(p.ST, p.Npad, W, E, p.WIp);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int16_t* pot_s = kResident ? pot_res : reinterpret_cast<int16_t*>(smem + L.pot);
  uint32_t* pk = reinterpret_cast<uint32_t*>(smem + L.pk);
  uint32_t* raw = reinterpret_cast<uint32_t*>(smem + L.raw);
  uint32_t* lines_s = reinterpret_cast<uint32_t*>(smem + L.lines);
  const int cur = (int)(p.t & p.rp_mask);
  const uint32_t tile_bytes = (uint32_t)ns * p.Npad * 2;
  int16_t* pot_g = p.pot + ((size_t)cl * p.S + s0) * p.Npad;
  // RANC_DEBUG_PHASES: per-phase cycle sums over all CTAs (f4 profile)
  const bool prof = !kResident && p.dbg && tid == 0;
  long long ck = prof ? clock64() : 0;
  auto phase_mark = [&](int k) {
    if (prof) {
      const long long now = clock64();
      atomicAdd(reinterpret_cast<unsigned long long*>(p.dbg) + k, (unsigned long long)(now - ck));
      ck = now;
    }
  };

  // stream the tile's potentials in (TMA bulk copy) while the spikes are staged
  if (!kResident && !p.fresh && tid == 0) {
    ptx::mbar_arrive_expect_tx(bar, tile_bytes);
    ptx::bulk_g2s(pot_s, pot_g, tile_bytes, bar);
  }
  // a1: stage the current scheduler rows of (core c, samples s0..) and clear
  // them (the row is free again for spikes due at t + Rp).
  uint32_t* row = p.ring + (((size_t)cur * p.G_loc + cl) * p.Sr + s0) * W;
  for (int i = tid; i < ns * W; i += blockDim.x) {
    raw[i] = row[i];
    row[i] = 0u;
  }
  const bool inject = p.t < p.T_in && p.has_in[c];
  if (inject) {
    const uint32_t* lg = p.lines + ((size_t)p.t * p.Sr + s0) * p.WIp;   // [T_in][Sr][WIp]
    for (int i = tid; i < ns * p.WIp; i += blockDim.x) lines_s[i] = lg[i];
  }
  __syncthreads();
  phase_mark(0);   // a1 scheduler read + clear (and the line rows staged)
  // a2: external input lines arriving at tick t (G8).  Thread <-> permuted
  // axon a'; one warp ballot builds one 32-axon ring word, so the OR into the
  // staged row needs no atomics.
  if (inject) {
    for (int ap0 = tid - lane; ap0 < W * 32; ap0 += blockDim.x) {
      const int ap = ap0 + lane;
      const int32_t ln = ap < p.A ? p.inl[(size_t)c * p.A + ap] : -1;
      const int lw = ln >> 5, lb = ln & 31;
      for (int s = 0; s < ns; ++s) {
        const bool bit = ln >= 0 && ((lines_s[s * p.WIp + lw] >> lb) & 1u);
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
        if (lane == 0) raw[s * W + (ap0 >> 5)] |= m;
      }
    }
    __syncthreads();
  }
  if (p.spkin)   // RANC_TRACE_STATE_DIGEST: the axon spikes integrated this tick
    for (int i = tid; i < ns * W; i += blockDim.x)
      p.spkin[((size_t)(s0 + i / W) * p.G_loc + cl) * W + i % W] = raw[i];
  phase_mark(1);   // a2 input injection
  // expand to one spike word per piece
  const uint8_t* pword = p.pword + (size_t)c * E;
  for (int i = tid; i < ns * E; i += blockDim.x) {
    const int s = i / E, e = i - s * E;
    pk[i] = raw[s * W + pword[e]];
  }
  __syncthreads();
  phase_mark(2);   // spike words per crossbar piece
  if (!kResident && !p.fresh) {
    ptx::mbar_wait(bar, phase);
    phase ^= 1u;
  }
  phase_mark(3);   // potential tile load (TMA) not hidden by a1-a2

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
    const int init = p.init[(size_t)c * p.Npad + n];
    const uint32_t kind = route_kind(rt.x);
    const bool lin = route_lin(rt.x);
    const bool valid = n < p.N;
    const int leak = prm.x, pth = prm.y, nth = prm.z, rst = prm.w;
    // a route to a core of another rank is delivered by the exchange step
    const uint32_t dloc = rt.y - (uint32_t)p.c_lo;
    const bool route_here = kind == RK_ROUTE && dloc < (uint32_t)p.G_loc;
    const bool exporting = p.fired && p.exports[c];
#pragma unroll 2
    for (int s = 0; s < ns; ++s) {
      // a3: integration
      const uint4* sw = reinterpret_cast<const uint4*>(pk + s * E);
      int acc = 0;
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        const uint4 v4 = sw[q];
        acc += wp[4 * q + 0] * __popc(xp[4 * q + 0] & v4.x);
        acc += wp[4 * q + 1] * __popc(xp[4 * q + 1] & v4.y);
        acc += wp[4 * q + 2] * __popc(xp[4 * q + 2] & v4.z);
        acc += wp[4 * q + 3] * __popc(xp[4 * q + 3] & v4.w);
      }
      // a4: leak, thresholds, reset, saturate once (G1-G5)
      const int pot = p.fresh ? init : (int)pot_s[s * p.Npad + n];
      const int v = pot + acc + leak;
      const bool fire = v >= pth;
      const bool neg = v < nth;
      const int rv = lin ? v - (fire ? pth : nth) : (fire ? rst : -rst);
      int nv = (fire || neg) ? rv : v;
      nv = min(max(nv, p.pot_lo), p.pot_hi);
      pot_s[s * p.Npad + n] = (int16_t)nv;
      // a5 / a6: route into the destination ring row of tick t+delay, or count
      if (fire && valid) {
        if (route_here) {
          const uint32_t ax = route_axon(rt.x);
          const int slot = (int)((p.t + route_delay(rt.x)) & p.rp_mask);
          atomicOr(p.ring + (((size_t)slot * p.G_loc + dloc) * p.Sr + s0 + s) * W + (ax >> 5), 1u << (ax & 31));
        } else if (kind == RK_OUTPUT) {
          atomicAdd(p.counts + (size_t)(s0 + s) * p.C + rt.y, 1);
        }
      }
      if (p.raster || exporting) {
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, fire && valid);
        if (lane == 0 && (n >> 5) < p.Wn) {
          if (p.raster)
            p.raster[(((size_t)(p.t - p.raster_t0) * p.S + s0 + s) * p.G_loc + cl) * p.Wn + (n >> 5)] = m;
          if (exporting) p.fired[((size_t)cl * p.Sr + s0 + s) * p.Wn + (n >> 5)] = m;
        }
      }
    }
  }
  if (kResident) {
    __syncthreads();   // the staging buffers are reused by the next tile
    return;
  }
  // stream the updated tile back (TMA bulk store)
  ptx::fence_proxy_async_smem();
  __syncthreads();
  phase_mark(4);   // a3-a6: integration, LIF, routing + output bus (fused per sample)
  if (tid == 0) {
    ptx::bulk_s2g(pot_g, pot_s, tile_bytes);
    ptx::bulk_commit();
    ptx::bulk_wait_read0();
  }
  phase_mark(5);   // potential tile store
}

__device__ __forceinline__ void init_tile_barrier(uint8_t* smem) {
  if (threadIdx.x == 0) {
    ptx::mbar_init(reinterpret_cast<uint64_t*>(smem), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
}

template <int E>
__global__ void __launch_bounds__(kThreads, (E <= 12 ? 4 : (E <= 16 ? 3 : 2))) tick_popc_kernel(const TickParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  init_tile_barrier(smem);
  uint32_t phase = 0;
  popc_tile<E, false>(p, blockIdx.x, blockIdx.y, smem, phase, nullptr);
}

// Streaming mode (one long stream, few samples): all
// ticks of a ranc_run_ticks call in one cooperative launch.  CTA b owns the
// (core, tile) items b, b + grid, ...; their potentials stay in shared memory
// for the whole run (loaded before the first tick, stored after the last),
// so a tick only touches the scheduler rings (L2) and the input lines.  The
// grid barrier is the tick barrier (a7): it orders the ring ORs of
// tick t before the row reads of tick t+1.
template <int E>
__global__ void __launch_bounds__(kThreads, 1) tick_stream_kernel(TickParams p, int nticks, int n_tiles,
                                                                  uint32_t res_off) {
  extern __shared__ __align__(16) uint8_t smem[];
  init_tile_barrier(smem);
  uint32_t phase = 0;
  cg::grid_group grid = cg::this_grid();
  const int items = p.G_loc * n_tiles;
  const size_t tile_elems = (size_t)p.ST * p.Npad;
  int16_t* res = reinterpret_cast<int16_t*>(smem + res_off);
  if (!p.fresh) {
    int j = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++j) {
      const int cl = w % p.G_loc, s0 = (w / p.G_loc) * p.ST, ns = min(p.ST, p.S - s0);
      const int16_t* g = p.pot + ((size_t)cl * p.S + s0) * p.Npad;
      for (int i = threadIdx.x; i < ns * p.Npad; i += blockDim.x) res[j * tile_elems + i] = g[i];
    }
    __syncthreads();
  }
  for (int it = 0; it < nticks; ++it) {
    int j = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++j)
      popc_tile<E, true>(p, w % p.G_loc, w / p.G_loc, smem, phase, res + j * tile_elems);
    p.fresh = 0;
    ++p.t;
    if (p.fault != 1) grid.sync();   // (RANC_OPT_DEBUG_FAULT 1: the mutation test's missing barrier)
  }
  int j = 0;
  for (int w = blockIdx.x; w < items; w += gridDim.x, ++j) {
    const int cl = w % p.G_loc, s0 = (w / p.G_loc) * p.ST, ns = min(p.ST, p.S - s0);
    int16_t* g = p.pot + ((size_t)cl * p.S + s0) * p.Npad;
    for (int i = threadIdx.x; i < ns * p.Npad; i += blockDim.x) g[i] = res[j * tile_elems + i];
  }
}

// Streaming mode, one (core, sample tile) item per CTA (the common case:
// S = 1 and at most ~4 x 148 cores): thread = neuron, the neuron's crossbar
// pieces, weights and routing word stay in registers and the tile's
// potentials in shared memory for the whole run, so a tick is: read + clear
// the scheduler rows, OR in the input lines, integrate + LIF + route, grid
// barrier (the tick barrier, a7).
template <int E>
__global__ void __launch_bounds__(kThreads, (E <= 12 ? 4 : (E <= 16 ? 3 : 2)))
    tick_stream1_kernel(TickParams p, int nticks) {
  extern __shared__ __align__(16) uint8_t smem[];
  cg::grid_group grid = cg::this_grid();
  const int cl = blockIdx.x % p.G_loc, tile = blockIdx.x / p.G_loc;
  const int c = p.c_lo + cl;
  const int s0 = tile * p.ST, ns = min(p.ST, p.S - s0);
  const int tid = threadIdx.x, lane = tid & 31, W = p.W, n = tid;
  uint32_t* raw = reinterpret_cast<uint32_t*>(smem);                       // [ST][W]
  int16_t* pot_s = reinterpret_cast<int16_t*>(smem + (size_t)p.ST * W * 4);  // [ST][Npad]
  const bool has_n = n < p.Npad;
  uint32_t xp[E];
  int wp[E], pw[E];
  short4 prm = make_short4(0, 0, 0, 0);
  uint2 rt = make_uint2(0u, 0u);
  int init = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    xp[e] = has_n ? p.xp[((size_t)c * E + e) * p.Npad + n] : 0u;
    wp[e] = has_n ? p.wp[((size_t)c * E + e) * p.Npad + n] : 0;
    pw[e] = p.pword[(size_t)c * E + e];
  }
  if (has_n) {
    prm = p.prm[(size_t)c * p.Npad + n];
    rt = p.route[(size_t)c * p.Npad + n];
    init = p.init[(size_t)c * p.Npad + n];
  }
  const uint32_t kind = route_kind(rt.x);
  const bool lin = route_lin(rt.x);
  const bool valid = n < p.N;
  const int leak = prm.x, pth = prm.y, nth = prm.z, rst = prm.w;
  const uint32_t dloc = rt.y - (uint32_t)p.c_lo;
  const bool route_here = kind == RK_ROUTE && dloc < (uint32_t)p.G_loc;
  const uint32_t ax = route_axon(rt.x);
  if (has_n)
    for (int s = 0; s < ns; ++s)
      pot_s[s * p.Npad + n] = p.fresh ? (int16_t)init : p.pot[((size_t)cl * p.S + s0 + s) * p.Npad + n];
  const bool has_in = p.has_in[c];
  // one sample and one axon per thread (the streaming case): the input bit
  // of tick t+1 is fetched before tick t's barrier, off the critical path
  const bool fast_in = has_in && ns == 1 && W * 32 <= (int)blockDim.x;
  const int32_t my_ln = (fast_in && tid < p.A) ? p.inl[(size_t)c * p.A + tid] : -1;
  auto line_bit = [&](int64_t tt) -> bool {
    return my_ln >= 0 && tt < p.T_in &&
           ((p.lines[((size_t)tt * p.Sr + s0) * p.WIp + (my_ln >> 5)] >> (my_ln & 31)) & 1u);
  };
  bool next_bit = fast_in ? line_bit(p.t) : false;
  for (int it = 0; it < nticks; ++it) {
    const int64_t t = p.t + it;
    const int cur = (int)(t & p.rp_mask);
    // a1: rows due now; clear the words that hold spikes
    uint32_t* row = p.ring + (((size_t)cur * p.G_loc + cl) * p.Sr + s0) * W;
    for (int i = tid; i < ns * W; i += blockDim.x) {
      const uint32_t v = row[i];
      raw[i] = v;
      if (v) row[i] = 0u;
    }
    __syncthreads();
    // a2: input lines arriving now, one ballot per 32-axon word
    if (fast_in) {
      const bool bit = next_bit;
      next_bit = line_bit(t + 1);   // prefetch for the next tick
      if (t < p.T_in && tid < W * 32) {
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
        if (lane == 0 && m) raw[tid >> 5] |= m;
      }
      __syncthreads();
    } else if (t < p.T_in && has_in) {
      const uint32_t* lg = p.lines + ((size_t)t * p.Sr + s0) * p.WIp;
      for (int ap0 = tid - lane; ap0 < W * 32; ap0 += blockDim.x) {
        const int ap = ap0 + lane;
        const int32_t ln = ap < p.A ? p.inl[(size_t)c * p.A + ap] : -1;
        for (int s = 0; s < ns; ++s) {
          const bool bit = ln >= 0 && ((lg[s * p.WIp + (ln >> 5)] >> (ln & 31)) & 1u);
          const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
          if (lane == 0 && m) raw[s * W + (ap0 >> 5)] |= m;
        }
      }
      __syncthreads();
    }
    if (has_n) {
      for (int s = 0; s < ns; ++s) {
        int acc = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) acc += wp[e] * __popc(xp[e] & raw[s * W + pw[e]]);
        const int v = (int)pot_s[s * p.Npad + n] + acc + leak;
        const bool fire = v >= pth;
        const bool neg = v < nth;
        const int rv = lin ? v - (fire ? pth : nth) : (fire ? rst : -rst);
        int nv = (fire || neg) ? rv : v;
        nv = min(max(nv, p.pot_lo), p.pot_hi);
        pot_s[s * p.Npad + n] = (int16_t)nv;
        if (fire && valid) {
          if (route_here) {
            const int slot = (int)((t + route_delay(rt.x)) & p.rp_mask);
            atomicOr(p.ring + (((size_t)slot * p.G_loc + dloc) * p.Sr + s0 + s) * W + (ax >> 5), 1u << (ax & 31));
          } else if (kind == RK_OUTPUT) {
            atomicAdd(p.counts + (size_t)(s0 + s) * p.C + rt.y, 1);
          }
        }
        if (p.raster) {
          const uint32_t m = __ballot_sync(0xFFFFFFFFu, fire && valid);
          if (lane == 0 && (n >> 5) < p.Wn)
            p.raster[(((size_t)(t - p.raster_t0) * p.S + s0 + s) * p.G_loc + cl) * p.Wn + (n >> 5)] = m;
        }
      }
    }
    if (p.fault != 1) grid.sync();   // a7: tick t's deliveries are visible to tick t+1's row reads
  }
  if (has_n)
    for (int s = 0; s < ns; ++s) p.pot[((size_t)cl * p.S + s0 + s) * p.Npad + n] = pot_s[s * p.Npad + n];
}

// RANC_TRACE_STATE_DIGEST: one block per sample sums,
// mod 2^64, mix() of every (neuron, potential), every fired neuron and every
// integrated axon spike of this context's cores (original indices).
__device__ __forceinline__ uint64_t digest_mix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void digest_kernel(const int16_t* __restrict__ pot, int tc_layout, const uint32_t* __restrict__ raster,
                              const uint32_t* __restrict__ spkin, const int32_t* __restrict__ perm, int c_lo,
                              int G_loc, int S, int N, int Npad, int A, int W, int Wn, uint64_t* __restrict__ out) {
  const uint64_t K1 = 0x243F6A8885A308D3ull, K2 = 0x13198A2E03707344ull;
  constexpr int TNT = 64;   // tensor-core potential tile (tick_tc.cu NT)
  const int nT = (S + TNT - 1) / TNT;
  for (int s = blockIdx.x; s < S; s += gridDim.x) {
    uint64_t d = 0;
    for (int i = threadIdx.x; i < G_loc * N; i += blockDim.x) {
      const int cl = i / N, n = i - cl * N;
      const uint64_t id = (uint64_t)(c_lo + cl) * N + n;
      const size_t pi = tc_layout
                            ? ((((size_t)cl * nT + s / TNT) * (TNT / 8) + (s % TNT) / 8) * Npad + n) * 8 + s % 8
                            : ((size_t)cl * S + s) * Npad + n;
      d += digest_mix((id << 32) | (uint32_t)(int32_t)pot[pi]);
      if ((raster[((size_t)s * G_loc + cl) * Wn + (n >> 5)] >> (n & 31)) & 1u) d += digest_mix(K1 ^ id);
    }
    for (int i = threadIdx.x; i < G_loc * W * 32; i += blockDim.x) {
      const int cl = i / (W * 32), ap = i - cl * W * 32;
      if (ap < A && ((spkin[((size_t)s * G_loc + cl) * W + (ap >> 5)] >> (ap & 31)) & 1u)) {
        const int c = c_lo + cl;
        d += digest_mix(K2 ^ (uint64_t)((size_t)c * A + perm[(size_t)c * A + ap]));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xFFFFFFFFu, d, o);
    __shared__ uint64_t part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += part[w];
      out[s] = tot;
    }
    __syncthreads();
  }
}

// [S][T_in][WI] -> [T_in][Sr][WIp] (padding words stay zero)
__global__ void transpose_lines_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int S, int T,
                                       int WI, int Sr, int WIp) {
  const size_t total = (size_t)S * T * WI;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t w = i % WI, st = i / WI;
    const size_t t = st % T, s = st / T;
    out[(t * Sr + s) * WIp + w] = in[i];
  }
}

template <int E>
cudaError_t launch_one(const TickParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured))
    cudaFuncSetAttribute(tick_popc_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  tick_popc_kernel<E><<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

// grid and shared memory of the streaming kernel: as many CTAs as can be
// co-resident (cooperative launch), each holding its items' potentials
struct StreamPlan {
  int grid = 0;
  uint32_t res_off = 0;
  size_t smem = 0;
};

template <int E>
StreamPlan plan_stream_e(const TickParams& p, size_t scratch, int n_tiles, int num_sms) {
  StreamPlan pl;
  const int items = p.G_loc * n_tiles;
  const size_t tile_bytes = (size_t)p.ST * p.Npad * 2;
  pl.res_off = (uint32_t)((scratch + 15) & ~(size_t)15);
  static const int force = getenv("RANC_STREAM_CTAS") ? atoi(getenv("RANC_STREAM_CTAS")) : 0;
  for (int per_sm = 4; per_sm >= 1; --per_sm) {
    const int grid = std::max(1, std::min(items, force > 0 ? force : per_sm * num_sms));
    const size_t smem = pl.res_off + (size_t)((items + grid - 1) / grid) * tile_bytes;
    if (smem > 200 * 1024) continue;
    int fit = 0;
    cudaFuncSetAttribute(tick_stream_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, tick_stream_kernel<E>, kThreads, smem) != cudaSuccess)
      return pl;
    if ((int64_t)fit * num_sms < grid) continue;
    pl.grid = grid;
    pl.smem = smem;
    return pl;
  }
  return pl;   // grid 0: not possible (too many potentials to keep resident)
}

template <int E>
cudaError_t launch_stream_e(TickParams p, int nticks, size_t scratch, int n_tiles, int num_sms, cudaStream_t st,
                            bool dry, bool* ok) {
  static const bool no1 = getenv("RANC_STREAM_MULTI") != nullptr;   // experiment: force the multi-item kernel
  const int items = p.G_loc * n_tiles;
  if (p.Npad <= kThreads && !no1) {
    const size_t smem1 = (size_t)p.ST * p.W * 4 + (size_t)p.ST * p.Npad * 2;
    int fit = 0;
    if (smem1 <= 48 * 1024 &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, tick_stream1_kernel<E>, kThreads, smem1) == cudaSuccess &&
        (int64_t)fit * num_sms >= items) {
      *ok = true;
      if (dry) return cudaSuccess;
      void* args[] = {&p, &nticks};
      return cudaLaunchCooperativeKernel((const void*)tick_stream1_kernel<E>, dim3(items), dim3(kThreads), args,
                                         smem1, st);
    }
  }
  const StreamPlan pl = plan_stream_e<E>(p, scratch, n_tiles, num_sms);
  *ok = pl.grid > 0;
  if (dry || !*ok) return cudaSuccess;
  uint32_t res_off = pl.res_off;
  void* args[] = {&p, &nticks, &n_tiles, &res_off};
  return cudaLaunchCooperativeKernel((const void*)tick_stream_kernel<E>, dim3(pl.grid), dim3(kThreads), args,
                                     pl.smem, st);
}

}  // namespace

int pieces_template(int E) {
  const int opts[] = {4, 8, 12, 16, 24, 36};
  for (int o : opts)
    if (E <= o) return o;
  return 36;
}

int choose_sample_tile(const Compiled& n, int64_t S) {
  // as many samples per CTA as the potential tile budget allows (<= 64), but
  // enough CTAs to fill the 148 SMs several times over
  int64_t cap = std::max<int64_t>(1, kPotTileBytes / (n.Npad * 2));
  int64_t want = (int64_t)n.G * S / (4 * 148);
  want = std::max<int64_t>(1, std::min<int64_t>({want, 64, cap, S}));
  return (int)want;
}

cudaError_t transpose_lines(ranc_ctx* ctx, const uint32_t* staging) {
  const Compiled& n = ctx->net;
  const size_t total = (size_t)ctx->S * ctx->T_in * n.WI;
  if (!total) return cudaSuccess;
  int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 8);
  cudaError_t e = cudaMemsetAsync(ctx->d_lines.p, 0, ctx->d_lines.bytes, ctx->stream);
  if (e != cudaSuccess) return e;
  transpose_lines_kernel<<<blocks, 256, 0, ctx->stream>>>(staging, (uint32_t*)ctx->d_lines.p, (int)ctx->S,
                                                          ctx->T_in, n.WI, (int)ctx->Sr, n.WIp);
  ctx->launches++;
  return cudaGetLastError();
}

cudaError_t launch_reset(ranc_ctx* ctx) {
  // potentials are re-initialised by the first tick (p.fresh), so a reset only
  // empties the rings and the class counts
  cudaError_t e;
  if ((e = cudaMemsetAsync(ctx->d_ring.p, 0, ctx->d_ring.bytes, ctx->stream)) != cudaSuccess) return e;
  if (ctx->d_counts.bytes)
    if ((e = cudaMemsetAsync(ctx->d_counts.p, 0, ctx->d_counts.bytes, ctx->stream)) != cudaSuccess) return e;
  ctx->fresh = true;
  return cudaSuccess;
}

namespace {

TickParams make_params(ranc_ctx* ctx) {
  const Compiled& n = ctx->net;
  TickParams p{};
  p.G = n.G; p.S = (int)ctx->S; p.Sr = (int)ctx->Sr; p.WIp = n.WIp; p.N = n.N; p.Npad = n.Npad; p.A = n.A;
  p.W = n.W; p.E = n.E; p.Wn = n.Wn; p.C = n.C; p.T_in = ctx->T_in; p.WI = n.WI; p.ST = ctx->sample_tile;
  p.c_lo = ctx->c_lo; p.G_loc = ctx->G_loc;
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
  p.init = (const int16_t*)ctx->d_init.p;
  p.lines = (const uint32_t*)ctx->d_lines.p;
  p.pot = (int16_t*)ctx->d_pot.p;
  p.ring = (uint32_t*)ctx->d_ring.p;
  p.counts = (int32_t*)ctx->d_counts.p;
  p.raster = (uint32_t*)ctx->d_raster.p;
  p.raster_t0 = ctx->raster_t0;
  p.fired = ctx->shard_mode == RANC_SHARD_CORES ? (uint32_t*)ctx->d_fired.p : nullptr;
  p.spkin = (ctx->trace_flags & RANC_TRACE_STATE_DIGEST) ? (uint32_t*)ctx->d_spkin.p : nullptr;
  p.exports = (const uint8_t*)ctx->d_exports.p;
  p.Kp = n.Kp;
  p.wfold = (const uint8_t*)ctx->d_wfold.p;
  p.t = ctx->now;
  p.fresh = ctx->fresh ? 1 : 0;
  p.fault = ctx->fault;
  return p;
}

}  // namespace

namespace {

cudaError_t stream_dispatch(ranc_ctx* ctx, int64_t num_ticks, bool dry, bool* ok) {
  const Compiled& n = ctx->net;
  TickParams p = make_params(ctx);
  const int n_tiles = (int)((ctx->S + p.ST - 1) / p.ST);
  const size_t scratch = smem_layout(p.ST, n.Npad, n.W, n.E, n.WIp).total;
  const int nt = (int)std::min<int64_t>(num_ticks, 1 << 30);
  switch (n.E) {
    case 4: return launch_stream_e<4>(p, nt, scratch, n_tiles, ctx->num_sms, ctx->stream, dry, ok);
    case 8: return launch_stream_e<8>(p, nt, scratch, n_tiles, ctx->num_sms, ctx->stream, dry, ok);
    case 12: return launch_stream_e<12>(p, nt, scratch, n_tiles, ctx->num_sms, ctx->stream, dry, ok);
    case 16: return launch_stream_e<16>(p, nt, scratch, n_tiles, ctx->num_sms, ctx->stream, dry, ok);
    case 24: return launch_stream_e<24>(p, nt, scratch, n_tiles, ctx->num_sms, ctx->stream, dry, ok);
    default: return launch_stream_e<36>(p, nt, scratch, n_tiles, ctx->num_sms, ctx->stream, dry, ok);
  }
}

}  // namespace

bool stream_eligible(ranc_ctx* ctx, int64_t num_ticks) {
  if (ctx->kernel_active == RANC_KERNEL_TC) return tc_multi_eligible(ctx, num_ticks);
  if (ctx->kernel_active != RANC_KERNEL_POPC || ctx->shard_mode == RANC_SHARD_CORES || num_ticks < 2) return false;
  if (ctx->stream_opt == 1) return false;
  if (ctx->stream_opt == 0) {
    // automatic: few (core, tile) items per tick, where per-tick launches dominate
    const int64_t tiles = (ctx->S + ctx->sample_tile - 1) / ctx->sample_tile;
    if ((int64_t)ctx->G_loc * tiles > 4 * 148 * 4) return false;
  }
  bool ok = false;
  return stream_dispatch(ctx, num_ticks, true, &ok) == cudaSuccess && ok;
}

cudaError_t launch_stream(ranc_ctx* ctx, int64_t num_ticks) {
  bool ok = false;
  cudaError_t e;
  if (ctx->kernel_active == RANC_KERNEL_TC) {
    e = launch_tc_multi(ctx, make_params(ctx), num_ticks);
    ok = true;
  } else {
    e = stream_dispatch(ctx, num_ticks, false, &ok);
  }
  ctx->launches++;
  if (e != cudaSuccess) return e;
  if (!ok) return cudaErrorCooperativeLaunchTooLarge;
  const int nt = (int)std::min<int64_t>(num_ticks, 1 << 30);
  ctx->fresh = false;
  ctx->now += nt;
  return cudaSuccess;
}

cudaError_t launch_digest(ranc_ctx* ctx, int64_t tick_index) {
  const Compiled& n = ctx->net;
  const uint32_t* raster = (const uint32_t*)ctx->d_raster.p + (size_t)tick_index * ctx->S * ctx->G_loc * n.Wn;
  uint64_t* out = (uint64_t*)ctx->d_digest.p + (size_t)tick_index * ctx->S;
  const int grid = (int)std::min<int64_t>(ctx->S, 148 * 8);
  digest_kernel<<<grid, 256, 0, ctx->stream>>>((const int16_t*)ctx->d_pot.p, ctx->kernel_active == RANC_KERNEL_TC ? 1 : 0,
                                               raster, (const uint32_t*)ctx->d_spkin.p,
                                               (const int32_t*)ctx->d_perm_dig.p, ctx->c_lo, ctx->G_loc, (int)ctx->S,
                                               n.N, n.Npad, n.A, n.W, n.Wn, out);
  ctx->launches++;
  return cudaGetLastError();
}

cudaError_t launch_one_tick(ranc_ctx* ctx) {
  const Compiled& n = ctx->net;
  TickParams p = make_params(ctx);
  cudaError_t e;
  if (ctx->kernel_active == RANC_KERNEL_TC) {
    e = launch_tick_tc(ctx, p);
  } else {
    const dim3 grid(ctx->G_loc, (unsigned)((ctx->S + p.ST - 1) / p.ST));
    const size_t smem = smem_layout(p.ST, n.Npad, n.W, n.E, n.WIp).total;
    static const bool phases = getenv("RANC_DEBUG_PHASES") != nullptr;
    if (phases) {
      if (!ctx->d_dbg.p) dev_alloc(ctx, &ctx->d_dbg, 4096 * 8);
      cudaMemsetAsync(ctx->d_dbg.p, 0, 8 * 8, ctx->stream);
      p.dbg = (unsigned long long*)ctx->d_dbg.p;
    }
    switch (n.E) {
      case 4: e = launch_one<4>(p, grid, smem, ctx->stream); break;
      case 8: e = launch_one<8>(p, grid, smem, ctx->stream); break;
      case 12: e = launch_one<12>(p, grid, smem, ctx->stream); break;
      case 16: e = launch_one<16>(p, grid, smem, ctx->stream); break;
      case 24: e = launch_one<24>(p, grid, smem, ctx->stream); break;
      default: e = launch_one<36>(p, grid, smem, ctx->stream); break;
    }
  }
  ctx->launches++;
  if (e != cudaSuccess) return e;
  if (p.dbg && ctx->kernel_active != RANC_KERNEL_TC) {
    unsigned long long h[6];
    cudaMemcpyAsync(h, ctx->d_dbg.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    fprintf(stderr, "phases t=%lld cycles (sum over CTAs): a1 %llu a2 %llu expand %llu potwait %llu a3-a6 %llu store %llu\n",
            (long long)p.t, h[0], h[1], h[2], h[3], h[4], h[5]);
  }
  ctx->fresh = false;
  ctx->now += 1;
  return cudaSuccess;
}

}  // namespace ranc
