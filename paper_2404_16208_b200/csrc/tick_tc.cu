// tick_tc.cu -- the tick kernel with synaptic integration on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM).  SURVEY.md 8(f) row f1.
//
// Integration (Alg. 1 l.10-13) of one core over a tile of NT
// samples is the integer matrix product
//     acc[n][s] = sum_a' Wfold[n][a'] * spike[s][a'],
//     Wfold[n][a'] = conn[n][a'] * w[n][type(a')]
// exact in int32 (|w| <= 127 checked at load, K <= 256 terms).  M = 128
// neurons per MMA (two halves for 256 neurons), N = NT samples, K = 32 axons
// per instruction.  Wfold is pre-arranged on the host in the canonical
// K-major core-matrix layout (tc.h) and lands in shared memory with one TMA
// bulk copy; the spike bits of the tile are expanded to 0/1 bytes in the same
// layout.  The epilogue (thread = neuron = TMEM lane) adds the accumulator to
// the potential, applies leak / thresholds / reset (Alg. 1 l.14) and routes
// the spikes exactly like the popcount kernel (tick.cu), which stays the path
// for networks outside the int8 envelope.
//
// Potential layout of this kernel: tile-blocked [G][nT][Np][NT] int16, so a
// thread's 32 samples of one neuron are 64 contiguous bytes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"
#include "ptx.h"
#include "tc.h"

namespace ranc {

namespace {

constexpr int kThreadsTC = 256;

struct TcLayout {
  uint32_t w, b, raw, lines, total;
};

__host__ __device__ inline TcLayout tc_layout(int Np, int Kp, int NT, int W, int WI) {
  TcLayout L;
  uint32_t o = 64;                          // mbarriers + TMEM address holder
  L.w = 1024;  o = L.w + (uint32_t)Np * Kp; // Wfold, canonical layout
  o = (o + 127) & ~127u;
  L.b = o;     o += (uint32_t)NT * Kp;      // spikes as bytes, canonical layout
  o = (o + 15) & ~15u;
  L.raw = o;   o += (uint32_t)NT * W * 4;   // staged ring rows
  o = (o + 15) & ~15u;
  L.lines = o; o += (uint32_t)NT * WI * 4;  // staged input lines
  L.total = (o + 127) & ~127u;
  return L;
}

template <int NT>
__global__ void __launch_bounds__(kThreadsTC, 2) tick_tc_kernel(const TickParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar_w = reinterpret_cast<uint64_t*>(smem);
  uint64_t* bar_mma = reinterpret_cast<uint64_t*>(smem + 8);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + 16);
  const int Np = p.Npad, Kp = p.Kp, W = p.W;
  const TcLayout L = tc_layout(Np, Kp, NT, W, p.WI);
  uint8_t* w_s = smem + L.w;
  uint8_t* b_s = smem + L.b;
  uint32_t* raw = reinterpret_cast<uint32_t*>(smem + L.raw);
  uint32_t* lines_s = reinterpret_cast<uint32_t*>(smem + L.lines);

  const int c = blockIdx.x;
  const int tile = blockIdx.y;
  const int s0 = tile * NT;
  const int ns = min(NT, p.S - s0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cur = (int)(p.t & p.rp_mask);
  const int Mh = Np / 128;
  const int nT = (p.S + NT - 1) / NT;

  if (warp == 0) tc::alloc(tmem_holder, 2 * NT >= 32 ? 2 * NT : 32);
  if (tid == 32) {
    ptx::mbar_init(bar_w, 1);
    ptx::mbar_init(bar_mma, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 32) {
    const uint32_t bytes = (uint32_t)Np * Kp;
    ptx::mbar_arrive_expect_tx(bar_w, bytes);
    ptx::bulk_g2s(w_s, p.wfold + (size_t)c * bytes, bytes, bar_w);
  }

  // epilogue identity: neuron n = TMEM lane, half h
  const int h = warp >> 2, q = warp & 3;
  const int n = h * 128 + q * 32 + lane;
  const bool in_tile = h < Mh;
  // prefetch this thread's potentials for the whole tile (2*NT bytes)
  uint32_t potw[NT / 2];   // 2 x int16 per word, samples in order
  int16_t* pot_row = p.pot + (((size_t)c * nT + tile) * Np + (in_tile ? n : 0)) * NT;
  if (in_tile && !p.fresh) {
#pragma unroll
    for (int i = 0; i < NT / 8; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(pot_row)[i];
      potw[4 * i + 0] = v.x;
      potw[4 * i + 1] = v.y;
      potw[4 * i + 2] = v.z;
      potw[4 * i + 3] = v.w;
    }
  }

  // a1: stage + clear the scheduler rows due now
  uint32_t* row = p.ring + (((size_t)cur * p.G + c) * p.S + s0) * W;
  for (int i = tid; i < ns * W; i += blockDim.x) {
    raw[i] = row[i];
    row[i] = 0u;
  }
  for (int i = ns * W + tid; i < NT * W; i += blockDim.x) raw[i] = 0u;  // tail samples: no spikes
  const bool inject = p.t < p.T_in && p.has_in[c];
  if (inject) {
    const uint32_t* lg = p.lines + ((size_t)p.t * p.S + s0) * p.WI;
    for (int i = tid; i < ns * p.WI; i += blockDim.x) lines_s[i] = lg[i];
  }
  __syncthreads();
  // a2: input lines (ballot per 32-axon word, as in tick.cu)
  if (inject) {
    for (int ap0 = tid - lane; ap0 < W * 32; ap0 += blockDim.x) {
      const int ap = ap0 + lane;
      const int32_t ln = ap < p.A ? p.inl[(size_t)c * p.A + ap] : -1;
      const int lw = ln >> 5, lb = ln & 31;
      for (int s = 0; s < ns; ++s) {
        const bool bit = ln >= 0 && ((lines_s[s * p.WI + lw] >> lb) & 1u);
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
        if (lane == 0) raw[s * W + (ap0 >> 5)] |= m;
      }
    }
    __syncthreads();
  }
  // spikes -> 0/1 bytes in the canonical K-major layout (B operand, N = samples)
  const int K16 = Kp >> 4;
  for (int i = tid; i < NT * K16; i += blockDim.x) {
    const int s = i / K16, k16 = i - s * K16;
    const uint32_t wv = raw[s * W + (k16 >> 1)];
    const uint32_t bits = (k16 & 1) ? (wv >> 16) : (wv & 0xFFFFu);
    uint4 v;
    v.x = tc::nib2bytes(bits & 15u);
    v.y = tc::nib2bytes((bits >> 4) & 15u);
    v.z = tc::nib2bytes((bits >> 8) & 15u);
    v.w = tc::nib2bytes((bits >> 12) & 15u);
    *reinterpret_cast<uint4*>(b_s + tc::operand_offset(s, k16 * 16, Kp)) = v;
  }
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  // a3: integration on the tensor cores
  if (tid == 0) {
    ptx::mbar_wait(bar_w, 0);
    const uint32_t id = tc::idesc_i8(128, NT);
    const uint32_t sbo = (uint32_t)Kp * 8;
    for (int hh = 0; hh < Mh; ++hh)
      for (int kk = 0; kk < Kp / 32; ++kk) {
        const uint64_t ad = tc::smem_desc(ptx::smem_u32(w_s + hh * 128 * Kp + kk * 256), 128, sbo);
        const uint64_t bd = tc::smem_desc(ptx::smem_u32(b_s + kk * 256), 128, sbo);
        tc::mma_i8(tmem + hh * NT, ad, bd, id, kk > 0 ? 1u : 0u);
      }
    tc::commit(bar_mma);
  }
  ptx::mbar_wait(bar_mma, 0);
  tc::fence_after();

  // a4-a6: epilogue, thread = neuron, 32 samples per TMEM load
  if (in_tile) {
    const short4 prm = p.prm[(size_t)c * Np + n];
    const uint2 rt = p.route[(size_t)c * Np + n];
    const int init = p.init[(size_t)c * Np + n];
    const uint32_t kind = route_kind(rt.x);
    const bool lin = route_lin(rt.x);
    const bool valid = n < p.N;
    const int leak = prm.x, pth = prm.y, nth = prm.z, rst = prm.w;
    const uint32_t ax = route_axon(rt.x);
    const int slot = (int)((p.t + route_delay(rt.x)) & p.rp_mask);
    uint32_t* ring_dst = p.ring + (((size_t)slot * p.G + rt.y) * p.S) * W + (ax >> 5);
    const uint32_t axbit = 1u << (ax & 31);
#pragma unroll
    for (int j = 0; j < NT / 32; ++j) {
      uint32_t acc[32];
      tc::ld32(tmem + ((uint32_t)(q * 32) << 16) + h * NT + j * 32, acc);
      tc::wait_ld();
      uint32_t outw[16];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t word = potw[(j * 32 + i) >> 1];
        const int pot = p.fresh ? init : (int)(int16_t)((i & 1) ? (word >> 16) : (word & 0xFFFFu));
        const int v = pot + (int)acc[i] + leak;
        const bool fire = v >= pth;
        const bool neg = v < nth;
        const int rv = lin ? v - (fire ? pth : nth) : (fire ? rst : -rst);
        int nv = (fire || neg) ? rv : v;
        nv = min(max(nv, p.pot_lo), p.pot_hi);
        if (i & 1) outw[i >> 1] |= ((uint32_t)nv & 0xFFFFu) << 16;
        else outw[i >> 1] = (uint32_t)nv & 0xFFFFu;
        const int s = j * 32 + i;
        const bool real = s < ns;
        if (fire && valid && real && kind != RK_NONE) {
          if (kind == RK_ROUTE) atomicOr(ring_dst + (size_t)(s0 + s) * W, axbit);
          else atomicAdd(p.counts + (size_t)(s0 + s) * p.C + rt.y, 1);
        }
        if (p.raster) {
          const uint32_t m = __ballot_sync(0xFFFFFFFFu, fire && valid);
          if (lane == 0 && real && (n >> 5) < p.Wn)
            p.raster[(((size_t)(p.t - p.raster_t0) * p.S + s0 + s) * p.G + c) * p.Wn + (n >> 5)] = m;
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(pot_row) + j * 4;
      dst[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
      dst[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
      dst[2] = make_uint4(outw[8], outw[9], outw[10], outw[11]);
      dst[3] = make_uint4(outw[12], outw[13], outw[14], outw[15]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 2 * NT >= 32 ? 2 * NT : 32);
}

}  // namespace

int tc_tile() { return 64; }

size_t tc_smem_bytes(const Compiled& n, int NT) { return tc_layout(n.Npad, n.Kp, NT, n.W, n.WI).total; }

cudaError_t launch_ticks_tc(ranc_ctx* ctx, TickParams p, int64_t num_ticks) {
  const Compiled& n = ctx->net;
  constexpr int NT = 64;
  p.ST = NT;
  const dim3 grid(n.G, (unsigned)((ctx->S + NT - 1) / NT));
  const size_t smem = tc_smem_bytes(n, NT);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tick_tc_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  for (int64_t i = 0; i < num_ticks; ++i) {
    p.t = ctx->now + i;
    p.fresh = ctx->fresh ? 1 : 0;
    tick_tc_kernel<NT><<<grid, kThreadsTC, smem, ctx->stream>>>(p);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ctx->fresh = false;
  }
  return cudaSuccess;
}

}  // namespace ranc
