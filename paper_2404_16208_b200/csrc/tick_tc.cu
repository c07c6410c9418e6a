// tick_tc.cu -- the tick kernel with synaptic integration on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM).  SURVEY.md 8(f) row f1.
//
// Integration (Alg. 1 l.10-13) of one core over a tile of NT = 64
// samples is the integer matrix product
//     acc[n][s] = sum_a' Wfold[n][a'] * spike[s][a'],
//     Wfold[n][a'] = conn[n][a'] * w[n][type(a')]
// exact in int32 (|w| <= 127 checked at load, K <= 1024 terms).  M = 128
// neurons per MMA (two halves for 256 neurons), N = 64 samples, K = 32 axons
// per instruction.  Wfold is pre-arranged on the host in the canonical
// K-major core-matrix layout (tc.h).
//
// Persistent, warp-specialised: one CTA per SM walks a contiguous range of
// (core, sample-tile) work items; the roles overlap through mbarriers (NS = 4
// spike stages, up to 4 TMEM accumulator stages), so that the next tiles are
// loaded, expanded and multiplied while the epilogue of this one runs:
//   warps 0-15  epilogue, thread = neuron = TMEM lane (warp % 4 = lane
//               quarter; neuron half and 32-sample half from the warp id):
//               potentials streamed HBM -> shared (cp.async, one tile ahead)
//               -> registers -> HBM, leak / thresholds / reset (a4), routing
//               and output bus (a5, a6)
//   warps 16-19 spike stage: clear the rows read (a1), input injection (a2),
//               bits -> 0/1 bytes in the operand layout
//   warp 20     producer: TMA bulk loads of Wfold (on a core change) and of
//               the tile's scheduler rows and decoded input words
//   warp 21     MMA issuer (one elected thread) + TMEM allocation
// A tick is one launch; the kernel boundary is the tick barrier (a7).
//
// Potential layout: tile-blocked [G][nT][8][Np][8] int16 (tile, 8-sample chunk,
// neuron, sample in chunk): every 16-byte access of a warp is coalesced.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include "internal.h"
#include "ptx.h"
#include "tc.h"

#ifdef RANC_POT_STCS
#define POT_STORE(ptr, v) ptx::st16_cs(ptr, v)
#else
#define POT_STORE(ptr, v) (*reinterpret_cast<uint4*>(ptr) = (v))
#endif

namespace ranc {

namespace cg = cooperative_groups;

namespace {

constexpr int NT = 64;                 // samples per tile (MMA N)
constexpr int NS = 4;                  // spike-stage pipeline depth
constexpr int kExpWarps = 4;
constexpr int kEpiWarps = 16;
// Warp ids (SMSP = warp % 4): 0..15 epilogue (TMEM lane quarter = warp % 4,
// so every SMSP holds four epilogue warps to hide the LIF's dependency
// latencies); 16..19 spike stage; 20 producer; 21 MMA issuer.
constexpr int kFirstEpi = 0;
constexpr int kThreadsTC = 32 * (2 + kExpWarps + kEpiWarps);  // 704
// history-scheduler launches with the compact operand: 8 spike warps in two
// groups of 4 that take alternate work items (their per-item chain --
// position ORs, B operand, operand expansion -- is the longest one; 832
// threads keep 72 registers per thread; config 5 95.7 -> 84 us per tick; the
// folded VMM-1024 launch was 1-2 % slower with them, so it keeps 4)
constexpr int kExpWarpsHist = 8;
constexpr int kThreadsHist = 32 * (2 + kExpWarpsHist + kEpiWarps);  // 832
__host__ __device__ constexpr int tc_threads(bool hist) { return hist ? kThreadsHist : kThreadsTC; }
constexpr int kExpThreads = 32 * kExpWarps;
constexpr int kSub = 16;               // samples per TMEM load / LIF pass of an epilogue warp
static_assert(kExpThreads == 2 * NT, "spike stage maps thread -> (sample, 16-bit half)");

enum Bar { FULL0 = 0, SEMPTY0 = 4, BFULL0 = 8, BEMPTY0 = 12, ACCFULL0 = 16, ACCEMPTY0 = 20, WFULL = 24, WFREE = 25,
           WFULL1 = 26, WFREE1 = 27, NBARS = 28 };

struct TcLayout {
  uint32_t w, runs, lut, tsel, potbuf, cplanes, pmask, stage, b, raw, lines, pull, paoff, hcnt, stage_bytes, total;
};

// WIp: input-line row words (multiple of 4)
// wide: weights beyond int8 are split w = 256*hi + lo (lo the unsigned low
// byte, hi in [-128,127]); the two folded operands double the weight buffer and the
// spike pipeline keeps 2 stages (NS_WIDE) to stay inside 227 KB
constexpr int NS_WIDE = 2;
// multi-tick launch: 3 spike stages (its ticks are a latency chain; the
// freed 20 KB hold the bit-sliced output counters of two items)
constexpr int NS_MULTI = 3;
// neuron-group launch (cores of more than 256 neurons or more than 256
// axons): one spike stage feeds several groups' MMAs, and a B stage holds up
// to 512 axons, so 2 stages
constexpr int NS_GRP = 2;
// neuron groups beyond 512 axons: the group's operand is split into K chunks
// of 512 axons (one 64 KB buffer load each, accumulated in TMEM) and the
// 64 KB spike stage is single (TickParams::grp_ns = 1)
constexpr int kKChunk = 512;
// compact-operand launch: two expanded operand buffers (the next core's is
// expanded while this one's MMAs run) leave room for 2 spike stages
constexpr int NS_COMP = 2;
// pot_items: potential tiles kept on chip (multi-tick launch with up to two
// work items per CTA: one region each)
// cnt_planes: per-thread bit-sliced output-bus counters (multi-tick launch)
constexpr int kCntPlanes = 8;   // counts < 256 between flushes
// wrows: operand rows held in shared memory (Npad, or the group size of a
// neuron-group launch, grp)
__host__ __device__ inline TcLayout tc_layout(int wrows, int Kp, int W, int WIp, int rmax, bool wide, int pot_items = 1,
                                              bool cnt_planes = false, bool multi = false, int grp = 0,
                                              int pull_emax = -1, bool comp = false) {
  // grp: spike stages of a neuron-group launch (0: not grouped); its operand
  // buffer holds one K chunk of at most kKChunk axons.  History launches
  // (pull_emax >= 0) with the compact operand run two spike groups: their
  // runs, type selectors and per-axon masks are per group; history launches
  // without input lines stage no ring rows or input words.
  const bool pull = pull_emax >= 0;
  const uint32_t ng = pull && comp ? 2u : 1u;
  const bool stage_rows = !pull || WIp > 0;
  TcLayout L;
  L.w = 1024;
  uint32_t o = L.w + (uint32_t)wrows * (grp ? (Kp < kKChunk ? Kp : kKChunk) : Kp) * (wide || comp ? 2u : 1u);
  L.runs = o;                                 // int2 [rmax] + int32 [W] of the current core
  o += ((uint32_t)rmax * 8 + (uint32_t)W * 4) * ng;
  o = (o + 15) & ~15u;
  L.lut = o;                                  // u32 [16]: nibble -> four 0/1 bytes
  o += 256 * 8;
  L.tsel = o;                                 // compact operand: u32 [Kp/4] the core's prmt type selectors
  if (comp) o += (uint32_t)Kp * ng;
  o = (o + 127) & ~127u;
  L.potbuf = o;                               // uint4 [NT/8][epilogue threads]: next tile's potentials
  o += (NT / 8) * (32 * 8) * 16 * (uint32_t)pot_items;   // = 4 chunks x 512 epilogue threads per item
  L.cplanes = o;                              // u32 [items][kCntPlanes][512 epilogue threads]
  if (cnt_planes) o += (uint32_t)pot_items * kCntPlanes * 512 * 4;
  o = (o + 15) & ~15u;
  L.pmask = o;                                // history scheduler: u64 [Kp] spike masks per axon (64 samples)
  if (pull) o += (uint32_t)Kp * 8 * ng;
  L.stage = (o + 1023) & ~1023u;
  uint32_t q = 0;
  L.b = q;     q += (uint32_t)NT * Kp;       // spikes as 0/1 bytes, canonical layout
  q = (q + 15) & ~15u;
  L.raw = q;   if (stage_rows) q += (uint32_t)NT * W * 4;    // scheduler rows due now (TMA)
  q = (q + 15) & ~15u;
  L.lines = q; if (stage_rows) q += (uint32_t)NT * (WIp > W ? WIp : W) * 4;  // input line rows or decoded words (TMA)
  q = (q + 15) & ~15u;
  L.paoff = q;                                // history: u16 [emax] destination axon per position (TMA)
  if (pull_emax >= 0) q += (uint32_t)pull_emax * 2;
  q = (q + 15) & ~15u;
  L.hcnt = q;                                 // history: u32 the core's position count (producer)
  if (pull_emax >= 0) q += 16;
  q = (q + 15) & ~15u;
  L.pull = q;                                 // history: u64 [emax] the positions' words of this tile (TMA)
  if (pull_emax >= 0) q += (uint32_t)pull_emax * 8;
  L.stage_bytes = (q + 1023) & ~1023u;
  L.total = L.stage + (grp ? grp : wide ? NS_WIDE : multi ? NS_MULTI : comp ? NS_COMP : NS) * L.stage_bytes;
  return L;
}

// optional per-tile timeline of CTA 0 (debug builds of a run: p.dbg != nullptr)
__device__ __forceinline__ void stamp(const TickParams& p, int k, int slot) {
  if (p.dbg && blockIdx.x == 0 && k < 64) p.dbg[k * 16 + slot] = (unsigned long long)clock64();
}

// 32x32 bit transpose across a warp: lane l holds row l (bit i = entry (l, i));
// returns row `lane` of the transpose (bit l = entry (l, lane)).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int j = 16 >> st;
    const uint32_t M = masks[st];
    const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, x, j);
    x = (lane & j) ? (((o >> j) & M) | (x & ~M)) : ((x & M) | ((o & M) << j));
  }
  return x;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Potential tile layout [chunk q = s/8][neuron n][s%8] (int16): chunk q of
// neuron n is the 16-byte uint4 at index q*Npad + n, so the 32 lanes (= 32
// consecutive neurons) of a warp access 512 contiguous bytes per chunk.
__device__ __forceinline__ uint4* pot_tile(const TickParams& p, int c, int tile, int nT, int n) {
  return reinterpret_cast<uint4*>(p.pot + ((size_t)c * nT + tile) * (size_t)p.Npad * NT) + n;
}

// a4 for NE samples of one neuron (Alg. 1 l.14-24): v = V + acc +
// leak; fire if v >= theta+, negative reset if v < theta-; reset to R / -R
// (ABS) or v - theta (LIN); saturate to pb bits once (G8).  Returns the fired
// mask and the 32 new potentials packed as s16 pairs.  The reset is one IMAD:
// r = v * lin + (fire ? bf : bn).  kSat16 (pb = 16): the saturation and the
// packing of two potentials are one cvt.pack.sat.s16.s32.
// `one` is 1 at run time but opaque to the compiler, so that the "no change"
// move stays a predicated IMAD (FMA pipe) instead of becoming an ALU select.
template <bool kSat16, int NE>
__device__ __forceinline__ uint32_t lif(const uint4 (&cur)[NE / 8], const uint32_t (&acc)[NE], int leak, int pth,
                                        int nth, int linmul, int bf, int bn, int lo, int hi, int one,
                                        uint32_t (&outw)[NE / 2]) {
  uint32_t fired = 0u;
#pragma unroll
  for (int i2 = 0; i2 < NE / 2; ++i2) {
    const uint4 v4 = cur[i2 >> 2];
    const uint32_t w32 = (i2 & 3) == 0 ? v4.x : (i2 & 3) == 1 ? v4.y : (i2 & 3) == 2 ? v4.z : v4.w;
    int nvp[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 2 * i2 + e;
      // the sign-extended half plus the input: one LEA.HI.SX32 (the low half
      // is first moved up with an IMAD on the FMA pipe)
      uint32_t src = w32;
      if (!e) asm("mul.lo.u32 %0, %1, 65536;" : "=r"(src) : "r"(w32));   // IMAD.SHL (FMA pipe)
      const int v = ((int)src >> 16) + ((int)acc[i] + leak);
      // fire / change predicates; the reset value is selected with
      // predicated IMADs (FMA pipe) instead of ALU selects:
      //   r = v*lin + bn; fire: r = v*lin + bf; no change: r = v
      int nv;
      asm("{\n\t.reg .pred pf, pc;\n\t"
          "setp.ge.s32 pf, %2, %3;\n\t"
          "setp.lt.or.s32 pc, %2, %4, pf;\n\t"
          "mad.lo.s32 %0, %2, %5, %7;\n\t"
          "@pf mad.lo.s32 %0, %2, %5, %6;\n\t"
          "@!pc mad.lo.s32 %0, %2, %9, 0;\n\t"
          "@pf add.u32 %1, %1, %8;\n\t}"
          : "=&r"(nv), "+r"(fired)
          : "r"(v), "r"(pth), "r"(nth), "r"(linmul), "r"(bf), "r"(bn), "r"(1u << i), "r"(one));
      if (!kSat16) nv = min(max(nv, lo), hi);
      nvp[e] = nv;
    }
    if (kSat16) {
      uint32_t d;
      asm("cvt.pack.sat.s16.s32 %0, %1, %2;" : "=r"(d) : "r"(nvp[1]), "r"(nvp[0]));
      outw[i2] = d;
    } else {
      outw[i2] = __byte_perm((uint32_t)nvp[0], (uint32_t)nvp[1], 0x5410u);
    }
  }
  return fired;
}

// nticks > 1 (cooperative launch, at most one work item per CTA): all ticks
// of a ranc_run_ticks call in one launch; the grid barrier is the tick
// barrier (a7) and each epilogue thread keeps its potentials in
// registers between ticks (stored once, after the last tick).
// kWm: word-major scheduler rings (compile-time, so each instantiation only
// carries its own layout's code)
// kWide: 16-bit weights split into a u8 low byte and an s8 high byte, two MMAs and two TMEM
// accumulators per tile, acc = acc_lo + 256 * acc_hi in the epilogue
// kGrp: cores of up to 1024 neurons / 512 axons.  The neurons are processed in
// groups of p.grp_rows (256 or 128) rows: per (core, sample tile) work item
// the spike operand is built once and multiplied with each group's Wfold
// (loaded in turn into the one operand buffer), every group filling its own
// accumulator stage and being retired by the epilogue like a work item of
// its own (a sub-item).  Per-tick launches only.
// kPull: the history scheduler (word-major networks, per-tick launches).
// Every routing neuron owns a position in its destination core's list
// (compile.cpp); each tick the epilogue stores the neuron's fired bits of the
// tile's samples at that position in the history slot of the ARRIVAL tick
// t + delay (plain stores, zero or not), and the producer of the destination
// loads the core's contiguous positions of slot t with one bulk copy; the
// spike stage ORs each position's word into its axon's mask and transposes
// the masks into the staged ring-word layout.  No atomics in global memory,
// no clears: position i of slot t was written at tick t - d_i.
template <bool kMulti, bool kDebug, bool kWm, bool kWide, bool kGrp = false, bool kPull = false, bool kComp = false>
__global__ void __launch_bounds__(tc_threads(kPull && kComp), 1) tick_tc_kernel(const TickParams p, const int nticks_arg) {
  static_assert(!kGrp || !kMulti, "neuron groups are a per-tick launch");
  static_assert(!kComp || (!kMulti && !kWide && !kGrp), "the compact operand is a per-tick int8 launch");
  static_assert(!kPull || (!kMulti && kWm && !kGrp), "the history scheduler is a per-tick word-major launch");
  const int nticks = kMulti ? nticks_arg : 1;
  // kDebug: the RANC_DEBUG_TIMELINE instrumentation (a separate instantiation,
  // so that the product kernel issues none of it)
  auto stamp_k = [&](int k, int slot) {
    if (kDebug) stamp(p, k, slot);
  };
  const bool dbg_on = kDebug && p.dbg;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + 8 * NBARS);
  const int Np = p.Npad, Kp = p.Kp, W = p.W, WIp = p.WIp;
  // operand rows per sub-item and sub-items (neuron groups) per work item
  const int GS = kGrp ? p.grp_rows : Np;
  const int nGrp = kGrp ? Np / GS : 1;
  const TcLayout L = tc_layout(GS, Kp, W, WIp, p.rmax, kWide, kMulti ? p.pot_items : 1, kMulti && p.out_planes,
                               kMulti, kGrp ? p.grp_ns : 0, kPull ? p.hist_emax : -1, kComp);
  constexpr int NS = kGrp ? NS_GRP : kWide ? NS_WIDE : kMulti ? NS_MULTI : kComp ? NS_COMP : ranc::NS;   // spike stages (at most)
  const int nsr = kGrp ? p.grp_ns : NS;   // spike stages in use
  const int nK = kGrp ? (Kp + kKChunk - 1) / kKChunk : 1;   // K chunks of a group's operand
  uint8_t* w_s = smem + L.w;
  const int Mh = GS >> 7;
  const int nT = (p.S + NT - 1) / NT;
  const int total = p.G_loc * nT;
  // this CTA's contiguous range of (core, tile) work items: equal shares, or
  // (per-tick launches, p.part) the cost-balanced partition of the previous
  // ticks -- written only by the rebalance kernel, after which the next tick
  // is launched without programmatic dependency (so it is complete here)
  const int lo = (!kMulti && p.part) ? p.part[blockIdx.x] : (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int hi = (!kMulti && p.part) ? p.part[blockIdx.x + 1] : (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const int nwork = hi - lo;
  // Serpentine order (per-tick launches, p.serp): odd ticks walk the CTA's
  // items backwards, so a tick starts on the items whose potentials, ring
  // rows and operands the previous tick touched last and are still in L2.
  // Items of one tick are independent, so the order is invisible.
  // (word-major instantiations only: on the layered nets' sample-major path
  // the reverse walk buys no L2 hits and its branches cost the issue-bound
  // epilogue ~1.5 %, measured)
  const bool rev = !kMulti && kWm && p.serp && (p.t & 1);
  const int first_idx = rev ? hi - 1 : lo;
  auto adv = [&](int& cl_, int& tile_) {   // the next item in walking order
    if (!rev) {
      if (++tile_ == nT) { tile_ = 0; ++cl_; }
    } else if (--tile_ < 0) {
      tile_ = nT - 1;
      --cl_;
    }
  };
  auto next_cl_of = [&](int cl_, int tile_) { return !rev ? (tile_ + 1 == nT ? cl_ + 1 : cl_) : (tile_ == 0 ? cl_ - 1 : cl_); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM columns per accumulator stage (wide: the hi accumulator follows the lo one)
  const uint32_t acc_stride = (uint32_t)Mh * NT * (kWide ? 2u : 1u);
  constexpr int NA = kWide ? 2 : 4;                        // accumulator stages (Np <= 256: 512 columns)
  const uint32_t tcols = acc_stride * NA;
  // a7: the grid barrier orders tick t's ring deposits before tick t+1's
  // reads.  A network without routes has no cross-CTA state (each CTA owns
  // one (core, tile) and its potentials), so its ticks need no barrier and
  // the roles' mbarrier pipelines overlap consecutive ticks.
  auto tick_barrier = [&]() {
    if (kMulti && p.any_route && p.fault != 1) cg::this_grid().sync();
  };
  // pipeline waits: sleeping (issue slots left to the working warps) in the
  // throughput kernel; spinning in the multi-tick kernel, whose ticks are a
  // latency chain (producer -> spike stage -> MMA -> epilogue -> barrier)
  // (measured: spinning stays best in the multi-tick launch even when its
  // ticks overlap, i.e. without routes)
  constexpr bool spin = kMulti;
  auto wait = [&](uint64_t* bar, uint32_t parity) {
    if (spin) ptx::mbar_wait(bar, parity);
    else ptx::mbar_wait_sleep(bar, parity, 2000);
  };

  // role warps
  // spike warps: 4 (8 with the history scheduler), then the producer and MMA warps
  constexpr int kEW = kPull && kComp ? kExpWarpsHist : kExpWarps;
  constexpr int SET = 32 * kEW;   // spike threads
  const int prod_warp = kEpiWarps + kEW, mma_warp = kEpiWarps + kEW + 1;
  if (warp == mma_warp) tc::alloc(tmem_holder, tcols < 32 ? 32 : tcols);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&bars[FULL0 + i], 1);
      ptx::mbar_init(&bars[SEMPTY0 + i], 1);
      ptx::mbar_init(&bars[BFULL0 + i], 1);
      ptx::mbar_init(&bars[BEMPTY0 + i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&bars[ACCFULL0 + i], 1);
      ptx::mbar_init(&bars[ACCEMPTY0 + i], kEpiWarps);
    }
    // (compact operand expanded by the epilogue: one arrival per epilogue warp)
    ptx::mbar_init(&bars[WFULL], 1);
    ptx::mbar_init(&bars[WFREE], 1);
    ptx::mbar_init(&bars[WFULL1], 1);
    ptx::mbar_init(&bars[WFREE1], 1);
    ptx::fence_mbar_init();
  }
  // programmatic dependent launch (per-tick launches): let the next tick's
  // grid be scheduled now, so its CTAs start (launch, TMEM allocation,
  // barrier set-up) as soon as this grid's CTAs leave their SMs; then wait
  // until the previous tick's grid has completed and its writes (potentials,
  // ring deposits, counts) are visible.  Both are no-ops without PDL.
  if (!kMulti) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;
  unsigned long long gt_start = 0;
  if ((dbg_on || p.cta_ns) && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_start));

  if (warp == prod_warp) {
    // ------------------------------------------------------------ producer (TMA)
    // the whole warp walks the work list (convergent waits); lane 0 issues
    int prev_core = -1, jw = -1;
    for (int it = 0; it < nticks; ++it) {
    const int64_t t = p.t + it;
    const int cur = (int)(t & p.rp_mask);
    int cl = first_idx / nT, tile = first_idx - (first_idx / nT) * nT;   // advanced incrementally
    for (int k0 = 0; k0 < nwork; ++k0, adv(cl, tile)) {
      const int k = it * nwork + k0;                 // pipeline index (barrier phases)
      const int c = p.c_lo + cl;
      const int s = k % nsr, u = k / nsr;
      if (lane == 0) stamp_k(k, 0);
      wait(&bars[SEMPTY0 + s], (u & 1) ^ 1);
      if (lane == 0) {
        stamp_k(k, 1);
        uint8_t* st = smem + L.stage + s * L.stage_bytes;
        const int s0 = tile * NT;
        const bool inject = t < p.T_in && p.nruns[c] > 0;
        // decoded inputs: the tile's input words in ring-row layout; else the raw line rows
        const int slot = p.inw ? p.inslot[cl] : -1;
        const uint32_t ring_bytes = (!kPull && p.incoming[c]) ? (uint32_t)NT * W * 4 : 0u;
        const uint32_t line_bytes = !inject ? 0u : (p.inw ? (uint32_t)NT * W * 4 : (uint32_t)NT * WIp * 4);
        // history scheduler: the core's positions (axons, and their words of
        // slot t for this tile); a multiple of 8 positions, 16-byte aligned
        const uint32_t hb0 = kPull ? p.hbase[c] : 0u, hcnt = kPull ? p.hbase[c + 1] - hb0 : 0u;
        if (kPull) *reinterpret_cast<uint32_t*>(st + L.hcnt) = hcnt;   // released by the arrive below
        ptx::mbar_arrive_expect_tx(&bars[FULL0 + s], ring_bytes + line_bytes + hcnt * 10u);
        if (kPull && hcnt) {
          ptx::bulk_g2s(st + L.paoff, p.hax + hb0, hcnt * 2u, &bars[FULL0 + s]);
          ptx::bulk_g2s(st + L.pull, p.hist + (((size_t)cur * nT + tile) * p.hist_P + hb0) * 2, hcnt * 8u,
                        &bars[FULL0 + s]);
        }
        // ring rows and decoded inputs: sample-major [..][Sr][W] is one bulk
        // copy per tile, staged [NT][W]; word-major [..][W][Sr] one copy of
        // the tile's 64 samples per ring word, staged [W][NT]
        const size_t rrow0 = (size_t)cur * p.G_loc + cl, irow0 = (size_t)t * p.n_inslots + slot;
        if (ring_bytes) {
          if (!kWm)
            ptx::bulk_g2s(st + L.raw, p.ring + (rrow0 * p.Sr + s0) * W, ring_bytes, &bars[FULL0 + s]);
          else
            for (int w = 0; w < W; ++w)
              ptx::bulk_g2s(st + L.raw + w * NT * 4, p.ring + (rrow0 * W + w) * p.Sr + s0, NT * 4, &bars[FULL0 + s]);
        }
        if (inject && p.inw && !kWm)
          ptx::bulk_g2s(st + L.lines, p.inw + (irow0 * p.Sr + s0) * W, line_bytes, &bars[FULL0 + s]);
        else if (inject && p.inw)
          for (int w = 0; w < W; ++w)
            ptx::bulk_g2s(st + L.lines + w * NT * 4, p.inw + (irow0 * W + w) * p.Sr + s0, NT * 4, &bars[FULL0 + s]);
        else if (inject)
          ptx::bulk_g2s(st + L.lines, p.lines + ((size_t)t * p.Sr + s0) * WIp, line_bytes, &bars[FULL0 + s]);
      }
      __syncwarp();
      // a new core's operand, once the previous core's MMAs have read the
      // buffer.  Issued AFTER this item's ring rows / gathers, so that their
      // latency overlaps the previous item's MMAs instead of following them
      // (one tile per core at config 5: every item waits here).
      if (!kGrp && !kComp && c != prev_core) {
        ++jw;
        if (jw > 0) wait(&bars[WFREE], (jw - 1) & 1);
        if (lane == 0) {
          const uint32_t wb = (uint32_t)Np * Kp * (kWide ? 2u : 1u);   // wide: [lo | hi]
          ptx::mbar_arrive_expect_tx(&bars[WFULL], wb);
          ptx::bulk_g2s(w_s, p.wfold + (size_t)c * wb, wb, &bars[WFULL]);
        }
        prev_core = c;
        __syncwarp();
      }
      if (kGrp) {
        // the groups' operands in turn (K chunk by K chunk beyond 512 axons),
        // each once the MMAs of the previous one have read the buffer
        // (Wfold per core: nGrp blocks of gb bytes; chunk kc of a block at
        // kc * 512 * GS * parts, [lo | hi] parts of KSc columns each)
        const uint32_t parts = kWide ? 2u : 1u, gb = (uint32_t)GS * Kp * parts;
        for (int g = 0; g < nGrp; ++g)
          for (int kc = 0; kc < nK; ++kc) {
            const uint32_t ksc = (uint32_t)min(kKChunk, Kp - kc * kKChunk);
            const uint32_t wb = (uint32_t)GS * ksc * parts;
            ++jw;
            if (jw > 0) wait(&bars[WFREE], (jw - 1) & 1);
            if (lane == 0) {
              ptx::mbar_arrive_expect_tx(&bars[WFULL], wb);
              ptx::bulk_g2s(w_s, p.wfold + ((size_t)c * nGrp + g) * gb + (size_t)kc * kKChunk * GS * parts, wb,
                            &bars[WFULL]);
            }
            __syncwarp();
          }
      }
    }
    tick_barrier();
    // the next tick's ring rows were written through the generic proxy
    // (other CTAs' atomicOr deposits, this CTA's clears Rp ticks ago) and are
    // read below with cp.async.bulk (async proxy): order the two proxies
    // after the grid barrier (per-tick launches: the kernel boundary does)
    if (kMulti) ptx::fence_proxy_async_global();
    }
  } else if (warp == mma_warp) {
    // ------------------------------------------------------------ MMA issuer
    // convergent warp loop; one elected thread issues the tcgen05 operations
    // history scheduler: the B operand is MN-major (instruction descriptor
    // bit 16; descriptor LBO = 512 between 8-axon groups, SBO = 128 between
    // 16-sample groups, the same 2 KB per 32-axon K step)
    const uint32_t bmn = kPull ? (1u << 16) : 0u;
    const uint32_t id = tc::idesc_i8(128, NT) | bmn;
    // wide weights: w = 256*hi + lo, lo the UNSIGNED low byte, hi signed
    const uint32_t id_lo = kWide ? (tc::idesc_i8(128, NT, false) | bmn) : id;
    const uint32_t lbo_a = (uint32_t)GS * 16, lbo_b = (uint32_t)NT * 16;   // tc.h layout
    int prev_core = -1, jw = -1;
    for (int it = 0; it < nticks; ++it) {
    int cl = first_idx / nT, tile = first_idx - (first_idx / nT) * nT;
    for (int k0 = 0; k0 < nwork; ++k0, adv(cl, tile)) {
      const int k = it * nwork + k0;
      const int c = cl;
      const int s = k % nsr, u = k / nsr;
      if (!kGrp && c != prev_core) {
        ++jw;
        // compact operand: core jw's expanded operand is buffer jw & 1
        if (kComp) wait(&bars[(jw & 1) ? WFULL1 : WFULL], (jw >> 1) & 1);
        else wait(&bars[WFULL], jw & 1);
        prev_core = c;
      }
      wait(&bars[BFULL0 + s], u & 1);
      if (lane == 0) stamp_k(k, 5);
      for (int g = 0; g < nGrp; ++g) {
      const int j = k * nGrp + g;          // sub-item: accumulator ring index
      const int a = j % NA, ua = j / NA;
      wait(&bars[ACCEMPTY0 + a], (ua & 1) ^ 1);
      for (int kc = 0; kc < nK; ++kc) {
      const int ksc = kGrp ? min(kKChunk, Kp - kc * kKChunk) : Kp;   // axons of this operand chunk
      if (kGrp) {   // every group (K chunk) is a new operand
        ++jw;
        wait(&bars[WFULL], jw & 1);
      }
      tc::fence_after();
      if (lane == 0) {
        stamp_k(k, 6);
        const uint8_t* b_s = smem + L.stage + s * L.stage_bytes + L.b;
        const uint8_t* a_s = kComp ? w_s + (jw & 1) * (uint32_t)(GS * Kp) : w_s;
        const uint32_t acc = tmem + a * acc_stride;
        const int kk0 = kc * (kKChunk / 32);   // K step of the spike operand
        for (int hh = 0; hh < Mh; ++hh)
          for (int kk = 0; kk < ksc / 32; ++kk) {
            const uint32_t accum = (kc > 0 || kk > 0) ? 1u : 0u;
            const uint64_t ad = tc::smem_desc(ptx::smem_u32(a_s + hh * 2048 + kk * 2 * lbo_a), lbo_a, 128);
            const uint64_t bd = kPull ? tc::smem_desc(ptx::smem_u32(b_s + (kk0 + kk) * 2048), 512, 128)
                                      : tc::smem_desc(ptx::smem_u32(b_s + (kk0 + kk) * 2 * lbo_b), lbo_b, 128);
            tc::mma_i8(acc + hh * NT, ad, bd, id_lo, accum);
            if (kWide) {
              const uint64_t ah = tc::smem_desc(ptx::smem_u32(w_s + GS * ksc + hh * 2048 + kk * 2 * lbo_a), lbo_a, 128);
              tc::mma_i8(acc + (Mh + hh) * NT, ah, bd, id, accum);
            }
          }
        if (g + 1 == nGrp && kc + 1 == nK) tc::commit(&bars[BEMPTY0 + s]);
        if (kc + 1 == nK) tc::commit(&bars[ACCFULL0 + a]);
        stamp_k(k, 7);
        // the next item (in a multi-tick launch: cyclically, the CTA's first
        // item of the next tick) belongs to another core, or this is the end
        // (neuron groups: every sub-item / K chunk has its own operand)
        const bool last_item = k0 + 1 == nwork;
        const int next_cl = last_item ? first_idx / nT : next_cl_of(cl, tile);
        if (kGrp || (last_item && it + 1 == nticks) || next_cl != cl) tc::commit(&bars[(kComp && (jw & 1)) ? WFREE1 : WFREE]);
      }
      __syncwarp();
      }
      }
    }
    tick_barrier();
    }
  } else if (warp >= kEpiWarps && warp < kEpiWarps + kEW) {
    // ------------------------------------------------------------ spike stage
    // history launches: two independent spike groups of 4 warps take
    // alternate work items (their own spike stages, per-axon masks, type
    // selectors and named barrier), so that two items' chains overlap
    constexpr int kSG = kPull && kComp ? 2 : 1;             // spike groups
    constexpr int GT = 128;                                 // threads per group
    const int gi = (warp - kEpiWarps) >> 2;                 // this warp's group
    const int et = 32 * ((warp - kEpiWarps) & 3) + lane;    // thread within the group
    const int gbar = 2 + gi;                                // the group's named barrier
    int runs_core = -1;
    const uint32_t runs_off = (uint32_t)gi * ((uint32_t)p.rmax * 8 + (uint32_t)W * 4);
    uint32_t* const gmsk = reinterpret_cast<uint32_t*>(smem + L.pmask) + (size_t)gi * 2 * Kp;
    // nibble -> four 0/1 bytes; a 16-entry u32 table spans 16 distinct banks,
    // so the lookups never conflict
    uint32_t* lut = reinterpret_cast<uint32_t*>(smem + L.lut);
    if (gi == 0)
      for (int b = et; b < 16; b += GT) lut[b] = tc::nib2bytes((uint32_t)b);
    if (kPull)   // the per-axon masks start (and stay between items) zero
      for (int i = et; i < 2 * Kp; i += GT) gmsk[i] = 0u;
    named_sync(4, SET);
    // kComp: the spike warps expand each core's compact operand (crossbar
    // bits, type weights, axon types) into Wfold[n][a'] = conn * w[n][type(a')]
    // in the canonical layout, into operand buffer j & 1 for the
    // CTA's j-th core, one core ahead of the MMAs; the compact operand of the
    // core after that is prefetched into registers meanwhile (L2 evict_last:
    // every core's operand is read again next tick).
    constexpr int kNH = 2;   // neurons per thread (Np <= 256)
    uint32_t cx[kNH][8], cw[kNH], cts = 0u;
#pragma unroll
    for (int h = 0; h < kNH; ++h) cw[h] = 0u;
    const uint64_t pol_keep = kComp ? ptx::policy_evict_last() : 0ull;
    int ncores = 0, jcore = 0;
    const int core0 = first_idx / nT, core_dir = rev ? -1 : 1;
    if (kComp && nwork > 0) ncores = abs((rev ? lo : hi - 1) / nT - core0) + 1;
    auto comp_load = [&](int j) {   // registers <- the compact operand of the CTA's j-th core
      if (j >= ncores) return;
      const int cg = p.c_lo + core0 + core_dir * j;
#pragma unroll
      for (int h = 0; h < kNH; ++h) {
        const int nn = et + GT * h;
#pragma unroll
        for (int w = 0; w < 8; ++w)
          cx[h][w] = (nn < Np && w < W) ? ptx::ldg_hint(p.xbits + ((size_t)cg * W + w) * Np + nn, pol_keep) : 0u;
        cw[h] = nn < Np ? ptx::ldg_hint(p.wq + (size_t)cg * Np + nn, pol_keep) : 0u;
      }
      if (et < (Kp >> 2)) cts = ptx::ldg_hint(p.tsel + (size_t)cg * (Kp >> 2) + et, pol_keep);
    };
    auto comp_expand = [&](int j) {   // operand buffer j & 1 <- the j-th core's expanded operand
      const int b = j & 1;
      if (j >= 2) wait(&bars[b ? WFREE1 : WFREE], ((j >> 1) - 1) & 1);   // core j - 2's MMAs are done
      if (et == 0 && j > 0) stamp_k(j - 1, 12);   // (timeline: slots 12 / 13 = expansion start / end)
      uint32_t* ts = reinterpret_cast<uint32_t*>(smem + L.tsel + (uint32_t)gi * Kp);
      if (et < (Kp >> 2)) ts[et] = cts;
      named_sync(gbar, GT);
      uint4* const abuf = reinterpret_cast<uint4*>(w_s + b * (uint32_t)(Np * Kp));
#pragma unroll
      for (int h = 0; h < kNH; ++h) {
        const int nn = et + GT * h;
        if (nn >= Np) break;   // Np = 128 or 256: warp-uniform
        const uint32_t wv = cw[h];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (w >= W) break;
          // chunk kc = 2w + (m >> 2) (16 axons) of row nn sits at (kc * Np + nn) * 16
          // bytes (tc.h); byte j of word m: axon 32w + 4m + j, its weight byte
          // selected by type (selector nibble j = type) unless the synapse is
          // absent (nibble bit 2 set: a byte of the zero operand) -- one shift,
          // one lop3 and one prmt per four synapses
          const uint32_t x = cx[h][w];
          const uint4 s0 = reinterpret_cast<const uint4*>(ts)[2 * w];
          const uint4 s1 = reinterpret_cast<const uint4*>(ts)[2 * w + 1];
          const uint32_t sel[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
          uint32_t o[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const uint32_t z = m < 2 ? x << (2 - m) : m < 4 ? x >> (m - 2) : x >> (14 + (m & 3));
            o[m] = ptx::prmt(wv, 0u, (z & 0x4444u) | sel[m]);
          }
          abuf[(2 * w) * Np + nn] = make_uint4(o[0], o[1], o[2], o[3]);
          abuf[(2 * w + 1) * Np + nn] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
      ptx::fence_proxy_async_smem();   // generic writes -> the tensor core's (async proxy) reads
      named_sync(gbar, GT);
      if (et == 0) {
        ptx::mbar_arrive(&bars[b ? WFULL1 : WFULL]);
        if (j > 0) stamp_k(j - 1, 13);
      }
    };
    // one group: core j + 1 is expanded after the last item of core j (one
    // core ahead).  Two groups: the group of a core's first item expands
    // it after that item's B operand (the other group's item overlaps), the
    // compact operand of the group's next core prefetched meanwhile.
    // (walking order: a core starts at tile 0, or at tile nT - 1 reversed)
    int cx_j = -1;   // the core whose compact operand is in cx
    auto core_start = [&](int k0_, int tile_) { return k0_ == 0 || (rev ? tile_ == nT - 1 : tile_ == 0); };
    if (kComp && ncores > 0) {
      if (kSG == 1) {
        comp_load(0);
        comp_expand(0);
        comp_load(1);
      } else {
        int ccl = first_idx / nT, ctile = first_idx - (first_idx / nT) * nT;
        for (int i = 0; i < gi; ++i) adv(ccl, ctile);
        if (gi < nwork && core_start(gi, ctile)) {
          cx_j = abs(ccl - core0);
          comp_load(cx_j);
        }
      }
    }
    for (int it = 0; it < nticks; ++it) {
    const int64_t t = p.t + it;
    const int cur = (int)(t & p.rp_mask);
    int cl = first_idx / nT, tile = first_idx - (first_idx / nT) * nT;
    for (int i = 0; i < gi; ++i) adv(cl, tile);
    for (int k0 = gi; k0 < nwork; k0 += kSG) {
      const int k = it * nwork + k0;
      const int c = p.c_lo + cl;
      const int s = k % nsr, u = k / nsr;
      const int s0 = tile * NT, ns = min(NT, p.S - s0);
      uint8_t* st = smem + L.stage + s * L.stage_bytes;
      uint32_t* raw = reinterpret_cast<uint32_t*>(st + L.raw);
      const uint32_t* lines = reinterpret_cast<const uint32_t*>(st + L.lines);
      // a1: the scheduler rows due now were staged by the producer (TMA);
      // clear them in global memory (free again for spikes due at t + Rp)
      wait(&bars[FULL0 + s], u & 1);
      if (et == 0) stamp_k(k, 2);
      // staged rows: raw[sm * W + w] (sample-major) or raw[w * NT + sm]
      // (word-major) = ring word w of sample s0 + sm
      constexpr bool wm = kWm;
      if (kPull) {
        // a1 (history scheduler): the spikes due now on axon a' are the OR of
        // the words its sources stored for tick t (idempotent OR, P:158,
        // G11), collected in the per-axon 64-sample masks msk (zero between
        // items: the B emission below clears what it reads).  The B operand
        // is MN-major (per axon, 64 contiguous sample bytes), so the masks
        // become operand bytes without a bit transpose.
        const uint2* gat = reinterpret_cast<const uint2*>(st + L.pull);
        const uint16_t* hax = reinterpret_cast<const uint16_t*>(st + L.paoff);
        uint32_t* msk = gmsk;
        const int hcnt = (int)*reinterpret_cast<const uint32_t*>(st + L.hcnt);
        for (int e = et; e < hcnt; e += GT) {
          const uint2 v = gat[e];
          if (v.x | v.y) {
            const int ap = hax[e];
            if (v.x) atomicOr(msk + 2 * ap, v.x);
            if (v.y) atomicOr(msk + 2 * ap + 1, v.y);
          }
        }
        // a2: external inputs as ring words raw[w * NT + sample] (decoded at
        // load, or gathered from the line runs), bit-transposed into msk
        const bool inj = t < p.T_in && p.nruns[c] > 0;
        if (inj) {
          if (p.inw) {
            for (int i = et; i < NT * W; i += GT) raw[i] = lines[i];
          } else {
            int2* runs = reinterpret_cast<int2*>(smem + L.runs + runs_off);
            int32_t* wr = reinterpret_cast<int32_t*>(smem + L.runs + runs_off + (uint32_t)p.rmax * 8);
            if (c != runs_core) {
              named_sync(gbar, GT);
              for (int i = et; i < p.nruns[c]; i += GT) runs[i] = p.runs[(size_t)c * p.rmax + i];
              for (int i = et; i < W; i += GT) wr[i] = p.word_runs[(size_t)c * W + i];
              named_sync(gbar, GT);
              runs_core = c;
            }
            for (int i = et; i < NT * W; i += GT) {
              const int w = i / NT, sm = i % NT;
              uint32_t acc = 0u;
              const int32_t fr = wr[w];
              const uint32_t* lr = lines + sm * WIp;
              for (int r = fr & 0xFFFF; r < (fr & 0xFFFF) + (fr >> 16); ++r) {
                const int2 rn = runs[r];
                const int ap = rn.x & 0xFFFF, len = rn.x >> 16, ln = rn.y;
                const int lw = ln >> 5, lb = ln & 31;
                uint32_t x = lr[lw] >> lb;
                if (lb + len > 32) x |= lr[lw + 1] << (32 - lb);
                if (len < 32) x &= (1u << len) - 1u;
                const int off = ap - 32 * w;
                acc |= off >= 0 ? (x << off) : (x >> (-off));
              }
              raw[i] = acc;
            }
          }
          named_sync(gbar, GT);
          for (int b = et >> 5; b < 2 * W; b += 4) {
            const int w = b >> 1, hf = b & 1;
            const uint32_t x = transpose32(raw[w * NT + 32 * hf + lane], lane);
            if (x) atomicOr(msk + 2 * (32 * w + lane) + hf, x);
          }
        }
        named_sync(gbar, GT);
        if (p.spkin)   // RANC_TRACE_STATE_DIGEST: the axon spikes integrated this tick
          for (int b = et >> 5; b < 2 * W; b += 4) {
            const int w = b >> 1, hf = b & 1, sm = 32 * hf + lane;
            const uint32_t y = transpose32(msk[2 * (32 * w + lane) + hf], lane);
            if (sm < ns) p.spkin[((size_t)(s0 + sm) * p.G_loc + cl) * W + w] = y;
          }
        wait(&bars[BEMPTY0 + s], (u & 1) ^ 1);
        if (et == 0) stamp_k(k, 3);
        // MN-major B: axon a', samples 16g..16g+15 at (a'/8)*512 + g*128 + (a'%8)*16
        // (tcgen05 MN-major core matrices: LBO = 512 between 8-axon groups,
        // SBO = 128 between 16-sample groups); samples >= ns get no spikes
        uint8_t* b_s = st + L.b;
        const uint64_t keep = ns >= 64 ? ~0ull : ((1ull << ns) - 1ull);
        for (int ap = et; ap < Kp; ap += GT) {
          uint2* mp = reinterpret_cast<uint2*>(msk) + ap;
          const uint2 mv = *mp;
          *mp = make_uint2(0u, 0u);
          const uint64_t m = (((uint64_t)mv.y << 32) | mv.x) & keep;
          uint8_t* bd = b_s + (ap >> 3) * 512 + (ap & 7) * 16;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t h16 = (uint32_t)(m >> (16 * g));
            *reinterpret_cast<uint4*>(bd + g * 128) =
                make_uint4(lut[h16 & 15u], lut[(h16 >> 4) & 15u], lut[(h16 >> 8) & 15u], lut[(h16 >> 12) & 15u]);
          }
        }
      } else if (p.incoming[c]) {
        // only the words that hold spikes need clearing
        if (!wm) {
          uint32_t* row = p.ring + (((size_t)cur * p.G_loc + cl) * p.Sr + s0) * W;
          for (int i = et; i < ns * W; i += kExpThreads)
            if (raw[i]) row[i] = 0u;
        } else {
          uint32_t* row = p.ring + ((size_t)cur * p.G_loc + cl) * W * p.Sr + s0;
          for (int i = et; i < NT * W; i += kExpThreads) {
            const int w = i / NT, sm = i % NT;
            if (sm < ns && raw[i]) row[(size_t)w * p.Sr + sm] = 0u;
          }
        }
      } else {
        // no neuron routes here: the ring stays zero and was not loaded
        for (int i = et; i < NT * W; i += kExpThreads) raw[i] = 0u;
      }
      if (et == 0 && !kComp) stamp_k(k, 12);
      if (!kPull) {
      // a2: external inputs.  Thread <-> (sample, ring word): OR in the line
      // runs overlapping that word (no atomics: every word has one owner)
      if (t < p.T_in && p.nruns[c] > 0 && p.inw) {
        // decoded input words (input decode done once at load, Alg. 1 l.1)
        // same layout as the staged ring rows; rows of samples >= ns are never read
        for (int i = et; i < NT * W; i += kExpThreads) raw[i] |= lines[i];
      } else if (t < p.T_in && p.nruns[c] > 0) {
        // the core's input runs live in shared memory while its tiles are processed
        int2* runs = reinterpret_cast<int2*>(smem + L.runs);
        int32_t* wr = reinterpret_cast<int32_t*>(smem + L.runs + (uint32_t)p.rmax * 8);
        if (c != runs_core) {
          named_sync(2, kExpThreads);
          for (int i = et; i < p.nruns[c]; i += kExpThreads) runs[i] = p.runs[(size_t)c * p.rmax + i];
          for (int i = et; i < W; i += kExpThreads) wr[i] = p.word_runs[(size_t)c * W + i];
          named_sync(2, kExpThreads);
          runs_core = c;
        }
        constexpr int B = 2;   // independent items in flight per thread
        for (int base = et; base < NT * W; base += B * kExpThreads) {
          uint32_t accs[B];
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const int i = base + b * kExpThreads;
            accs[b] = 0u;
            const int w = wm ? i / NT : i % W, sm = wm ? i % NT : i / W;
            if (i >= NT * W || sm >= ns) continue;
            const int32_t fr = wr[w];
            const int r0 = fr & 0xFFFF, nrw = fr >> 16;
            const uint32_t* lr = lines + sm * WIp;
            for (int r = r0; r < r0 + nrw; ++r) {
              const int2 rn = runs[r];
              const int ap = rn.x & 0xFFFF, len = rn.x >> 16, ln = rn.y;
              const int lw = ln >> 5, lb = ln & 31;
              uint32_t x = lr[lw] >> lb;
              if (lb + len > 32) x |= lr[lw + 1] << (32 - lb);
              if (len < 32) x &= (1u << len) - 1u;
              const int off = ap - 32 * w;   // bit position of the run inside word w
              accs[b] |= off >= 0 ? (x << off) : (x >> (-off));
            }
          }
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const int i = base + b * kExpThreads;
            if (i < NT * W && accs[b]) raw[i] |= accs[b];
          }
        }
      }
      if (p.spkin)   // RANC_TRACE_STATE_DIGEST: the axon spikes integrated this tick
        for (int i = et; i < NT * W; i += kExpThreads) {
          const int w = wm ? i / NT : i % W, sm = wm ? i % NT : i / W;
          if (sm < ns) p.spkin[((size_t)(s0 + sm) * p.G_loc + cl) * W + w] = raw[i];
        }
      if (et == 0 && !kComp) stamp_k(k, 13);
      named_sync(2, kExpThreads);
      if (et == 0) stamp_k(k, 14);
      // bits -> 0/1 bytes, canonical K-major operand (rows = samples);
      // samples >= ns of a tail tile get no spikes.  Lanes take consecutive
      // samples so each 8-lane phase of the 16-byte stores fills one core
      // matrix (bank-conflict free).
      wait(&bars[BEMPTY0 + s], (u & 1) ^ 1);
      if (et == 0) stamp_k(k, 3);
      uint8_t* b_s = st + L.b;
      {
        // thread <-> (sample sm, half hf): the 16-bit halves hf of the
        // sample's W ring words become K chunks 2w+hf; lanes take consecutive
        // samples so every 8-lane phase of the 16-byte stores fills one core
        // matrix (bank-conflict free); bytes via the nibble table
        const int sm = et % NT, hf = et / NT;   // kExpThreads == 2 * NT
        // word-major staging: lanes read consecutive words (conflict free);
        // K chunk 2w+hf of sample sm sits w * 2*NT*16 bytes after chunk hf
        const uint32_t* rcol = raw + sm;
        uint8_t* bdst = b_s + tc::operand_offset(sm, hf * 16, NT);
        const uint32_t sh = hf * 16;
        auto emit = [&](int w, uint32_t wv) {
          const uint32_t bits = (wv >> sh) & 0xFFFFu;
          *reinterpret_cast<uint4*>(bdst + w * (2 * NT * 16)) =
              make_uint4(lut[bits & 15u], lut[(bits >> 4) & 15u], lut[(bits >> 8) & 15u], lut[bits >> 12]);
        };
        if (sm >= ns) {   // tail samples of a ragged tile get no spikes
          for (int w = 0; w < W; ++w) *reinterpret_cast<uint4*>(bdst + w * (2 * NT * 16)) = make_uint4(0u, 0u, 0u, 0u);
        } else if (!wm && (W & 3) == 0) {
          // sample-major: 16-byte row loads, lanes 32 B apart (<= 2-way conflicts)
          const uint32_t* rrow = raw + sm * W;
#pragma unroll 1
          for (int w4 = 0; w4 < W; w4 += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(rrow + w4);
            emit(w4 + 0, v.x);
            emit(w4 + 1, v.y);
            emit(w4 + 2, v.z);
            emit(w4 + 3, v.w);
          }
        } else if (!wm) {
#pragma unroll 1
          for (int w = 0; w < W; ++w) emit(w, raw[sm * W + w]);
        } else if (W == 8) {   // A = 256 (the paper's core): fully unrolled
#pragma unroll
          for (int w = 0; w < 8; ++w) emit(w, rcol[w * NT]);
        } else {
#pragma unroll 4
          for (int w = 0; w < W; ++w) emit(w, rcol[w * NT]);
        }
      }
      }   // !kPull
      if (et == 0) stamp_k(k, 15);
      ptx::fence_proxy_async_smem();
      named_sync(gbar, GT);
      if (et == 0) {
        stamp_k(k, 4);
        ptx::mbar_arrive(&bars[BFULL0 + s]);
        ptx::mbar_arrive(&bars[SEMPTY0 + s]);   // raw/lines of this stage are consumed
      }
      if (kComp && kSG == 1 && k0 + 1 < nwork && next_cl_of(cl, tile) != cl) {   // the next item starts a new core
        comp_expand(++jcore);
        comp_load(jcore + 1);
      }
      // the group's next item
      int ncl = cl, ntile = tile;
      for (int i = 0; i < kSG; ++i) adv(ncl, ntile);
      if (kComp && kSG > 1 && core_start(k0, tile)) {   // this item starts its core: expand it
        const int j = abs(cl - core0);
        if (cx_j != j) comp_load(j);
        comp_expand(j);
        cx_j = -1;
        if (k0 + kSG < nwork && core_start(k0 + kSG, ntile)) {
          cx_j = abs(ncl - core0);
          comp_load(cx_j);
        }
      }
      cl = ncl;
      tile = ntile;
    }
    tick_barrier();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // warp ew: TMEM lane quarter q = ew % 4 (thread = neuron n), neuron half
    // h, sample half jj of the tile (32 samples, two LIF passes of kSub)
    const int ew = warp - kFirstEpi;
    const int q = warp & 3;
    const int h = (ew >> 2) & 1, jj = ew >> 3;
    // neuron of this thread in group g: n0 + g * GS (one group unless kGrp)
    const int n0 = h * 128 + q * 32 + lane;
    int n = n0;
    const bool active = h < Mh;
    bool valid = active && n < p.N;
    int prev_core = -1;   // key of the parameters in registers: core (* nGrp + group)
    int leak = 0, pth = 0, nth = 0, rst = 0, init = 0, bf = 0, bn = 0, linmul = 0;
    uint32_t kind = RK_NONE, cls = 0, axbit = 0, out_lanes = 0, out_peers = 0;
    bool route_here = false, exporting = false, block_route = false, block_identity = false, has_output = false;
    bool out_scatter = false;
    size_t ring_off = 0, warp_ring_off = 0;
    // Potentials stream HBM -> shared memory with cp.async one tile ahead:
    // pbuf[c * PB] holds 16-byte chunk c (8 samples) of this thread's 32
    // samples.  The chunks of pass sb of the next tile are requested right
    // after the same pass of the current tile has read them out, so every
    // load has about a tile of time to land; one commit group per pass,
    // waited with cp.async.wait_group 1.
    static_assert(NT == 64 && kSub == 16, "two 32-sample halves, two passes each");
    constexpr int kPass = 32 / kSub, kCh = kSub / 8;   // passes per half, chunks per pass
    uint4* pbuf = reinterpret_cast<uint4*>(smem + L.potbuf) + (threadIdx.x - 32 * kFirstEpi);
    constexpr int PB = 32 * kEpiWarps;   // uint4 stride between chunks in potbuf
    constexpr int kItem = kPass * kCh * PB;   // uint4 per item region (multi-tick launch): 32 KB
    // multi-tick launch: output-bus counts of this thread's 32 samples, bit-
    // sliced (plane b = bit b of every sample's count), flushed every 255
    // ticks and after the last one -- one add per (sample, neuron) per flush
    // instead of one per spike
    const bool planes = kMulti && p.out_planes;
    uint32_t* const cpl = reinterpret_cast<uint32_t*>(smem + L.cplanes) + (threadIdx.x - 32 * kFirstEpi);
    constexpr int kPl = kCntPlanes * 512;   // u32 per item
    if (planes)
      for (int i = 0; i < nwork * kCntPlanes; ++i) cpl[i * 512] = 0u;
    const bool load = active && !p.fresh;
    const bool sat16 = p.pot_lo == -32768 && p.pot_hi == 32767;
    const int one = 1 + (p.N >> 30);   // N <= 1024: 1 (see lif)
    uint4 initv = make_uint4(0u, 0u, 0u, 0u);
    // work item idx = cl * nT + tile, advanced incrementally (no divisions);
    // its potential tile is pot + idx * tile_stride (pot_tile); this warp's
    // chunks start at chunk 4*jj
    int cl = first_idx / nT, tile = first_idx - (first_idx / nT) * nT;
    const size_t tile_stride = (size_t)Np * NT / 8;   // uint4 per potential tile
    const ptrdiff_t dstep = rev ? -(ptrdiff_t)tile_stride : (ptrdiff_t)tile_stride;   // to the next item's tile
    uint4* dst = pot_tile(p, cl, tile, nT, n) + (size_t)(4 * jj) * Np;
    if (load && nwork > 0) {
#pragma unroll
      for (int sb = 0; sb < kPass; ++sb) {
#pragma unroll
        for (int i = 0; i < kCh; ++i)
          ptx::cp_async16(pbuf + (kCh * sb + i) * PB, dst + (size_t)(kCh * sb + i) * Np);
        ptx::cp_async_commit();
      }
    }
    long long dbg_wait = 0;
    const long long dbg_t0 = dbg_on ? clock64() : 0;
    const int cl0 = cl, tile0 = tile;
    // neuron parameters of the next work item's core (prefetched one item ahead)
    // (kept as the raw 8 bytes until use: unpacked right after the load, a
    // short4 made every prefetch wait for its own load -- 13 % of the stall
    // samples at config 5)
    uint2 nprm = make_uint2(0u, 0u);
    uint2 nrt = make_uint2(0u, 0u);
    int nini = 0;
    uint32_t nhp = 0u, hpos = 0u;   // history scheduler: this neuron's position
    if (!kMulti && active && nwork > 0) {
      const size_t nc = (size_t)(p.c_lo + cl0) * Np + n;
      nprm = *reinterpret_cast<const uint2*>(p.prm + nc);
      nrt = p.route[nc];
      nini = p.init[nc];
      if (kPull) nhp = p.hpos[nc];
    }
    // this thread's TMEM lane and column offset (the stage adds a * acc_stride)
    const uint32_t tmem_lane_base = tmem + ((uint32_t)(q * 32) << 16) + h * NT + jj * 32;
    // chunk c of this thread's 32 samples sits c * Np * 16 bytes after chunk 0
    const uint32_t chunk_bytes = (uint32_t)Np * 16u;
    uint4* const dst0 = dst;
    size_t ring_base = 0, warp_ring_base = 0;   // ring word offsets without the slot term
    int rdelay = 0, warp_rdelay = 0;
    // ring [Rp][G_loc][Sr][W] (sample stride W) or word-major [Rp][G_loc][W][Sr]
    // (sample stride 1: a ring word's samples are contiguous)
    const size_t slot_stride = (size_t)p.G_loc * p.Sr * W;
    constexpr bool wm = kWm;
    const uint32_t ss = wm ? 1u : (uint32_t)W;
    for (int it = 0; it < nticks; ++it) {
    const int64_t t = p.t + it;
    const bool first = it == 0, last = it + 1 == nticks;
    cl = cl0;
    tile = tile0;
    dst = dst0;
    for (int k0 = 0; k0 < nwork; ++k0, dst += dstep) {
      const int k = it * nwork + k0;
      const int s0 = tile * NT, ns = min(NT, p.S - s0);
      const int ncl = (k0 + 1 == nwork) ? cl0 : next_cl_of(cl, tile);   // next item's core
      for (int g = 0; g < nGrp; ++g) {
      const int j = k * nGrp + g;   // sub-item (neuron group g of item k): accumulator ring index
      const int c = p.c_lo + cl;
      const int key = kGrp ? c * nGrp + g : c;
      const int a = j % NA, ua = j / NA;
      n = n0 + g * GS;
      valid = active && n < p.N;
      uint4* const dsub = dst + g * GS;   // this group's rows of the potential tile
      const bool pf = load && (g + 1 < nGrp || k0 + 1 < nwork);
      const uint4* nsrc = g + 1 < nGrp ? dsub + GS : dst + dstep;
      const long long tw0 = dbg_on ? clock64() : 0;
      // a new core's neuron parameters were requested a whole work item
      // ahead (one tile per core at config 5: the loads would otherwise stall
      // the epilogue at every item); prefetch the next item's now
      // (the multi-tick launch, at most two items per CTA, loads them in place)
      uint2 prm = nprm;
      uint2 rt = nrt;
      int ini = nini;
      const uint32_t hp = nhp;
      if (kMulti && active && key != prev_core) {
        const size_t nc = (size_t)c * Np + n;
        prm = *reinterpret_cast<const uint2*>(p.prm + nc);
        rt = p.route[nc];
        ini = p.init[nc];
      }
      if (!kMulti && active) {
        const int nkc = g + 1 < nGrp ? cl : ncl;            // next sub-item: core, neuron
        const int nkn = g + 1 < nGrp ? n + GS : n0;
        if (nkc != cl || nkn != n) {
          const size_t nc = (size_t)(p.c_lo + nkc) * Np + nkn;
          nprm = *reinterpret_cast<const uint2*>(p.prm + nc);
          nrt = p.route[nc];
          nini = p.init[nc];
          if (kPull) nhp = p.hpos[nc];
        }
      }
      // one warp per lane quarter polls the accumulator barrier; the other
      // three wait on the quarter's named barrier (no issue slots spent)
      // back-off polling (measured best against the suspend-hint wait, a plain
      // spin and a per-quarter named barrier)
      if (spin) ptx::mbar_wait(&bars[ACCFULL0 + a], ua & 1);
      else if (kComp) ptx::mbar_wait_sleep(&bars[ACCFULL0 + a], ua & 1, 1000);   // (issue-bound compact launches: -1 %)
      else ptx::mbar_wait_backoff(&bars[ACCFULL0 + a], ua & 1, 128);
      if (dbg_on && blockIdx.x == 0) dbg_wait += clock64() - tw0;
      if (lane == 0 && ew == 0) stamp_k(k, 8);
      tc::fence_after();
      if (active) {
        if (key != prev_core) {
          leak = (int)(int16_t)(prm.x & 0xFFFFu); pth = (int)prm.x >> 16;   // short4 {leak, th+, th-, R}
          nth = (int)(int16_t)(prm.y & 0xFFFFu); rst = (int)prm.y >> 16;
          init = ini;
          hpos = hp;
          if (p.fresh && first) {
            // first tick after a reset: the pass inputs are the initial
            // potentials; pbuf is not refilled while this core's tiles run
            // (the new potentials go to HBM; a multi-tick launch fills each
            // item's region below and keeps its potentials there)
            const uint32_t ii = ((uint32_t)init & 0xFFFFu) * 0x10001u;
            initv = make_uint4(ii, ii, ii, ii);
            if (!kMulti) {
#pragma unroll
              for (int i = 0; i < kPass * kCh; ++i) pbuf[i * PB] = initv;
            }
          }
          kind = valid ? route_kind(rt.x) : RK_NONE;
          const bool lin = route_lin(rt.x);
          // nv = fire ? v*linmul + bf : neg ? v*linmul + bn : v
          linmul = lin ? 1 : 0;
          bf = lin ? -pth : rst;
          bn = lin ? -nth : -rst;
          cls = rt.y;
          const uint32_t ax = route_axon(rt.x);
          axbit = 1u << (ax & 31);
          rdelay = (int)route_delay(rt.x);
          // a route to a core of another rank is delivered by the exchange step
          const uint32_t dloc = rt.y - (uint32_t)p.c_lo;
          route_here = kind == RK_ROUTE && dloc < (uint32_t)p.G_loc;
          exporting = p.fired && p.exports[c];
          if (!kPull) {   // ring deposits (the history scheduler stores at positions instead)
            ring_base = wm ? ((size_t)dloc * W + (ax >> 5)) * p.Sr : (size_t)dloc * p.Sr * W + (ax >> 5);
            const uint32_t wf = p.wflags ? p.wflags[(size_t)c * (Np >> 5) + (n >> 5)] : 0u;
            block_route = wf & 1u;
            block_identity = (wf & 3u) == 3u;
            const uint32_t rmask = __ballot_sync(0xFFFFFFFFu, route_here);
            // block routes: all routing lanes share the destination word and delay
            warp_ring_base = rmask ? __shfl_sync(0xFFFFFFFFu, ring_base, __ffs(rmask) - 1) : 0;
            warp_rdelay = rmask ? __shfl_sync(0xFFFFFFFFu, rdelay, __ffs(rmask) - 1) : 0;
            if (!kMulti) {   // one tick: the slots are fixed for the launch
              ring_off = ring_base + (size_t)((p.t + rdelay) & p.rp_mask) * slot_stride;
              warp_ring_off = warp_ring_base + (size_t)((p.t + warp_rdelay) & p.rp_mask) * slot_stride;
            }
          }
          out_lanes = __ballot_sync(0xFFFFFFFFu, kind == RK_OUTPUT);
          has_output = out_lanes != 0u;
          out_peers = 0u;
          out_scatter = false;
          if (has_output) {   // (warp-uniform)
            // lanes of the same output class (classes are < C, never ~0u)
            out_peers = __match_any_sync(0xFFFFFFFFu, kind == RK_OUTPUT ? cls : 0xFFFFFFFFu);
            // more than 8 class groups: per-lane adds (see the output bus below)
            out_scatter = __popc(__ballot_sync(0xFFFFFFFFu, kind == RK_OUTPUT && __ffs(out_peers) - 1 == lane)) > 8;
          }
          prev_core = key;
        }
        // this item's potential region: the multi-tick launch keeps one per
        // item (pb) and prefetches the next item's into its own (pbn)
        uint4* const pb = kMulti ? pbuf + k0 * kItem : pbuf;
        uint4* const pbn = kMulti ? pb + kItem : pbuf;
        if (kMulti && p.fresh && first) {
#pragma unroll
          for (int i = 0; i < kPass * kCh; ++i) pb[i * PB] = initv;
        }
        if (kMulti) {   // ring slot of tick t + delay
          ring_off = ring_base + (size_t)((t + rdelay) & p.rp_mask) * slot_stride;
          warp_ring_off = warp_ring_base + (size_t)((t + warp_rdelay) & p.rp_mask) * slot_stride;
        }
        const uint32_t acc_addr = tmem_lane_base + a * acc_stride;
        uint32_t fired = 0u;
#pragma unroll
        for (int sb = 0; sb < kPass; ++sb) {
          uint32_t acc[kSub];
          tc::ld16(acc_addr + sb * kSub, acc);
          if (kWide) {   // acc = lo + 256 * hi (exact in int32: |acc| < 2^26 for A <= 1024)
            uint32_t hi[kSub];
            tc::ld16(acc_addr + Mh * NT + sb * kSub, hi);
            tc::wait_ld();
#pragma unroll
            for (int i = 0; i < kSub; ++i) acc[i] += hi[i] << 8;
          }
          // this pass's potentials are in pbuf: prefetched a tile ago
          // (cp.async), kept from the previous tick (multi-tick launch), or
          // the initial potentials (first tick after a reset, filled below)
          if (first && load) ptx::cp_async_wait<1>();   // this pass's group has landed
          uint4 cur[kCh];
#pragma unroll
          for (int i = 0; i < kCh; ++i) cur[i] = pb[(kCh * sb + i) * PB];
          if (first && load) {
            // request the same chunks of the next tile into the slots just read
            if (pf) {
              const char* nb = reinterpret_cast<const char*>(nsrc);
#pragma unroll
              for (int i = 0; i < kCh; ++i)
                ptx::cp_async16(pbn + (kCh * sb + i) * PB, nb + (uint32_t)((kCh * sb + i) * chunk_bytes));
            }
            ptx::cp_async_commit();   // (possibly empty) group: keeps the wait_group 1 accounting
          }
          tc::wait_ld();
          if (lane == 0 && ew == 0) stamp_k(k, 9 + sb);
          // a4: leak / thresholds / reset per sample
          uint32_t outw[kSub / 2];
          const uint32_t fb = sat16 ? lif<true, kSub>(cur, acc, leak, pth, nth, linmul, bf, bn, 0, 0, one, outw)
                                    : lif<false, kSub>(cur, acc, leak, pth, nth, linmul, bf, bn, p.pot_lo, p.pot_hi,
                                                       one, outw);
          fired |= fb << (sb * kSub);
#pragma unroll
          for (int cc = 0; cc < kCh; ++cc) {
            const uint4 o = make_uint4(outw[4 * cc + 0], outw[4 * cc + 1], outw[4 * cc + 2], outw[4 * cc + 3]);
            if (!last) pb[(kCh * sb + cc) * PB] = o;   // kept on chip for the next tick
            else POT_STORE(reinterpret_cast<char*>(dsub) + (uint32_t)((kCh * sb + cc) * chunk_bytes), o);
          }
        }
        // a5 / a6: route or count the spikes of real samples
        const int sj = s0 + jj * 32;          // first sample of this warp's half
        const int lim = ns - jj * 32;
        const uint32_t f = lim >= 32 ? fired : (lim > 0 ? fired & ((1u << lim) - 1u) : 0u);
        if (kPull) {
          // a5 (history scheduler): store this neuron's fired bits of the 32
          // samples of this half at its position in the slot of tick t + delay
          if (route_here) p.hist[((((size_t)((t + rdelay) & p.rp_mask)) * nT + tile) * p.hist_P + hpos) * 2 + jj] = f;
        } else if (block_identity) {
          // every routing lane l of this warp deposits bit l of one ring
          // word: a 32x32 bit transpose turns the per-lane sample masks into
          // per-sample deposit words, one RED per (sample, word) issued by
          // the lane of that sample (idempotent OR, G11)
          const uint32_t m = transpose32(route_here ? f : 0u, lane);
          if (m) atomicOr(p.ring + warp_ring_off + (sj + lane) * ss, m);
        } else if (block_route) {
          // every routing lane targets the same ring word: the OR-reduced
          // deposit of sample i is kept by lane i, then one coalesced RED
          uint32_t any = __reduce_or_sync(0xFFFFFFFFu, route_here ? f : 0u);
          uint32_t mine = 0u;
          while (any) {
            const int i = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t m = __reduce_or_sync(0xFFFFFFFFu, (route_here && ((f >> i) & 1u)) ? axbit : 0u);
            if (lane == i) mine = m;
          }
          if (mine) atomicOr(p.ring + warp_ring_off + (sj + lane) * ss, mine);
        } else if (!wm) {
          if (route_here) {
            uint32_t g = f;
            while (g) {
              const int i = __ffs(g) - 1;
              g &= g - 1;
              atomicOr(p.ring + ring_off + (size_t)(sj + i) * W, axbit);
            }
          }
        } else {
          // per-neuron destinations: lane i receives the routing neurons
          // (lanes) fired in sample i; for each such neuron the warp issues
          // one RED over its 32 contiguous sample words (one 128-byte line)
          uint32_t src = __ballot_sync(0xFFFFFFFFu, route_here && f != 0u);
          const uint32_t m = src ? transpose32(route_here ? f : 0u, lane) : 0u;
          while (src) {
            const int l = __ffs(src) - 1;
            src &= src - 1;
            const size_t off = __shfl_sync(0xFFFFFFFFu, ring_off, l);
            const uint32_t bit = __shfl_sync(0xFFFFFFFFu, axbit, l);
            if ((m >> l) & 1u) atomicOr(p.ring + off + sj + lane, bit);
          }
        }
        if (has_output && planes && out_scatter) {   // (few classes: the grouped adds below are cheaper)
          uint32_t* const pl = cpl + k0 * kPl;
          uint32_t carry = kind == RK_OUTPUT ? f : 0u;
          for (int b = 0; b < kCntPlanes && carry; ++b) {   // ripple-carry add of one per fired sample
            const uint32_t x = pl[b * 512];
            pl[b * 512] = x ^ carry;
            carry &= x;
          }
          if (kind == RK_OUTPUT && (last || (it + 1) % 255 == 0)) {
            uint32_t v[kCntPlanes];
#pragma unroll
            for (int b = 0; b < kCntPlanes; ++b) {
              v[b] = pl[b * 512];
              pl[b * 512] = 0u;
            }
            for (int i = 0; i < 32; ++i) {
              int cnt = 0;
#pragma unroll
              for (int b = 0; b < kCntPlanes; ++b) cnt |= (int)((v[b] >> i) & 1u) << b;
              if (cnt) atomicAdd(p.counts + (size_t)(sj + i) * p.C + cls, cnt);
            }
          }
        } else if (has_output && out_scatter) {
          // a6 output bus, many classes in the warp (e.g. VMM: one class per
          // neuron): each lane adds its own fired samples; the lanes' classes
          // are neighbouring words of one counts row, so a warp's add touches
          // one or two lines instead of 32
          uint32_t g = kind == RK_OUTPUT ? f : 0u;
          while (g) {
            const int i = __ffs(g) - 1;
            g &= g - 1;
            atomicAdd(p.counts + (size_t)(sj + i) * p.C + cls, 1);
          }
        } else if (has_output) {
          // a6 output bus: lane i receives the output neurons (lanes) fired
          // in sample i; one add per (sample, class group of lanes)
          const uint32_t m = transpose32(kind == RK_OUTPUT ? f : 0u, lane);
          uint32_t rem = out_lanes;
          while (rem) {
            const int l = __ffs(rem) - 1;
            const uint32_t grp = __shfl_sync(0xFFFFFFFFu, out_peers, l);
            const uint32_t cg = __shfl_sync(0xFFFFFFFFu, cls, l);
            rem &= ~grp;
            const int cnt = __popc(m & grp);
            if (cnt) atomicAdd(p.counts + (size_t)(sj + lane) * p.C + cg, cnt);
          }
        }
        if (p.raster || exporting) {
          // lane i receives the fired word (32 neurons) of sample i
          const uint32_t m = transpose32(valid ? fired : 0u, lane);
          if (lane < lim && (n >> 5) < p.Wn) {
            const int sg = sj + lane;
            if (p.raster) p.raster[(((size_t)(t - p.raster_t0) * p.S + sg) * p.G_loc + cl) * p.Wn + (n >> 5)] = m;
            if (exporting) p.fired[((size_t)cl * p.Sr + sg) * p.Wn + (n >> 5)] = m;
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0 && ew == 0) stamp_k(k, 11);
      if (lane == 0) ptx::mbar_arrive(&bars[ACCEMPTY0 + a]);
      }
      adv(cl, tile);
    }
    tick_barrier();
    }
    if (dbg_on && blockIdx.x == 0 && lane == 0) {
      p.dbg[64 * 16 + 2 * ew] = (unsigned long long)dbg_wait;
      p.dbg[64 * 16 + 2 * ew + 1] = (unsigned long long)(clock64() - dbg_t0);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == mma_warp) tc::dealloc(tmem, tcols < 32 ? 32 : tcols);
  if (p.cta_ns && threadIdx.x == 0) {   // this CTA's busy time, for the partition
    unsigned long long gt_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_end));
    p.cta_ns[blockIdx.x] = (uint32_t)min(gt_end - gt_start, 0xFFFFFFFFull);
  }
  if (dbg_on && threadIdx.x == 0 && blockIdx.x < 256) {
    unsigned long long gt_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_end));
    p.dbg[64 * 16 + 64 + 2 * blockIdx.x] = gt_start;
    p.dbg[64 * 16 + 64 + 2 * blockIdx.x + 1] = gt_end;
  }
}

// Input decode (Alg. 1 l.1, "Initial setup and input decode"): the line
// bits of every (tick, input core, sample) are mapped once onto the core's
// ring-word layout, inw [T_in][slots][Sr][W], so the per-tick spike stage only
// ORs a TMA-loaded row into the scheduler row.
// grid (sample blocks, slots, T_in); the core's runs are staged in shared memory
__global__ void decode_inputs_kernel(const uint32_t* __restrict__ lines, uint32_t* __restrict__ inw,
                                     const int32_t* __restrict__ slot_core, const int2* __restrict__ runs,
                                     const int32_t* __restrict__ word_runs, int S, int Sr, int W, int WIp,
                                     int rmax, int wmajor, int n_slots, int slot0, int t0) {
  extern __shared__ int2 dec_sm[];
  const int slot = slot0 + blockIdx.y, t = t0 + blockIdx.z;
  const int c = slot_core[slot];
  int2* rs = dec_sm;
  int32_t* wr = reinterpret_cast<int32_t*>(dec_sm + rmax);
  for (int i = threadIdx.x; i < rmax; i += blockDim.x) rs[i] = runs[(size_t)c * rmax + i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) wr[i] = word_runs[(size_t)c * W + i];
  __syncthreads();
  const int per_block = (int)blockDim.x * 4;   // ring words per block
  const int total = S * W;
  for (int i = blockIdx.x * per_block + threadIdx.x; i < min(total, (blockIdx.x + 1) * per_block);
       i += blockDim.x) {
    // word-major: consecutive threads take consecutive samples of one word
    const int w = wmajor ? i / S : i % W, s = wmajor ? i - w * S : i / W;
    const int32_t fr = wr[w];
    const int r0 = fr & 0xFFFF, nrw = fr >> 16;
    const uint32_t* lr = lines + ((size_t)t * Sr + s) * WIp;
    uint32_t acc = 0u;
    for (int q = r0; q < r0 + nrw; ++q) {
      const int2 rn = rs[q];
      const int ap = rn.x & 0xFFFF, len = rn.x >> 16, ln = rn.y;
      const int lw = ln >> 5, lb = ln & 31;
      uint32_t x = lr[lw] >> lb;
      if (lb + len > 32) x |= lr[lw + 1] << (32 - lb);
      if (len < 32) x &= (1u << len) - 1u;
      const int off = ap - 32 * w;
      acc |= off >= 0 ? (x << off) : (x >> (-off));
    }
    const size_t row = (size_t)t * n_slots + slot;   // same layout as the ring
    inw[wmajor ? (row * W + w) * Sr + s : (row * Sr + s) * W + w] = acc;
  }
}

// Cost-balanced work partition of the per-tick launches (load balance only:
// the items of one tick are independent, so results do not depend on it).
// From the CTAs' measured busy times over their current ranges (a piecewise
// constant cost per item), the item sequence is cut into g pieces of equal
// estimated cost; the new bounds are averaged with the old ones (damping).
__global__ void rebalance_kernel(int32_t* part, const uint32_t* cta_ns, int g) {
  __shared__ int32_t nb[1025];
  if (threadIdx.x != 0 || g > 1024) return;
  double tot = 0.0, mx = 0.0;
  for (int b = 0; b < g; ++b) {
    tot += (double)cta_ns[b];
    mx = fmax(mx, (double)cta_ns[b]);
  }
  if (tot <= 0.0 || mx <= 1.03 * tot / g) return;   // balanced within 3 %: keep (uniform meshes: moving
                                                      // items only costs L2 locality)
  nb[0] = part[0];
  nb[g] = part[g];
  double cum = 0.0;
  int b = 0;
  for (int k = 1; k < g; ++k) {
    const double target = tot * k / g;
    while (b < g - 1 && cum + (double)cta_ns[b] < target) cum += (double)cta_ns[b++];
    const int items = part[b + 1] - part[b];
    const double f = cta_ns[b] > 0 ? (target - cum) / (double)cta_ns[b] : 0.0;
    int cut = part[b] + (int)(f * items + 0.5);
    nb[k] = cut;
  }
  for (int k = 1; k < g; ++k) {
    int v = (part[k] + nb[k] + 1) / 2;
    v = max(v, part[0] + k);                 // at least one item per CTA
    v = min(v, part[g] - (g - k));
    nb[k] = v;
  }
  for (int k = 1; k < g; ++k) part[k] = max(nb[k], part[k - 1] + 1);
}

__global__ void part_init_kernel(int32_t* part, int g, int total) {
  for (int b = threadIdx.x; b <= g; b += blockDim.x) part[b] = (int)((int64_t)b * total / g);
}

}  // namespace

cudaError_t decode_inputs_tc(ranc_ctx* ctx) {
  const Compiled& n = ctx->net;
  const int64_t words = (int64_t)ctx->S * n.W;
  if (words == 0 || ctx->n_inslots == 0 || ctx->T_in == 0) return cudaSuccess;
  if (words > INT32_MAX) return cudaErrorInvalidValue;
  const int threads = 256;
  const size_t smem = (size_t)n.rmax * sizeof(int2) + (size_t)n.W * sizeof(int32_t);
  // grid.y / grid.z are limited to 65535: long input streams and many input
  // slots are decoded in chunks
  constexpr int kMaxYZ = 65535;
  for (int t0 = 0; t0 < ctx->T_in; t0 += kMaxYZ)
    for (int s0 = 0; s0 < ctx->n_inslots; s0 += kMaxYZ) {
      const dim3 grid((unsigned)((words + threads * 4 - 1) / (threads * 4)),
                      (unsigned)std::min(kMaxYZ, ctx->n_inslots - s0), (unsigned)std::min(kMaxYZ, ctx->T_in - t0));
      decode_inputs_kernel<<<grid, threads, smem, ctx->stream>>>(
          (const uint32_t*)ctx->d_lines.p, (uint32_t*)ctx->d_inw.p, (const int32_t*)ctx->d_slot_core.p,
          (const int2*)ctx->d_runs.p, (const int32_t*)ctx->d_word_runs.p, (int)ctx->S, (int)ctx->Sr, n.W, n.WIp,
          n.rmax, ctx->ring_wmajor ? 1 : 0, ctx->n_inslots, s0, t0);
      ctx->launches++;
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

int tc_tile() { return NT; }

int grp_stages(const Compiled& n) { return !n.tc_grp ? 0 : n.Kp > kKChunk ? 1 : NS_GRP; }

size_t tc_smem_bytes(const Compiled& n) {
  return tc_layout(n.grp_rows, n.Kp, n.W, n.WIp, n.rmax, n.tc_wide, 1, false, false, grp_stages(n)).total;
}

// shared memory of the pull-scheduler launch (word-major, per-tick, no groups)
size_t tc_smem_bytes_pull(const Compiled& n) {
  return tc_layout(n.grp_rows, n.Kp, n.W, n.WIp, n.rmax, n.tc_wide, 1, false, false, 0, n.hist_emax).total;
}

// shared memory of the compact-operand launch (two expanded operand buffers)
size_t tc_smem_bytes_comp(const Compiled& n, bool pull) {
  return tc_layout(n.grp_rows, n.Kp, n.W, n.WIp, n.rmax, false, 1, false, false, 0, pull ? n.hist_emax : -1, true)
      .total;
}

namespace {

void tc_fill_params(ranc_ctx* ctx, TickParams& p) {
  const Compiled& n = ctx->net;
  p.ST = NT;
  p.route = (const uint2*)ctx->d_route_tc.p;
  p.wflags = (const uint8_t*)ctx->d_wflags_tc.p;
  p.incoming = (const uint8_t*)ctx->d_incoming.p;
  p.runs = (const int2*)ctx->d_runs.p;
  p.word_runs = (const int32_t*)ctx->d_word_runs.p;
  p.inw = ctx->inw_valid ? (const uint32_t*)ctx->d_inw.p : nullptr;
  p.inslot = (const int32_t*)ctx->d_inslot.p;
  p.n_inslots = ctx->n_inslots;
  p.nruns = (const int32_t*)ctx->d_nruns.p;
  p.rmax = n.rmax;
  p.grp_rows = n.grp_rows;
  p.grp_ns = grp_stages(n);
  p.wmajor = ctx->ring_wmajor ? 1 : 0;
  p.hist = (uint32_t*)ctx->d_hist.p;
  p.hpos = (const uint32_t*)ctx->d_hpos.p;
  p.hbase = (const uint32_t*)ctx->d_hbase.p;
  p.hax = (const uint16_t*)ctx->d_hax.p;
  p.hist_emax = n.hist_emax;
  p.hist_P = (int32_t)n.hbase.back();
  p.xbits = (const uint32_t*)ctx->d_xbits.p;
  p.wq = (const uint32_t*)ctx->d_wq.p;
  p.tsel = (const uint32_t*)ctx->d_tsel.p;
  p.any_route = n.any_route ? 1 : 0;
}

}  // namespace

bool tc_multi_eligible(const ranc_ctx* ctx, int64_t num_ticks) {
  if (ctx->kernel_active != RANC_KERNEL_TC || ctx->shard_mode == RANC_SHARD_CORES || num_ticks < 2) return false;
  if (ctx->stream_opt == 1 || getenv("RANC_DEBUG_TIMELINE") || ctx->net.tc_wide || ctx->net.tc_grp || ctx->ring_pull)
    return false;   // (_MULTI: kept)
  const int64_t total = (int64_t)ctx->G_loc * ((ctx->S + NT - 1) / NT);
  if (total <= ctx->num_sms) return true;   // one work item per CTA, one CTA per SM (cooperative launch)
  // two work items per CTA: both potential tiles stay in shared memory
  const Compiled& n = ctx->net;
  return total <= 2 * (int64_t)ctx->num_sms &&
         tc_layout(n.Npad, n.Kp, n.W, n.WIp, n.rmax, false, 2, false, true).total <= 227 * 1024;
}

// all ticks of a ranc_run_ticks call in one cooperative launch (small
// batches: at most two (core, 64-sample tile) items per SM, their
// potentials kept in shared memory between ticks)
// RANC_DEBUG_TIMELINE(_MULTI): per-tile stamps of CTA 0 (work items k < 64;
// in a multi-tick launch k = tick), per-warp wait / total cycles, CTA end times
constexpr int kDbg = 64 * 16 + 64 + 512;
void dump_timeline(ranc_ctx* ctx, int64_t t, int grid) {
    static unsigned long long h[kDbg];
    cudaMemcpyAsync(h, ctx->d_dbg.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    const unsigned long long t0 = h[0];
    fprintf(stderr, "timeline t=%lld grid=%d (cycles rel. to producer start)\n", (long long)t, grid);
    fprintf(stderr, "  k  prodW prodGo expFull expBempty expBfull mmaB mmaAccE mmaCommit | ew0: acc ld0 ld1 done | exp: cleared injected synced expanded\n");
    for (int k = 0; k < 64; ++k) {
      fprintf(stderr, "%3d", k);
      for (int j = 0; j < 16; ++j) fprintf(stderr, " %8lld", h[k * 16 + j] ? (long long)(h[k * 16 + j] - t0) : -1LL);
      fprintf(stderr, "\n");
    }
    fprintf(stderr, "epilogue warps of CTA 0: ACCFULL wait / total cycles\n");
    for (int w = 0; w < kEpiWarps; ++w)
      fprintf(stderr, "  ew%-2d %10llu %10llu\n", w, h[64 * 16 + 2 * w], h[64 * 16 + 2 * w + 1]);
    unsigned long long s_min = ~0ull, e_min = ~0ull, e_max = 0;
    for (int b = 0; b < std::min(grid, 256); ++b) {
      s_min = std::min(s_min, h[64 * 16 + 64 + 2 * b]);
      e_min = std::min(e_min, h[64 * 16 + 64 + 2 * b + 1]);
      e_max = std::max(e_max, h[64 * 16 + 64 + 2 * b + 1]);
    }
    fprintf(stderr, "CTA end times (ns after first start), by CTA:");
    for (int b = 0; b < std::min(grid, 256); ++b)
      fprintf(stderr, "%s%llu", b % 16 ? " " : "\n  ", h[64 * 16 + 64 + 2 * b + 1] - s_min);
    fprintf(stderr, "\nCTA end times (ns after first start): min %llu max %llu; slowest CTAs:", e_min - s_min,
            e_max - s_min);
    for (int b = 0; b < std::min(grid, 256); ++b)
      if (h[64 * 16 + 64 + 2 * b + 1] + 20000 > e_max) fprintf(stderr, " %d", b);
    fprintf(stderr, "\n");
  }

cudaError_t launch_tc_multi(ranc_ctx* ctx, TickParams p, int64_t num_ticks) {
  const Compiled& n = ctx->net;
  tc_fill_params(ctx, p);
  const int64_t total = (int64_t)ctx->G_loc * ((ctx->S + NT - 1) / NT);
  p.pot_items = total <= ctx->num_sms ? 1 : 2;
  ctx->operand_used = 1;
  const int grid = (int)((total + p.pot_items - 1) / p.pot_items);   // contiguous items: mostly the same core
  // bit-sliced output counters when the network has an output bus and they fit
  p.out_planes =
      n.any_output && tc_layout(n.Npad, n.Kp, n.W, n.WIp, n.rmax, false, p.pot_items, true, true).total <= 227 * 1024;
  const size_t smem = tc_layout(n.Npad, n.Kp, n.W, n.WIp, n.rmax, false, p.pot_items, p.out_planes, true).total;
  static const bool dbg = getenv("RANC_DEBUG_TIMELINE_MULTI") != nullptr;
  if (dbg && !ctx->d_dbg.p) dev_alloc(ctx, &ctx->d_dbg, kDbg * 8);
  p.dbg = dbg ? (unsigned long long*)ctx->d_dbg.p : nullptr;
  if (dbg) cudaMemsetAsync(ctx->d_dbg.p, 0, kDbg * 8, ctx->stream);
  const void* fn = dbg ? (p.wmajor ? (const void*)tick_tc_kernel<true, true, true, false>
                                   : (const void*)tick_tc_kernel<true, true, false, false>)
                       : (p.wmajor ? (const void*)tick_tc_kernel<true, false, true, false>
                                   : (const void*)tick_tc_kernel<true, false, false, false>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int nt = (int)std::min<int64_t>(num_ticks, 1 << 30);
  void* args[] = {&p, &nt};
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreadsTC), args, smem, ctx->stream);
  if (dbg && e == cudaSuccess) dump_timeline(ctx, p.t, grid);
  return e;
}

cudaError_t launch_tick_tc(ranc_ctx* ctx, TickParams p) {
  const Compiled& n = ctx->net;
  tc_fill_params(ctx, p);
  const int64_t total = (int64_t)ctx->G_loc * ((ctx->S + NT - 1) / NT);
  const int grid = (int)std::min<int64_t>(total, ctx->num_sms);
  // compact operand: requested, or automatic with at most two sample tiles
  // per core (the folded operand would be re-read for every 64 samples)
  const int64_t nT = (ctx->S + NT - 1) / NT;
  // (automatic: with the history scheduler, whose two spike groups expand
  // the operands; measured on config 5)
  const bool comp = n.tc_comp_ok && (ctx->operand == 2 || (ctx->operand == 0 && nT <= 2 && ctx->ring_pull)) &&
                    tc_smem_bytes_comp(n, ctx->ring_pull) <= 227 * 1024;
  ctx->operand_used = comp ? 2 : 1;
  const size_t smem = comp ? tc_smem_bytes_comp(n, ctx->ring_pull)
                           : ctx->ring_pull ? tc_smem_bytes_pull(n) : tc_smem_bytes(n);
  static const bool no_serp = getenv("RANC_DEBUG_NO_SERP") != nullptr;   // (timing comparisons)
  p.serp = no_serp ? 0 : 1;
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    const void* fns[] = {(const void*)tick_tc_kernel<false, false, false, false>,
                         (const void*)tick_tc_kernel<false, true, false, false>,
                         (const void*)tick_tc_kernel<false, false, true, false>,
                         (const void*)tick_tc_kernel<false, true, true, false>,
                         (const void*)tick_tc_kernel<false, false, false, true>,
                         (const void*)tick_tc_kernel<false, false, true, true>,
                         (const void*)tick_tc_kernel<false, false, false, false, true>,
                         (const void*)tick_tc_kernel<false, false, true, false, true>,
                         (const void*)tick_tc_kernel<false, false, false, true, true>,
                         (const void*)tick_tc_kernel<false, false, true, true, true>,
                         (const void*)tick_tc_kernel<false, false, true, true, false, true>,
                         (const void*)tick_tc_kernel<false, true, true, false, false, true>,
                         (const void*)tick_tc_kernel<false, false, true, false, false, true>,
                         (const void*)tick_tc_kernel<false, false, false, false, false, false, true>,
                         (const void*)tick_tc_kernel<false, false, true, false, false, false, true>,
                         (const void*)tick_tc_kernel<false, false, true, false, false, true, true>,
                         (const void*)tick_tc_kernel<false, true, true, false, false, true, true>};
    for (const void* f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  static const bool dbg_env = getenv("RANC_DEBUG_TIMELINE") != nullptr;
  const bool dbg = dbg_env && !n.tc_wide && !n.tc_grp && (!comp || ctx->ring_pull);
  if (dbg && !ctx->d_dbg.p) dev_alloc(ctx, &ctx->d_dbg, kDbg * 8);
  p.dbg = dbg ? (unsigned long long*)ctx->d_dbg.p : nullptr;
  if (dbg) cudaMemsetAsync(ctx->d_dbg.p, 0, kDbg * 8, ctx->stream);
  // cost-balanced partition: measured on the first ticks and every 64th,
  // rebalanced by a one-thread kernel after the measured tick
  static const bool no_bal = getenv("RANC_DEBUG_NO_BALANCE") != nullptr;
  bool measure = false;
  if (!no_bal && grid > 1 && grid <= 1024 && total >= 2 * (int64_t)grid) {
    const int64_t key = total * 4096 + grid;
    if (ctx->part_key != key) {
      if (dev_alloc(ctx, &ctx->d_part, (size_t)(grid + 1) * 4) != RANC_OK ||
          dev_alloc(ctx, &ctx->d_cta_ns, (size_t)grid * 4) != RANC_OK)
        return cudaErrorMemoryAllocation;
      part_init_kernel<<<1, 256, 0, ctx->stream>>>((int32_t*)ctx->d_part.p, grid, (int)total);
      ctx->launches++;
      ctx->part_key = key;
      ctx->part_ticks = 0;
      ctx->part_fresh = true;
    }
    p.part = (const int32_t*)ctx->d_part.p;
    measure = ctx->part_ticks < 6 || (ctx->part_ticks & 63) == 0;
    p.cta_ns = measure ? (uint32_t*)ctx->d_cta_ns.p : nullptr;
    ++ctx->part_ticks;
  }
  const bool pull = ctx->ring_pull;
  const void* fn = comp ? (pull ? (dbg ? (const void*)tick_tc_kernel<false, true, true, false, false, true, true>
                                       : (const void*)tick_tc_kernel<false, false, true, false, false, true, true>)
                                : p.wmajor ? (const void*)tick_tc_kernel<false, false, true, false, false, false, true>
                                           : (const void*)tick_tc_kernel<false, false, false, false, false, false, true>)
                   : pull ? (n.tc_wide ? (const void*)tick_tc_kernel<false, false, true, true, false, true>
                                     : dbg ? (const void*)tick_tc_kernel<false, true, true, false, false, true>
                                           : (const void*)tick_tc_kernel<false, false, true, false, false, true>)
                   : n.tc_grp ? (n.tc_wide ? (p.wmajor ? (const void*)tick_tc_kernel<false, false, true, true, true>
                                                      : (const void*)tick_tc_kernel<false, false, false, true, true>)
                                         : (p.wmajor ? (const void*)tick_tc_kernel<false, false, true, false, true>
                                                      : (const void*)tick_tc_kernel<false, false, false, false, true>))
                   : n.tc_wide ? (p.wmajor ? (const void*)tick_tc_kernel<false, false, true, true>   // wide: no timeline
                                          : (const void*)tick_tc_kernel<false, false, false, true>)
                   : dbg ? (p.wmajor ? (const void*)tick_tc_kernel<false, true, true, false>
                                     : (const void*)tick_tc_kernel<false, true, false, false>)
                         : (p.wmajor ? (const void*)tick_tc_kernel<false, false, true, false>
                                     : (const void*)tick_tc_kernel<false, false, false, false>);
  // programmatic dependent launch: consecutive tick launches overlap the
  // next grid's start-up with this one's tail (griddepcontrol in the kernel)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc_threads(pull && comp));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const bool no_pdl = getenv("RANC_DEBUG_NO_PDL") != nullptr;
  // (not right after a rebalance: the kernel reads the partition at its start)
  attr[0].val.programmaticStreamSerializationAllowed = (ctx->pdl && !no_pdl && !ctx->part_fresh) ? 1 : 0;
  ctx->part_fresh = measure;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int one = 1;
  void* args[] = {&p, &one};
  const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return e;
  if (measure) {
    rebalance_kernel<<<1, 32, 0, ctx->stream>>>((int32_t*)ctx->d_part.p, (const uint32_t*)ctx->d_cta_ns.p, grid);
    ctx->launches++;
  }
  if (dbg) dump_timeline(ctx, p.t, grid);
  return cudaGetLastError();
}

}  // namespace ranc
