// internal.h -- context, compiled-network layout and kernel parameter block of
// libranc.so.  Not part of the ABI (include/ranc.h is).
//
// Device layout, per context:
//   compiled network (uploaded once), L2-resident at the paper's sizes:
//     xp    u32 [G][E][Npad]   popcount piece words: crossbar column of neuron n
//                              restricted to one axon-type segment of one
//                              32-axon word, after the per-core axon type-sort
//     wp    i16 [G][E][Npad]   weight of that piece's axon type for neuron n
//     pword u8  [G][E]         ring word index of piece e
//     prm   short4 [G][Npad]   {leak, pos_threshold, neg_threshold, reset}
//     route uint2  [G][Npad]   x: kind | lin<<2 | delay<<3 | axon'<<8 ; y: dest core or class
//     inl   i32 [G][A]         input line of permuted axon a' (-1 none)
//   state (streamed every tick):
//     pot   i16 [G][S][Npad]   membrane potentials (pb <= 16), popcount kernel;
//           i16 [G][nT][NT/8][Npad][8] tile-blocked, tensor-core kernel (NT = 64)
//     ring  u32 [Rp][G][Sr][W] scheduler rings, W = ceil(A/32) words per row;
//           u32 [Rp][G][W][Sr] word-major (tensor-core kernel, networks with per-neuron
//                              routes: the 32 sample words a warp deposits for one
//                              route are one 128-byte line; RANC_OPT_RING_LAYOUT),
//                              Sr = S rounded up to 64 (TMA-aligned tiles),
//                              slot of tick t = t & (Rp-1), Rp = next_pow2(D+1)
//     counts i32 [S][C]        output-bus class counts
//     lines u32 [T_in][Sr][WIp] external input line bits (transposed at load so a
//                              tile's rows of one tick are contiguous; WIp = WI
//                              rounded up to 4 words)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include <string>
#include <vector>

#include "../../include/ranc.h"

namespace ranc {

// route word fields
enum : uint32_t { RK_NONE = 0, RK_ROUTE = 1, RK_OUTPUT = 2 };
__host__ __device__ inline uint32_t route_kind(uint32_t x) { return x & 3u; }
__host__ __device__ inline uint32_t route_lin(uint32_t x) { return (x >> 2) & 1u; }
__host__ __device__ inline uint32_t route_delay(uint32_t x) { return (x >> 3) & 31u; }
__host__ __device__ inline uint32_t route_axon(uint32_t x) { return (x >> 8) & 0x7FFu; }

// Function attributes (cudaFuncSetAttribute) are per device: true the first
// time `mask` sees the current device (contexts on several GPUs in one
// process each configure their device's copy of a kernel).
inline bool first_use_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  return !(mask.fetch_or(bit) & bit);
}

struct TickParams {
  int32_t G, S, N, Npad, A, W, E, Wn, C, T_in, WI, ST;
  int32_t Sr;               // sample stride of ring rows and input lines (S rounded up to 64)
  int32_t c_lo, G_loc;      // cores [c_lo, c_lo+G_loc) are simulated here (core-sharded mode)
  int32_t WIp;              // u32 words per input-line row (WI rounded up to 4: 16-byte rows)
  int32_t rp_mask;          // Rp - 1
  int32_t pot_lo, pot_hi;   // saturation range of pb bits
  int32_t fresh;            // first tick after a reset: potentials start at init
  int32_t wmajor;           // tensor-core path: ring and decoded inputs word-major [..][W][Sr]
  int32_t any_route;        // some neuron routes (multi-tick tensor-core launch needs the grid barrier)
  int32_t pot_items;        // multi-tick tensor-core launch: work items (potential tiles) per CTA, 1 or 2
  int32_t out_planes;       // multi-tick tensor-core launch: bit-sliced per-thread output counters in shared memory
  int32_t Kp;               // tensor-core path: K bytes per operand row (= 32*W)
  int32_t grp_rows;         // tensor-core path: rows per neuron group (Compiled::grp_rows)
  int32_t grp_ns;           // neuron-group launch: spike stages (2, or 1 beyond 512 axons)
  int32_t serp;             // tensor-core per-tick launches: odd ticks walk each CTA's items backwards
  int32_t fault;            // RANC_OPT_DEBUG_FAULT (mutation tests): 1 = skip the grid barrier of
                            // cooperative multi-tick launches
  int64_t t;                // tick being executed
  int64_t raster_t0;        // first tick of the raster buffer
  const uint8_t* wfold;     // tensor-core path: [G][Npad*Kp] canonical-layout int8
  const int2* runs;         // tensor-core path: input runs [G][rmax]
  const int32_t* word_runs; // [G][W]: runs overlapping ring word w: first | count << 16
  const uint32_t* inw;      // decoded inputs [T_in][n_inslots][Sr][W] or [..][W][Sr] (the ring's layout), or nullptr
  const int32_t* inslot;    // [G_loc] input slot of a local core (-1: no input lines)
  int32_t n_inslots;
  const int32_t* nruns;     // [G]
  int32_t rmax;
  const uint32_t* xp;
  const int16_t* wp;
  const uint8_t* pword;
  const short4* prm;
  const uint2* route;
  const int32_t* inl;
  const uint8_t* has_in;
  const int16_t* init;      // [G][Npad] initial potentials
  const uint32_t* lines;    // [T_in][S][WI]
  int16_t* pot;
  uint32_t* ring;
  int32_t* counts;
  uint32_t* raster;         // [T][S][G_loc][Wn] or nullptr
  uint32_t* fired;          // core-sharded: [G_loc][Sr][Wn] fired bits of this tick (export cores)
  const uint8_t* exports;   // [G] core has a neuron routing to another rank
  unsigned long long* dbg;  // optional pipeline timeline (RANC_DEBUG_TIMELINE)
  const uint8_t* wflags;    // [G][Npad/32] per-warp flags (bit 0: block route), or nullptr
  const uint8_t* incoming;  // [G] 1 if any neuron of the network routes to the core (its ring can be non-zero)
  uint32_t* spkin;          // RANC_TRACE_STATE_DIGEST: [S][G_loc][W] axon spikes integrated this tick, or nullptr
  // history scheduler (tensor-core path, RANC_OPT_RING_LAYOUT 3): fired-bit
  // history u32 [Rp][nT][P][2] (slot = arrival tick & (Rp-1); position i of
  // the destination-ordered list; word j = samples 32j..32j+31 of the tile)
  // and the position tables (Compiled::h*)
  uint32_t* hist;
  const uint32_t* hpos;
  const uint32_t* hbase;
  const uint16_t* hax;
  int32_t hist_emax;
  int32_t hist_P;
  // compact operand (tensor-core path, RANC_OPT_OPERAND): Compiled::xbits / wq / tsel
  const uint32_t* xbits;
  const uint32_t* wq;
  const uint32_t* tsel;
  // cost-balanced partition of per-tick launches: CTA b takes items
  // [part[b], part[b+1]) (nullptr: equal shares) and, when cta_ns is set,
  // stores its busy time in ns
  const int32_t* part;
  uint32_t* cta_ns;
};

// Host copy of the compiled network.
struct Compiled {
  int32_t G = 0, A = 0, N = 0, Npad = 0, K = 0, D = 0, C = 0, I = 0, W = 0, E = 0, Wn = 0, WI = 0;
  int32_t grid_w = 0, grid_h = 0, pb = 16, Rp = 2;
  int32_t Kp = 0;               // 32 * W
  int32_t WIp = 0;              // WI rounded up to 4
  bool tc_ok = false;           // eligible for the tcgen05 kind::i8 path
  bool tc_grp = false;          // tensor-core path in neuron groups (Npad > 256 or Npad*Kp > 64 KB)
  int32_t grp_rows = 0;         // rows per neuron group (Npad unless tc_grp: 256 or 128)
  bool any_route = false;       // some neuron has dest_kind ROUTE
  bool any_output = false;      // some neuron has dest_kind OUTPUT
  bool tc_wide = false;         // some weight outside [-128,127]: Wfold split w = 256*hi + lo, [G][2][Npad*Kp] (u8 lo, s8 hi)
  bool tc_hist = false;         // automatic ring layout: the history scheduler when a third of all neurons
                                // are such routers (and a tick runs as per-tick launches)
  bool tc_wmajor = false;       // automatic ring layout: word-major when most routing neurons sit in
                                // warps without a shared destination word (per-neuron routes)
  std::vector<int8_t> wfold;    // [G][Npad*Kp] canonical operand layout, tensor-core axon order
  std::vector<int32_t> perm_tc, inv_tc;   // tensor-core axon order (sorted by input line)
  std::vector<uint2> route_tc;  // route words with tensor-core destination axons
  std::vector<int2> runs;       // [G][rmax] input runs: x = a'start | len<<16, y = first line
  std::vector<int32_t> nruns;   // [G]
  std::vector<int32_t> word_runs;  // [G][W] first run | count << 16 (runs overlapping word w)
  std::vector<uint8_t> incoming;   // [G] 1 if some neuron routes to the core
  bool tc_comp_ok = false;         // the compact operand applies (int8 weights, Npad <= 256, A <= 256)
  std::vector<uint32_t> xbits;     // [G][W][Npad] crossbar bits, expansion bit order (compile.cpp)
  std::vector<uint32_t> wq;        // [G][Npad] the K type weights of neuron n as int8 bytes
  std::vector<uint32_t> tsel;      // [G][Kp/4] prmt selectors: nibble j = type of axon a' = 4g + j
  std::vector<uint32_t> hbase;     // [G+1] history scheduler: first position of destination core c (compile.cpp)
  std::vector<uint32_t> hpos;      // [G][Npad] position of routing neuron (c, n), ~0u otherwise
  std::vector<uint16_t> hax;       // [P] destination axon a' of a position
  std::vector<uint8_t> hdel;       // [P] delay of a position (0: padding)
  int32_t hist_emax = 0;           // most positions of one destination core
  std::vector<uint8_t> wflags_tc;  // [G][Npad/32] bit 0: all routing neurons of the warp share one
                                   // (dest core, ring word, delay) in the tensor-core axon order
  int32_t rmax = 0;
  std::vector<uint32_t> xp;     // [G][E][Npad]
  std::vector<int16_t> wp;      // [G][E][Npad]
  std::vector<uint8_t> pword;   // [G][E]
  std::vector<short4> prm;      // [G][Npad]
  std::vector<uint2> route;     // [G][Npad]
  std::vector<int32_t> inl;     // [G][A]
  std::vector<uint8_t> has_in;  // [G]
  std::vector<int16_t> init;    // [G][Npad]
  std::vector<int32_t> perm;    // [G][A]  a' -> a
  std::vector<int32_t> inv;     // [G][A]  a -> a'
  std::vector<uint8_t> kind;    // [G][N]
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool user = false;   // allocated by the ranc_set_allocator callback (freed by it too)
};

}  // namespace ranc

struct ranc_group;

struct ranc_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  void* (*user_alloc)(size_t, void*) = nullptr;
  void (*user_free)(void*, void*) = nullptr;
  void* user = nullptr;
  std::string err;
  ranc::Compiled net;
  // device: compiled network
  ranc::DevBuf d_xp, d_wp, d_pword, d_prm, d_route, d_inl, d_has_in, d_init, d_wfold, d_route_tc, d_runs, d_nruns, d_wflags_tc, d_incoming,
      d_word_runs;
  int num_sms = 148;
  // device: state
  ranc::DevBuf d_pot, d_ring, d_counts, d_lines, d_stage, d_raster;
  // inputs from pinned host memory: H2D on a copy stream into one of two
  // staging buffers, overlapping the work already queued on the context stream
  ranc::DevBuf d_stage2;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied = nullptr, ev_stage_free[2] = {nullptr, nullptr};
  int stage_flip = 0;
  bool fresh = false;            // no tick since the last reset: d_pot is stale, potentials = init
  int64_t S = 0, first_sample = 0;
  int64_t Sr = 0;                // S rounded up to 64
  int32_t T_in = 0;
  bool have_inputs = false;
  int64_t now = 0;
  int32_t sample_tile = 0;       // in use (set by ranc_run_ticks)
  int32_t sample_tile_opt = 0;   // RANC_OPT_SAMPLE_TILE, 0 = automatic
  int32_t input_decode = 1;      // RANC_OPT_INPUT_DECODE
  int32_t pdl = 1;               // programmatic dependent launch of per-tick tensor-core launches
                                 // (RANC_DEBUG_NO_PDL=1 disables it, for timing comparisons)
  int32_t stream_opt = 0;        // RANC_OPT_STREAM: 0 auto, 1 off, 2 on
  int32_t kernel = 0;            // RANC_OPT_KERNEL request: 0 auto, 1 popcount, 2 tensor core
  int32_t kernel_active = 1;     // latched at every reset (the potential layout depends on it)
  int32_t ring_layout = 0;       // RANC_OPT_RING_LAYOUT request: 0 auto, 1 sample-major, 2 word-major
  bool ring_wmajor = false;      // latched at every reset: tensor-core ring word-major [Rp][G][W][Sr]
  int64_t launches = 0;
  int64_t device_bytes = 0;
  uint32_t trace_flags = 0;
  int64_t raster_t0 = 0, raster_ticks = 0;
  // multi-GPU
  void* nccl_comm = nullptr;
  int world = 1, rank = 0;
  int shard_mode = 0;            // RANC_SHARD_SAMPLES or RANC_SHARD_CORES
  int32_t c_lo = 0, G_loc = 0;   // local core range (G_loc = G unless core-sharded)
  ranc_group* group = nullptr;   // loopback group (several contexts, one process)
  bool group_broken = false;     // a member of the loopback group was destroyed
  // core-sharded exchange
  std::vector<std::vector<int32_t>> send_cores, recv_cores;  // per peer: local / global core ids
  std::vector<int64_t> send_off, recv_off;                   // per peer, in u32 words
  ranc::DevBuf d_fired, d_exports, d_send, d_recv, d_send_list, d_recv_list, d_recv_peer;
  ranc::DevBuf d_gsend, d_grecv;   // sample-sharded gather: padded shard, root's [world][Smax][C]
  int64_t n_send_words = 0, n_recv_words = 0, n_recv_rows = 0;
  int64_t exchange_bytes = 0;    // bytes sent per tick (introspection)
  ranc::DevBuf d_dbg;            // RANC_DEBUG_TIMELINE
  // tensor-core path: input decode (once per ranc_load_inputs)
  ranc::DevBuf d_inw, d_inslot, d_slot_core;
  // tensor-core path: history scheduler (latched at reset, RANC_OPT_RING_LAYOUT 3)
  ranc::DevBuf d_hist, d_hpos, d_hbase, d_hax;
  bool ring_pull = false;
  // tensor-core path: compact operand (RANC_OPT_OPERAND; chosen per launch)
  ranc::DevBuf d_xbits, d_wq, d_tsel;
  int32_t operand = 0;           // RANC_OPT_OPERAND request: 0 auto, 1 folded, 2 compact
  int32_t operand_used = 0;      // operand of the last tensor-core launch (1 folded, 2 compact)
  // cost-balanced work partition of the per-tick tensor-core launches
  ranc::DevBuf d_part, d_cta_ns;
  int64_t part_key = -1;         // (items, grid) the partition was made for
  int64_t part_ticks = 0;        // ticks run with it
  bool part_fresh = false;       // a rebalance kernel was queued after the last tick (no PDL for the next)
  // RANC_TRACE_STATE_DIGEST
  ranc::DevBuf d_spkin, d_digest, d_perm_dig;
  int32_t perm_dig_kernel = 0;   // kernel whose axon order d_perm_dig holds
  int32_t n_inslots = 0;
  bool inw_valid = false;
  int32_t fault = 0;             // RANC_OPT_DEBUG_FAULT (mutation tests only)
};

struct ranc_group {
  std::vector<ranc_ctx*> ctxs;
};

namespace ranc {
enum { RANC_KERNEL_AUTO = 0, RANC_KERNEL_POPC = 1, RANC_KERNEL_TC = 2 };
// comm.cpp
struct CoreShardPlan {
  int32_t c_lo = 0, G_loc = 0;                   // this rank's cores [c_lo, c_lo + G_loc)
  std::vector<uint8_t> exports;                  // [G] core has a route into another rank's band
  std::vector<std::vector<int32_t>> send_cores;  // per peer: local ids of the cores whose fired bits it needs
  std::vector<std::vector<int32_t>> recv_cores;  // per peer: global ids of the peer's cores routing here
};
ranc_status plan_core_shards(const Compiled& c, int world, int rank, CoreShardPlan* out, std::string* err);
ranc_status setup_core_shards(ranc_ctx* ctx, int world, int rank);
void clear_core_shards(ranc_ctx* ctx);
ranc_status alloc_exchange(ranc_ctx* ctx);
ranc_status exchange_nccl(ranc_ctx* ctx, int64_t t);
ranc_status exchange_loopback(ranc_group* g, int64_t t);
// compile.cpp
ranc_status validate_and_compile(const ranc_network_desc* d, Compiled* out, std::string* err);
// tick.cu
cudaError_t launch_reset(ranc_ctx* ctx);
cudaError_t transpose_lines(ranc_ctx* ctx, const uint32_t* staging);

cudaError_t launch_one_tick(ranc_ctx* ctx);          // the tick kernel for tick ctx->now (no exchange)
cudaError_t launch_pack(ranc_ctx* ctx);              // core-sharded: fired rows -> send buffer
cudaError_t launch_unpack(ranc_ctx* ctx, int64_t t); // core-sharded: received rows -> local rings
int choose_sample_tile(const Compiled& n, int64_t S);
int pieces_template(int E);
// tick_tc.cu
int tc_tile();
size_t tc_smem_bytes(const Compiled& n);
size_t tc_smem_bytes_pull(const Compiled& n);
size_t tc_smem_bytes_comp(const Compiled& n, bool pull);
cudaError_t launch_tick_tc(ranc_ctx* ctx, TickParams p);
cudaError_t decode_inputs_tc(ranc_ctx* ctx);
bool stream_eligible(ranc_ctx* ctx, int64_t num_ticks);
bool tc_multi_eligible(const ranc_ctx* ctx, int64_t num_ticks);
cudaError_t launch_tc_multi(ranc_ctx* ctx, TickParams p, int64_t num_ticks);
cudaError_t launch_digest(ranc_ctx* ctx, int64_t tick_index);
cudaError_t launch_stream(ranc_ctx* ctx, int64_t num_ticks);
// api.cpp
ranc_status dev_alloc(ranc_ctx* ctx, DevBuf* b, size_t bytes);
void dev_free(ranc_ctx* ctx, DevBuf* b);
ranc_status set_cuda_error(ranc_ctx* ctx, cudaError_t e, const char* where);
void set_load_error(const std::string& m);   // the thread-local message of ranc_last_error(NULL)
}  // namespace ranc
