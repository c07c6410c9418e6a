/*
 * ranc.h -- C ABI of the B200-native tick-accurate RANC core-update library
 * (libranc.so, built from paper_2404_16208_b200/csrc).
 *
 * The library simulates the method of GPU-RANC (Hassan et al., arXiv
 * 2404.16208): a 2-D mesh of neuromorphic cores (section II), each with
 * axons, a binary synaptic crossbar, LIF neurons whose weight is selected by
 * the axon type ("sets of four weights per neuron"), a scheduler ring
 * of future input spikes (section III-E) and a router that writes
 * each spike into the destination core's scheduler at (tick offset, axon)
 * (section III-D).  One call to ranc_run_ticks advances every core
 * of every sample by whole ticks of Algorithm 1.
 *
 * Citations: "P:NN" = line NN of the paper text, "S:NN" = line NN
 * of SPEC.md; G-numbers are the readings listed in DESIGN.md section 3.
 *
 * Conventions (all entry points):
 *   - every call returns ranc_status; RANC_OK == 0.  On failure a located,
 *     human-readable message is available from ranc_last_error(ctx) (or
 *     ranc_last_error(NULL) for a failed ranc_load_network).
 *   - host arrays passed in are BORROWED for the duration of the call only
 *     (the library copies what it needs); output buffers are caller-allocated
 *     with an explicit element count, a wrong count returns RANC_E_SIZE.
 *   - the library owns the context and all device memory (cudaMallocAsync on
 *     the context stream, or the allocator installed by ranc_set_allocator).
 *   - work is stream-ordered on the context stream; calls that return data
 *     to the host synchronise that stream.  Asynchronous kernel failures are
 *     reported (RANC_E_CUDA) by the next synchronising call.
 *   - results are bit-identical regardless of sample tiling, GPU count, or
 *     splitting ranc_run_ticks into pieces ("RANC contains no
 *     stochastic effects").
 *   - one context per host thread at a time; distinct contexts are
 *     independent.  There is no CPU fallback: without a usable CUDA device
 *     ranc_load_network fails with RANC_E_CUDA.
 */
#ifndef RANC_H
#define RANC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RANC_ABI_VERSION 1

typedef struct ranc_ctx ranc_ctx;

typedef enum {
  RANC_OK = 0,
  RANC_E_ARG = 1,       /* NULL pointer / bad argument                          */
  RANC_E_CONFIG = 2,    /* unsupported configuration (counts out of range, G20) */
  RANC_E_BITWIDTH = 3,  /* a value does not fit its signed bitwidth    */
  RANC_E_RANGE = 4,     /* type >= K, axon >= A, delay not in [1,D], class >= C,
                           line >= I, reset_mode/dest_kind invalid, padding bit */
  RANC_E_OFFGRID = 5,   /* route destination outside the grid (G17)      */
  RANC_E_BOUND = 6,     /* the int32 accumulator could overflow (G3)           */
  RANC_E_STATE = 7,     /* wrong call order (e.g. run before inputs)           */
  RANC_E_SIZE = 8,      /* caller buffer element count mismatch                */
  RANC_E_CUDA = 9,      /* CUDA error (message carries cudaGetErrorString)     */
  RANC_E_OOM = 10,      /* device allocation failed                            */
  RANC_E_NCCL = 11      /* NCCL error / comm not initialised                   */
} ranc_status;

/* Network description.  All arrays: host, caller-owned,
 * row-major, read during ranc_load_network only.  G = grid_w*grid_h; core
 * c = y*grid_w + x (P:61, 2-D mesh).  Ranges are validated; every violation
 * is reported with its location, e.g.
 *   "core (3,1) neuron 17: weight[2]=300 exceeds weight_bits=9".           */
typedef struct {
  int32_t abi_version;           /* RANC_ABI_VERSION                                  */
  int32_t grid_w, grid_h;        /* >= 1, G <= 65536                                  */
  int32_t axons, neurons;        /* A, N in [1, 1024] (configurable)     */
  int32_t num_types;             /* K in [1, 4] ("sets of four weights")        */
  int32_t max_delay;             /* D in [1, 15]: packet tick offsets 1..D (G6, G7)   */
  int32_t num_classes;           /* C >= 0 output-bus classes (G13)                   */
  int32_t num_lines;             /* I >= 0 external input lines (G8)                  */
  int32_t potential_bits, weight_bits, leak_bits, threshold_bits, reset_bits;
                                 /* each in [2, 16] (P:42 configurable bitwidths; G20) */
  const uint8_t*  axon_type;     /* [G][A]  < K (axon type per core, G12)       */
  const int32_t*  input_line;    /* [G][A]  -1 or [0, I): line feeding this axon      */
  const uint32_t* crossbar;      /* [G][N][ceil(A/32)]: bit (a&31) of word a>>5 is the
                                    synaptic connection axon a -> neuron n;
                                    bits >= A must be 0                               */
  const int16_t*  weight;        /* [G][N][K]   fits weight_bits                      */
  const int16_t*  leak;          /* [G][N]      fits leak_bits                        */
  const int16_t*  pos_threshold; /* [G][N]      fits threshold_bits (fire iff v >= it, G1) */
  const int16_t*  neg_threshold; /* [G][N]      fits threshold_bits (v < it: negative reset, G4) */
  const int16_t*  reset_potential;   /* [G][N]  fits reset_bits (R; -R on the negative side) */
  const int16_t*  initial_potential; /* [G][N]  fits potential_bits (G15)             */
  const uint8_t*  reset_mode;    /* [G][N] 0 absolute (R / -R), 1 linear (v - threshold) */
  const uint8_t*  dest_kind;     /* [G][N] 0 none, 1 route, 2 output bus (G13, G16)   */
  const int16_t*  dest_dx;       /* [G][N] route only: destination core (x+dx, y+dy)  */
  const int16_t*  dest_dy;       /*        must be on the grid (G17)                  */
  const int16_t*  dest_axon;     /* [G][N] route only: [0, A)                         */
  const uint8_t*  dest_delay;    /* [G][N] route only: [1, D] ticks (P:154 tick offset) */
  const uint16_t* out_class;     /* [G][N] output only: [0, C)                        */
} ranc_network_desc;

/* Input stream of S_local independent samples (G14). */
typedef struct {
  int32_t  num_samples;          /* S_local >= 1                                      */
  int64_t  first_sample;         /* global index of local sample 0 (sharding, traces) */
  int32_t  num_input_ticks;      /* T_in >= 0; ticks >= T_in receive no input         */
  const uint32_t* line_bits;     /* [S_local][T_in][ceil(I/32)]: bit i of row (s,t) =
                                    line i spikes ARRIVE at tick t (G8; Alg. 1 l.5-9,
                                    P:82-90).  May be NULL when I == 0 or T_in == 0.  */
} ranc_inputs_desc;

/* Validate and compile the network (per-core axon type-sort, route words,
 * bound check) and upload it once to `cuda_device` ("allocated and
 * copied to the GPU global memory once").  *out receives the new context.
 * Errors: RANC_E_ARG/CONFIG/BITWIDTH/RANGE/OFFGRID/BOUND/CUDA/OOM. */
ranc_status ranc_load_network(const ranc_network_desc* net, int cuda_device, ranc_ctx** out);

/* Copy the input stream to the device and reset the simulation state:
 * potentials = initial_potential, scheduler rings empty, class counts 0,
 * tick = 0 (Alg. 1 l.1).  Stream-ordered; the host array is staged
 * before the call returns.  From page-locked (pinned) host memory the copy
 * runs on the context's copy stream into one of two staging buffers, so it
 * overlaps work still queued on the context stream (a running batch) and the
 * call returns as soon as the copy is done; from pageable memory the call
 * waits for the context stream.  Errors: RANC_E_ARG/RANGE/SIZE/CUDA/OOM. */
ranc_status ranc_load_inputs(ranc_ctx* ctx, const ranc_inputs_desc* in);

/* Reset the state exactly as ranc_load_inputs does, keeping the inputs
 * already on the device.  Errors: RANC_E_STATE (no inputs loaded). */
ranc_status ranc_reset_state(ranc_ctx* ctx);

/* Advance every core of every sample by num_ticks >= 0 ticks of Alg. 1
 * (P:77-113): scheduler read (l.3-5), input injection (l.6-9), synaptic
 * integration + leak/threshold/reset (l.10-14), routing of fired spikes into
 * destination scheduler rows or the output bus (l.15-20).  Stream-ordered and
 * asynchronous; resumable (run(a); run(b) == run(a+b)).
 * Errors: RANC_E_STATE (no inputs), RANC_E_ARG (num_ticks < 0), RANC_E_CUDA. */
ranc_status ranc_run_ticks(ranc_ctx* ctx, int64_t num_ticks);

/* Current tick (number of ticks executed since the last reset). */
ranc_status ranc_now(const ranc_ctx* ctx, int64_t* tick);

/* Output-bus spike counts per (sample, class) (P:250 output file; G13):
 * counts[S_local][C] int32.  n must equal S_local*C.  Synchronises. */
ranc_status ranc_read_outputs(ranc_ctx* ctx, int32_t* counts, size_t n);

/* Parity / debug readers, in the ORIGINAL axon and neuron order.
 * Potentials: [S_local][G][N] int32.  Pending: [S_local][G][D][ceil(A/32)]
 * u32 bitmaps, row j = spikes due at tick now+j (j = 0..D-1).  Synchronise. */
ranc_status ranc_read_potentials(ranc_ctx* ctx, int32_t* pot, size_t n);
ranc_status ranc_read_pending(ranc_ctx* ctx, uint32_t* bits, size_t n);

/* Tracing.  flags: RANC_TRACE_SPIKE_RASTER records, for every tick of each
 * subsequent ranc_run_ticks call, the fired bit of every neuron:
 * raster [ticks][S_local][G][ceil(N/32)] u32 (bit n&31 of word n>>5).
 * RANC_TRACE_OUTPUT_EVENTS is derived from the raster: records of 5 int64
 * (sample, tick, x, y, neuron) of output-bus spikes, canonical order
 * (sample, tick, y, x, neuron).  Reading refers to the most recent
 * ranc_run_ticks call.  *written receives the bytes required/written;
 * a too-small buffer returns RANC_E_SIZE with *written = bytes required.
 * RANC_TRACE_STATE_DIGEST (per-tick parity at sizes where
 * state dumps are too large): uint64 [ticks][S_local], per (tick, sample) the
 * mod-2^64 sum over this context's cores of mix(((c*N+n)<<32) | (u32)pot)
 * for every neuron after the tick, mix(K1 ^ (c*N+n)) for every neuron that
 * fired in it and mix(K2 ^ (c*A+a)) for every axon spike it integrated
 * (original indices; mix = SplitMix64 finaliser, K1 = 0x243F6A8885A308D3,
 * K2 = 0x13198A2E03707344).  Sums over core shards add up to the whole
 * network's digest.  Forces per-tick launches while enabled. */
#define RANC_TRACE_SPIKE_RASTER 1u
#define RANC_TRACE_OUTPUT_EVENTS 2u
#define RANC_TRACE_STATE_DIGEST 4u
ranc_status ranc_set_trace(ranc_ctx* ctx, uint32_t flags);
ranc_status ranc_read_trace(ranc_ctx* ctx, uint32_t kind, void* buf, size_t bytes, size_t* written);

/* Runtime plumbing.  ranc_set_stream: use this cudaStream_t for all work
 * (e.g. torch.cuda.current_stream().cuda_stream); NULL restores the context's
 * own stream.  Switching synchronises the previous stream first, so work and
 * stream-ordered allocations queued there never race the new stream.  Buffers
 * of a user allocator are released only after the context stream has drained.  ranc_set_allocator: device allocations made from now on use
 * alloc(bytes, user) / dealloc(ptr, user) (e.g. the torch caching allocator);
 * must be called before ranc_load_inputs. */
ranc_status ranc_set_stream(ranc_ctx* ctx, void* cuda_stream);
ranc_status ranc_set_allocator(ranc_ctx* ctx, void* (*alloc)(size_t, void*),
                               void (*dealloc)(void*, void*), void* user);

/* Tuning knobs (no effect on results).  RANC_OPT_SAMPLE_TILE: samples per CTA
 * of the popcount tick kernel (default chosen from S).  RANC_OPT_INPUT_DECODE:
 * tensor-core kernel only -- 1 (default): decode the input lines into per-core
 * scheduler words once per ranc_load_inputs (Alg. 1 l.1, "input decode";
 * T_in x input cores x S x ceil(A/32) x 4 bytes of device memory, skipped when
 * that exceeds a quarter of the free memory); 0: gather the line runs every
 * tick.  Takes effect at the next ranc_load_inputs / ranc_reset_state.
 * RANC_OPT_KERNEL: 0 automatic (tensor core when the network is eligible,
 * unless S < 64 and cores x S <= 592, where the popcount path's streaming
 * launch is faster), 1 popcount, 2 tensor core (see ranc_info.kernel).
 * Tensor-core eligibility: N <= 1024 neurons and A <= 1024 axons (cores with
 * more than 256 neurons or 32*ceil(A/32)*Npad > 64 KB run in neuron groups
 * of 256 or 128 rows, one Wfold operand each, split into K chunks of 512
 * axons beyond 512), weights of any valid width (-128..127: one s8 operand;
 * 16-bit: w = 256*hi + lo, a u8 low byte and an s8 high byte, two MMAs),
 * and the kernel's shared memory within 227 KB (16-bit weights on more than
 * ~800 axons do not fit); otherwise RANC_E_CONFIG for value 2. */
#define RANC_OPT_SAMPLE_TILE 1
#define RANC_OPT_INPUT_DECODE 2
/* RANC_OPT_STREAM (streaming mode: one long stream of inputs,
 * ~1 image per tick): 0 (default) automatic -- when the popcount
 * kernel is active, the context is not core-sharded and a tick has few
 * (core, sample-tile) items, a ranc_run_ticks call of >= 2 ticks runs as ONE
 * cooperative launch whose grid barrier is the tick barrier;
 * 1 always per-tick launches; 2 always the cooperative launch when possible.
 * Results are identical either way. */
#define RANC_OPT_STREAM 4
#define RANC_OPT_KERNEL 3
/* RANC_OPT_RING_LAYOUT (tensor-core kernel only; device memory layout of the
 * scheduler rings, Alg. 1 l.3-5 and l.15-20, P:79-82 / P:102-110): 0 (default)
 * automatic -- the history scheduler (3) when more than 1/3 of all neurons
 * route to their own destination word (the random mesh of config 5, VMM)
 * and a tick has more than two 64-sample tiles per SM (per-tick launches);
 * else word-major when more than 2/3 do; otherwise sample-major (layered
 * MNIST nets deposit whole words together); 1 sample-major
 * [Rp][G][S][W]; 2 word-major [Rp][G][W][S] (a warp's deposits for 32 samples
 * of one route hit one 128-byte line); 3 history scheduler: no ring -- every
 * routing neuron owns a position in its destination core's list and each
 * tick stores its fired bits there, in the history slot of the arrival tick
 * t + delay; every core reads its contiguous positions of slot t with one
 * bulk copy (RANC_E_CONFIG when neuron groups or core sharding are in use).  Takes
 * effect at the next ranc_load_inputs / ranc_reset_state.  Results are
 * identical either way. */
#define RANC_OPT_RING_LAYOUT 5
/* RANC_OPT_DEBUG_FAULT (mutation tests only, "deliberately
 * fault-injected parallel build (skip barrier) -> FAIL with located
 * divergence"; CHANGES RESULTS): 0 (default) none; 1 the cooperative
 * multi-tick launches skip their per-tick grid barrier (the tick barrier a7,
 * P:70); 2 every route of delay >= 2 delivers one tick early (a wrong
 * scheduler offset).  Parity tests must fail with either set. */
#define RANC_OPT_DEBUG_FAULT 6
/* RANC_OPT_OPERAND (tensor-core kernel, per-tick launches; the integration
 * operand Wfold[n][a'] = conn[n][a'] * w[n][type(a')]): 0 (default)
 * automatic -- compact when eligible, the history scheduler is in use and
 * every core has at most two 64-sample tiles (S <= 128: the 64 KB folded
 * operand would be re-read from HBM for every 64 samples); 1 folded: the host-folded int8 operand is loaded per
 * core; 2 compact: the crossbar bits, the K weights per neuron and the axon
 * types (9.3 KB per 256 x 256 core) are read and expanded on chip
 * (RANC_E_CONFIG unless the weights fit int8 and the cores have at most 256
 * neurons and 256 axons).  Results are identical either way. */
#define RANC_OPT_OPERAND 7
ranc_status ranc_set_option(ranc_ctx* ctx, int option, int64_t value);

/* Introspection of the compiled network and of the last run. */
typedef struct {
  int32_t grid_w, grid_h, axons, neurons, num_types, max_delay, num_classes, num_lines;
  int32_t ring_rows;          /* physical ring rows Rp = next_pow2(D+1)                 */
  int32_t ring_words;         /* u32 words per ring row, ceil(A/32)                     */
  int32_t pieces;             /* popcount pieces per neuron after the type-sort         */
  int32_t sample_tile;        /* samples per CTA in use                                 */
  int64_t num_samples;        /* S_local                                                */
  int64_t device_bytes;       /* device memory held by the context                      */
  int64_t kernel_launches;    /* kernels launched by the library since load             */
  int32_t kernel;             /* kernel variant in use: 1 popcount, 2 tensor core       */
  int32_t core_lo;            /* first global core simulated by this context            */
  int32_t cores_local;        /* number of cores simulated by this context              */
  int32_t shard_mode;         /* RANC_SHARD_* (0 without a communicator)                */
  int64_t exchange_bytes;     /* core-sharded: bytes sent per tick                      */
  int32_t ring_layout;        /* scheduler ring layout in use: 1 sample-major, 2 word-major (RANC_OPT_RING_LAYOUT) */
  int32_t operand;            /* operand of the last tensor-core launch: 1 folded, 2 compact, 0 none (RANC_OPT_OPERAND) */
} ranc_info;
ranc_status ranc_get_info(const ranc_ctx* ctx, ranc_info* info);

/* Multi-GPU (one process per GPU).
 *
 * ranc_comm_init joins an NCCL communicator from a 128-byte ncclUniqueId
 * (distributed by the caller, e.g. over torch.distributed), `world` ranks,
 * this `rank`.  Modes:
 *   RANC_SHARD_SAMPLES: every rank simulates its own samples of the
 *     replicated network (independent simulations, G14); no collective on
 *     the tick path.
 *   RANC_SHARD_CORES: every rank simulates the cores of a band of grid rows
 *     (rows [r*H/world, (r+1)*H/world)) for ALL samples.  After every tick the
 *     fired bits of cores whose routes cross a band boundary are exchanged
 *     with grouped ncclSend/ncclRecv and applied to the receivers' scheduler
 *     rows (Alg. 1 l.15-20).  Must be called before
 *     ranc_load_inputs.  The readers (potentials, pending, outputs, trace)
 *     then cover the local cores only ([S][G_local]..., local output counts);
 *     ranc_get_info reports core_lo / cores_local.
 * ranc_gather_outputs: every rank calls it, with the same n.  Sample mode:
 * the ranks hold the contiguous shards of S_total = n / C samples (sizes
 * differ by at most one, lower ranks first: rank r owns [r*b + min(r, m),
 * ...) with b = S_total / world, m = S_total % world, and its
 * ranc_inputs_desc.first_sample says so); every rank pads its counts to
 * ceil(S_total / world) rows and ONE ncclGather delivers them to `root`, which
 * receives the class counts of all samples in order ([S_total][C]) in
 * counts_global (may be NULL off-root).  A rank whose shard differs returns
 * RANC_E_SIZE naming both ranges.  Core mode: n = S*C; `root` receives the
 * element-wise sum ([S][C]) of one ncclReduce.  Synchronises.
 * Errors: RANC_E_NCCL, RANC_E_STATE, RANC_E_SIZE, RANC_E_ARG. */
#define RANC_SHARD_SAMPLES 0
#define RANC_SHARD_CORES 1
ranc_status ranc_comm_init(ranc_ctx* ctx, const void* nccl_unique_id, int world, int rank, int mode);
ranc_status ranc_gather_outputs(ranc_ctx* ctx, int32_t* counts_global, size_t n, int root);
/* Fill a 128-byte buffer with a fresh ncclUniqueId (call on one rank). */
ranc_status ranc_comm_unique_id(void* out128);

/* Host-only planner of RANC_SHARD_CORES (no device needed; the same code
 * ranc_comm_init runs): validates and compiles `net`, then reports rank
 * `rank`'s band of cores [*core_lo, *core_lo + *cores_local) of `world` and
 * its per-tick exchange lists.  send_counts[p] / recv_counts[p] (caller
 * arrays of `world` entries) receive the list lengths; send_cores receives,
 * peer by peer, the LOCAL ids of this rank's cores with a route into peer
 * p's band (their fired bits are sent to p every tick, Alg. 1 l.15-20,
 * P:102-110), recv_cores the GLOBAL ids of peer p's cores with a route into
 * this band.  Capacities are in entries; too small -> RANC_E_SIZE (counts
 * still written).  Errors as ranc_load_network, message via
 * ranc_last_error(NULL). */
ranc_status ranc_plan_core_shards(const ranc_network_desc* net, int world, int rank, int32_t* core_lo,
                                  int32_t* cores_local, int32_t* send_counts, int32_t* recv_counts,
                                  int32_t* send_cores, size_t send_cap, int32_t* recv_cores, size_t recv_cap);

/* Loopback group: n contexts of this process (same device, same network)
 * act as the n ranks of a core-sharded run, exchanging spikes with device
 * copies instead of NCCL (mode must be RANC_SHARD_CORES).  Such contexts are
 * advanced together with ranc_run_ticks_loopback (ranc_run_ticks on a member
 * returns RANC_E_STATE); everything else is per context as above. */
ranc_status ranc_comm_init_loopback(ranc_ctx* const* ctxs, int n, int mode);
ranc_status ranc_run_ticks_loopback(ranc_ctx* const* ctxs, int n, int64_t num_ticks);

/* Last error message of ctx, or (ctx == NULL) of the calling thread's last
 * failed ranc_load_network.  Never NULL. */
const char* ranc_last_error(const ranc_ctx* ctx);

/* Release the context and all its device memory.  NULL is a no-op. */
void ranc_destroy(ranc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* RANC_H */
