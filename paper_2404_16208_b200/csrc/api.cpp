// api.cpp -- the extern "C" entry points of include/ranc.h: context lifetime,
// device memory, call-order checks, readback (permutations undone) and
// tracing.  Every step of the simulation itself runs in tick.cu kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "internal.h"

namespace {
thread_local std::string g_load_err;
}

namespace ranc {

void set_load_error(const std::string& m) { g_load_err = m; }

ranc_status set_cuda_error(ranc_ctx* ctx, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  if (ctx) ctx->err = m;
  else g_load_err = m;
  return (e == cudaErrorMemoryAllocation) ? RANC_E_OOM : RANC_E_CUDA;
}

ranc_status dev_alloc(ranc_ctx* ctx, DevBuf* b, size_t bytes) {
  dev_free(ctx, b);
  if (bytes == 0) return RANC_OK;
  void* p = nullptr;
  if (ctx->user_alloc) {
    p = ctx->user_alloc(bytes, ctx->user);
    if (!p) {
      ctx->err = "user allocator returned NULL for " + std::to_string(bytes) + " bytes";
      return RANC_E_OOM;
    }
  } else {
    cudaError_t e = cudaMallocAsync(&p, bytes, ctx->stream);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "cudaMallocAsync");
  }
  b->p = p;
  b->bytes = bytes;
  b->user = ctx->user_alloc != nullptr;
  ctx->device_bytes += (int64_t)bytes;
  return RANC_OK;
}

void dev_free(ranc_ctx* ctx, DevBuf* b) {
  if (!b->p) return;
  // a buffer is released by the allocator that made it (network buffers are
  // allocated before ranc_set_allocator may be called).  A user allocator
  // (e.g. torch's caching allocator) may hand the block to someone else at
  // once, so the context's queued work that can still touch it must finish
  // first; cudaFreeAsync is stream-ordered on the context stream, which every
  // user of the buffer ran on (ranc_set_stream drains the previous stream).
  if (b->user) {
    cudaStreamSynchronize(ctx->stream);
    ctx->user_free(b->p, ctx->user);
  } else {
    cudaFreeAsync(b->p, ctx->stream);
  }
  ctx->device_bytes -= (int64_t)b->bytes;
  b->p = nullptr;
  b->bytes = 0;
}

}  // namespace ranc

using namespace ranc;

#define CK(call, where)                                         \
  do {                                                          \
    cudaError_t _e = (call);                                    \
    if (_e != cudaSuccess) return set_cuda_error(ctx, _e, where); \
  } while (0)

#define TRY(call)                      \
  do {                                 \
    ranc_status _s = (call);           \
    if (_s != RANC_OK) return _s;      \
  } while (0)

namespace {

template <class T>
ranc_status upload(ranc_ctx* ctx, DevBuf* b, const std::vector<T>& v) {
  TRY(dev_alloc(ctx, b, v.size() * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpyAsync(b->p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream),
                     "upload");
  return RANC_OK;
}

ranc_status check_ctx(const ranc_ctx* ctx) { return ctx ? RANC_OK : RANC_E_ARG; }

ranc_status sync(ranc_ctx* ctx, const char* where) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, where);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(ctx, e, where);
  return RANC_OK;
}

void free_all(ranc_ctx* ctx) {
  DevBuf* bufs[] = {&ctx->d_xp, &ctx->d_wp, &ctx->d_pword, &ctx->d_prm, &ctx->d_route, &ctx->d_inl,
                    &ctx->d_has_in, &ctx->d_init, &ctx->d_wfold, &ctx->d_route_tc, &ctx->d_runs,
                    &ctx->d_nruns, &ctx->d_wflags_tc, &ctx->d_incoming, &ctx->d_word_runs, &ctx->d_pot, &ctx->d_ring, &ctx->d_counts, &ctx->d_lines,
                    &ctx->d_stage, &ctx->d_stage2, &ctx->d_raster, &ctx->d_fired, &ctx->d_exports, &ctx->d_send, &ctx->d_recv,
                    &ctx->d_send_list, &ctx->d_recv_list, &ctx->d_dbg, &ctx->d_inw, &ctx->d_inslot,
                    &ctx->d_slot_core, &ctx->d_spkin, &ctx->d_digest, &ctx->d_perm_dig, &ctx->d_gsend, &ctx->d_grecv,
                    &ctx->d_hist, &ctx->d_hpos, &ctx->d_hbase, &ctx->d_hax, &ctx->d_xbits, &ctx->d_wq, &ctx->d_tsel,
                    &ctx->d_part, &ctx->d_cta_ns};
  for (DevBuf* b : bufs) dev_free(ctx, b);
}

}  // namespace

namespace {

// Tensor-core path input decode (Alg. 1 l.1): lines -> per-core ring words,
// kept while the inputs stay loaded.  Input cores with the same line -> axon
// map (identical runs) share one decoded slot.  Skipped (the kernel gathers
// the line runs every tick instead) when the decoded array would exceed its
// budget.
ranc_status prepare_inputs_tc(ranc_ctx* ctx) {
  const Compiled& c = ctx->net;
  if (ctx->inw_valid || !ctx->input_decode || ctx->kernel_active != RANC_KERNEL_TC || ctx->T_in == 0) return RANC_OK;
  std::vector<int32_t> inslot(ctx->G_loc, -1), slot_core;
  std::map<std::vector<int32_t>, int32_t> seen;
  for (int g = 0; g < ctx->G_loc; ++g) {
    const int core = ctx->c_lo + g;
    const int nr = c.nruns[core];
    if (nr == 0) continue;
    std::vector<int32_t> key;
    key.reserve(2 * nr + c.W);
    for (int q = 0; q < nr; ++q) {
      key.push_back(c.runs[(size_t)core * c.rmax + q].x);
      key.push_back(c.runs[(size_t)core * c.rmax + q].y);
    }
    for (int w = 0; w < c.W; ++w) key.push_back(c.word_runs[(size_t)core * c.W + w]);
    auto it = seen.find(key);
    if (it == seen.end()) {
      it = seen.emplace(std::move(key), (int32_t)slot_core.size()).first;
      slot_core.push_back(core);
    }
    inslot[g] = it->second;
  }
  ctx->n_inslots = (int32_t)slot_core.size();
  if (slot_core.empty()) return RANC_OK;
  const size_t bytes = (size_t)ctx->T_in * slot_core.size() * ctx->Sr * c.W * 4;
  if (ctx->d_inw.bytes != bytes) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (bytes > (free_b + ctx->d_inw.bytes) / 4) return RANC_OK;   // keep the per-tick gather path
    TRY(dev_alloc(ctx, &ctx->d_inw, bytes));
  }
  TRY(upload(ctx, &ctx->d_inslot, inslot));
  TRY(upload(ctx, &ctx->d_slot_core, slot_core));
  // rows s >= S of the last tile are never consumed (the kernel ORs i < ns*W)
  CK(decode_inputs_tc(ctx), "decode_inputs");
  ctx->inw_valid = true;
  return RANC_OK;
}

// The history scheduler needs the tensor-core path without neuron groups,
// all sources in this context (not core-sharded), and its staged positions
// within 227 KB of shared memory.
bool pull_eligible(const ranc_ctx* ctx) {
  const Compiled& c = ctx->net;
  return c.tc_ok && !c.tc_grp && ctx->shard_mode != RANC_SHARD_CORES && tc_smem_bytes_pull(c) <= 227 * 1024;
}

}  // namespace

extern "C" {

ranc_status ranc_load_network(const ranc_network_desc* net, int cuda_device, ranc_ctx** out) {
  g_load_err.clear();
  if (!out) {
    g_load_err = "out pointer is NULL";
    return RANC_E_ARG;
  }
  *out = nullptr;
  ranc_ctx* ctx = new (std::nothrow) ranc_ctx();
  if (!ctx) return RANC_E_OOM;
  // host-side validation first (located errors do not need a GPU)
  ranc_status s = validate_and_compile(net, &ctx->net, &g_load_err);
  if (s != RANC_OK) {
    delete ctx;
    return s;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    g_load_err = std::string("no CUDA device available (") + (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                 "); libranc has no CPU fallback";
    delete ctx;
    return RANC_E_CUDA;
  }
  if (cuda_device < 0 || cuda_device >= ndev) {
    g_load_err = "cuda_device " + std::to_string(cuda_device) + " out of range (" + std::to_string(ndev) + " devices)";
    delete ctx;
    return RANC_E_ARG;
  }
  ctx->device = cuda_device;
  e = cudaSetDevice(cuda_device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    set_cuda_error(nullptr, e, "ranc_load_network");
    delete ctx;
    return RANC_E_CUDA;
  }
  ctx->stream = ctx->own_stream;
  ctx->c_lo = 0;
  ctx->G_loc = ctx->net.G;
  const Compiled& c = ctx->net;
  s = upload(ctx, &ctx->d_xp, c.xp);
  if (!s) s = upload(ctx, &ctx->d_wp, c.wp);
  if (!s) s = upload(ctx, &ctx->d_pword, c.pword);
  if (!s) s = upload(ctx, &ctx->d_prm, c.prm);
  if (!s) s = upload(ctx, &ctx->d_route, c.route);
  if (!s) s = upload(ctx, &ctx->d_inl, c.inl);
  if (!s) s = upload(ctx, &ctx->d_has_in, c.has_in);
  if (!s) s = upload(ctx, &ctx->d_init, c.init);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_wfold, c.wfold);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_route_tc, c.route_tc);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_runs, c.runs);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_nruns, c.nruns);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_wflags_tc, c.wflags_tc);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_incoming, c.incoming);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_word_runs, c.word_runs);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_hpos, c.hpos);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_hbase, c.hbase);
  if (!s && c.tc_ok) s = upload(ctx, &ctx->d_hax, c.hax);
  if (!s && c.tc_comp_ok) s = upload(ctx, &ctx->d_xbits, c.xbits);
  if (!s && c.tc_comp_ok) s = upload(ctx, &ctx->d_wq, c.wq);
  if (!s && c.tc_comp_ok) s = upload(ctx, &ctx->d_tsel, c.tsel);
  if (!s) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device) == cudaSuccess && sms > 0)
      ctx->num_sms = sms;
  }
  if (!s) s = sync(ctx, "ranc_load_network");
  if (s) {
    g_load_err = ctx->err;
    free_all(ctx);
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return s;
  }
  *out = ctx;
  return RANC_OK;
}

ranc_status ranc_load_inputs(ranc_ctx* ctx, const ranc_inputs_desc* in) {
  TRY(check_ctx(ctx));
  if (!in) {
    ctx->err = "inputs descriptor is NULL";
    return RANC_E_ARG;
  }
  if (in->num_samples < 1 || in->num_input_ticks < 0) {
    ctx->err = "num_samples=" + std::to_string(in->num_samples) + " num_input_ticks=" +
               std::to_string(in->num_input_ticks) + ": need num_samples >= 1, num_input_ticks >= 0";
    return RANC_E_RANGE;
  }
  const Compiled& c = ctx->net;
  const size_t line_words = (size_t)in->num_samples * in->num_input_ticks * c.WI;
  if (line_words && !in->line_bits) {
    ctx->err = "line_bits is NULL but num_lines*num_input_ticks > 0";
    return RANC_E_ARG;
  }
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int64_t S = in->num_samples;
  const int64_t Sr = (S + 63) / 64 * 64;   // ring / line sample stride (TMA-aligned tiles)
  if (S != ctx->S || !ctx->d_pot.p) {
    // room for either potential layout: [G][S][Npad] or [G][nT][Npad][NT]
    TRY(dev_alloc(ctx, &ctx->d_pot, (size_t)ctx->G_loc * Sr * c.Npad * sizeof(int16_t)));
    // padding rows (samples >= S of the popcount layout) are never written;
    // zero them once so readback copies no uninitialised bytes (initcheck)
    CK(cudaMemsetAsync(ctx->d_pot.p, 0, ctx->d_pot.bytes, ctx->stream), "potential buffer clear");
    TRY(dev_alloc(ctx, &ctx->d_ring, (size_t)c.Rp * ctx->G_loc * Sr * c.W * sizeof(uint32_t)));
    TRY(dev_alloc(ctx, &ctx->d_counts, (size_t)S * c.C * sizeof(int32_t)));
  }
  const size_t dev_line_words = (size_t)in->num_input_ticks * Sr * c.WIp;
  if (ctx->d_lines.bytes != dev_line_words * sizeof(uint32_t)) TRY(dev_alloc(ctx, &ctx->d_lines, dev_line_words * 4));
  ctx->inw_valid = false;
  ctx->S = S;
  ctx->Sr = Sr;
  ctx->first_sample = in->first_sample;
  ctx->T_in = in->num_input_ticks;
  TRY(alloc_exchange(ctx));
  if (line_words) {
    // H2D into a staging buffer, then a device transpose to [T_in][S][WI].
    // The host buffer is borrowed for the call only.  From pinned memory the
    // copy runs on a copy stream into one of two staging buffers, so it
    // overlaps the batch still queued on the context stream (which waits for
    // it with an event), and the call returns when the copy is done -- not
    // when the previous batch is.  From pageable memory: copy, transpose, sync.
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, in->line_bits) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();   // (a pageable pointer may leave an error behind on old drivers)
    if (pinned) {
      if (!ctx->copy_stream) {
        CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
        CK(cudaEventCreateWithFlags(&ctx->ev_copied, cudaEventDisableTiming), "copy event");
        for (cudaEvent_t& e : ctx->ev_stage_free) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "copy event");
        CK(cudaEventRecord(ctx->ev_stage_free[0], ctx->stream), "copy event");
        CK(cudaEventRecord(ctx->ev_stage_free[1], ctx->stream), "copy event");
      }
      const int f = ctx->stage_flip;
      DevBuf* st = f ? &ctx->d_stage2 : &ctx->d_stage;
      if (st->bytes != line_words * sizeof(uint32_t)) {
        CK(cudaStreamSynchronize(ctx->copy_stream), "copy stream");
        TRY(dev_alloc(ctx, st, line_words * 4));   // stream-ordered on the context stream:
        CK(cudaEventRecord(ctx->ev_stage_free[f], ctx->stream), "ranc_load_inputs");   // (ordered below)
      }
      // the transpose that last read this staging buffer has run
      CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_stage_free[f], 0), "ranc_load_inputs");
      CK(cudaMemcpyAsync(st->p, in->line_bits, line_words * 4, cudaMemcpyHostToDevice, ctx->copy_stream),
         "ranc_load_inputs H2D");
      CK(cudaEventRecord(ctx->ev_copied, ctx->copy_stream), "ranc_load_inputs");
      CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied, 0), "ranc_load_inputs");
      CK(transpose_lines(ctx, (const uint32_t*)st->p), "transpose_lines");
      CK(cudaEventRecord(ctx->ev_stage_free[f], ctx->stream), "ranc_load_inputs");
      ctx->stage_flip ^= 1;
      CK(cudaEventSynchronize(ctx->ev_copied), "ranc_load_inputs H2D");
    } else {
      if (ctx->d_stage.bytes != line_words * sizeof(uint32_t)) TRY(dev_alloc(ctx, &ctx->d_stage, line_words * 4));
      CK(cudaMemcpyAsync(ctx->d_stage.p, in->line_bits, line_words * 4, cudaMemcpyHostToDevice, ctx->stream),
         "ranc_load_inputs H2D");
      CK(transpose_lines(ctx, (const uint32_t*)ctx->d_stage.p), "transpose_lines");
      CK(cudaStreamSynchronize(ctx->stream), "ranc_load_inputs sync");
    }
  }
  ctx->have_inputs = true;
  return ranc_reset_state(ctx);
}

ranc_status ranc_reset_state(ranc_ctx* ctx) {
  TRY(check_ctx(ctx));
  if (!ctx->have_inputs) {
    ctx->err = "ranc_reset_state before ranc_load_inputs";
    return RANC_E_STATE;
  }
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  CK(launch_reset(ctx), "reset kernel");
  // latch the kernel variant (the potential layout is re-initialised here)
  // automatic choice: the tensor-core path unless the batch is a few samples
  // of a small net (e.g. streaming, S = 1): then the popcount path runs all
  // ticks of a call in one cooperative launch (one (core, sample) per CTA)
  const bool tc_auto = ctx->kernel == 0 && !(ctx->S < 64 && (int64_t)ctx->G_loc * ctx->S <= 4 * 148);
  ctx->kernel_active = (ctx->kernel == RANC_KERNEL_POPC || (ctx->kernel == 0 && !tc_auto) || !ctx->net.tc_ok ||
                        tc_smem_bytes(ctx->net) > 227 * 1024)
                           ? RANC_KERNEL_POPC
                           : RANC_KERNEL_TC;
  // the history scheduler (layout 3) replaces the ring on request, and
  // automatically for networks with many per-neuron routes whose ticks run as
  // per-tick launches anyway (more than two 64-sample tiles per SM: no
  // cooperative multi-tick launch), e.g. config 5 (126 -> 97 us per tick)
  // and VMM-1024
  const int64_t tc_items = (int64_t)ctx->G_loc * ((ctx->S + tc_tile() - 1) / tc_tile());
  const bool pull = ctx->kernel_active == RANC_KERNEL_TC && pull_eligible(ctx) &&
                    (ctx->ring_layout == 3 ||
                     (ctx->ring_layout == 0 && ctx->net.tc_hist && tc_items > 2 * (int64_t)ctx->num_sms));
  const bool wmajor = ctx->kernel_active == RANC_KERNEL_TC &&
                      (pull || ctx->ring_layout == 2 || (ctx->ring_layout == 0 && ctx->net.tc_wmajor));
  if (wmajor != ctx->ring_wmajor) ctx->inw_valid = false;   // decoded inputs follow the ring layout
  ctx->ring_wmajor = wmajor;
  ctx->ring_pull = pull;
  if (pull) {
    // fired-bit history [Rp][nT][P][2] u32, empty (no spikes before tick 0)
    const size_t hb = (size_t)ctx->net.Rp * ((ctx->S + tc_tile() - 1) / tc_tile()) * ctx->net.hbase.back() * 8;
    if (ctx->d_hist.bytes != hb) TRY(dev_alloc(ctx, &ctx->d_hist, hb));
    CK(cudaMemsetAsync(ctx->d_hist.p, 0, hb, ctx->stream), "history clear");
  }
  TRY(prepare_inputs_tc(ctx));
  ctx->now = 0;
  ctx->raster_ticks = 0;
  return RANC_OK;
}

namespace {

ranc_status prepare_run(ranc_ctx* ctx, int64_t num_ticks) {
  if (num_ticks < 0) {
    ctx->err = "num_ticks < 0";
    return RANC_E_ARG;
  }
  if (!ctx->have_inputs) {
    ctx->err = "ranc_run_ticks before ranc_load_inputs";
    return RANC_E_STATE;
  }
  if (ctx->group_broken) {
    ctx->err = "a member of this loopback group was destroyed";
    return RANC_E_STATE;
  }
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->sample_tile = ctx->sample_tile_opt > 0 ? ctx->sample_tile_opt : choose_sample_tile(ctx->net, ctx->S);
  if (ctx->sample_tile > ctx->S) ctx->sample_tile = (int)ctx->S;
  if (ctx->trace_flags) {
    const size_t bytes = (size_t)num_ticks * ctx->S * ctx->G_loc * ctx->net.Wn * 4;
    if (ctx->d_raster.bytes < bytes) TRY(dev_alloc(ctx, &ctx->d_raster, bytes));
    if (bytes) CK(cudaMemsetAsync(ctx->d_raster.p, 0, bytes, ctx->stream), "raster clear");
    ctx->raster_t0 = ctx->now;
    ctx->raster_ticks = num_ticks;
    if (ctx->trace_flags & RANC_TRACE_STATE_DIGEST) {
      const Compiled& c = ctx->net;
      const size_t sp = (size_t)ctx->S * ctx->G_loc * c.W * 4;
      if (ctx->d_spkin.bytes < sp) TRY(dev_alloc(ctx, &ctx->d_spkin, sp));
      const size_t db = std::max<size_t>(8, (size_t)num_ticks * ctx->S * 8);
      if (ctx->d_digest.bytes < db) TRY(dev_alloc(ctx, &ctx->d_digest, db));
      // a' -> a of the active kernel's axon order
      if (!ctx->d_perm_dig.p || ctx->perm_dig_kernel != ctx->kernel_active) {
        TRY(upload(ctx, &ctx->d_perm_dig, ctx->kernel_active == RANC_KERNEL_TC ? c.perm_tc : c.perm));
        ctx->perm_dig_kernel = ctx->kernel_active;
      }
    }
  } else if (ctx->d_raster.p) {
    dev_free(ctx, &ctx->d_raster);
    ctx->raster_ticks = 0;
  }
  return RANC_OK;
}

}  // namespace

ranc_status ranc_run_ticks(ranc_ctx* ctx, int64_t num_ticks) {
  TRY(check_ctx(ctx));
  if (ctx->group) {
    ctx->err = "this context belongs to a loopback group: use ranc_run_ticks_loopback";
    return RANC_E_STATE;
  }
  TRY(prepare_run(ctx, num_ticks));
  const bool exchange = ctx->shard_mode == RANC_SHARD_CORES && ctx->nccl_comm && ctx->world > 1;
  const bool digest = (ctx->trace_flags & RANC_TRACE_STATE_DIGEST) != 0;
  if (!exchange && !digest && stream_eligible(ctx, num_ticks)) {
    // streaming mode: every tick of this call in one cooperative launch
    int64_t left = num_ticks;
    while (left > 0) {
      const int64_t chunk = std::min<int64_t>(left, 1 << 30);
      CK(launch_stream(ctx, chunk), "stream kernel launch");
      left -= chunk;
    }
    return RANC_OK;
  }
  for (int64_t i = 0; i < num_ticks; ++i) {
    const int64_t t = ctx->now;
    CK(launch_one_tick(ctx), "tick kernel launch");
    if (exchange) TRY(exchange_nccl(ctx, t));
    if (digest) CK(launch_digest(ctx, i), "digest kernel launch");
  }
  return RANC_OK;
}

ranc_status ranc_run_ticks_loopback(ranc_ctx* const* ctxs, int n, int64_t num_ticks) {
  if (!ctxs || n < 1 || !ctxs[0]) return RANC_E_ARG;
  ranc_group* g = ctxs[0]->group;
  if (!g || (int)g->ctxs.size() != n) {
    ctxs[0]->err = "contexts are not one loopback group";
    return RANC_E_STATE;
  }
  for (int i = 0; i < n; ++i)
    if (g->ctxs[i] != ctxs[i]) {
      ctxs[0]->err = "contexts must be passed in group (rank) order";
      return RANC_E_ARG;
    }
  for (int i = 0; i < n; ++i) {
    TRY(prepare_run(ctxs[i], num_ticks));
    if (ctxs[i]->now != ctxs[0]->now || ctxs[i]->S != ctxs[0]->S) {
      ctxs[0]->err = "loopback members must be at the same tick with the same samples";
      return RANC_E_STATE;
    }
  }
  // one stream for the whole group (the exchange orders the members); work
  // queued on the members' own streams (allocations, raster clears, input
  // decode, ring / count resets) is ordered before it with events
  std::vector<cudaStream_t> saved(n);
  for (int i = 1; i < n; ++i)
    if (ctxs[i]->stream != ctxs[0]->stream) {
      cudaEvent_t ev;
      cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventRecord(ev, ctxs[i]->stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ctxs[0]->stream, ev, 0);
      if (e == cudaSuccess) e = cudaEventDestroy(ev);
      if (e != cudaSuccess) return set_cuda_error(ctxs[i], e, "ranc_run_ticks_loopback (stream ordering)");
    }
  for (int i = 0; i < n; ++i) {
    saved[i] = ctxs[i]->stream;
    ctxs[i]->stream = ctxs[0]->stream;
  }
  ranc_status st = RANC_OK;
  for (int64_t k = 0; k < num_ticks && st == RANC_OK; ++k) {
    const int64_t t = ctxs[0]->now;
    for (int i = 0; i < n && st == RANC_OK; ++i) {
      cudaError_t e = launch_one_tick(ctxs[i]);
      if (e != cudaSuccess) st = set_cuda_error(ctxs[i], e, "tick kernel launch");
    }
    if (st == RANC_OK && n > 1) st = exchange_loopback(g, t);
    for (int i = 0; i < n && st == RANC_OK; ++i)
      if (ctxs[i]->trace_flags & RANC_TRACE_STATE_DIGEST) {
        cudaError_t e = launch_digest(ctxs[i], k);
        if (e != cudaSuccess) st = set_cuda_error(ctxs[i], e, "digest kernel launch");
      }
  }
  for (int i = 0; i < n; ++i) ctxs[i]->stream = saved[i];
  if (st == RANC_OK) {
    cudaError_t e = cudaStreamSynchronize(ctxs[0]->stream);
    if (e != cudaSuccess) st = set_cuda_error(ctxs[0], e, "ranc_run_ticks_loopback");
  }
  return st;
}

ranc_status ranc_now(const ranc_ctx* ctx, int64_t* tick) {
  if (!ctx || !tick) return RANC_E_ARG;
  *tick = ctx->now;
  return RANC_OK;
}

ranc_status ranc_read_outputs(ranc_ctx* ctx, int32_t* counts, size_t n) {
  TRY(check_ctx(ctx));
  if (!ctx->have_inputs) {
    ctx->err = "ranc_read_outputs before ranc_load_inputs";
    return RANC_E_STATE;
  }
  const size_t want = (size_t)ctx->S * ctx->net.C;
  if (n != want) {
    ctx->err = "counts buffer has " + std::to_string(n) + " elements, need S*C = " + std::to_string(want);
    return RANC_E_SIZE;
  }
  if (want && !counts) return RANC_E_ARG;
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (want) CK(cudaMemcpyAsync(counts, ctx->d_counts.p, want * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H counts");
  return sync(ctx, "ranc_read_outputs");
}

ranc_status ranc_read_potentials(ranc_ctx* ctx, int32_t* pot, size_t n) {
  TRY(check_ctx(ctx));
  if (!ctx->have_inputs) {
    ctx->err = "ranc_read_potentials before ranc_load_inputs";
    return RANC_E_STATE;
  }
  const Compiled& c = ctx->net;
  const int GL = ctx->G_loc;
  const size_t want = (size_t)ctx->S * GL * c.N;
  if (n != want || !pot) {
    ctx->err = "potentials buffer has " + std::to_string(n) + " elements, need S*G_local*N = " + std::to_string(want);
    return RANC_E_SIZE;
  }
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (ctx->fresh) {  // no tick since the reset: potentials are the initial ones
    TRY(sync(ctx, "ranc_read_potentials"));
    for (int64_t s = 0; s < ctx->S; ++s)
      for (int g = 0; g < GL; ++g)
        for (int j = 0; j < c.N; ++j)
          pot[((size_t)s * GL + g) * c.N + j] = c.init[(size_t)(ctx->c_lo + g) * c.Npad + j];
    return RANC_OK;
  }
  std::vector<int16_t> h(ctx->d_pot.bytes / 2);
  CK(cudaMemcpyAsync(h.data(), ctx->d_pot.p, h.size() * 2, cudaMemcpyDeviceToHost, ctx->stream), "D2H pot");
  TRY(sync(ctx, "ranc_read_potentials"));
  const int64_t NT = tc_tile(), nT = (ctx->S + NT - 1) / NT;
  for (int64_t s = 0; s < ctx->S; ++s)
    for (int g = 0; g < GL; ++g)
      for (int j = 0; j < c.N; ++j)
        pot[((size_t)s * GL + g) * c.N + j] =
            ctx->kernel_active == RANC_KERNEL_TC
                ? h[(((size_t)g * nT + s / NT) * (NT / 8) + (s % NT) / 8) * c.Npad * 8 + (size_t)j * 8 + s % 8]
                : h[((size_t)g * ctx->S + s) * c.Npad + j];
  return RANC_OK;
}

ranc_status ranc_read_pending(ranc_ctx* ctx, uint32_t* bits, size_t n) {
  TRY(check_ctx(ctx));
  if (!ctx->have_inputs) {
    ctx->err = "ranc_read_pending before ranc_load_inputs";
    return RANC_E_STATE;
  }
  const Compiled& c = ctx->net;
  const int GL = ctx->G_loc;
  const size_t want = (size_t)ctx->S * GL * c.D * c.W;
  if (n != want || !bits) {
    ctx->err = "pending buffer has " + std::to_string(n) + " elements, need S*G*D*ceil(A/32) = " +
               std::to_string(want);
    return RANC_E_SIZE;
  }
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (ctx->ring_pull) {
    // history scheduler: the spikes due at tick now+j on position i (delay
    // d) were stored at tick now+j-d; they are pending iff that tick has run
    // (d > j) -- otherwise the slot still holds the word of Rp ticks earlier
    std::vector<uint32_t> hh(ctx->d_hist.bytes / 4);
    CK(cudaMemcpyAsync(hh.data(), ctx->d_hist.p, ctx->d_hist.bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H hist");
    TRY(sync(ctx, "ranc_read_pending"));
    std::memset(bits, 0, want * 4);
    const int64_t nT = (ctx->S + tc_tile() - 1) / tc_tile();
    const size_t P = c.hbase.back();
    for (int g = 0; g < GL; ++g)
      for (uint32_t i = c.hbase[g]; i < c.hbase[g + 1]; ++i) {
        const int d = c.hdel[i];
        if (!d) continue;   // padding
        const int a = c.perm_tc[(size_t)g * c.A + c.hax[i]];
        for (int j = 0; j < std::min(d, c.D); ++j) {
          if (ctx->now + j - d < 0) continue;
          const uint32_t* hs = &hh[(size_t)((ctx->now + j) & (c.Rp - 1)) * nT * P * 2];
          for (int64_t s = 0; s < ctx->S; ++s) {
            const uint32_t w = hs[((size_t)(s / 64) * P + i) * 2 + (s % 64) / 32];
            if ((w >> (s % 32)) & 1u) bits[(((size_t)s * GL + g) * c.D + j) * c.W + (a >> 5)] |= 1u << (a & 31);
          }
        }
      }
    return RANC_OK;
  }
  std::vector<uint32_t> h((size_t)c.Rp * GL * ctx->Sr * c.W);
  CK(cudaMemcpyAsync(h.data(), ctx->d_ring.p, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H ring");
  TRY(sync(ctx, "ranc_read_pending"));
  std::memset(bits, 0, want * 4);
  for (int j = 0; j < c.D; ++j) {
    const int slot = (int)((ctx->now + j) & (c.Rp - 1));
    for (int64_t s = 0; s < ctx->S; ++s)
      for (int g = 0; g < GL; ++g) {
        // ring [Rp][G][Sr][W], or word-major [Rp][G][W][Sr]
        const bool wmajor = ctx->ring_wmajor;
        const size_t base = wmajor ? ((size_t)slot * GL + g) * c.W * ctx->Sr + s
                                   : (((size_t)slot * GL + g) * ctx->Sr + s) * c.W;
        const size_t wst = wmajor ? (size_t)ctx->Sr : 1;
        uint32_t* dst = bits + (((size_t)s * GL + g) * c.D + j) * c.W;
        const int gg = ctx->c_lo + g;
        const int32_t* perm = ctx->kernel_active == RANC_KERNEL_TC ? &c.perm_tc[(size_t)gg * c.A]
                                                                   : &c.perm[(size_t)gg * c.A];
        for (int ap = 0; ap < c.A; ++ap)
          if ((h[base + (ap >> 5) * wst] >> (ap & 31)) & 1u) {
            const int a = perm[ap];
            dst[a >> 5] |= 1u << (a & 31);
          }
      }
  }
  return RANC_OK;
}

ranc_status ranc_set_trace(ranc_ctx* ctx, uint32_t flags) {
  TRY(check_ctx(ctx));
  if (flags & ~(RANC_TRACE_SPIKE_RASTER | RANC_TRACE_OUTPUT_EVENTS | RANC_TRACE_STATE_DIGEST)) {
    ctx->err = "unknown trace flags";
    return RANC_E_ARG;
  }
  ctx->trace_flags = flags;
  return RANC_OK;
}

ranc_status ranc_read_trace(ranc_ctx* ctx, uint32_t kind, void* buf, size_t bytes, size_t* written) {
  TRY(check_ctx(ctx));
  if (!written) return RANC_E_ARG;
  *written = 0;
  if (!(ctx->trace_flags & kind) ||
      (kind != RANC_TRACE_SPIKE_RASTER && kind != RANC_TRACE_OUTPUT_EVENTS && kind != RANC_TRACE_STATE_DIGEST)) {
    ctx->err = "trace kind not enabled (ranc_set_trace) or unknown";
    return RANC_E_STATE;
  }
  const Compiled& c = ctx->net;
  const int GL = ctx->G_loc;
  if (kind == RANC_TRACE_STATE_DIGEST) {
    const size_t dbytes = (size_t)ctx->raster_ticks * ctx->S * 8;
    *written = dbytes;
    if (bytes < dbytes || (!buf && dbytes)) {
      ctx->err = "digest buffer too small";
      return RANC_E_SIZE;
    }
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (dbytes) CK(cudaMemcpyAsync(buf, ctx->d_digest.p, dbytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H digest");
    return sync(ctx, "ranc_read_trace");
  }
  const size_t rbytes = (size_t)ctx->raster_ticks * ctx->S * GL * c.Wn * 4;
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (kind == RANC_TRACE_SPIKE_RASTER) {
    *written = rbytes;
    if (bytes < rbytes || (!buf && rbytes)) {
      ctx->err = "raster buffer too small";
      return RANC_E_SIZE;
    }
    if (rbytes) CK(cudaMemcpyAsync(buf, ctx->d_raster.p, rbytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H raster");
    return sync(ctx, "ranc_read_trace");
  }
  std::vector<uint32_t> r(rbytes / 4);
  if (rbytes) CK(cudaMemcpyAsync(r.data(), ctx->d_raster.p, rbytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H raster");
  TRY(sync(ctx, "ranc_read_trace"));
  // canonical order (sample, tick, y, x, neuron)
  std::vector<int64_t> ev;
  for (int64_t s = 0; s < ctx->S; ++s)
    for (int64_t t = 0; t < ctx->raster_ticks; ++t)
      for (int gl = 0; gl < GL; ++gl) {
        const int g = ctx->c_lo + gl;
        const uint32_t* w = &r[(((size_t)t * ctx->S + s) * GL + gl) * c.Wn];
        for (int j = 0; j < c.N; ++j)
          if (((w[j >> 5] >> (j & 31)) & 1u) && c.kind[(size_t)g * c.N + j] == RK_OUTPUT) {
            ev.push_back(ctx->first_sample + s);
            ev.push_back(ctx->raster_t0 + t);
            ev.push_back(g % c.grid_w);
            ev.push_back(g / c.grid_w);
            ev.push_back(j);
          }
      }
  *written = ev.size() * sizeof(int64_t);
  if (bytes < *written || (!buf && *written)) {
    ctx->err = "events buffer too small";
    return RANC_E_SIZE;
  }
  if (!ev.empty()) std::memcpy(buf, ev.data(), *written);
  return RANC_OK;
}

ranc_status ranc_set_stream(ranc_ctx* ctx, void* cuda_stream) {
  TRY(check_ctx(ctx));
  const cudaStream_t next = cuda_stream ? (cudaStream_t)cuda_stream : ctx->own_stream;
  if (next != ctx->stream) {
    // everything queued on the old stream (uploads, input decode, stream-
    // ordered allocations and frees) completes before work on the new one
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaStreamSynchronize(ctx->stream), "ranc_set_stream (draining the previous stream)");
  }
  ctx->stream = next;
  return RANC_OK;
}

ranc_status ranc_set_allocator(ranc_ctx* ctx, void* (*alloc)(size_t, void*), void (*dealloc)(void*, void*),
                               void* user) {
  TRY(check_ctx(ctx));
  if ((alloc == nullptr) != (dealloc == nullptr)) {
    ctx->err = "alloc and dealloc must both be set or both be NULL";
    return RANC_E_ARG;
  }
  if (ctx->have_inputs) {
    ctx->err = "ranc_set_allocator must be called before ranc_load_inputs";
    return RANC_E_STATE;
  }
  ctx->user_alloc = alloc;
  ctx->user_free = dealloc;
  ctx->user = user;
  return RANC_OK;
}

ranc_status ranc_set_option(ranc_ctx* ctx, int option, int64_t value) {
  TRY(check_ctx(ctx));
  switch (option) {
    case RANC_OPT_SAMPLE_TILE:
      if (value < 0 || value > 256) {
        ctx->err = "sample tile must be in [0,256] (0 = automatic)";
        return RANC_E_ARG;
      }
      ctx->sample_tile_opt = (int32_t)value;
      return RANC_OK;
    case RANC_OPT_INPUT_DECODE:
      ctx->input_decode = value ? 1 : 0;
      ctx->inw_valid = false;
      return RANC_OK;
    case RANC_OPT_STREAM:
      if (value < 0 || value > 2) {
        ctx->err = "stream option must be 0 (auto), 1 (per-tick launches) or 2 (one cooperative launch per run)";
        return RANC_E_ARG;
      }
      ctx->stream_opt = (int32_t)value;
      return RANC_OK;
    case RANC_OPT_KERNEL:
      if (value < 0 || value > 2) {
        ctx->err = "kernel variant must be 0 (auto), 1 (popcount) or 2 (tensor core)";
        return RANC_E_ARG;
      }
      if (value == RANC_KERNEL_TC && (!ctx->net.tc_ok || tc_smem_bytes(ctx->net) > 227 * 1024)) {
        ctx->err = "network is outside the tensor-core envelope (<= 1024 neurons and axons, whose operands and stages fit 227 KB of shared memory; 16-bit weights on the widest cores do not)";
        return RANC_E_CONFIG;
      }
      ctx->kernel = (int32_t)value;  // takes effect at the next ranc_load_inputs / ranc_reset_state
      return RANC_OK;
    case RANC_OPT_RING_LAYOUT:
      if (value < 0 || value > 3) {
        ctx->err = "ring layout must be 0 (auto), 1 (sample-major), 2 (word-major) or 3 (history scheduler); "
                   "tensor-core path";
        return RANC_E_ARG;
      }
      if (value == 3 && !pull_eligible(ctx)) {
        ctx->err = "the history scheduler needs the tensor-core path without neuron groups, no core sharding and "
                   "per-core position lists within the shared-memory budget";
        return RANC_E_CONFIG;
      }
      ctx->ring_layout = (int32_t)value;  // takes effect at the next ranc_load_inputs / ranc_reset_state
      return RANC_OK;
    case RANC_OPT_OPERAND:
      if (value < 0 || value > 2) {
        ctx->err = "operand must be 0 (auto), 1 (folded Wfold) or 2 (compact, expanded on chip)";
        return RANC_E_ARG;
      }
      if (value == 2 && !ctx->net.tc_comp_ok) {
        ctx->err = "the compact operand needs the tensor-core path with int8 weights and cores of at most 256 "
                   "neurons and 256 axons";
        return RANC_E_CONFIG;
      }
      ctx->operand = (int32_t)value;  // chosen per launch (per-tick tensor-core launches)
      return RANC_OK;
    case RANC_OPT_DEBUG_FAULT: {
      if (value < 0 || value > 2) {
        ctx->err = "debug fault must be 0 (none), 1 (skip the multi-tick grid barrier) or 2 (routes one tick early)";
        return RANC_E_ARG;
      }
      ctx->fault = (int32_t)value;
      // fault 2: every route of delay >= 2 delivers one tick early (a wrong
      // scheduler offset); the compiled route words are re-uploaded
      const Compiled& c = ctx->net;
      CK(cudaSetDevice(ctx->device), "cudaSetDevice");
      auto early = [&](std::vector<uint2> v) {
        if (value == 2)
          for (uint2& r : v)
            if (route_kind(r.x) == RK_ROUTE && route_delay(r.x) >= 2) r.x -= 1u << 3;
        return v;
      };
      TRY(upload(ctx, &ctx->d_route, early(c.route)));
      if (c.tc_ok) TRY(upload(ctx, &ctx->d_route_tc, early(c.route_tc)));
      return sync(ctx, "ranc_set_option");
    }
    default:
      ctx->err = "unknown option";
      return RANC_E_ARG;
  }
}

ranc_status ranc_get_info(const ranc_ctx* ctx, ranc_info* info) {
  if (!ctx || !info) return RANC_E_ARG;
  std::memset(info, 0, sizeof *info);
  const Compiled& c = ctx->net;
  info->grid_w = c.grid_w; info->grid_h = c.grid_h; info->axons = c.A; info->neurons = c.N;
  info->num_types = c.K; info->max_delay = c.D; info->num_classes = c.C; info->num_lines = c.I;
  info->ring_rows = c.Rp; info->ring_words = c.W; info->pieces = c.E;
  info->sample_tile = ctx->sample_tile; info->num_samples = ctx->S;
  info->device_bytes = ctx->device_bytes; info->kernel_launches = ctx->launches;
  info->kernel = ctx->kernel_active;
  info->ring_layout = ctx->ring_pull ? 3 : ctx->ring_wmajor ? 2 : 1;
  info->operand = ctx->operand_used;
  info->core_lo = ctx->c_lo;
  info->cores_local = ctx->G_loc;
  info->shard_mode = (ctx->nccl_comm || ctx->group) ? ctx->shard_mode : 0;
  info->exchange_bytes = ctx->exchange_bytes;
  return RANC_OK;
}

const char* ranc_last_error(const ranc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_load_err.c_str(); }

void ranc_comm_destroy_internal(ranc_ctx* ctx);

void ranc_destroy(ranc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  ranc_comm_destroy_internal(ctx);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  free_all(ctx);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->copy_stream) {
    cudaStreamDestroy(ctx->copy_stream);
    cudaEventDestroy(ctx->ev_copied);
    for (cudaEvent_t e : ctx->ev_stage_free) cudaEventDestroy(e);
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

}  // extern "C"
