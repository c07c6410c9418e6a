// comm.cpp -- multi-GPU plumbing over NCCL (NVLink 5 / NVSwitch on B200).
//
// Sample-sharded mode: every rank holds the whole network
// and simulates its own contiguous shard of the samples; the only collective
// on the path is one gather of the class counts to the root at the end of a
// run (north_star: "one NCCL gather of class spike counts").
// Core-sharded mode (networks too large for one GPU): every rank simulates a
// band of grid rows for all samples; after every tick the fired bits of the
// cores whose routes cross a band boundary are exchanged with grouped
// ncclSend/ncclRecv (exchange.cu applies them on the receiver), and the class
// counts are summed with one ncclReduce at the end.  A loopback group runs
// the same exchange between several contexts of one process (device copies),
// which is how the core-sharded logic is tested on a single GPU.
// The communicator is built from an ncclUniqueId that the caller distributes
// (the Python binding uses torch.distributed.broadcast_object_list).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace ranc;

namespace {
ranc_status nccl_err(ranc_ctx* ctx, ncclResult_t r, const char* where) {
  if (ctx) ctx->err = std::string(where) + ": " + ncclGetErrorString(r);
  return RANC_E_NCCL;
}
}  // namespace

#define NK(call, where)                                   \
  do {                                                    \
    ncclResult_t _r = (call);                             \
    if (_r != ncclSuccess) return nccl_err(ctx, _r, where); \
  } while (0)

namespace ranc {

// Row-band partition of the cores over `world` ranks and the export / import
// lists of `rank` (computed identically on every rank from the replicated
// network; host only, so ranc_plan_core_shards can expose it without a GPU).
ranc_status plan_core_shards(const Compiled& c, int world, int rank, CoreShardPlan* out, std::string* err) {
  if (world < 1 || rank < 0 || rank >= world) {
    *err = "bad world/rank (world=" + std::to_string(world) + ", rank=" + std::to_string(rank) + ")";
    return RANC_E_ARG;
  }
  if (world > c.grid_h) {
    *err = "core-sharded mode needs at least one grid row per rank (grid_h=" + std::to_string(c.grid_h) +
           ", world=" + std::to_string(world) + ")";
    return RANC_E_CONFIG;
  }
  auto row_lo = [&](int r) { return (int)((int64_t)r * c.grid_h / world); };
  std::vector<int> owner(c.G);
  for (int r = 0; r < world; ++r)
    for (int y = row_lo(r); y < row_lo(r + 1); ++y)
      for (int x = 0; x < c.grid_w; ++x) owner[y * c.grid_w + x] = r;
  out->c_lo = row_lo(rank) * c.grid_w;
  out->G_loc = (row_lo(rank + 1) - row_lo(rank)) * c.grid_w;
  // to[dest rank][src core]: some neuron of src routes to a core of dest rank
  out->exports.assign(c.G, 0);
  std::vector<std::vector<uint8_t>> to(world, std::vector<uint8_t>(c.G, 0));
  for (int g = 0; g < c.G; ++g)
    for (int j = 0; j < c.N; ++j) {
      const uint2 rt = c.route[(size_t)g * c.Npad + j];
      if (route_kind(rt.x) != RK_ROUTE) continue;
      const int dr = owner[rt.y];
      if (dr != owner[g]) {
        out->exports[g] = 1;
        to[dr][g] = 1;
      }
    }
  out->send_cores.assign(world, {});
  out->recv_cores.assign(world, {});
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    for (int g = 0; g < c.G; ++g) {
      if (owner[g] == rank && to[p][g]) out->send_cores[p].push_back(g - out->c_lo);   // local id
      if (owner[g] == p && to[rank][g]) out->recv_cores[p].push_back(g);              // global id
    }
  }
  return RANC_OK;
}

ranc_status setup_core_shards(ranc_ctx* ctx, int world, int rank) {
  const Compiled& c = ctx->net;
  if (ctx->have_inputs) {
    ctx->err = "core-sharded communicators must be set up before ranc_load_inputs";
    return RANC_E_STATE;
  }
  CoreShardPlan plan;
  ranc_status s = plan_core_shards(c, world, rank, &plan, &ctx->err);
  if (s) return s;
  s = dev_alloc(ctx, &ctx->d_exports, (size_t)c.G);
  if (s) return s;
  cudaError_t e = cudaMemcpyAsync(ctx->d_exports.p, plan.exports.data(), c.G, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "setup_core_shards");
  ctx->c_lo = plan.c_lo;
  ctx->G_loc = plan.G_loc;
  ctx->send_cores = std::move(plan.send_cores);
  ctx->recv_cores = std::move(plan.recv_cores);
  return RANC_OK;
}

// undo setup_core_shards (a failed group set-up)
void clear_core_shards(ranc_ctx* ctx) {
  ctx->c_lo = 0;
  ctx->G_loc = ctx->net.G;
  ctx->send_cores.clear();
  ctx->recv_cores.clear();
  dev_free(ctx, &ctx->d_exports);
}

// Size the exchange buffers for S samples (called by ranc_load_inputs).
ranc_status alloc_exchange(ranc_ctx* ctx) {
  if (ctx->shard_mode != RANC_SHARD_CORES) return RANC_OK;
  const Compiled& c = ctx->net;
  const int world = ctx->world;
  const int64_t per = ctx->S * c.Wn;
  std::vector<int32_t> sl, rl;
  ctx->send_off.assign(world + 1, 0);
  ctx->recv_off.assign(world + 1, 0);
  for (int p = 0; p < world; ++p) {
    ctx->send_off[p] = (int64_t)sl.size() * per;
    ctx->recv_off[p] = (int64_t)rl.size() * per;
    sl.insert(sl.end(), ctx->send_cores[p].begin(), ctx->send_cores[p].end());
    rl.insert(rl.end(), ctx->recv_cores[p].begin(), ctx->recv_cores[p].end());
  }
  ctx->send_off[world] = (int64_t)sl.size() * per;
  ctx->recv_off[world] = (int64_t)rl.size() * per;
  ctx->n_send_words = (int64_t)sl.size() * per;
  ctx->n_recv_words = (int64_t)rl.size() * per;
  ctx->n_recv_rows = (int64_t)rl.size();
  ctx->exchange_bytes = ctx->n_send_words * 4;
  ranc_status s = dev_alloc(ctx, &ctx->d_fired, (size_t)ctx->G_loc * ctx->Sr * c.Wn * 4);
  if (!s) s = dev_alloc(ctx, &ctx->d_send, (size_t)ctx->n_send_words * 4);
  if (!s) s = dev_alloc(ctx, &ctx->d_recv, (size_t)ctx->n_recv_words * 4);
  if (!s) s = dev_alloc(ctx, &ctx->d_send_list, sl.size() * 4);
  if (!s) s = dev_alloc(ctx, &ctx->d_recv_list, rl.size() * 4);
  if (s) return s;
  cudaError_t e = cudaSuccess;
  if (!sl.empty()) e = cudaMemcpyAsync(ctx->d_send_list.p, sl.data(), sl.size() * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess && !rl.empty())
    e = cudaMemcpyAsync(ctx->d_recv_list.p, rl.data(), rl.size() * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "alloc_exchange");
  return RANC_OK;
}

// One tick's exchange over NCCL (grouped point-to-point, NVLink / NVSwitch).
ranc_status exchange_nccl(ranc_ctx* ctx, int64_t t) {
  cudaError_t e = launch_pack(ctx);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "pack");
  ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
  NK(ncclGroupStart(), "ncclGroupStart");
  for (int p = 0; p < ctx->world; ++p) {
    if (p == ctx->rank) continue;
    const size_t ns = (size_t)(ctx->send_off[p + 1] - ctx->send_off[p]);
    const size_t nr = (size_t)(ctx->recv_off[p + 1] - ctx->recv_off[p]);
    if (ns) NK(ncclSend((uint32_t*)ctx->d_send.p + ctx->send_off[p], ns, ncclUint32, p, comm, ctx->stream), "ncclSend");
    if (nr) NK(ncclRecv((uint32_t*)ctx->d_recv.p + ctx->recv_off[p], nr, ncclUint32, p, comm, ctx->stream), "ncclRecv");
  }
  NK(ncclGroupEnd(), "ncclGroupEnd");
  e = launch_unpack(ctx, t);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "unpack");
  return RANC_OK;
}

// One tick's exchange inside a loopback group: device copies between contexts.
ranc_status exchange_loopback(ranc_group* g, int64_t t) {
  const int n = (int)g->ctxs.size();
  for (ranc_ctx* c : g->ctxs) {
    cudaError_t e = launch_pack(c);
    if (e != cudaSuccess) return set_cuda_error(c, e, "pack");
  }
  for (int r = 0; r < n; ++r)
    for (int p = 0; p < n; ++p) {
      if (p == r) continue;
      ranc_ctx* src = g->ctxs[r];
      ranc_ctx* dst = g->ctxs[p];
      const size_t words = (size_t)(src->send_off[p + 1] - src->send_off[p]);
      if (!words) continue;
      cudaError_t e = cudaMemcpyAsync((uint32_t*)dst->d_recv.p + dst->recv_off[r],
                                      (const uint32_t*)src->d_send.p + src->send_off[p], words * 4,
                                      cudaMemcpyDeviceToDevice, src->stream);
      if (e != cudaSuccess) return set_cuda_error(src, e, "loopback copy");
    }
  for (ranc_ctx* c : g->ctxs) {
    cudaError_t e = launch_unpack(c, t);
    if (e != cudaSuccess) return set_cuda_error(c, e, "unpack");
  }
  return RANC_OK;
}

}  // namespace ranc

extern "C" {

ranc_status ranc_comm_unique_id(void* out128) {
  if (!out128) return RANC_E_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RANC_E_NCCL;
  std::memcpy(out128, &id, sizeof id);
  return RANC_OK;
}

ranc_status ranc_comm_init(ranc_ctx* ctx, const void* nccl_unique_id, int world, int rank, int mode) {
  if (!ctx || !nccl_unique_id) return RANC_E_ARG;
  if (world < 1 || rank < 0 || rank >= world) {
    ctx->err = "bad world/rank";
    return RANC_E_ARG;
  }
  if (mode != RANC_SHARD_SAMPLES && mode != RANC_SHARD_CORES) {
    ctx->err = "unsupported shard mode";
    return RANC_E_ARG;
  }
  if (ctx->nccl_comm || ctx->group) {
    ctx->err = "communicator already initialised";
    return RANC_E_STATE;
  }
  if (mode == RANC_SHARD_CORES) {
    ranc_status st = setup_core_shards(ctx, world, rank);
    if (st) return st;
  }
  cudaSetDevice(ctx->device);
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof id);
  ncclComm_t comm = nullptr;
  NK(ncclCommInitRank(&comm, world, id, rank), "ncclCommInitRank");
  ctx->nccl_comm = comm;
  ctx->world = world;
  ctx->rank = rank;
  ctx->shard_mode = mode;
  return RANC_OK;
}

ranc_status ranc_gather_outputs(ranc_ctx* ctx, int32_t* counts_global, size_t n, int root) {
  if (!ctx) return RANC_E_ARG;
  if (!ctx->nccl_comm) {
    ctx->err = "ranc_gather_outputs before ranc_comm_init";
    return RANC_E_NCCL;
  }
  if (!ctx->have_inputs) {
    ctx->err = "ranc_gather_outputs before ranc_load_inputs";
    return RANC_E_STATE;
  }
  if (root < 0 || root >= ctx->world) return RANC_E_ARG;
  ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
  cudaSetDevice(ctx->device);
  const int C = ctx->net.C;
  if (ctx->shard_mode == RANC_SHARD_CORES) {
    // every rank counted the output-bus spikes of its own cores: sum them
    if (ctx->rank == root && n != (size_t)(ctx->S * C)) {
      ctx->err = "counts_global has " + std::to_string(n) + " elements, need S*C = " + std::to_string(ctx->S * C);
      return RANC_E_SIZE;
    }
    if (C == 0) return RANC_OK;
    DevBuf sum;
    if (ctx->rank == root) {
      ranc_status s = dev_alloc(ctx, &sum, (size_t)ctx->S * C * 4);
      if (s) return s;
    }
    NK(ncclReduce(ctx->d_counts.p, sum.p, (size_t)ctx->S * C, ncclInt32, ncclSum, root, comm, ctx->stream),
       "ncclReduce");
    if (ctx->rank == root) {
      if (!counts_global) return RANC_E_ARG;
      cudaMemcpyAsync(counts_global, sum.p, (size_t)ctx->S * C * 4, cudaMemcpyDeviceToHost, ctx->stream);
    }
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    dev_free(ctx, &sum);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "reduce");
    return RANC_OK;
  }
  // Sample mode: the shards are the contiguous partition of S_total = n / C
  // samples (sizes differ by at most one, lower ranks first; the binding's
  // shard_range), so every rank knows every shard size without a message.
  // Each rank pads its counts to Smax rows and ONE ncclGather collects the
  // [world][Smax][C] block on the root, which copies the S_r rows of each
  // rank to the host.
  if (C == 0) return RANC_OK;
  if (n % (size_t)C) {
    ctx->err = "counts_global has " + std::to_string(n) + " elements, not a multiple of C = " + std::to_string(C);
    return RANC_E_SIZE;
  }
  const int64_t S_total = (int64_t)(n / C);
  const int world = ctx->world;
  auto shard_lo = [&](int r) {
    const int64_t base = S_total / world, rem = S_total % world;
    return r * base + std::min<int64_t>(r, rem);
  };
  const int64_t mine = shard_lo(ctx->rank + 1) - shard_lo(ctx->rank);
  if (ctx->S != mine || ctx->first_sample != shard_lo(ctx->rank)) {
    ctx->err = "rank " + std::to_string(ctx->rank) + " holds samples [" + std::to_string(ctx->first_sample) + ", " +
               std::to_string(ctx->first_sample + ctx->S) + "), but the contiguous shard of " +
               std::to_string(S_total) + " samples over " + std::to_string(world) + " ranks is [" +
               std::to_string(shard_lo(ctx->rank)) + ", " + std::to_string(shard_lo(ctx->rank + 1)) + ")";
    return RANC_E_SIZE;
  }
  if (ctx->rank == root && !counts_global) return RANC_E_ARG;
  const int64_t Smax = (S_total + world - 1) / world;
  const size_t chunk = (size_t)Smax * C;   // int32 elements per rank
  if (ctx->d_gsend.bytes != chunk * 4) {
    ranc_status s = dev_alloc(ctx, &ctx->d_gsend, chunk * 4);
    if (s) return s;
  }
  if (ctx->rank == root && ctx->d_grecv.bytes != chunk * world * 4) {
    ranc_status s = dev_alloc(ctx, &ctx->d_grecv, chunk * world * 4);
    if (s) return s;
  }
  cudaError_t e = cudaMemcpyAsync(ctx->d_gsend.p, ctx->d_counts.p, (size_t)ctx->S * C * 4, cudaMemcpyDeviceToDevice,
                                  ctx->stream);
  if (e == cudaSuccess && (size_t)ctx->S * C < chunk)
    e = cudaMemsetAsync((int32_t*)ctx->d_gsend.p + (size_t)ctx->S * C, 0, (chunk - (size_t)ctx->S * C) * 4,
                        ctx->stream);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "gather staging");
  NK(ncclGather(ctx->d_gsend.p, ctx->rank == root ? ctx->d_grecv.p : nullptr, chunk, ncclInt32, root, comm,
                ctx->stream),
     "ncclGather");
  if (ctx->rank == root)
    for (int r = 0; r < world && e == cudaSuccess; ++r) {
      const int64_t lo = shard_lo(r), rows = shard_lo(r + 1) - lo;
      if (rows)
        e = cudaMemcpyAsync(counts_global + (size_t)lo * C, (const int32_t*)ctx->d_grecv.p + (size_t)r * chunk,
                            (size_t)rows * C * 4, cudaMemcpyDeviceToHost, ctx->stream);
    }
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "gather");
  return RANC_OK;
}

ranc_status ranc_comm_init_loopback(ranc_ctx* const* ctxs, int n, int mode) {
  if (!ctxs || n < 1) return RANC_E_ARG;
  for (int i = 0; i < n; ++i)
    if (!ctxs[i]) return RANC_E_ARG;
  if (mode != RANC_SHARD_CORES) {
    ctxs[0]->err = "loopback groups support RANC_SHARD_CORES only";
    return RANC_E_ARG;
  }
  for (int i = 0; i < n; ++i) {
    if (ctxs[i]->nccl_comm || ctxs[i]->group) {
      ctxs[i]->err = "communicator already initialised";
      return RANC_E_STATE;
    }
    if (ctxs[i]->device != ctxs[0]->device || ctxs[i]->net.G != ctxs[0]->net.G) {
      ctxs[i]->err = "loopback contexts must share one device and one network shape";
      return RANC_E_ARG;
    }
  }
  // set every member up before any of them joins the group; on failure the
  // members set up so far are rolled back and nothing is left half-sharded
  for (int i = 0; i < n; ++i) {
    ranc_status st = setup_core_shards(ctxs[i], n, i);
    if (st) {
      if (i > 0) ctxs[0]->err = ctxs[i]->err;
      for (int j = 0; j < i; ++j) clear_core_shards(ctxs[j]);
      return st;
    }
  }
  ranc_group* g = new ranc_group();
  g->ctxs.assign(ctxs, ctxs + n);
  for (int i = 0; i < n; ++i) {
    ctxs[i]->world = n;
    ctxs[i]->rank = i;
    ctxs[i]->shard_mode = RANC_SHARD_CORES;
    ctxs[i]->group = g;
  }
  return RANC_OK;
}

ranc_status ranc_plan_core_shards(const ranc_network_desc* net, int world, int rank, int32_t* core_lo,
                                  int32_t* cores_local, int32_t* send_counts, int32_t* recv_counts,
                                  int32_t* send_cores, size_t send_cap, int32_t* recv_cores, size_t recv_cap) {
  static thread_local std::string perr;
  if (!net || !core_lo || !cores_local || !send_counts || !recv_counts) return RANC_E_ARG;
  Compiled c;
  std::string err;
  ranc_status s = validate_and_compile(net, &c, &err);
  if (s == RANC_OK) {
    CoreShardPlan plan;
    s = plan_core_shards(c, world, rank, &plan, &err);
    if (s == RANC_OK) {
      size_t ns = 0, nr = 0;
      for (int p = 0; p < world; ++p) {
        send_counts[p] = (int32_t)plan.send_cores[p].size();
        recv_counts[p] = (int32_t)plan.recv_cores[p].size();
        ns += plan.send_cores[p].size();
        nr += plan.recv_cores[p].size();
      }
      *core_lo = plan.c_lo;
      *cores_local = plan.G_loc;
      if (ns > send_cap || nr > recv_cap || (ns && !send_cores) || (nr && !recv_cores)) {
        err = "list buffers too small: need " + std::to_string(ns) + " send and " + std::to_string(nr) +
              " receive entries";
        s = RANC_E_SIZE;
      } else {
        for (int p = 0; p < world; ++p) {
          for (int32_t v : plan.send_cores[p]) *send_cores++ = v;
          for (int32_t v : plan.recv_cores[p]) *recv_cores++ = v;
        }
      }
    }
  }
  set_load_error(err);
  return s;
}

void ranc_comm_destroy_internal(ranc_ctx* ctx) {
  if (ctx && ctx->nccl_comm) {
    ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
  }
  if (ctx && ctx->group) {
    ranc_group* g = ctx->group;
    for (ranc_ctx*& m : g->ctxs)
      if (m == ctx) m = nullptr;
    ctx->group = nullptr;
    bool empty = true;
    for (ranc_ctx* m : g->ctxs)
      if (m) empty = false;
    if (empty) delete g;
    else
      for (ranc_ctx* m : g->ctxs)
        if (m) m->group_broken = true;
  }
}

}  // extern "C"
