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
// lists of this rank (computed identically on every rank from the replicated
// network).
ranc_status setup_core_shards(ranc_ctx* ctx, int world, int rank) {
  const Compiled& c = ctx->net;
  if (ctx->have_inputs) {
    ctx->err = "core-sharded communicators must be set up before ranc_load_inputs";
    return RANC_E_STATE;
  }
  if (world > c.grid_h) {
    ctx->err = "core-sharded mode needs at least one grid row per rank (grid_h=" + std::to_string(c.grid_h) +
               ", world=" + std::to_string(world) + ")";
    return RANC_E_CONFIG;
  }
  auto row_lo = [&](int r) { return (int)((int64_t)r * c.grid_h / world); };
  std::vector<int> owner(c.G);
  for (int r = 0; r < world; ++r)
    for (int y = row_lo(r); y < row_lo(r + 1); ++y)
      for (int x = 0; x < c.grid_w; ++x) owner[y * c.grid_w + x] = r;
  ctx->c_lo = row_lo(rank) * c.grid_w;
  ctx->G_loc = (row_lo(rank + 1) - row_lo(rank)) * c.grid_w;
  // needs[src core][dest rank]
  std::vector<uint8_t> exports(c.G, 0);
  std::vector<std::vector<uint8_t>> to(world, std::vector<uint8_t>(c.G, 0));
  for (int g = 0; g < c.G; ++g)
    for (int j = 0; j < c.N; ++j) {
      const uint2 rt = c.route[(size_t)g * c.Npad + j];
      if (route_kind(rt.x) != RK_ROUTE) continue;
      const int dr = owner[rt.y];
      if (dr != owner[g]) {
        exports[g] = 1;
        to[dr][g] = 1;
      }
    }
  ctx->send_cores.assign(world, {});
  ctx->recv_cores.assign(world, {});
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    for (int g = 0; g < c.G; ++g) {
      if (owner[g] == rank && to[p][g]) ctx->send_cores[p].push_back(g - ctx->c_lo);   // local id
      if (owner[g] == p && to[rank][g]) ctx->recv_cores[p].push_back(g);              // global id
    }
  }
  ranc_status s = dev_alloc(ctx, &ctx->d_exports, (size_t)c.G);
  if (s) return s;
  cudaError_t e = cudaMemcpyAsync(ctx->d_exports.p, exports.data(), c.G, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "setup_core_shards");
  return RANC_OK;
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
  // 1) every rank's sample count
  DevBuf sizes;
  {
    ranc_status s = dev_alloc(ctx, &sizes, sizeof(int64_t) * (ctx->world + 1));
    if (s) return s;
  }
  int64_t mine = ctx->S;
  cudaMemcpyAsync((int64_t*)sizes.p + ctx->world, &mine, 8, cudaMemcpyHostToDevice, ctx->stream);
  NK(ncclAllGather((int64_t*)sizes.p + ctx->world, sizes.p, 1, ncclInt64, comm, ctx->stream), "ncclAllGather");
  std::vector<int64_t> hs(ctx->world);
  cudaMemcpyAsync(hs.data(), sizes.p, 8 * ctx->world, cudaMemcpyDeviceToHost, ctx->stream);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  dev_free(ctx, &sizes);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "gather sizes");
  int64_t total = 0;
  for (int64_t v : hs) total += v;
  if (ctx->rank == root && n != (size_t)(total * C)) {
    ctx->err = "counts_global has " + std::to_string(n) + " elements, need (sum S_local)*C = " +
               std::to_string(total * C);
    return RANC_E_SIZE;
  }
  if (C == 0) return RANC_OK;
  // 2) point-to-point gather into a device buffer on the root
  DevBuf all;
  if (ctx->rank == root) {
    ranc_status s = dev_alloc(ctx, &all, (size_t)total * C * 4);
    if (s) return s;
  }
  NK(ncclGroupStart(), "ncclGroupStart");
  if (ctx->rank == root) {
    int64_t off = 0;
    for (int r = 0; r < ctx->world; ++r) {
      NK(ncclRecv((int32_t*)all.p + off * C, (size_t)hs[r] * C, ncclInt32, r, comm, ctx->stream), "ncclRecv");
      off += hs[r];
    }
  }
  NK(ncclSend(ctx->d_counts.p, (size_t)ctx->S * C, ncclInt32, root, comm, ctx->stream), "ncclSend");
  NK(ncclGroupEnd(), "ncclGroupEnd");
  if (ctx->rank == root) {
    if (!counts_global) return RANC_E_ARG;
    cudaMemcpyAsync(counts_global, all.p, (size_t)total * C * 4, cudaMemcpyDeviceToHost, ctx->stream);
  }
  e = cudaStreamSynchronize(ctx->stream);
  dev_free(ctx, &all);
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
  ranc_group* g = new ranc_group();
  g->ctxs.assign(ctxs, ctxs + n);
  for (int i = 0; i < n; ++i) {
    ranc_status st = setup_core_shards(ctxs[i], n, i);
    if (st) return st;
    ctxs[i]->world = n;
    ctxs[i]->rank = i;
    ctxs[i]->shard_mode = RANC_SHARD_CORES;
    ctxs[i]->group = g;
  }
  return RANC_OK;
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
