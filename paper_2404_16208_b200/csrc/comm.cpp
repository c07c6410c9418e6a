// comm.cpp -- multi-GPU plumbing over NCCL (NVLink 5 / NVSwitch on B200).
//
// Sample-sharded mode: every rank holds the whole network
// and simulates its own contiguous shard of the samples; the only collective
// on the path is one gather of the class counts to the root at the end of a
// run (north_star: "one NCCL gather of class spike counts").  The
// communicator is built from an ncclUniqueId that the caller distributes
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
  if (mode != RANC_SHARD_SAMPLES) {
    ctx->err = "unsupported shard mode";
    return RANC_E_ARG;
  }
  cudaSetDevice(ctx->device);
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof id);
  ncclComm_t comm = nullptr;
  NK(ncclCommInitRank(&comm, world, id, rank), "ncclCommInitRank");
  ctx->nccl_comm = comm;
  ctx->world = world;
  ctx->rank = rank;
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

void ranc_comm_destroy_internal(ranc_ctx* ctx) {
  if (ctx && ctx->nccl_comm) {
    ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
  }
}

}  // extern "C"
