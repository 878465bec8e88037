// comm_nccl.cu — ipi_comm over an NCCL communicator (the sharded driver's two
// exchanges on NVLink / NVSwitch):
//
//   * allgather_blocks: the value vector from the ranks' make_partition blocks.
//     Equal blocks: one ncclAllGather straight into the full vector; unequal
//     blocks (n mod R != 0): one ncclBroadcast per rank inside a group (each
//     rank is the root of its own block), the usual all-gather-v.
//   * allgather: R x count partial dots, one ncclAllGather.
//
// libnccl.so.2 is resolved with dlopen at the first use (the library torch
// already loaded), so libipi_b200.so has no link-time NCCL dependency and the
// single-GPU path never touches it.
#include <dlfcn.h>

#include <cstdlib>

#include <mutex>
#include <string>
#include <vector>

#include "handle.cuh"

namespace {

typedef int nccl_result;  // ncclResult_t; 0 = ncclSuccess
constexpr int kNcclFloat64 = 8;  // ncclDataType_t ncclFloat64 (nccl.h)

struct NcclApi {
  nccl_result (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  nccl_result (*broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  nccl_result (*group_start)() = nullptr;
  nccl_result (*group_end)() = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.all_gather && api.broadcast && api.group_start && api.group_end;
  });
  return api;
}

struct NcclCtx {
  void* comm;
  int rank, world;
  std::vector<int64_t> start;
  bool equal;
  bool local;  // one rank and no communicator (or not forced): plain device copies
};

int nccl_fail(nccl_result r, const char* what) {
  const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
  return ipi::fail(IPI_ECUDA, std::string(what) + ": " + msg);
}

int nccl_allgather_blocks(void* ctx, const double* local, double* full, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  NcclApi& api = nccl();
  cudaStream_t st = (cudaStream_t)stream;
  if (c->local) {
    if (full != local) {
      const cudaError_t e = cudaMemcpyAsync(full, local, sizeof(double) * (c->start[1] - c->start[0]),
                                            cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return ipi::fail(IPI_ECUDA, cudaGetErrorString(e));
    }
    return IPI_OK;
  }
  if (c->equal) {
    const nccl_result r = api.all_gather(local, full, (size_t)(c->start[1] - c->start[0]),
                                         kNcclFloat64, c->comm, st);
    return r ? nccl_fail(r, "ncclAllGather (V blocks)") : IPI_OK;
  }
  nccl_result r = api.group_start();
  for (int q = 0; q < c->world && !r; ++q) {
    const int64_t lo = c->start[q], cnt = c->start[q + 1] - lo;
    r = api.broadcast(q == c->rank ? local : nullptr, full + lo, (size_t)cnt, kNcclFloat64, q,
                      c->comm, st);
  }
  const nccl_result r2 = api.group_end();
  if (r) return nccl_fail(r, "ncclBroadcast (V block)");
  return r2 ? nccl_fail(r2, "ncclGroupEnd") : IPI_OK;
}

int nccl_allgather(void* ctx, const double* send, double* out, int64_t count, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  if (c->local) {
    const cudaError_t e = cudaMemcpyAsync(out, send, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                                          (cudaStream_t)stream);
    return e != cudaSuccess ? ipi::fail(IPI_ECUDA, cudaGetErrorString(e)) : IPI_OK;
  }
  const nccl_result r = nccl().all_gather(send, out, (size_t)count, kNcclFloat64, c->comm,
                                          (cudaStream_t)stream);
  return r ? nccl_fail(r, "ncclAllGather (partials)") : IPI_OK;
}

}  // namespace

extern "C" {

int ipi_comm_nccl(void* nccl_comm, int32_t rank, int32_t world, const int64_t* block_start,
                  ipi_comm* out) {
  if (!out || !block_start) return ipi::fail(IPI_EVALIDATION, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return ipi::fail(IPI_EVALIDATION, "bad rank / world");
  if (world > 1 && !nccl_comm) return ipi::fail(IPI_EVALIDATION, "null NCCL communicator");
  // One rank normally needs no NCCL at all; IPI_COMM_FORCE_NCCL=1 sends a
  // one-rank communicator's exchanges through ncclAllGather / ncclBroadcast
  // anyway (how the binding is exercised on a single-GPU box).
  const bool force = nccl_comm && getenv("IPI_COMM_FORCE_NCCL") && atoi(getenv("IPI_COMM_FORCE_NCCL")) != 0;
  const bool use_nccl = world > 1 || force;
  if (use_nccl && !nccl().ok)
    return ipi::fail(IPI_ECUDA, "libnccl.so.2 not found (load torch.distributed's NCCL first)");
  auto* c = new NcclCtx{nccl_comm, rank, world, std::vector<int64_t>(block_start, block_start + world + 1),
                        true, !use_nccl};
  if (force && world == 1 && getenv("IPI_COMM_FORCE_NCCL")[0] == '2') c->equal = false;  // the broadcast path
  for (int q = 1; q < world; ++q)
    if (c->start[q + 1] - c->start[q] != c->start[1] - c->start[0]) c->equal = false;
  out->ctx = c;
  out->rank = rank;
  out->world = world;
  out->allgather_blocks = nccl_allgather_blocks;
  out->allgather = nccl_allgather;
  return IPI_OK;
}

void ipi_comm_nccl_destroy(ipi_comm* c) {
  if (c && c->ctx) {
    delete static_cast<NcclCtx*>(c->ctx);
    c->ctx = nullptr;
  }
}

}  // extern "C"
