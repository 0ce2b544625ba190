// SPDX-License-Identifier: Apache-2.0
// vest_nccl.cpp -- native NCCL exchanges for the sharded (multi-GPU) driver.
// The library's two exchange points (vest_ctx_set_comm: allreduce_sum,
// allgather_rows) served by an NCCL communicator owned by the context, the
// collectives issued directly on the context's stream: no host callback per
// exchange.  NCCL is opened at run time (dlopen "libnccl.so.2": the copy the
// process already loaded, e.g. torch's, or the system one), so the library
// has no link-time NCCL dependency.  The unique id is distributed by the
// caller (paper_1904_02603_b200/sharded.py: torch.distributed).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "vest_internal.h"

namespace vest {
namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a = [] {
    NcclApi r;
    r.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!r.so) r.so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!r.so) return r;
    auto sym = [&](const char* n) { return dlsym(r.so, n); };
    r.GetUniqueId = reinterpret_cast<decltype(r.GetUniqueId)>(sym("ncclGetUniqueId"));
    r.CommInitRank = reinterpret_cast<decltype(r.CommInitRank)>(sym("ncclCommInitRank"));
    r.CommDestroy = reinterpret_cast<decltype(r.CommDestroy)>(sym("ncclCommDestroy"));
    r.AllReduce = reinterpret_cast<decltype(r.AllReduce)>(sym("ncclAllReduce"));
    r.Broadcast = reinterpret_cast<decltype(r.Broadcast)>(sym("ncclBroadcast"));
    r.AllGather = reinterpret_cast<decltype(r.AllGather)>(sym("ncclAllGather"));
    r.GroupStart = reinterpret_cast<decltype(r.GroupStart)>(sym("ncclGroupStart"));
    r.GroupEnd = reinterpret_cast<decltype(r.GroupEnd)>(sym("ncclGroupEnd"));
    r.GetErrorString = reinterpret_cast<decltype(r.GetErrorString)>(sym("ncclGetErrorString"));
    return r;
  }();
  if (!a.so || !a.CommInitRank || !a.AllReduce || !a.Broadcast || !a.AllGather)
    throw std::runtime_error("NCCL not available (dlopen libnccl.so.2 failed)");
  return a;
}

void nccl_check(ncclResult_t r, const char* where) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL ") + where + ": " +
                             (api().GetErrorString ? api().GetErrorString(r) : "error"));
}

struct NcclState {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  std::vector<std::vector<uint64_t>> bounds;  // per mode: world + 1 row bounds
  bool broadcast = false;                     // VEST_NCCL_ROWS=broadcast: one broadcast per rank (A/B)
  double* send = nullptr;                     // padded all-gather staging
  double* recv = nullptr;
  size_t cap = 0;                             // doubles per rank slot
};

int hook_allreduce(void* user, double* p, uint64_t n, void* stream) {
  auto* s = static_cast<NcclState*>(user);
  if (n == 0) return 0;
  return api().AllReduce(p, p, n, ncclDouble, ncclSum, s->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess
             ? 0
             : 1;
}

// rows [b[r], b[r+1]) of a row-major buffer (ld doubles per row) come from
// rank r: one broadcast per rank, grouped
int hook_allgather_rows(void* user, int mode, double* base, uint64_t ld, void* stream) {
  auto* s = static_cast<NcclState*>(user);
  const auto& b = s->bounds[mode];
  const NcclApi& A = api();
  if (A.GroupStart() != ncclSuccess) return 1;
  for (int r = 0; r < s->world; ++r) {
    const uint64_t lo = b[r] * ld, hi = b[r + 1] * ld;
    if (hi > lo &&
        A.Broadcast(base + lo, base + lo, hi - lo, ncclDouble, r, s->comm, static_cast<cudaStream_t>(stream)) !=
            ncclSuccess) {
      A.GroupEnd();
      return 1;
    }
  }
  return A.GroupEnd() == ncclSuccess ? 0 : 1;
}

// The same exchange as ONE ncclAllGather: every rank's row range padded to
// the longest range of the mode (ranges differ by the work balancing), its own
// rows staged into the send slot, the gathered slots copied back into place
// (stream-ordered device copies).
int hook_allgather_rows_padded(void* user, int mode, double* base, uint64_t ld, void* stream) {
  auto* s = static_cast<NcclState*>(user);
  const auto& b = s->bounds[mode];
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t maxr = 0;
  for (int r = 0; r < s->world; ++r) maxr = std::max<uint64_t>(maxr, b[r + 1] - b[r]);
  const size_t slot = (size_t)maxr * ld;
  if (slot == 0) return 0;
  if (slot > s->cap) {
    cudaStreamSynchronize(st);
    cudaFree(s->send);
    cudaFree(s->recv);
    s->send = s->recv = nullptr;
    if (cudaMalloc(&s->send, slot * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->recv, slot * s->world * sizeof(double)) != cudaSuccess)
      return 1;
    s->cap = slot;
  }
  const uint64_t own = (b[s->rank + 1] - b[s->rank]) * ld;
  if (own && cudaMemcpyAsync(s->send, base + b[s->rank] * ld, own * sizeof(double), cudaMemcpyDeviceToDevice, st) !=
                 cudaSuccess)
    return 1;
  if (api().AllGather(s->send, s->recv, slot, ncclDouble, s->comm, st) != ncclSuccess) return 1;
  for (int r = 0; r < s->world; ++r) {
    const uint64_t n = (b[r + 1] - b[r]) * ld;
    if (r == s->rank || n == 0) continue;
    if (cudaMemcpyAsync(base + b[r] * ld, s->recv + (size_t)r * slot, n * sizeof(double), cudaMemcpyDeviceToDevice,
                        st) != cudaSuccess)
      return 1;
  }
  return 0;
}

void free_state(void* user) {
  auto* s = static_cast<NcclState*>(user);
  if (s->comm) api().CommDestroy(s->comm);
  cudaFree(s->send);
  cudaFree(s->recv);
  delete s;
}

}  // namespace

// Install an NCCL communicator on a shard context (see vest.h).
void ctx_set_nccl(Ctx& c, int rank, int world, const void* id, const uint64_t* bounds) {
  if (world < 1 || rank < 0 || rank >= world) throw ArgError{"bad rank/world"};
  const NcclApi& A = api();
  auto st = std::make_unique<NcclState>();
  st->rank = rank;
  st->world = world;
  if (const char* e = getenv("VEST_NCCL_ROWS")) st->broadcast = std::string(e) == "broadcast";
  st->bounds.resize(c.N);
  for (int n = 0; n < c.N; ++n) st->bounds[n].assign(bounds + (size_t)n * (world + 1), bounds + (size_t)(n + 1) * (world + 1));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  check(cudaSetDevice(c.device), "device");
  nccl_check(A.CommInitRank(&st->comm, world, uid, rank), "CommInitRank");
  const bool st_broadcast = st->broadcast;
  if (c.comm_free) c.comm_free(c.comm.user);
  c.comm.user = st.release();
  c.comm.allreduce_sum = hook_allreduce;
  c.comm.allgather_rows = st_broadcast ? hook_allgather_rows : hook_allgather_rows_padded;
  c.comm_free = free_state;
  c.comm_capturable = true;  // NCCL collectives are stream operations: an iteration graph may hold them
}

void nccl_unique_id(void* out) {
  ncclUniqueId uid;
  nccl_check(api().GetUniqueId(&uid), "GetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

}  // namespace vest
