// fvb_mgpu.cu -- the C-ABI's multi-GPU entry points:
// the step's one exchange, a MAX all-reduce of the global wave speed over NCCL
// (NVLink / NVSwitch), for hosts that do not go through torch.distributed.
//
// Two process models:
//   * one process driving ndev GPUs:  fvb_mgpu_init(ndev, devs)  (ncclCommInitAll);
//     fvb_mgpu_allreduce_max_all() issues every rank's all-reduce in one NCCL
//     group; fvb_mgpu_allreduce_max(rank, ...) serves one-thread-per-GPU callers;
//   * one process per GPU (the Python driver's model, torchrun-style):
//     fvb_mgpu_unique_id() on rank 0, broadcast by the caller, then
//     fvb_mgpu_init_rank(nranks, rank, id) on every rank.
// NCCL is opened at run time (dlopen "libnccl.so.2": the copy torch already
// loaded when there is one), so the library has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "../../include/fvb200.h"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

constexpr int kMaxComms = 64;
std::mutex g_mu;
Nccl g_nccl;
ncclComm_t g_comms[kMaxComms];
int g_ncomms = 0;      // communicators owned by this process
int g_rank_base = 0;   // global rank of g_comms[0] (one-process-per-GPU model: the caller's rank)

bool load_nccl() {
  if (g_nccl.h) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  Nccl n;
  n.h = h;
  n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  n.commInitAll = reinterpret_cast<decltype(n.commInitAll)>(dlsym(h, "ncclCommInitAll"));
  n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(h, "ncclCommInitRank"));
  n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(h, "ncclCommDestroy"));
  n.allReduce = reinterpret_cast<decltype(n.allReduce)>(dlsym(h, "ncclAllReduce"));
  n.groupStart = reinterpret_cast<decltype(n.groupStart)>(dlsym(h, "ncclGroupStart"));
  n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(dlsym(h, "ncclGroupEnd"));
  n.getErrorString = reinterpret_cast<decltype(n.getErrorString)>(dlsym(h, "ncclGetErrorString"));
  if (!n.getUniqueId || !n.commInitAll || !n.commInitRank || !n.commDestroy || !n.allReduce || !n.groupStart ||
      !n.groupEnd) {
    dlclose(h);
    return false;
  }
  g_nccl = n;
  return true;
}

int nccl_rc(ncclResult_t r) { return r == ncclSuccess ? FVB_OK : FVB_ERR_CUDA; }

}  // namespace

extern "C" {

int fvb_mgpu_unique_id(uint8_t* id_out) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!id_out) return FVB_ERR_CONTRACT;
  if (!load_nccl()) return FVB_ERR_CUDA;
  ncclUniqueId id;
  const int rc = nccl_rc(g_nccl.getUniqueId(&id));
  if (rc == FVB_OK) memcpy(id_out, id.internal, FVB_MGPU_ID_BYTES);
  return rc;
}

int fvb_mgpu_init_rank(int nranks, int rank, const uint8_t* id_in) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (nranks < 1 || rank < 0 || rank >= nranks || !id_in || g_ncomms) return FVB_ERR_CONTRACT;
  if (!load_nccl()) return FVB_ERR_CUDA;
  ncclUniqueId id;
  memcpy(id.internal, id_in, FVB_MGPU_ID_BYTES);
  const int rc = nccl_rc(g_nccl.commInitRank(&g_comms[0], nranks, id, rank));   // on the current device
  if (rc == FVB_OK) {
    g_ncomms = 1;
    g_rank_base = rank;
  }
  return rc;
}

int fvb_mgpu_init(int ndev, const int* devs) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (ndev < 1 || ndev > kMaxComms || !devs || g_ncomms) return FVB_ERR_CONTRACT;
  if (!load_nccl()) return FVB_ERR_CUDA;
  const int rc = nccl_rc(g_nccl.commInitAll(g_comms, ndev, devs));
  if (rc == FVB_OK) {
    g_ncomms = ndev;
    g_rank_base = 0;
  }
  return rc;
}

int fvb_mgpu_allreduce_max(int rank, double* buf, void* stream) {
  const int k = rank - g_rank_base;
  if (!buf || k < 0 || k >= g_ncomms) return FVB_ERR_CONTRACT;
  return nccl_rc(g_nccl.allReduce(buf, buf, 1, ncclFloat64, ncclMax, g_comms[k],
                                  reinterpret_cast<cudaStream_t>(stream)));
}

int fvb_mgpu_allreduce_max_all(double* const* bufs, void* const* streams) {
  if (!bufs || !streams || g_ncomms < 1) return FVB_ERR_CONTRACT;
  int rc = nccl_rc(g_nccl.groupStart());
  for (int k = 0; k < g_ncomms && rc == FVB_OK; ++k)
    rc = nccl_rc(g_nccl.allReduce(bufs[k], bufs[k], 1, ncclFloat64, ncclMax, g_comms[k],
                                  reinterpret_cast<cudaStream_t>(streams[k])));
  const int rc2 = nccl_rc(g_nccl.groupEnd());
  return rc != FVB_OK ? rc : rc2;
}

int fvb_mgpu_finalize(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc = FVB_OK;
  for (int k = 0; k < g_ncomms; ++k)
    if (g_nccl.commDestroy(g_comms[k]) != ncclSuccess) rc = FVB_ERR_CUDA;
  g_ncomms = 0;
  g_rank_base = 0;
  return rc;
}

}  // extern "C"
