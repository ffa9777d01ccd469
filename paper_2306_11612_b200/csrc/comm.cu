// comm.cu -- NCCL for sharded contexts, resolved at run time (dlopen of libnccl.so.2: the
// library has no link-time NCCL dependency, and inside a PyTorch process it binds to the
// NCCL that torch already loaded).  Only the types and enums come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "dvl_internal.h"

namespace dvl {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather &&
             api.allReduce && api.groupStart && api.groupEnd && api.errorString;
  });
  return api;
}

static const char* nccl_msg(ncclResult_t r) {
  return nccl().errorString ? nccl().errorString(r) : "NCCL error";
}

const char* nccl_unique_id(void* id128) {
  if (!nccl().ok) return "libnccl.so.2 not found";
  ncclUniqueId id;
  const ncclResult_t r = nccl().getUniqueId(&id);
  if (r != ncclSuccess) return nccl_msg(r);
  memcpy(id128, &id, sizeof(id));
  return nullptr;
}

const char* nccl_comm_init(void** comm, int nranks, int rank, const void* id128) {
  if (!nccl().ok) return "libnccl.so.2 not found";
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().commInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_msg(r);
  *comm = c;
  return nullptr;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().commDestroy((ncclComm_t)comm);
}

// the two exchanges of a sharded edit: the Q totals of all shards, and the
// merge of the accumulator exports (MAX over the first `max_words`, SUM over the next
// `sum_words`, both int64, in place, as one NCCL group)
const char* nccl_gather_totals(void* comm, const uint64_t* total, uint64_t* totals,
                               cudaStream_t st) {
  const ncclResult_t r = nccl().allGather(total, totals, 1, ncclUint64, (ncclComm_t)comm, st);
  return r == ncclSuccess ? nullptr : nccl_msg(r);
}

const char* nccl_merge_export(void* comm, int64_t* buf, size_t max_words, size_t sum_words,
                              cudaStream_t st) {
  ncclResult_t r = nccl().groupStart();
  if (r == ncclSuccess)
    r = nccl().allReduce(buf, buf, max_words, ncclInt64, ncclMax, (ncclComm_t)comm, st);
  if (r == ncclSuccess)
    r = nccl().allReduce(buf + max_words, buf + max_words, sum_words, ncclInt64, ncclSum,
                         (ncclComm_t)comm, st);
  const ncclResult_t r2 = nccl().groupEnd();
  if (r == ncclSuccess) r = r2;
  return r == ncclSuccess ? nullptr : nccl_msg(r);
}

}  // namespace dvl
