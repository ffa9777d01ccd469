// comm.cu -- the collectives of a sharded context, behind one interface with
// two transports:
//   * NCCL, resolved at run time (dlopen of libnccl.so.2: the library has no link-time NCCL
//     dependency, and inside a PyTorch process it binds to the NCCL torch already loaded);
//     one process per GPU, NVLink / NVSwitch between them.  Only the types and enums come
//     from nccl.h.
//   * an in-process group: G contexts driven by G host threads of one process (on one or
//     several devices); the exchanges are device-to-device copies between the posted
//     buffers, ordered by a host barrier.  It exists so that the whole distributed path --
//     sample-sort build and sharded edits -- runs through the C ABI on a single GPU (NCCL
//     cannot put two ranks on one device), with the same code above this interface.
// Every operation is collective and issued on the caller's stream; the in-process group
// synchronises the host, NCCL does not.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "dvl_internal.h"

namespace dvl {

// ----------------------------------------------------------------------------- NCCL
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
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
    api.send = (decltype(api.send))dlsym(h, "ncclSend");
    api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather &&
             api.allReduce && api.send && api.recv && api.groupStart && api.groupEnd &&
             api.errorString;
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

static ncclDataType_t nccl_type(RedType t) {
  return t == kU32 ? ncclUint32 : t == kI64 ? ncclInt64 : ncclUint64;
}

static ncclRedOp_t nccl_op(RedOp o) { return o == kMin ? ncclMin : o == kMax ? ncclMax : ncclSum; }

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c && nccl().ok) nccl().commDestroy(c);
  }
  const char* allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    const ncclResult_t r = nccl().allGather(send, recv, bytes, ncclInt8, c, st);
    return r == ncclSuccess ? nullptr : nccl_msg(r);
  }
  const char* allreduce(void* buf, size_t count, RedType t, RedOp op, cudaStream_t st) override {
    const ncclResult_t r = nccl().allReduce(buf, buf, count, nccl_type(t), nccl_op(op), c, st);
    return r == ncclSuccess ? nullptr : nccl_msg(r);
  }
  const char* merge_export(int64_t* buf, size_t max_words, size_t sum_words,
                           cudaStream_t st) override {
    ncclResult_t r = nccl().groupStart();
    if (r == ncclSuccess) r = nccl().allReduce(buf, buf, max_words, ncclInt64, ncclMax, c, st);
    if (r == ncclSuccess)
      r = nccl().allReduce(buf + max_words, buf + max_words, sum_words, ncclInt64, ncclSum, c, st);
    const ncclResult_t r2 = nccl().groupEnd();
    if (r == ncclSuccess) r = r2;
    return r == ncclSuccess ? nullptr : nccl_msg(r);
  }
  const char* alltoallv(const void* const* send, const size_t* sbytes, void* const* recv,
                        const size_t* rbytes, cudaStream_t st) override {
    ncclResult_t r = nccl().groupStart();
    for (int p = 0; p < nranks && r == ncclSuccess; ++p) {
      if (sbytes[p]) r = nccl().send(send[p], sbytes[p], ncclInt8, p, c, st);
      if (r == ncclSuccess && rbytes[p]) r = nccl().recv(recv[p], rbytes[p], ncclInt8, p, c, st);
    }
    const ncclResult_t r2 = nccl().groupEnd();
    if (r == ncclSuccess) r = r2;
    return r == ncclSuccess ? nullptr : nccl_msg(r);
  }
};

Comm* make_nccl_comm(int nranks, int rank, const void* id128, const char** err) {
  *err = nullptr;
  if (!nccl().ok) {
    *err = "libnccl.so.2 not found";
    return nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().commInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) {
    *err = nccl_msg(r);
    return nullptr;
  }
  NcclComm* cm = new NcclComm();
  cm->c = c;
  cm->nranks = nranks;
  cm->rank = rank;
  return cm;
}

// ------------------------------------------------------------------ in-process group
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int refs = 1;
  std::vector<const void*> ptr;                 // posted buffer of each rank
  std::vector<const void* const*> ptrs;         // posted per-peer send buffers
  std::vector<const size_t*> sizes;             // ... and their byte counts
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

LocalGroup* local_group_create(int n) {
  LocalGroup* g = new LocalGroup();
  g->n = n;
  g->ptr.assign(n, nullptr);
  g->ptrs.assign(n, nullptr);
  g->sizes.assign(n, nullptr);
  return g;
}

int local_group_size(const LocalGroup* g) { return g->n; }

void local_group_release(LocalGroup* g) {
  if (!g) return;
  bool last;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    last = --g->refs == 0;
  }
  if (last) delete g;
}

static const char* cuda_msg(cudaError_t e) { return e == cudaSuccess ? nullptr : cudaGetErrorString(e); }

struct LocalComm final : Comm {
  LocalGroup* g = nullptr;
  ~LocalComm() override { local_group_release(g); }

  const char* allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    cudaError_t e = cudaStreamSynchronize(st);   // the send buffer is complete
    g->ptr[rank] = send;
    g->barrier();
    for (int p = 0; p < nranks && e == cudaSuccess; ++p)
      e = cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)p * bytes, g->ptr[p], bytes,
                          cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    g->barrier();                                // every peer has read our buffer
    return cuda_msg(e);
  }

  template <typename T>
  static void reduce_into(T* acc, const T* v, size_t count, RedOp op) {
    for (size_t i = 0; i < count; ++i)
      acc[i] = op == kSum ? (T)(acc[i] + v[i]) : op == kMin ? (v[i] < acc[i] ? v[i] : acc[i])
                                                             : (v[i] > acc[i] ? v[i] : acc[i]);
  }

  // host reduction of the posted buffers (the operands are small: totals, counts, ranges,
  // the per-pixel accumulator export)
  template <typename T>
  const char* reduce_t(T* buf, size_t count, RedOp op, size_t sum_from, cudaStream_t st) {
    cudaError_t e = cudaStreamSynchronize(st);
    g->ptr[rank] = buf;
    g->barrier();
    std::vector<T> acc(count), v(count);
    for (int p = 0; p < nranks && e == cudaSuccess; ++p) {
      e = cudaMemcpy(p == 0 ? acc.data() : v.data(), g->ptr[p], count * sizeof(T), cudaMemcpyDefault);
      if (p > 0 && e == cudaSuccess) {
        reduce_into(acc.data(), v.data(), sum_from, op);
        reduce_into(acc.data() + sum_from, v.data() + sum_from, count - sum_from, kSum);
      }
    }
    g->barrier();                                // all peers have read before anyone writes
    if (e == cudaSuccess) e = cudaMemcpy(buf, acc.data(), count * sizeof(T), cudaMemcpyDefault);
    g->barrier();
    return cuda_msg(e);
  }

  const char* allreduce(void* buf, size_t count, RedType t, RedOp op, cudaStream_t st) override {
    if (t == kU32) return reduce_t(static_cast<uint32_t*>(buf), count, op, count, st);
    if (t == kI64) return reduce_t(static_cast<int64_t*>(buf), count, op, count, st);
    return reduce_t(static_cast<uint64_t*>(buf), count, op, count, st);
  }

  const char* merge_export(int64_t* buf, size_t max_words, size_t sum_words,
                           cudaStream_t st) override {
    return reduce_t(buf, max_words + sum_words, kMax, max_words, st);
  }

  const char* alltoallv(const void* const* send, const size_t* sbytes, void* const* recv,
                        const size_t* rbytes, cudaStream_t st) override {
    cudaError_t e = cudaStreamSynchronize(st);
    g->ptrs[rank] = send;
    g->sizes[rank] = sbytes;
    g->barrier();
    const char* bad = nullptr;
    for (int p = 0; p < nranks && e == cudaSuccess; ++p) {
      if (g->sizes[p][rank] != rbytes[p]) bad = "alltoallv: send / receive sizes differ";
      else if (rbytes[p])
        e = cudaMemcpyAsync(recv[p], g->ptrs[p][rank], rbytes[p], cudaMemcpyDefault, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    g->barrier();
    return bad ? bad : cuda_msg(e);
  }
};

Comm* make_local_comm(LocalGroup* g, int rank) {
  {
    std::lock_guard<std::mutex> lk(g->mu);
    ++g->refs;
  }
  LocalComm* c = new LocalComm();
  c->g = g;
  c->nranks = g->n;
  c->rank = rank;
  return c;
}

}  // namespace dvl
