// Transports of the slab decomposition (comm.hpp): NCCL resolved at run time
// from libnccl.so.2 (the copy torch already loaded, else the system one) and
// the in-process thread team.
#include "comm.hpp"

#include <dlfcn.h>

#include <chrono>
#include <cstdlib>
#include <thread>
#include <cstring>

#include "blas.cuh"

namespace ipmg {

bool Team::barrier(double timeout_s) {
  std::unique_lock<std::mutex> lk(mu);
  if (broken) return false;
  const long long gen = generation;
  if (++waiting == n) {
    waiting = 0;
    ++generation;
    cv.notify_all();
    return true;
  }
  const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                              [&] { return generation != gen || broken; });
  if (!ok) {   // a peer never arrived (failed call): break the team instead of hanging
    broken = true;
    cv.notify_all();
    return false;
  }
  return generation != gen;
}

namespace {

constexpr double kTimeout = 120.0;

// ------------------------------------------------------------ in-process team
struct LocalComm : ipmg_comm {
  std::shared_ptr<Team> team;
  int device = 0;
  const char* kind() const override { return "local"; }
  bool capturable() const override { return false; }   // host barriers

  bool fail(const char* what, cudaError_t e = cudaSuccess) {
    err = std::string("local comm: ") + what + (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : "");
    {
      std::lock_guard<std::mutex> lk(team->mu);
      team->broken = true;
    }
    team->cv.notify_all();
    return false;
  }
#define LC_CK(call, what)                    \
  do {                                       \
    cudaError_t e_ = (call);                 \
    if (e_ != cudaSuccess) return fail(what, e_); \
  } while (0)

  Team::Slot& me() { return team->slots[rank]; }
  Team::Slot& of(int r) { return team->slots[r]; }

  bool halo(const void* lo_src, const void* hi_src, void* lo_dst, void* hi_dst, size_t bytes,
            cudaStream_t s) override {
    LC_CK(cudaSetDevice(device), "set device");
    me().a = lo_src;
    me().b = hi_src;
    LC_CK(cudaEventRecord(me().ready, s), "record");
    if (!team->barrier(kTimeout)) return fail("barrier (halo post)");
    if (rank > 0 && lo_dst) {
      LC_CK(cudaStreamWaitEvent(s, of(rank - 1).ready, 0), "wait");
      LC_CK(cudaMemcpyAsync(lo_dst, of(rank - 1).b, bytes, cudaMemcpyDefault, s), "copy lo");
    }
    if (rank + 1 < nranks && hi_dst) {
      LC_CK(cudaStreamWaitEvent(s, of(rank + 1).ready, 0), "wait");
      LC_CK(cudaMemcpyAsync(hi_dst, of(rank + 1).a, bytes, cudaMemcpyDefault, s), "copy hi");
    }
    LC_CK(cudaEventRecord(me().done, s), "record");
    if (!team->barrier(kTimeout)) return fail("barrier (halo done)");
    // the neighbours' reads of MY layers must finish before I overwrite them
    if (rank > 0) LC_CK(cudaStreamWaitEvent(s, of(rank - 1).done, 0), "wait");
    if (rank + 1 < nranks) LC_CK(cudaStreamWaitEvent(s, of(rank + 1).done, 0), "wait");
    return true;
  }

  bool allgather(const void* src, void* dst, size_t bytes, cudaStream_t s) override {
    LC_CK(cudaSetDevice(device), "set device");
    me().a = src;
    LC_CK(cudaEventRecord(me().ready, s), "record");
    if (!team->barrier(kTimeout)) return fail("barrier (allgather post)");
    for (int r = 0; r < nranks; ++r) {
      if (r != rank) LC_CK(cudaStreamWaitEvent(s, of(r).ready, 0), "wait");
      LC_CK(cudaMemcpyAsync((char*)dst + r * bytes, of(r).a, bytes, cudaMemcpyDefault, s), "copy");
    }
    LC_CK(cudaEventRecord(me().done, s), "record");
    if (!team->barrier(kTimeout)) return fail("barrier (allgather done)");
    for (int r = 0; r < nranks; ++r)
      if (r != rank) LC_CK(cudaStreamWaitEvent(s, of(r).done, 0), "wait");
    return true;
  }

  bool allreduce_sum(void* buf, size_t n, int prec, cudaStream_t s) override {
    LC_CK(cudaSetDevice(device), "set device");
    const size_t bytes = n * (prec == 0 ? 8 : 4);
    const size_t need = bytes * (size_t)(nranks - 1);
    if (me().scratch_bytes < need) {
      if (me().scratch) cudaFree(me().scratch);
      me().scratch = nullptr;
      me().scratch_bytes = 0;
      LC_CK(cudaMalloc(&me().scratch, need), "scratch alloc");
      me().scratch_bytes = need;
    }
    me().a = buf;
    LC_CK(cudaEventRecord(me().ready, s), "record");
    if (!team->barrier(kTimeout)) return fail("barrier (allreduce post)");
    int j = 0;
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      LC_CK(cudaStreamWaitEvent(s, of(r).ready, 0), "wait");
      LC_CK(cudaMemcpyAsync((char*)me().scratch + (size_t)j * bytes, of(r).a, bytes, cudaMemcpyDefault, s), "copy");
      ++j;
    }
    LC_CK(cudaEventRecord(me().done, s), "record");
    if (!team->barrier(kTimeout)) return fail("barrier (allreduce done)");
    for (int r = 0; r < nranks; ++r)
      if (r != rank) LC_CK(cudaStreamWaitEvent(s, of(r).done, 0), "wait");
    LC_CK(sum_ranks(prec, buf, me().scratch, nranks, rank, (long long)n, s), "sum");
    return true;
  }
#undef LC_CK

  ~LocalComm() override {
    Team::Slot& m = team->slots[rank];
    if (m.ready) cudaEventDestroy(m.ready);
    if (m.done) cudaEventDestroy(m.done);
    if (m.scratch) cudaFree(m.scratch);
    m.ready = m.done = nullptr;
    m.scratch = nullptr;
  }
};

// ------------------------------------------------------------ NCCL (run-time resolved)
typedef int ncclResult_t;
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { ncclUint8 = 1, ncclFloat32 = 7, ncclFloat64 = 8 };
enum { ncclSum = 0 };

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy, if loaded
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      a.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return a;
    }
    bool all = true;
    auto sym = [&](const char* name) {
      void* p = dlsym(lib, name);
      if (!p) all = false;
      return p;
    };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    a.CommGetAsyncError = (decltype(a.CommGetAsyncError))sym("ncclCommGetAsyncError");
    a.CommAbort = (decltype(a.CommAbort))sym("ncclCommAbort");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

struct NcclComm : ipmg_comm {
  ncclComm_t comm = nullptr;
  int device = 0;
  const char* kind() const override { return "nccl"; }
  bool capturable() const override { return true; }
  bool ck(ncclResult_t r, const char* what) {
    if (r == 0) return true;
    err = std::string("nccl ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
    return false;
  }
  bool halo(const void* lo_src, const void* hi_src, void* lo_dst, void* hi_dst, size_t bytes,
            cudaStream_t s) override {
    if (nranks == 1) return true;
    const NcclApi& a = nccl();
    if (!ck(a.GroupStart(), "group start")) return false;
    // record the first failure but always close the group: an open group would swallow
    // every later NCCL call of this thread (torch's included)
    bool ok = true;
    if (rank > 0) {
      ok = ok && ck(a.Send(lo_src, bytes, ncclUint8, rank - 1, comm, s), "send lo");
      ok = ok && ck(a.Recv(lo_dst, bytes, ncclUint8, rank - 1, comm, s), "recv lo");
    }
    if (rank + 1 < nranks) {
      ok = ok && ck(a.Send(hi_src, bytes, ncclUint8, rank + 1, comm, s), "send hi");
      ok = ok && ck(a.Recv(hi_dst, bytes, ncclUint8, rank + 1, comm, s), "recv hi");
    }
    const std::string first = err;
    const bool closed = ck(a.GroupEnd(), "group end");
    if (!ok) err = first;
    return ok && closed;
  }
  bool wait(cudaStream_t s) override {
    const NcclApi& a = nccl();
    static const double limit = [] {
      const char* e = std::getenv("IPMG_NCCL_TIMEOUT");
      const double v = e ? std::atof(e) : 0.0;
      return v > 0 ? v : 120.0;
    }();
    if (!comm) {
      err = "nccl communicator was aborted";
      return false;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (long spin = 0;; ++spin) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) return true;
      if (q != cudaErrorNotReady) {
        err = std::string("stream wait: ") + cudaGetErrorString(q);
        return false;
      }
      ncclResult_t ae = 0;
      if (a.CommGetAsyncError && a.CommGetAsyncError(comm, &ae) == 0 && ae != 0 && ae != 7 /* ncclInProgress */) {
        err = std::string("nccl async error: ") + (a.GetErrorString ? a.GetErrorString(ae) : "?");
        if (a.CommAbort) a.CommAbort(comm);
        comm = nullptr;
        return false;
      }
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
        err = "nccl: no progress for IPMG_NCCL_TIMEOUT seconds (peer failed or stalled); communicator aborted";
        if (a.CommAbort) a.CommAbort(comm);
        comm = nullptr;
        return false;
      }
      if (spin > 2000) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
  bool allgather(const void* src, void* dst, size_t bytes, cudaStream_t s) override {
    return ck(nccl().AllGather(src, dst, bytes, ncclUint8, comm, s), "allgather");
  }
  bool allreduce_sum(void* buf, size_t n, int prec, cudaStream_t s) override {
    return ck(nccl().AllReduce(buf, buf, n, prec == 0 ? ncclFloat64 : ncclFloat32, ncclSum, comm, s), "allreduce");
  }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
};

}  // namespace

ipmg_comm* make_local_comm(std::shared_ptr<Team> team, int rank, int device, std::string* err) {
  LocalComm* c = new LocalComm();
  c->team = team;
  c->rank = rank;
  c->nranks = team->n;
  c->device = device;
  Team::Slot& m = team->slots[rank];
  m.device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&m.done, cudaEventDisableTiming) != cudaSuccess) {
    *err = "local comm: event creation failed";
    delete c;
    return nullptr;
  }
  return c;
}

bool nccl_unique_id(void* out128, std::string* err) {
  const NcclApi& a = nccl();
  if (!a.ok) {
    *err = a.why;
    return false;
  }
  ncclUniqueId id;
  const ncclResult_t r = a.GetUniqueId(&id);
  if (r != 0) {
    *err = std::string("ncclGetUniqueId: ") + a.GetErrorString(r);
    return false;
  }
  std::memcpy(out128, &id, sizeof(id));
  return true;
}

ipmg_comm* make_nccl_comm(const void* unique_id, int rank, int nranks, int device, std::string* err) {
  const NcclApi& a = nccl();
  if (!a.ok) {
    *err = a.why;
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    *err = "cudaSetDevice failed";
    return nullptr;
  }
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  const ncclResult_t r = a.CommInitRank(&c->comm, nranks, id, rank);
  if (r != 0) {
    *err = std::string("ncclCommInitRank: ") + a.GetErrorString(r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

}  // namespace ipmg

bool ipmg_comm::wait(cudaStream_t s) {
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) return true;
  err = std::string("stream wait: ") + cudaGetErrorString(e);
  return false;
}
