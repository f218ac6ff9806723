// Communicators of the slab decomposition (SURVEY.md
// 8(e)): the three exchanges the distributed path needs, stream-ordered on the
// caller's stream.
//   halo           neighbour exchange of one ghost parent layer per side
//                  (ranks r-1 and r+1 along the slowest axis)
//   allgather      fixed-size blocks (the per-rank partial dot products of CG)
//   allreduce_sum  vectors on the distributed -> replicated level transition
//                  (every entry has exactly one non-zero contribution)
// Two transports: NCCL (one process per GPU, libnccl.so.2 resolved at run
// time) and an in-process team of host threads (one handle per thread, any
// GPUs, copies over UVA) used to test the distributed path on one device.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

struct ipmg_comm {
  int rank = 0, nranks = 1;
  std::string err;
  virtual ~ipmg_comm() {}
  virtual const char* kind() const = 0;
  // send lo_src to rank-1 and hi_src to rank+1; receive rank-1's hi_src into
  // lo_dst and rank+1's lo_src into hi_dst (absent neighbours skipped)
  virtual bool halo(const void* lo_src, const void* hi_src, void* lo_dst, void* hi_dst, size_t bytes,
                    cudaStream_t s) = 0;
  // dst[r * bytes ..] = block of rank r
  virtual bool allgather(const void* src, void* dst, size_t bytes, cudaStream_t s) = 0;
  // buf = sum over ranks (prec 0 double, 1 float)
  virtual bool allreduce_sum(void* buf, size_t n, int prec, cudaStream_t s) = 0;
  virtual bool capturable() const = 0;   // may be recorded into a CUDA graph
  // host wait for stream s (the solvers' per-iteration scalar reads).  NCCL: polls the
  // stream and ncclCommGetAsyncError; a communicator error, or no progress for
  // IPMG_NCCL_TIMEOUT seconds (default 120), aborts the communicator (ncclCommAbort, so
  // a kernel blocked on a dead peer returns) and fails with err set.
  virtual bool wait(cudaStream_t s);
};

namespace ipmg {

// shared state of an in-process team
struct Team {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int waiting = 0;
  long long generation = 0;
  bool broken = false;
  struct Slot {
    const void* a = nullptr;
    const void* b = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    void* scratch = nullptr;     // allreduce staging: (n-1) * bytes, owned by the rank
    size_t scratch_bytes = 0;
    int device = 0;
  };
  std::vector<Slot> slots;
  // returns false on timeout / broken team (a peer failed): never hangs forever
  bool barrier(double timeout_s);
};

ipmg_comm* make_local_comm(std::shared_ptr<Team> team, int rank, int device, std::string* err);
ipmg_comm* make_nccl_comm(const void* unique_id, int rank, int nranks, int device, std::string* err);
bool nccl_unique_id(void* out128, std::string* err);

}  // namespace ipmg
