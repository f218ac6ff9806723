// C ABI of the ipmg library: handle, host setup, V-cycle and PCG drivers.
// The declarations and their contracts are in include/ipmg.h.
#include "ipmg.h"

#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "blas.cuh"
#include "comm.hpp"
#include "common.cuh"
#include "fe1d.hpp"

ipmg::KernelSet ipmg_kernel_set_k1();
ipmg::KernelSet ipmg_kernel_set_k2();
ipmg::KernelSet ipmg_kernel_set_k3();
ipmg::KernelSet ipmg_kernel_set_k4();
ipmg::KernelSet ipmg_kernel_set_k5();
ipmg::KernelSet ipmg_kernel_set_k6();
ipmg::KernelSet ipmg_kernel_set_k7();
ipmg::KernelSet ipmg_kernel_set_dir_k1();
ipmg::KernelSet ipmg_kernel_set_dir_k2();
ipmg::KernelSet ipmg_kernel_set_dir_k3();
ipmg::KernelSet ipmg_kernel_set_dir_k4();
ipmg::KernelSet ipmg_kernel_set_dir_k5();
ipmg::KernelSet ipmg_kernel_set_dir_k6();
ipmg::KernelSet ipmg_kernel_set_dir_k7();

namespace {

std::string g_create_error;

// partition rule of the slab decomposition (ipmg.h ipmg_partition)
// min_local_dofs: a level is only distributed if every rank keeps at least this
// many dofs of it (coarser levels are replicated: their halo exchanges would cost
// more latency than computing them redundantly); 0 = distribute whenever possible
void partition_rule(int dim, const int cc[3], int l, int nranks, int rank, int out[4], int degree = 1,
                    long long min_local_dofs = 0) {
  const int S = dim - 1;
  const long long ng = (long long)cc[S] << l;
  long long layer_dofs = 1;
  for (int a = 0; a < dim - 1; ++a) layer_dofs *= (long long)cc[a] << l;
  for (int a = 0; a < dim; ++a) layer_dofs *= degree + 1;
  const bool big = ng / (nranks > 0 ? nranks : 1) * layer_dofs >= min_local_dofs;
  const int dist = nranks == 1 ? 1 : (l >= 1 && ng % (2LL * nranks) == 0 && big ? 1 : 0);
  out[0] = dist;
  out[3] = (int)ng;
  out[2] = dist ? (int)(ng / nranks) : (int)ng;
  out[1] = dist ? rank * out[2] : 0;
}

ipmg::KernelSet kernel_set(int k) {
  switch (k) {
    case 1: return ipmg_kernel_set_k1();
    case 2: return ipmg_kernel_set_k2();
    case 3: return ipmg_kernel_set_k3();
    case 4: return ipmg_kernel_set_k4();
    case 5: return ipmg_kernel_set_k5();
    case 6: return ipmg_kernel_set_k6();
    default: return ipmg_kernel_set_k7();
  }
}
ipmg::KernelSet kernel_set_dir(int k) {
  switch (k) {
    case 1: return ipmg_kernel_set_dir_k1();
    case 2: return ipmg_kernel_set_dir_k2();
    case 3: return ipmg_kernel_set_dir_k3();
    case 4: return ipmg_kernel_set_dir_k4();
    case 5: return ipmg_kernel_set_dir_k5();
    case 6: return ipmg_kernel_set_dir_k6();
    default: return ipmg_kernel_set_dir_k7();
  }
}

}  // namespace

enum KClass { KC_SMOOTH = 0, KC_VMULT = 1, KC_RESTRICT = 2, KC_PROLONG = 3, KC_COARSE = 4, KC_BLAS = 5,
              KC_ADDITIVE = 6, KC_BELOW = 7, KC_N = 8 };

struct ipmg_handle {
  ipmg_config cfg{};
  int dim = 3, k = 1, nc = 2, cell = 8, nlev = 1;
  cudaStream_t stream = nullptr;
  ipmg::KernelSet ks{};
  ipmg::KernelSet ksd{};              // Dirichlet-kernel smoother (cfg.kernel == IPMG_KERNEL_DIRICHLET)
  ipmg::FE1D fe;
  std::vector<ipmg::LevelGeom> geom;
  std::vector<long long> ndofs;
  std::vector<double> hsize;
  // V-cycle / API workspace: [prec][level]
  std::vector<void*> vx0[2], vx1[2], vb[2], scratch[2];
  // coarse FD tables per precision and direction
  void* cS[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  void* cL[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  ipmg::CoarseDesc cdesc{};
  // PCG workspace (finest level, fp64)
  double *r = nullptr, *p = nullptr, *q = nullptr, *z = nullptr;
  double *partial = nullptr, *scal = nullptr, *hpin = nullptr, *pattern = nullptr;
  double *hpin_dev = nullptr, *ghpin_dev = nullptr;   // device aliases of the mapped pinned buffers
  long long partial_len = 0;
  std::vector<void*> allocs;
  std::string err;
  // ---- slab decomposition
  ipmg_comm* comm = nullptr;
  int rank = 0, nranks = 1;
  std::vector<int> dist;              // level distributed over the ranks (1) or replicated (0)
  std::vector<long long> ghost;       // elements of one ghost parent layer (0: no ghosts)
  double* gbuf = nullptr;             // allgathered per-rank scalars
  // halo/compute overlap: the exchange runs on cstream while the interior patch
  // blocks (which never touch ghosts) run on the main stream
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool overlap = true;
  std::vector<void*> gsc[2][3];       // ghosted copies of caller vectors (API calls), [prec][slot][level]
  // ---- the finest-level V-cycle captured as a CUDA graph per precision
  // ---- GMRES workspace (finest level, fp64): Krylov basis V, preconditioned Z
  std::vector<double*> gV, gZ;
  double *gw = nullptr, *ghcol = nullptr, *gy = nullptr, *ghpin = nullptr;
  const double** gzptr = nullptr;
  int gcap = 0;
  cudaGraphExec_t vgraph[2] = {nullptr, nullptr};
  long long vgraph_launches[2] = {0, 0};
  bool use_graphs = true;
  // ---- instrumentation: launch counter and (optional) CUDA-event timing of
  // the finest-level kernels, per kernel class (ipmg_profile*)
  long long n_launches = 0;
  bool prof_on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  struct Rec { int cls; double bytes; };
  std::vector<Rec> recs;

  template <class F>
  ipmg_status run(int cls, int level, double bytes, int nlaunch, F&& f, const char* what) {
    n_launches += nlaunch;
    const bool rec = prof_on && level == nlev - 1;
    std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
    if (rec) {
      if (recs.size() == ev_pool.size()) {
        std::pair<cudaEvent_t, cudaEvent_t> p;
        cudaEventCreate(&p.first);
        cudaEventCreate(&p.second);
        ev_pool.push_back(p);
      }
      ev = &ev_pool[recs.size()];
      cudaEventRecord(ev->first, stream);
    }
    cudaError_t e = f();
    if (rec) {
      cudaEventRecord(ev->second, stream);
      recs.push_back(Rec{cls, bytes});
    }
    return cuda(e, what);
  }
  // algorithmic HBM bytes of one smoother colour pass:
  // covered dofs read b and x_in and write x_out, uncovered dofs are copied
  double smooth_bytes(int level, int prec, int colour, bool has_x) const {
    long long covered = 1;
    for (int a = 0; a < dim; ++a) covered *= ((colour >> a) & 1) ? geom[level].n[a] - 2 : geom[level].n[a];
    const double cov = (double)covered * cell, unc = (double)ndofs[level] - cov;
    return esize(prec) * (cov * (2 + (has_x ? 1 : 0)) + unc * (1 + (has_x ? 1 : 0)));
  }

  // host wait on the handle's stream: through the communicator when there is one (the
  // NCCL transport polls for asynchronous errors and aborts on a stalled peer)
  ipmg_status host_sync(cudaStream_t s) {
    if (comm) {
      if (comm->wait(s)) return IPMG_OK;
      err = comm->err;
      return IPMG_ERR_NCCL;
    }
    return cuda(cudaStreamSynchronize(s), "sync");
  }
  std::vector<double*> sin_tab;   // ipmg_rhs kind 1: per level, 3 global 1D moment tables

  ipmg_status fail(ipmg_status st, const std::string& msg) {
    err = msg;
    return st;
  }
  ipmg_status cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return IPMG_OK;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return IPMG_ERR_CUDA;
  }
  void* dalloc(size_t bytes) {
    void* ptr = nullptr;
    if (cudaMalloc(&ptr, bytes) != cudaSuccess) return nullptr;
    allocs.push_back(ptr);
    return ptr;
  }
  size_t esize(int prec) const { return prec == IPMG_FP64 ? 8 : 4; }
  // level vector with a ghost parent layer before and after the local range
  // (distributed levels with several ranks; plain otherwise)
  void* valloc(int level, int prec) {
    const long long gh = ghost[level];
    char* base = (char*)dalloc((size_t)(ndofs[level] + 2 * gh) * esize(prec));
    return base ? base + gh * esize(prec) : nullptr;
  }
  ipmg_status ensure_scratch(int prec, int level) {
    if (scratch[prec][level]) return IPMG_OK;
    scratch[prec][level] = valloc(level, prec);
    return scratch[prec][level] ? IPMG_OK : fail(IPMG_ERR_OUT_OF_MEMORY, "scratch allocation failed");
  }
  // ------------------------------------------------------------ communication
  // ghost parent layers of x from the neighbour ranks (x: a valloc'ed vector)
  ipmg_status halo(int level, int prec, const void* x) {
    if (!comm || ghost[level] == 0) return IPMG_OK;
    const size_t es = esize(prec), gb = (size_t)ghost[level] * es, nb = (size_t)ndofs[level] * es;
    char* xb = (char*)const_cast<void*>(x);
    if (!comm->halo(xb, xb + nb - gb, xb - gb, xb + nb, gb, stream)) return fail(IPMG_ERR_NCCL, comm->err);
    return IPMG_OK;
  }
  // halo exchange of x followed by a patch kernel that reads x's ghosts:
  // kernel(g) launches with the level geometry g; with several ranks the halo is
  // forked onto cstream, the interior blocks (zsel 1) run meanwhile, and the first
  // and last blocks (zsel 2) after the join.  bytes: algorithmic bytes (profiling).
  template <class K>
  ipmg_status halo_then(int level, int prec, const void* x, int cls, double bytes, K&& kernel, const char* what) {
    if (!comm || ghost[level] == 0)
      return run(cls, level, bytes, 1, [&] { return kernel(geom[level]); }, what);
    if (!overlap || !cstream) {
      ipmg_status st = halo(level, prec, x);
      if (st != IPMG_OK) return st;
      return run(cls, level, bytes, 1, [&] { return kernel(geom[level]); }, what);
    }
    ipmg::LevelGeom gi = geom[level], gb = geom[level];
    gi.zsel = 1;
    gb.zsel = 2;
    ipmg_status st = cuda(cudaEventRecord(ev_fork, stream), "fork");
    if (st != IPMG_OK) return st;
    st = cuda(cudaStreamWaitEvent(cstream, ev_fork, 0), "fork");
    if (st != IPMG_OK) return st;
    {
      const size_t es = esize(prec), gbs = (size_t)ghost[level] * es, nb = (size_t)ndofs[level] * es;
      char* xb = (char*)const_cast<void*>(x);
      if (!comm->halo(xb, xb + nb - gbs, xb - gbs, xb + nb, gbs, cstream)) return fail(IPMG_ERR_NCCL, comm->err);
    }
    st = cuda(cudaEventRecord(ev_join, cstream), "join");
    if (st != IPMG_OK) return st;
    st = run(cls, level, 0.0, 1, [&] { return kernel(gi); }, what);   // bytes booked on the second launch
    if (st != IPMG_OK) return st;
    st = cuda(cudaStreamWaitEvent(stream, ev_join, 0), "join");
    if (st != IPMG_OK) return st;
    return run(cls, level, bytes, 1, [&] { return kernel(gb); }, what);
  }
  // device scalar -> its sum over the ranks (rank order, identical everywhere)
  ipmg_status allsum(double* slot) {
    if (!comm || nranks == 1) return IPMG_OK;
    if (!comm->allgather(slot, gbuf, sizeof(double), stream)) return fail(IPMG_ERR_NCCL, comm->err);
    n_launches += 1;
    return cuda(ipmg::gather_sum(gbuf, nranks, 1, slot, stream), "gather_sum");
  }
  // restriction into a replicated level from a distributed one: every rank
  // writes its parents into a zeroed vector, the sum over ranks assembles it
  bool transition(int l) const { return nranks > 1 && l >= 1 && dist[l] && !dist[l - 1]; }
  // caller vector -> ghosted copy with current ghosts (distributed levels)
  ipmg_status ghosted(int level, int prec, int slot, const void* v, const void** out) {
    *out = v;
    if (!v || ghost[level] == 0) return IPMG_OK;
    std::vector<void*>& g = gsc[prec][slot];
    if (g.empty()) g.assign(nlev, nullptr);
    if (!g[level] && !(g[level] = valloc(level, prec))) return fail(IPMG_ERR_OUT_OF_MEMORY, "ghosted copy allocation failed");
    ipmg_status st = cuda(cudaMemcpyAsync(g[level], v, ndofs[level] * esize(prec), cudaMemcpyDeviceToDevice, stream), "copy");
    if (st != IPMG_OK) return st;
    st = halo(level, prec, g[level]);
    *out = g[level];
    return st;
  }
  ipmg_status ensure_vcycle(int prec) {
    if (!vx0[prec].empty() && vx0[prec][0]) return IPMG_OK;
    vx0[prec].assign(nlev, nullptr);
    vx1[prec].assign(nlev, nullptr);
    vb[prec].assign(nlev, nullptr);
    for (int l = 0; l < nlev; ++l) {
      vx0[prec][l] = valloc(l, prec);
      vx1[prec][l] = valloc(l, prec);
      vb[prec][l] = valloc(l, prec);
      if (!vx0[prec][l] || !vx1[prec][l] || !vb[prec][l])
        return fail(IPMG_ERR_OUT_OF_MEMORY, "V-cycle workspace allocation failed");
    }
    return IPMG_OK;
  }

  // ------------------------------------------------------------ building blocks
  // r.z fused into the V-cycle's last finest-level colour pass (mixed PCG): set by the
  // solver around vcycle_level(L); rz_nparts > 0 afterwards when the pass could fuse it
  const double* rz_r = nullptr;
  double* rz_part = nullptr;
  long long rz_nparts = 0;
  ipmg_status smooth_colour(int level, int prec, const void* xi, const void* b, void* xo, int colour) {
    return run(KC_SMOOTH, level, smooth_bytes(level, prec, colour, xi != nullptr), 1,
               [&] {
                 return (cfg.kernel != IPMG_KERNEL_FULL ? ksd : ks).smooth(dim, prec, xi, b, xo, geom[level], colour, stream);
               },
               "smooth_colour");
  }
  // colour pass whose x_in ghosts come from the neighbour ranks (halo overlapped)
  ipmg_status smooth_colour_halo(int level, int prec, const void* xi, const void* b, void* xo, int colour) {
    return halo_then(level, prec, xi, KC_SMOOTH, smooth_bytes(level, prec, colour, true),
                     [&](const ipmg::LevelGeom& g) {
                       return (cfg.kernel != IPMG_KERNEL_FULL ? ksd : ks).smooth(dim, prec, xi, b, xo, g, colour, stream);
                     },
                     "smooth_colour");
  }
  // multiplicative step: passes ping-pong between x and other; 2^d passes -> ends in x
  ipmg_status smooth_mult(int level, int prec, void* x, void* other, const void* b, bool reverse, bool x_is_zero) {
    const int ncol = 1 << dim;
    void* cur = x;
    void* nxt = other;
    for (int i = 0; i < ncol; ++i) {
      const int c = reverse ? ncol - 1 - i : i;
      const bool zero = i == 0 && x_is_zero;
      // every colour with x reads face traces (and straddling cells) of the neighbour slabs
      ipmg_status st;
      if (!zero && rz_r && i == ncol - 1 && level == nlev - 1 && cfg.kernel == IPMG_KERNEL_FULL && ks.smooth_rz) {
        long long np = 0;
        st = halo_then(level, prec, cur, KC_SMOOTH, smooth_bytes(level, prec, c, true) + 8.0 * ndofs[level],
                       [&](const ipmg::LevelGeom& g) {
                         return ks.smooth_rz(dim, prec, cur, b, nxt, g, c, rz_r, rz_part, &np, stream);
                       },
                       "smooth_colour");
        rz_nparts = np;
      } else {
        st = zero ? smooth_colour(level, prec, nullptr, b, nxt, c) : smooth_colour_halo(level, prec, cur, b, nxt, c);
      }
      if (st != IPMG_OK) return st;
      std::swap(cur, nxt);
    }
    return IPMG_OK;
  }
  double omega() const {
    return cfg.additive_omega > 0 ? cfg.additive_omega : 1.0 / (1 << dim);
  }
  // additive step: x += omega sum_j R_j^T A_j^{-1} R_j (b - A x); rbuf: residual scratch
  ipmg_status smooth_add(int level, int prec, void* x, void* rbuf, const void* b, bool x_is_zero) {
    const void* r = b;
    if (!x_is_zero) {
      ipmg_status st = halo_then(level, prec, x, KC_VMULT, 3.0 * esize(prec) * ndofs[level],
                                 [&](const ipmg::LevelGeom& g) { return ks.vmult(dim, prec, x, rbuf, g, b, nullptr, nullptr, stream); },
                                 "residual");
      if (st != IPMG_OK) return st;
      st = halo(level, prec, rbuf);   // straddling patches read r on the ghost cells
      if (st != IPMG_OK) return st;
      r = rbuf;
    } else {
      ipmg_status st = cuda(cudaMemsetAsync(x, 0, ndofs[level] * esize(prec), stream), "memset");
      if (st != IPMG_OK) return st;
    }
    for (int c = 0; c < (1 << dim); ++c) {
      ipmg_status st = run(KC_ADDITIVE, level, 3.0 * esize(prec) * ndofs[level] / (1 << dim), 1,
                           [&] { return ks.additive(dim, prec, r, x, geom[level], c, omega(), stream); }, "additive");
      if (st != IPMG_OK) return st;
    }
    return IPMG_OK;
  }
  ipmg_status coarse(int prec, const void* b, void* x) {
    const void* S[3] = {cS[prec][0], cS[prec][1], cS[prec][2]};
    const void* L[3] = {cL[prec][0], cL[prec][1], cL[prec][2]};
    return run(KC_COARSE, 0, 2.0 * esize(prec) * ndofs[0], 1,
               [&] { return ipmg::coarse_solve(prec, b, x, cdesc, S, L, stream); }, "coarse_solve");
  }
  // one V-cycle on level l of the workspace of precision prec: input vb[l],
  // output vx1[l]
  // r_c = P^T (b - A x) (x ghosts current), with the distributed -> replicated transition
  // x_halo: exchange x's ghosts first (overlapped with the interior parents)
  ipmg_status restrict_to(int l, int prec, const void* x, const void* b, void* rc, bool x_halo = false) {
    ipmg_status st;
    if (transition(l)) {
      st = cuda(cudaMemsetAsync(rc, 0, ndofs[l - 1] * esize(prec), stream), "memset");
      if (st != IPMG_OK) return st;
    }
    const double by = esize(prec) * (2.0 * ndofs[l] + ndofs[l - 1]);
    auto kern = [&](const ipmg::LevelGeom& g) { return ks.restrict_(dim, prec, x, b, rc, g, geom[l - 1], stream); };
    st = (x_halo && x) ? halo_then(l, prec, x, KC_RESTRICT, by, kern, "restrict")
                       : run(KC_RESTRICT, l, by, 1, [&] { return kern(geom[l]); }, "restrict");
    if (st != IPMG_OK || !transition(l)) return st;
    if (!comm->allreduce_sum(rc, ndofs[l - 1], prec, stream)) return fail(IPMG_ERR_NCCL, comm->err);
    return IPMG_OK;
  }
  ipmg_status vcycle_level(int l, int prec) {
    void* b = vb[prec][l];
    void* const x0 = vx0[prec][l];
    void* const x1 = vx1[prec][l];
    if (l == 0) return coarse(prec, b, x1);
    ipmg_status st = halo(l, prec, b);   // straddling patches read b on the ghost cells
    if (st != IPMG_OK) return st;
    const bool additive = cfg.smoother == IPMG_ADDITIVE;
    // (1) pre-smoothing from x = 0; smooth_* leave the result in their first buffer
    if (additive) st = smooth_add(l, prec, x1, x0, b, true);
    else st = smooth_mult(l, prec, x1, x0, b, false, true);
    if (st != IPMG_OK) return st;
    // (2) coarse-grid correction x1 += P P_{l-1}^{-1} P^T (b - A x1)
    st = restrict_to(l, prec, x1, b, vb[prec][l - 1], true);
    if (st != IPMG_OK) return st;
    st = l == nlev - 1 ? run_coarse_vcycle(prec) : vcycle_level(l - 1, prec);
    if (st != IPMG_OK) return st;
    st = run(KC_PROLONG, l, esize(prec) * (2.0 * ndofs[l] + ndofs[l - 1]), 1,
             [&] { return ks.prolong(dim, prec, vx1[prec][l - 1], x1, geom[l], geom[l - 1], stream); }, "prolong");
    if (st != IPMG_OK) return st;
    // (3) post-smoothing (colours reversed for a symmetric V-cycle, reading A7)
    if (additive) return smooth_add(l, prec, x1, x0, b, false);
    return smooth_mult(l, prec, x1, x0, b, cfg.post_smooth_reverse != 0, false);
  }
  // The coarse part of the V-cycle (levels L-1 .. 0, launch-latency bound:
  // ~100 small kernels) replayed from a CUDA graph captured on first use; the
  // finest level's kernels are launched directly (so ipmg_profile still times
  // them).  Not with a communicator that cannot be captured (in-process team).
  // timed as one record of class KC_BELOW (the levels below the finest, ipmg_profile)
  ipmg_status run_coarse_vcycle(int prec) {
    ipmg_status inner = IPMG_OK;
    const ipmg_status st = run(KC_BELOW, nlev - 1, 0.0, 0, [&] {
      inner = run_coarse_vcycle_impl(prec);
      return cudaSuccess;
    }, "levels below the finest");
    return inner != IPMG_OK ? inner : st;
  }
  ipmg_status run_coarse_vcycle_impl(int prec) {
    const int L = nlev - 2;
    if (!use_graphs || (comm && !comm->capturable())) return vcycle_level(L, prec);
    if (!vgraph[prec]) {
      cudaStream_t cap = nullptr;
      ipmg_status st = cuda(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
      if (st != IPMG_OK) return st;
      cudaStream_t saved = stream;
      stream = cap;
      const long long n0 = n_launches;
      cudaGraph_t gph = nullptr;
      cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        st = vcycle_level(L, prec);
        e = cudaStreamEndCapture(cap, &gph);
      }
      stream = saved;
      if (e == cudaSuccess && st == IPMG_OK) e = cudaGraphInstantiate(&vgraph[prec], gph, 0);
      if (gph) cudaGraphDestroy(gph);
      cudaStreamDestroy(cap);
      vgraph_launches[prec] = n_launches - n0;
      n_launches = n0;
      if (st != IPMG_OK) return st;
      if (e != cudaSuccess) {   // capture unsupported here: fall back to direct launches from now on
        vgraph[prec] = nullptr;
        use_graphs = false;
        cudaGetLastError();
        return vcycle_level(L, prec);
      }
    }
    n_launches += vgraph_launches[prec];
    return cuda(cudaGraphLaunch(vgraph[prec], stream), "graph launch");
  }
  // fp32 V-cycle on the finest level (input vb, output vx1) with r.z of the mixed PCG
  // fused into its last colour pass where the kernel supports it (rz_nparts > 0)
  ipmg_status vcycle_rz(int L) {
    static const bool fuse = [] {   // IPMG_RZ_FUSE=0: separate dot kernel (A/B runs)
      const char* e = std::getenv("IPMG_RZ_FUSE");
      return !(e && e[0] == '0');
    }();
    rz_r = fuse ? r : nullptr;
    rz_part = partial;
    rz_nparts = 0;
    const ipmg_status st = vcycle_level(L, IPMG_FP32);
    rz_r = nullptr;
    rz_part = nullptr;
    return st;
  }
  ipmg_status vcycle(const double* r, double* z, double* rz_partial) {
    const int prec = cfg.vcycle_precision;
    const int L = nlev - 1;
    ipmg_status st = ensure_vcycle(prec);
    if (st != IPMG_OK) return st;
    st = run(KC_BLAS, L, (8.0 + esize(prec)) * ndofs[L], prec == 0 ? 0 : 1,
             [&] { return ipmg::cast(0, prec, r, vb[prec][L], ndofs[L], stream); }, "cast in");
    if (st != IPMG_OK) return st;
    st = vcycle_level(L, prec);
    if (st != IPMG_OK) return st;
    if (rz_partial && prec == IPMG_FP32)
      return run(KC_BLAS, L, 20.0 * ndofs[L], 1,
                 [&] { return ipmg::cast_f2d_dot((const float*)vx1[prec][L], z, r, ndofs[L], rz_partial, stream); },
                 "cast out");
    st = run(KC_BLAS, L, (8.0 + esize(prec)) * ndofs[L], prec == 0 ? 0 : 1,
             [&] { return ipmg::cast(prec, 0, vx1[prec][L], z, ndofs[L], stream); }, "cast out");
    if (st != IPMG_OK || !rz_partial) return st;
    return run(KC_BLAS, L, 16.0 * ndofs[L], 1,
               [&] { return ipmg::dot_partial(0, 0, r, z, ndofs[L], rz_partial, stream); }, "dot");
  }
};

// Scoped device guard of every entry point that takes a handle: the handle's work runs on
// cfg.device whatever device the calling thread has current, and the caller's current
// device is restored on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const ipmg_handle* h) {
    if (!h) return;
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != h->cfg.device && cudaSetDevice(h->cfg.device) == cudaSuccess)
      prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

extern "C" {

void ipmg_config_default(ipmg_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->dim = 3;
  c->degree = 4;
  c->coarse_cells[0] = c->coarse_cells[1] = c->coarse_cells[2] = 2;
  c->n_levels = 3;
  c->h0 = 0.5;
  c->kernel = IPMG_KERNEL_FULL;
  c->smoother = IPMG_MULTIPLICATIVE;
  c->additive_omega = 0.0;
  c->post_smooth_reverse = 1;
  c->vcycle_precision = IPMG_FP32;
  c->penalty_scale = 1.0;
  c->basis = IPMG_BASIS_LAGRANGE;
  c->dist_min_dofs = 0;
  c->boundary_penalty_scale = 1.0;
  c->device = 0;
  c->cuda_stream = nullptr;
}

const char* ipmg_last_error(const ipmg_handle* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

ipmg_status ipmg_tables_1d(int k, double penalty_scale, int what, double* out, int cap, int* len) {
  if (k < 1 || k > 7) return IPMG_ERR_UNSUPPORTED;
  if (!out || !len || what < 0 || what > 31) return IPMG_ERR_INVALID_ARG;
  ipmg::FE1D fe = ipmg::build_fe1d(k, penalty_scale);
  const std::vector<double>* src = nullptr;
  if (what == 0) src = &fe.nodes;
  else if (what == 1) src = &fe.M;
  else if (what == 2) src = &fe.K;
  else if (what <= 6) src = &fe.LP[what - 3];
  else if (what <= 10) src = &fe.S[what - 7];
  else if (what <= 14) src = &fe.lam[what - 11];
  else if (what == 15) src = &fe.P;
  else if (what <= 19) src = &fe.LPR[what - 16];
  else if (what <= 23) src = &fe.SD[what - 20];
  else if (what <= 27) src = &fe.lamD[what - 24];
  else src = &fe.actD[what - 28];
  *len = (int)src->size();
  if ((int)src->size() > cap) return IPMG_ERR_SIZE_MISMATCH;
  std::memcpy(out, src->data(), src->size() * sizeof(double));
  return IPMG_OK;
}

ipmg_status ipmg_create(const ipmg_config* cfg, ipmg_handle** out) {
  if (!cfg || !out) { g_create_error = "null argument"; return IPMG_ERR_INVALID_ARG; }
  *out = nullptr;
  if (cfg->dim != 2 && cfg->dim != 3) { g_create_error = "dim must be 2 or 3"; return IPMG_ERR_INVALID_ARG; }
  if (cfg->degree < 1 || cfg->degree > 7) { g_create_error = "degree must be 1..7"; return IPMG_ERR_UNSUPPORTED; }
  if (cfg->n_levels < 1 || cfg->n_levels > 16 || !(cfg->h0 > 0)) {
    g_create_error = "n_levels must be 1..16 and h0 > 0";
    return IPMG_ERR_INVALID_ARG;
  }
  for (int a = 0; a < cfg->dim; ++a)
    if (cfg->coarse_cells[a] != 1 && cfg->coarse_cells[a] != 2) {
      g_create_error = "coarse_cells must be 1 or 2 per direction";
      return IPMG_ERR_INVALID_ARG;
    }
  if (cfg->kernel != IPMG_KERNEL_FULL && cfg->kernel != IPMG_KERNEL_DIRICHLET && cfg->kernel != IPMG_KERNEL_CLAMPED) {
    g_create_error = "kernel must be IPMG_KERNEL_FULL, _DIRICHLET or _CLAMPED";
    return IPMG_ERR_UNSUPPORTED;
  }
  if (cfg->kernel != IPMG_KERNEL_FULL && cfg->smoother != IPMG_MULTIPLICATIVE) {
    g_create_error = "the Dirichlet and clamped kernels are multiplicative smoothers (Algorithm 1)";
    return IPMG_ERR_UNSUPPORTED;
  }
  if (cfg->basis != IPMG_BASIS_LAGRANGE && cfg->basis != IPMG_BASIS_HERMITE) {
    g_create_error = "unknown basis";
    return IPMG_ERR_INVALID_ARG;
  }
  if ((cfg->kernel == IPMG_KERNEL_CLAMPED && cfg->basis != IPMG_BASIS_HERMITE) ||
      (cfg->kernel == IPMG_KERNEL_DIRICHLET && cfg->basis != IPMG_BASIS_LAGRANGE) ||
      (cfg->basis == IPMG_BASIS_HERMITE && cfg->degree < 3)) {
    g_create_error = "clamped kernel needs the Hermite-type basis, Dirichlet the Lagrange one; Hermite needs k >= 3";
    return IPMG_ERR_UNSUPPORTED;
  }
  if (cfg->smoother != IPMG_MULTIPLICATIVE && cfg->smoother != IPMG_ADDITIVE) {
    g_create_error = "unknown smoother";
    return IPMG_ERR_INVALID_ARG;
  }
  if (cfg->vcycle_precision != IPMG_FP32 && cfg->vcycle_precision != IPMG_FP64) {
    g_create_error = "unknown vcycle precision";
    return IPMG_ERR_INVALID_ARG;
  }
  ipmg_handle* h = new (std::nothrow) ipmg_handle();
  if (!h) { g_create_error = "host allocation failed"; return IPMG_ERR_OUT_OF_MEMORY; }
  h->cfg = *cfg;
  if (!(h->cfg.penalty_scale > 0)) h->cfg.penalty_scale = 1.0;
  h->dim = cfg->dim;
  h->k = cfg->degree;
  h->nc = cfg->degree + 1;
  h->cell = h->dim == 2 ? h->nc * h->nc : h->nc * h->nc * h->nc;
  h->nlev = cfg->n_levels;
  h->stream = (cudaStream_t)cfg->cuda_stream;
  {
    const char* ng = std::getenv("IPMG_NO_GRAPH");
    h->use_graphs = !(ng && ng[0] == '1');
  }
  auto bail = [&](ipmg_status st) {
    g_create_error = h->err;
    ipmg_destroy(h);
    return st;
  };
  if (cudaSetDevice(cfg->device) != cudaSuccess) { h->err = "cudaSetDevice failed"; return bail(IPMG_ERR_CUDA); }
  // ---- 1D tables and their upload
  if (!(h->cfg.boundary_penalty_scale > 0)) h->cfg.boundary_penalty_scale = 1.0;
  h->fe = ipmg::build_fe1d(h->k, h->cfg.penalty_scale, cfg->basis, cfg->kernel == IPMG_KERNEL_CLAMPED ? 2 : 1,
                           h->cfg.boundary_penalty_scale);
  if (!h->fe.even_odd) {   // the interior-patch fast path relies on the reflection symmetry
    h->err = "interior patch eigenvectors are not even/odd";
    return bail(IPMG_ERR_UNSUPPORTED);
  }
  h->ks = kernel_set(h->k);
  {
    ipmg_status st = h->cuda(h->ks.upload(h->fe), "table upload");
    if (st != IPMG_OK) return bail(st);
  }
  if (cfg->kernel == IPMG_KERNEL_DIRICHLET || cfg->kernel == IPMG_KERNEL_CLAMPED) {
    if (!h->fe.even_odd_dir) {
      h->err = "Dirichlet interior eigenvectors are not even/odd";
      return bail(IPMG_ERR_UNSUPPORTED);
    }
    h->ksd = kernel_set_dir(h->k);
    ipmg_status st = h->cuda(h->ksd.upload(h->fe), "Dirichlet table upload");
    if (st != IPMG_OK) return bail(st);
  }
  // ---- hierarchy, slab partition of every level
  h->comm = cfg->comm;
  if (h->comm) {
    h->rank = h->comm->rank;
    h->nranks = h->comm->nranks;
  }
  for (int l = 0; l < h->nlev; ++l) {
    ipmg::LevelGeom g{};
    g.n[2] = 1;
    for (int a = 0; a < h->dim; ++a) g.n[a] = cfg->coarse_cells[a] << l;
    int part[4];
    partition_rule(h->dim, cfg->coarse_cells, l, h->nranks, h->rank, part, h->k, cfg->dist_min_dofs);
    g.n[h->dim - 1] = part[2];
    g.zoff = part[1];
    g.nglob = part[3];
    h->dist.push_back(part[0]);
    const long long layer = h->dim == 2 ? g.n[0] : (long long)g.n[0] * g.n[1];
    h->ghost.push_back(h->nranks > 1 && part[0] ? 2 * layer * h->cell : 0);
    g.grouped = l >= 1 ? 1 : 0;
    g.ncells = (long long)g.n[0] * g.n[1] * g.n[2];
    const double hh = cfg->h0 / double(1LL << l);
    g.hs = std::pow(hh, h->dim - 2);
    g.hinv = 1.0 / g.hs;
    h->geom.push_back(g);
    h->ndofs.push_back(g.ncells * h->cell);
    h->hsize.push_back(hh);
  }
  if (h->nranks > 1 && !h->dist[h->nlev - 1]) {
    h->err = "too many ranks: the finest level has fewer than 2 cell layers per rank along the slowest axis";
    return bail(IPMG_ERR_INVALID_ARG);
  }
  // ---- coarse FD tables (global 1D eigenpairs on level 0)
  h->cdesc.dim = h->dim;
  h->cdesc.nc = h->nc;
  h->cdesc.scale = std::pow(cfg->h0, 2 - h->dim);
  for (int a = 0; a < 3; ++a) {
    const int n0 = a < h->dim ? cfg->coarse_cells[a] : 1;
    h->cdesc.n0[a] = n0;
    h->cdesc.N[a] = a < h->dim ? n0 * h->nc : 1;
  }
  for (int a = 0; a < 3; ++a) {
    std::vector<double> S, lam;
    const int N = h->cdesc.N[a];
    if (a < h->dim) {
      std::vector<double> L, M;
      ipmg::global_1d(h->fe, h->cdesc.n0[a], L, M);
      if (!ipmg::gen_eig(N, L, M, S, lam)) { h->err = "coarse eigen-decomposition failed"; return bail(IPMG_ERR_CUDA); }
    } else {
      S.assign(1, 1.0);
      lam.assign(1, 0.0);
    }
    std::vector<float> Sf(S.begin(), S.end()), lf(lam.begin(), lam.end());
    h->cS[0][a] = h->dalloc(S.size() * 8);
    h->cL[0][a] = h->dalloc(lam.size() * 8);
    h->cS[1][a] = h->dalloc(S.size() * 4);
    h->cL[1][a] = h->dalloc(lam.size() * 4);
    if (!h->cS[0][a] || !h->cL[0][a] || !h->cS[1][a] || !h->cL[1][a]) { h->err = "alloc"; return bail(IPMG_ERR_OUT_OF_MEMORY); }
    cudaMemcpy(h->cS[0][a], S.data(), S.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(h->cL[0][a], lam.data(), lam.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(h->cS[1][a], Sf.data(), Sf.size() * 4, cudaMemcpyHostToDevice);
    if (cudaMemcpy(h->cL[1][a], lf.data(), lf.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      h->err = "coarse table upload failed";
      return bail(IPMG_ERR_CUDA);
    }
  }
  for (int p = 0; p < 2; ++p) h->scratch[p].assign(h->nlev, nullptr);
  // ---- f == 1 right-hand side pattern per level (w x w (x w) * h^d)
  h->pattern = (double*)h->dalloc(sizeof(double) * h->cell * h->nlev);
  {
    long long np = 0;   // fused p.q partials of the finest fp64 operator (one per CTA)
    h->ks.vmult(h->dim, IPMG_FP64, nullptr, nullptr, h->geom[h->nlev - 1], nullptr, nullptr, &np, nullptr);
    h->partial_len = np > ipmg::RED_BLOCKS ? np : ipmg::RED_BLOCKS;
  }
  h->partial = (double*)h->dalloc(sizeof(double) * h->partial_len);
  h->scal = (double*)h->dalloc(sizeof(double) * 8);
  h->gbuf = (double*)h->dalloc(sizeof(double) * 4 * h->nranks);
  if (h->comm && h->nranks > 1) {
    const char* no = std::getenv("IPMG_NO_OVERLAP");
    h->overlap = !(no && no[0] == '1');
    if (cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
      h->err = "comm stream / events";
      return bail(IPMG_ERR_CUDA);
    }
  }
  if (!h->pattern || !h->partial || !h->scal || !h->gbuf) { h->err = "alloc"; return bail(IPMG_ERR_OUT_OF_MEMORY); }
  {
    std::vector<double> pat((size_t)h->cell * h->nlev);
    for (int l = 0; l < h->nlev; ++l)
      for (int e = 0; e < h->cell; ++e) {
        double v = std::pow(h->hsize[l], h->dim);
        int r = e;
        for (int a = 0; a < h->dim; ++a) {
          v *= h->fe.w[r % h->nc];
          r /= h->nc;
        }
        pat[(size_t)l * h->cell + e] = v;
      }
    if (cudaMemcpy(h->pattern, pat.data(), pat.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
      h->err = "pattern upload failed";
      return bail(IPMG_ERR_CUDA);
    }
  }
  if (cudaHostAlloc(&h->hpin, sizeof(double) * 8, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&h->hpin_dev, h->hpin, 0) != cudaSuccess) {
    h->err = "mapped pinned alloc";
    return bail(IPMG_ERR_OUT_OF_MEMORY);
  }
  ipmg_status st = h->ensure_vcycle(h->cfg.vcycle_precision);
  if (st != IPMG_OK) return bail(st);
  *out = h;
  return IPMG_OK;
}

ipmg_status ipmg_destroy(ipmg_handle* h) {
  DeviceGuard dg(h);
  if (!h) return IPMG_OK;
  if (h->cstream) cudaStreamDestroy(h->cstream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (int p = 0; p < 2; ++p)
    if (h->vgraph[p]) cudaGraphExecDestroy(h->vgraph[p]);
  for (auto& e : h->ev_pool) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (void* p : h->allocs) cudaFree(p);
  if (h->hpin) cudaFreeHost(h->hpin);
  if (h->ghpin) cudaFreeHost(h->ghpin);
  delete h;
  return IPMG_OK;
}

ipmg_status ipmg_partition(int dim, const int coarse_cells[3], int n_levels, int nranks, int rank, int level,
                           int degree, int64_t min_local_dofs, int out[4]) {
  if ((dim != 2 && dim != 3) || !coarse_cells || !out || n_levels < 1 || level < 0 || level >= n_levels ||
      nranks < 1 || rank < 0 || rank >= nranks)
    return IPMG_ERR_INVALID_ARG;
  for (int a = 0; a < dim; ++a)
    if (coarse_cells[a] != 1 && coarse_cells[a] != 2) return IPMG_ERR_INVALID_ARG;
  if (degree < 1 || degree > 7 || min_local_dofs < 0) return IPMG_ERR_INVALID_ARG;
  partition_rule(dim, coarse_cells, level, nranks, rank, out, degree, min_local_dofs);
  return IPMG_OK;
}

ipmg_status ipmg_level_partition(const ipmg_handle* h, int level, int* distributed, int* zoff, int* nglob) {
  if (!h || level < 0 || level >= h->nlev) return IPMG_ERR_INVALID_ARG;
  if (distributed) *distributed = h->dist[level];
  if (zoff) *zoff = h->geom[level].zoff;
  if (nglob) *nglob = h->geom[level].nglob;
  return IPMG_OK;
}

ipmg_status ipmg_nccl_unique_id(void* id128) {
  if (!id128) return IPMG_ERR_INVALID_ARG;
  std::string e;
  if (!ipmg::nccl_unique_id(id128, &e)) {
    g_create_error = e;
    return IPMG_ERR_NCCL;
  }
  return IPMG_OK;
}

ipmg_status ipmg_comm_create_nccl(const void* id128, int rank, int nranks, int device, ipmg_comm** out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return IPMG_ERR_INVALID_ARG;
  std::string e;
  *out = ipmg::make_nccl_comm(id128, rank, nranks, device, &e);
  if (!*out) {
    g_create_error = e;
    return IPMG_ERR_NCCL;
  }
  return IPMG_OK;
}

ipmg_status ipmg_comm_create_local(int nranks, const int* devices, ipmg_comm** out) {
  if (!out || nranks < 1) return IPMG_ERR_INVALID_ARG;
  auto team = std::make_shared<ipmg::Team>();
  team->n = nranks;
  team->slots.resize(nranks);
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  for (int r = 0; r < nranks; ++r) {
    std::string e;
    out[r] = ipmg::make_local_comm(team, r, devices ? devices[r] : 0, &e);
    if (!out[r]) {
      g_create_error = e;
      for (int q = 0; q < r; ++q) delete out[q];
      return IPMG_ERR_CUDA;
    }
  }
  return IPMG_OK;
}

ipmg_status ipmg_comm_destroy(ipmg_comm* c) {
  delete c;
  return IPMG_OK;
}

ipmg_status ipmg_level_info(const ipmg_handle* h, int level, int64_t* ndofs, int cells[3], double* hsize) {
  if (!h || level < 0 || level >= h->nlev) return IPMG_ERR_INVALID_ARG;
  if (ndofs) *ndofs = h->ndofs[level];
  if (cells)
    for (int a = 0; a < 3; ++a) cells[a] = h->geom[level].n[a];
  if (hsize) *hsize = h->hsize[level];
  return IPMG_OK;
}

static bool bad_prec(int p) { return p != IPMG_FP64 && p != IPMG_FP32; }

ipmg_status ipmg_vmult(ipmg_handle* h, int level, int precision, const void* x, void* y) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (level < 0 || level >= h->nlev || bad_prec(precision) || !x || !y || x == y)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_vmult: bad level/precision/pointers");
  if (level == 0 && h->nlev >= 1) {
    // level 0 may have odd cell counts; the patch-wise operator needs a 2x2(x2) tiling
    for (int a = 0; a < h->dim; ++a)
      if (h->geom[0].n[a] % 2) return h->fail(IPMG_ERR_UNSUPPORTED, "ipmg_vmult: level 0 with odd cell count");
  }
  const void* xg = nullptr;
  ipmg_status st = h->ghosted(level, precision, 0, x, &xg);
  if (st != IPMG_OK) return st;
  return h->run(KC_VMULT, level, 2.0 * h->esize(precision) * h->ndofs[level], 1,
                [&] { return h->ks.vmult(h->dim, precision, xg, y, h->geom[level], nullptr, nullptr, nullptr, h->stream); },
                "vmult");
}

ipmg_status ipmg_smooth_colour(ipmg_handle* h, int level, int precision, const void* x_in, const void* b,
                               void* x_out, int colour) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (level < 1 || level >= h->nlev || bad_prec(precision) || !b || !x_out || x_in == x_out || colour < 0 ||
      colour >= (1 << h->dim))
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_smooth_colour: bad arguments");
  const void *xg = nullptr, *bg = nullptr;
  ipmg_status st = h->ghosted(level, precision, 0, x_in, &xg);
  if (st != IPMG_OK) return st;
  st = h->ghosted(level, precision, 1, b, &bg);
  if (st != IPMG_OK) return st;
  return h->smooth_colour(level, precision, xg, bg, x_out, colour);
}

ipmg_status ipmg_smooth(ipmg_handle* h, int level, int precision, void* x, const void* b, int reverse) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (level < 1 || level >= h->nlev || bad_prec(precision) || !x || !b || x == b)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_smooth: bad arguments");
  ipmg_status st = h->ensure_scratch(precision, level);
  if (st != IPMG_OK) return st;
  if (h->ghost[level] > 0) {   // distributed: run on ghosted copies, copy the result back
    const void *xg = nullptr, *bg = nullptr;
    st = h->ghosted(level, precision, 0, x, &xg);
    if (st != IPMG_OK) return st;
    st = h->ghosted(level, precision, 1, b, &bg);
    if (st != IPMG_OK) return st;
    void* xw = const_cast<void*>(xg);
    st = h->cfg.smoother == IPMG_ADDITIVE ? h->smooth_add(level, precision, xw, h->scratch[precision][level], bg, false)
                                          : h->smooth_mult(level, precision, xw, h->scratch[precision][level], bg,
                                                           reverse != 0, false);
    if (st != IPMG_OK) return st;
    return h->cuda(cudaMemcpyAsync(x, xw, h->ndofs[level] * h->esize(precision), cudaMemcpyDeviceToDevice, h->stream),
                   "copy back");
  }
  if (h->cfg.smoother == IPMG_ADDITIVE) return h->smooth_add(level, precision, x, h->scratch[precision][level], b, false);
  return h->smooth_mult(level, precision, x, h->scratch[precision][level], b, reverse != 0, false);
}

ipmg_status ipmg_residual_restrict(ipmg_handle* h, int fine_level, int precision, const void* x, const void* b,
                                   void* r_c) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (fine_level < 1 || fine_level >= h->nlev || bad_prec(precision) || !b || !r_c)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_residual_restrict: bad arguments");
  const void* xg = nullptr;
  ipmg_status st = h->ghosted(fine_level, precision, 0, x, &xg);
  if (st != IPMG_OK) return st;
  return h->restrict_to(fine_level, precision, xg, b, r_c);
}

ipmg_status ipmg_prolongate_add(ipmg_handle* h, int fine_level, int precision, const void* e_c, void* x_f) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (fine_level < 1 || fine_level >= h->nlev || bad_prec(precision) || !e_c || !x_f)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_prolongate_add: bad arguments");
  return h->run(KC_PROLONG, fine_level, h->esize(precision) * (2.0 * h->ndofs[fine_level] + h->ndofs[fine_level - 1]), 1,
                [&] {
                  return h->ks.prolong(h->dim, precision, e_c, x_f, h->geom[fine_level], h->geom[fine_level - 1], h->stream);
                },
                "prolong");
}

ipmg_status ipmg_coarse_solve(ipmg_handle* h, int precision, const void* b0, void* x0) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (bad_prec(precision) || !b0 || !x0 || b0 == x0) return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_coarse_solve: bad arguments");
  return h->coarse(precision, b0, x0);
}

ipmg_status ipmg_vcycle(ipmg_handle* h, const double* r, double* z) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (!r || !z || (const void*)r == (const void*)z) return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_vcycle: bad pointers");
  return h->vcycle(r, z, nullptr);
}

ipmg_status ipmg_rhs(ipmg_handle* h, int level, int kind, double* b) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (level < 0 || level >= h->nlev || (kind != 0 && kind != 1) || !b)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_rhs: bad arguments");
  if (kind == 0) {
    h->n_launches += 1;
    return h->cuda(ipmg::pattern_fill(b, h->pattern + (size_t)level * h->cell, h->cell, h->ndofs[level], h->stream),
                   "rhs");
  }
  // kind 1: f = pi^2 sum_a 1/ell_a^2 prod_a sin(pi x_a / ell_a), ell_a the box extents;
  // b = f-moments, a product of 1D moment tables per cell (separable)
  if (h->cfg.basis != IPMG_BASIS_LAGRANGE)
    return h->fail(IPMG_ERR_UNSUPPORTED, "ipmg_rhs: kind 1 needs the Lagrange basis");
  if (h->sin_tab.empty()) h->sin_tab.assign((size_t)h->nlev * 3, nullptr);
  const ipmg::LevelGeom& g = h->geom[level];
  const double hh = h->hsize[level];
  const double pi = 3.14159265358979323846;
  double scale = 0.0;
  for (int a = 0; a < h->dim; ++a) {
    const double ell = h->cfg.coarse_cells[a] * h->cfg.h0;
    scale += pi * pi / (ell * ell);
    double*& t = h->sin_tab[(size_t)level * 3 + a];
    if (!t) {
      // global cells along a: the slowest axis may be a slab (nglob global layers)
      const int S = h->dim - 1;
      const int nglob = a == S ? g.nglob : g.n[a];
      const std::vector<double> m = ipmg::sin_moments(h->fe, nglob, 0, hh, ell);
      t = (double*)h->dalloc(m.size() * sizeof(double));
      if (!t) return h->fail(IPMG_ERR_OUT_OF_MEMORY, "ipmg_rhs: table");
      ipmg_status st = h->cuda(cudaMemcpy(t, m.data(), m.size() * sizeof(double), cudaMemcpyHostToDevice), "rhs table");
      if (st != IPMG_OK) return st;
    }
  }
  h->n_launches += 1;
  double* const* tb = &h->sin_tab[(size_t)level * 3];
  return h->cuda(ipmg::sep_fill(b, tb[0], tb[1], h->dim == 3 ? tb[2] : nullptr, g, h->nc, h->dim, scale,
                                h->ndofs[level], h->stream),
                 "rhs");
}

ipmg_status ipmg_to_cellwise(ipmg_handle* h, int level, int precision, const void* x_lib, void* x_cw) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (level < 0 || level >= h->nlev || bad_prec(precision) || !x_lib || !x_cw || x_lib == x_cw)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_to_cellwise: bad arguments");
  h->n_launches += 1;
  return h->cuda(ipmg::permute(precision, true, x_lib, x_cw, h->geom[level], h->cell, h->ndofs[level], h->stream), "permute");
}

ipmg_status ipmg_from_cellwise(ipmg_handle* h, int level, int precision, const void* x_cw, void* x_lib) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (level < 0 || level >= h->nlev || bad_prec(precision) || !x_lib || !x_cw || x_lib == x_cw)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_from_cellwise: bad arguments");
  h->n_launches += 1;
  return h->cuda(ipmg::permute(precision, false, x_cw, x_lib, h->geom[level], h->cell, h->ndofs[level], h->stream), "permute");
}

ipmg_status ipmg_synchronize(ipmg_handle* h) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  return h->host_sync(h->stream);
}

ipmg_status ipmg_cg_solve(ipmg_handle* h, const double* b, double* x, double rtol, int max_it, ipmg_solve_info* info) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (!b || !x || (const void*)b == (const void*)x || !(rtol > 0) || max_it < 1)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_cg_solve: bad arguments");
  const int L = h->nlev - 1;
  const long long n = h->ndofs[L];
  auto t0 = std::chrono::steady_clock::now();
  if (!h->r) {
    h->r = (double*)h->dalloc(n * 8);
    h->p = (double*)h->valloc(L, IPMG_FP64);   // read with ghosts by the operator
    h->q = (double*)h->dalloc(n * 8);
    h->z = (double*)h->dalloc(n * 8);
    if (!h->r || !h->p || !h->q || !h->z) {
      h->r = nullptr;
      return h->fail(IPMG_ERR_OUT_OF_MEMORY, "CG workspace allocation failed");
    }
  }
  cudaStream_t s = h->stream;
  ipmg_status st;
#define CK(call, what)                                 \
  do {                                                 \
    st = h->cuda((call), what);                        \
    if (st != IPMG_OK) return st;                      \
  } while (0)
  // the bandwidth-heavy vector kernels, timed as class KC_BLAS by ipmg_profile
#define TK(call, bytes, what)                                                         \
  do {                                                                              \
    st = h->run(KC_BLAS, L, (double)(bytes), 0, [&] { return (call); }, what);      \
    if (st != IPMG_OK) return st;                                                   \
  } while (0)
  std::vector<double> hist;
  // slots: 0/1 rz (alternating), 2 pq, 3 rr
  CK(cudaMemsetAsync(x, 0, n * 8, s), "memset x");
  CK(cudaMemcpyAsync(h->r, b, n * 8, cudaMemcpyDeviceToDevice, s), "copy r");
  h->n_launches += 2;
  CK(ipmg::dot_partial(0, 0, h->r, h->r, n, h->partial, s), "dot");
  CK(ipmg::finalize(h->partial, h->scal + 3, s), "finalize");
  if ((st = h->allsum(h->scal + 3)) != IPMG_OK) return st;
  CK(ipmg::to_host(h->hpin_dev, h->scal + 3, 1, s), "to host");
  h->n_launches += 1;
  if ((st = h->host_sync(s)) != IPMG_OK) return st;
  const double r0 = std::sqrt(h->hpin[0]);
  hist.push_back(r0);
  int it = 0;
  bool conv = (r0 == 0.0);
  if (!conv) {
    // mixed precision: the fp32 V-cycle input r32 is written by
    // the fused x/r update, z stays fp32 (p = (double) z + beta p), and p.q is
    // fused into the operator kernel.
    const bool mixed = h->cfg.vcycle_precision == IPMG_FP32;
    if (mixed) {
      st = h->ensure_vcycle(IPMG_FP32);
      if (st != IPMG_OK) return st;
    }
    float* r32 = mixed ? (float*)h->vb[IPMG_FP32][L] : nullptr;
    const float* z32 = mixed ? (const float*)h->vx1[IPMG_FP32][L] : nullptr;
    int cur = 0;
    if (mixed) {
      h->n_launches += 1;
      CK(ipmg::cast(0, 1, h->r, r32, n, s), "cast");
      if ((st = h->vcycle_rz(L)) != IPMG_OK) return st;
      h->n_launches += h->rz_nparts > 0 ? 2 : 3;
      if (h->rz_nparts == 0) TK(ipmg::dot_partial(0, 1, h->r, z32, n, h->partial, s), 12.0 * n, "dot");
      CK(ipmg::finalize(h->partial, h->scal + cur, s, h->rz_nparts > 0 ? h->rz_nparts : -1), "finalize");
      if ((st = h->allsum(h->scal + cur)) != IPMG_OK) return st;
      TK(ipmg::cg_update_p32(h->p, z32, n, h->scal, cur, -1, s), 12.0 * n, "p = z");
    } else {
      st = h->vcycle(h->r, h->z, h->partial);
      if (st != IPMG_OK) return st;
      h->n_launches += 1;
      CK(ipmg::finalize(h->partial, h->scal + cur, s), "finalize");
      if ((st = h->allsum(h->scal + cur)) != IPMG_OK) return st;
      CK(cudaMemcpyAsync(h->p, h->z, n * 8, cudaMemcpyDeviceToDevice, s), "copy p");
    }
    while (it < max_it) {
      long long nparts = 0;
      st = h->halo_then(L, IPMG_FP64, h->p, KC_VMULT, 16.0 * n,
                        [&](const ipmg::LevelGeom& g) {
                          return h->ks.vmult(h->dim, IPMG_FP64, h->p, h->q, g, nullptr, h->partial, &nparts, s);
                        },
                        "vmult");
      if (st != IPMG_OK) return st;
      h->n_launches += 3;
      CK(ipmg::finalize(h->partial, h->scal + 2, s, nparts), "finalize");
      if ((st = h->allsum(h->scal + 2)) != IPMG_OK) return st;
      // mixed: the solution update x += alpha p is deferred into the next direction
      // update (cg_update_xp32), or the final cg_update_x on convergence -- the same
      // fma on the same p, one pass over x and p fewer per iteration
      TK(ipmg::cg_update_xr(mixed ? nullptr : x, h->r, h->p, h->q, n, h->scal, cur, 2, h->partial, s, r32),
         (mixed ? 28.0 : 48.0) * n, "update");
      CK(ipmg::finalize(h->partial, h->scal + 3, s), "finalize");
      if ((st = h->allsum(h->scal + 3)) != IPMG_OK) return st;
      CK(ipmg::to_host(h->hpin_dev, h->scal + 3, 1, s), "to host");
      h->n_launches += 1;
      if ((st = h->host_sync(s)) != IPMG_OK) return st;
      ++it;
      const double rn = std::sqrt(h->hpin[0]);
      hist.push_back(rn);
      if (rn <= rtol * r0 || it == max_it) {
        // converged, or max_it reached: apply the pending x += alpha p (mixed) and stop --
        // no V-cycle whose direction update would never be used
        conv = rn <= rtol * r0;
        if (mixed) TK(ipmg::cg_update_x(x, h->p, n, h->scal, cur, 2, s), 24.0 * n, "update x");
        break;
      }
      if (mixed) {
        if ((st = h->vcycle_rz(L)) != IPMG_OK) return st;
        h->n_launches += h->rz_nparts > 0 ? 2 : 3;
        if (h->rz_nparts == 0) TK(ipmg::dot_partial(0, 1, h->r, z32, n, h->partial, s), 12.0 * n, "dot");
        CK(ipmg::finalize(h->partial, h->scal + (1 - cur), s, h->rz_nparts > 0 ? h->rz_nparts : -1), "finalize");
        if ((st = h->allsum(h->scal + (1 - cur))) != IPMG_OK) return st;
        TK(ipmg::cg_update_xp32(x, h->p, z32, n, h->scal, 1 - cur, cur, 2, s), 36.0 * n, "update x, p");
      } else {
        st = h->vcycle(h->r, h->z, h->partial);
        if (st != IPMG_OK) return st;
        h->n_launches += 2;
        CK(ipmg::finalize(h->partial, h->scal + (1 - cur), s), "finalize");
        if ((st = h->allsum(h->scal + (1 - cur))) != IPMG_OK) return st;
        CK(ipmg::cg_update_p(h->p, h->z, n, h->scal, 1 - cur, cur, s), "update p");
      }
      cur = 1 - cur;
    }
  }
#undef CK
#undef TK
  auto t1 = std::chrono::steady_clock::now();
  if (info) {
    info->iterations = it;
    info->rel_residual = r0 > 0 ? hist.back() / r0 : 0.0;
    info->nu = (it > 0 && info->rel_residual > 0) ? -8.0 * it / std::log10(info->rel_residual) : 0.0;
    info->seconds = std::chrono::duration<double>(t1 - t0).count();
    info->history_len = 0;
    if (info->history && info->history_cap > 0) {
      const int m = (int)hist.size() < info->history_cap ? (int)hist.size() : info->history_cap;
      for (int i = 0; i < m; ++i) info->history[i] = hist[i];
      info->history_len = m;
    }
  }
  if (!conv) return h->fail(IPMG_ERR_NOT_CONVERGED, "ipmg_cg_solve: max_it reached");
  return IPMG_OK;
}

ipmg_status ipmg_gmres_solve(ipmg_handle* h, const double* b, double* x, double rtol, int max_it,
                             ipmg_solve_info* info) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  if (!b || !x || (const void*)b == (const void*)x || !(rtol > 0) || max_it < 1 || max_it > 1000)
    return h->fail(IPMG_ERR_INVALID_ARG, "ipmg_gmres_solve: bad arguments");
  const int L = h->nlev - 1;
  const long long n = h->ndofs[L];
  auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = h->stream;
  const bool mixed = h->cfg.vcycle_precision == IPMG_FP32;
  ipmg_status st = h->ensure_vcycle(h->cfg.vcycle_precision);
  if (st != IPMG_OK) return st;
#define CK(call, what)                                 \
  do {                                                 \
    st = h->cuda((call), what);                        \
    if (st != IPMG_OK) return st;                      \
  } while (0)
  // workspace (grown on demand, kept for later solves)
  if (h->gcap < max_it) {
    if (!h->gw && !(h->gw = (double*)h->dalloc(n * 8))) return h->fail(IPMG_ERR_OUT_OF_MEMORY, "GMRES workspace");
    h->ghcol = (double*)h->dalloc(sizeof(double) * (max_it + 2));
    h->gy = (double*)h->dalloc(sizeof(double) * (max_it + 1));
    h->gzptr = (const double**)h->dalloc(sizeof(double*) * (max_it + 1));
    if (h->ghpin) cudaFreeHost(h->ghpin);
    h->ghpin = nullptr;
    if (!h->ghcol || !h->gy || !h->gzptr ||
        cudaHostAlloc(&h->ghpin, sizeof(double) * (max_it + 2), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&h->ghpin_dev, h->ghpin, 0) != cudaSuccess)
      return h->fail(IPMG_ERR_OUT_OF_MEMORY, "GMRES workspace");
    h->gcap = max_it;
  }
  auto vecV = [&](int j) -> double* {
    while ((int)h->gV.size() <= j) h->gV.push_back((double*)h->dalloc(n * 8));
    return h->gV[j];
  };
  auto vecZ = [&](int j) -> double* {   // operator input: ghosted
    while ((int)h->gZ.size() <= j) h->gZ.push_back((double*)h->valloc(L, IPMG_FP64));
    return h->gZ[j];
  };
  std::vector<double> hist;
  // beta0 = ||b||
  CK(ipmg::dot_partial(0, 0, b, b, n, h->partial, s), "dot");
  CK(ipmg::finalize(h->partial, h->scal + 3, s), "finalize");
  h->n_launches += 2;
  if ((st = h->allsum(h->scal + 3)) != IPMG_OK) return st;
  CK(ipmg::to_host(h->hpin_dev, h->scal + 3, 1, s), "to host");
  h->n_launches += 1;
  if ((st = h->host_sync(s)) != IPMG_OK) return st;
  const double beta0 = std::sqrt(h->hpin[0]);
  hist.push_back(beta0);
  int m = 0;
  bool conv = beta0 == 0.0;
  if (conv) {
    CK(cudaMemsetAsync(x, 0, n * 8, s), "memset x");
  } else {
    float* r32 = mixed ? (float*)h->vb[IPMG_FP32][L] : nullptr;
    const float* z32 = mixed ? (const float*)h->vx1[IPMG_FP32][L] : nullptr;
    if (!vecV(0)) return h->fail(IPMG_ERR_OUT_OF_MEMORY, "GMRES basis");
    CK(ipmg::scale_vec(vecV(0), b, n, nullptr, 1.0 / beta0, r32, s), "scale");   // v_0 = b / beta0
    h->n_launches += 1;
    // Hessenberg column j, Givens rotations and the rhs g (host, tiny)
    std::vector<double> H((size_t)(max_it + 1) * max_it, 0.0), cs(max_it), sn(max_it), g(max_it + 1, 0.0);
    auto Hij = [&](int i, int j) -> double& { return H[(size_t)j * (max_it + 1) + i]; };
    g[0] = beta0;
    for (int j = 0; j < max_it; ++j) {
      double* vj = h->gV[j];
      double* zj = vecZ(j);
      double* vn = vecV(j + 1);
      if (!zj || !vn) return h->fail(IPMG_ERR_OUT_OF_MEMORY, "GMRES basis");
      // z_j = P^{-1} v_j (right preconditioning; fp32 V-cycle input r32 = (float) v_j)
      if (mixed) {
        st = h->vcycle_level(L, IPMG_FP32);
        if (st != IPMG_OK) return st;
        CK(ipmg::cast(1, 0, z32, zj, n, s), "cast");
        h->n_launches += 1;
      } else {
        st = h->vcycle(vj, zj, nullptr);
        if (st != IPMG_OK) return st;
      }
      // w = A z_j
      st = h->halo_then(L, IPMG_FP64, zj, KC_VMULT, 16.0 * n,
                        [&](const ipmg::LevelGeom& g) {
                          return h->ks.vmult(h->dim, IPMG_FP64, zj, h->gw, g, nullptr, nullptr, nullptr, s);
                        },
                        "vmult");
      if (st != IPMG_OK) return st;
      // modified Gram-Schmidt: h_ij = w.v_i ; w -= h_ij v_i (each step fused with the next dot)
      CK(ipmg::dot_partial(0, 0, h->gw, h->gV[0], n, h->partial, s), "dot");
      CK(ipmg::finalize(h->partial, h->ghcol, s), "finalize");
      h->n_launches += 2;
      if ((st = h->allsum(h->ghcol)) != IPMG_OK) return st;
      for (int i = 0; i <= j; ++i) {
        CK(ipmg::mgs_axpy_dot(h->gw, h->gV[i], i < j ? h->gV[i + 1] : nullptr, n, h->ghcol, i, h->partial, s), "mgs");
        CK(ipmg::finalize(h->partial, h->ghcol + i + 1, s), "finalize");
        h->n_launches += 2;
        if ((st = h->allsum(h->ghcol + i + 1)) != IPMG_OK) return st;
      }
      // v_{j+1} = w / ||w|| (and its fp32 copy as the next V-cycle input)
      CK(ipmg::scale_vec(vn, h->gw, n, h->ghcol + j + 1, 0.0, r32, s), "scale");
      h->n_launches += 1;
      CK(ipmg::to_host(h->ghpin_dev, h->ghcol, j + 2, s), "to host");
      h->n_launches += 1;
      if ((st = h->host_sync(s)) != IPMG_OK) return st;
      for (int i = 0; i <= j; ++i) Hij(i, j) = h->ghpin[i];
      Hij(j + 1, j) = std::sqrt(h->ghpin[j + 1]);
      for (int i = 0; i < j; ++i) {   // previous rotations
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = Hij(j, j) / den;
      sn[j] = Hij(j + 1, j) / den;
      Hij(j, j) = den;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      hist.push_back(std::fabs(g[j + 1]));
      m = j + 1;
      if (std::fabs(g[j + 1]) <= rtol * beta0) {
        conv = true;
        break;
      }
    }
    // y = R^{-1} g (back substitution), x = sum_i y_i z_i
    std::vector<double> y(m);
    for (int i = m - 1; i >= 0; --i) {
      double t = g[i];
      for (int c = i + 1; c < m; ++c) t -= Hij(i, c) * y[c];
      y[i] = t / Hij(i, i);
    }
    std::vector<const double*> zp(h->gZ.begin(), h->gZ.begin() + m);
    CK(cudaMemcpyAsync(h->gy, y.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s), "h2d");
    CK(cudaMemcpyAsync(h->gzptr, zp.data(), sizeof(double*) * m, cudaMemcpyHostToDevice, s), "h2d");
    CK(ipmg::combine(x, h->gzptr, h->gy, m, n, s), "combine");
    h->n_launches += 1;
    if ((st = h->host_sync(s)) != IPMG_OK) return st;   // y, zp are host temporaries
  }
#undef CK
  auto t1 = std::chrono::steady_clock::now();
  if (info) {
    info->iterations = m;
    info->rel_residual = beta0 > 0 ? hist.back() / beta0 : 0.0;
    info->nu = (m > 0 && info->rel_residual > 0) ? -8.0 * m / std::log10(info->rel_residual) : 0.0;
    info->seconds = std::chrono::duration<double>(t1 - t0).count();
    info->history_len = 0;
    if (info->history && info->history_cap > 0) {
      const int c = (int)hist.size() < info->history_cap ? (int)hist.size() : info->history_cap;
      for (int i = 0; i < c; ++i) info->history[i] = hist[i];
      info->history_len = c;
    }
  }
  if (!conv) return h->fail(IPMG_ERR_NOT_CONVERGED, "ipmg_gmres_solve: max_it reached");
  return IPMG_OK;
}

ipmg_status ipmg_profile(ipmg_handle* h, int enable) {
  DeviceGuard dg(h);
  if (!h) return IPMG_ERR_INVALID_ARG;
  h->prof_on = enable != 0;
  if (h->prof_on) h->recs.clear();
  return IPMG_OK;
}

ipmg_status ipmg_profile_read(ipmg_handle* h, int kernel_class, int64_t* launches, double* total_ms,
                              double* total_bytes) {
  DeviceGuard dg(h);
  if (!h || kernel_class < 0 || kernel_class >= KC_N) return IPMG_ERR_INVALID_ARG;
  ipmg_status st = h->cuda(cudaStreamSynchronize(h->stream), "profile sync");
  if (st != IPMG_OK) return st;
  int64_t n = 0;
  double ms = 0.0, by = 0.0;
  for (size_t i = 0; i < h->recs.size(); ++i) {
    if (h->recs[i].cls != kernel_class) continue;
    float t = 0.f;
    st = h->cuda(cudaEventElapsedTime(&t, h->ev_pool[i].first, h->ev_pool[i].second), "event time");
    if (st != IPMG_OK) return st;
    ++n;
    ms += t;
    by += h->recs[i].bytes;
  }
  if (launches) *launches = n;
  if (total_ms) *total_ms = ms;
  if (total_bytes) *total_bytes = by;
  return IPMG_OK;
}

ipmg_status ipmg_launch_count(const ipmg_handle* h, int64_t* launches) {
  if (!h || !launches) return IPMG_ERR_INVALID_ARG;
  *launches = h->n_launches;
  return IPMG_OK;
}

}  // extern "C"
