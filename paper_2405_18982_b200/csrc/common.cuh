// Shared device-side definitions of the ipmg kernels (sm_100a).
//
// Geometry: a level has n[a] cubic cells per direction (n[2] = 1 in 2D), size
// h; the operator scales as A_h = h^(d-2) A_1 (mass ~ h, stiffness, penalty and
// traces ~ 1/h), so every table is a unit-h table and a level only carries the
// scalar hs = h^(d-2) (PAPER.md:118-126 Kronecker form with h-scaled 1D factors).
//
// Layout: cell chunks of (k+1)^d node values
// (lexicographic, x fastest).  Level l >= 1 groups the 2^d children of each
// level-(l-1) cell contiguously ("parent-grouped"); level 0 is lexicographic.
// A colour-0 vertex patch is exactly one parent cell, so its 2^d cells form one
// contiguous chunk; a shifted colour reads 2^d separate contiguous cell chunks.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ipmg {

// Slab decomposition: a rank owns the cells
// zoff..zoff+n[S]-1 of the slowest axis S = d-1 (y in 2D, z in 3D) out of
// nglob; zoff and n[S] are even, so the local cells are one contiguous range of
// the parent-grouped vector.  Internal vectors of a distributed level carry one
// ghost parent layer (2 cell layers) below and above the local range, addressed
// by the same cell_offset_cells with local coordinates -2..-1 and n[S]..n[S]+1
// (floor shifts give negative / past-the-end offsets).  A single GPU is the
// special case zoff = 0, nglob = n[S].
struct LevelGeom {
  int n[3];            // LOCAL cells per direction (n[2] = 1 in 2D)
  int grouped;         // 1: parent-grouped layout, 0: lexicographic cells
  long long ncells;    // local cells
  double hs;           // h^(d-2)
  double hinv;         // h^(2-d)
  int zoff;            // global index of local cell 0 along the slowest axis
  int nglob;           // global cells along the slowest axis
  // patch-block selection along the slowest axis (halo/compute overlap): 0 all,
  // 1 interior blocks (no ghost access), 2 the first and last block; znb = the
  // launch's full block count along that axis (set by the launchers)
  int zsel;
  int znb;
};

// "no neighbour" marker of patch neighbour offsets (ghost offsets are negative)
constexpr long long NO_NB = (long long)(-0x7fffffffffffffffLL - 1);

__host__ __device__ __forceinline__ long long cell_offset_cells(const LevelGeom& g, int cx, int cy,
                                                                int cz) {
  // index of the cell chunk (in units of cells)
  if (g.grouped) {
    const int PX = g.n[0] >> 1, PY = g.n[1] >> 1;
    const int qx = cx & 1, qy = cy & 1, qz = cz & 1;
    const long long plin = (long long)(cx >> 1) + (long long)PX * ((cy >> 1) + (long long)PY * (cz >> 1));
    const int nchild = (g.n[2] > 1) ? 8 : 4;   // 2^d (n[2] == 1 only in 2D)
    return plin * nchild + qx + 2 * qy + 4 * qz;
  }
  return (long long)cx + (long long)g.n[0] * (cy + (long long)g.n[1] * cz);
}

// Device-side 1D tables for degree K in precision T (unit h); one instance per
// precision lives in __constant__ memory of each per-degree translation unit.
// Rows are padded to a multiple of 4 entries and 16-byte aligned so that a
// kernel walking a row with compile-time indices loads 4 (fp32) / 2 (fp64)
// constants per uniform-register load (LDCU.128).  Every matrix is stored in
// the orientation it is applied in (out[i] = sum_j A[i][j] in[j], j contiguous).
template <int K, typename T>
struct TabData {
  static constexpr int NC = K + 1, NP = 2 * (K + 1);
  static constexpr int RC = (NC + 3) & ~3, RP = (NP + 3) & ~3;   // padded row lengths
  alignas(16) T M[NC][RC];          // cell mass
  alignas(16) T LP[4][NP][RP];      // 2-cell patch stiffness + face terms, variant v
  alignas(16) T S[4][NP][RP];       // eigenvectors, S[v][node][mode]
  alignas(16) T ST[4][NP][RP];      // transposed eigenvectors, ST[v][mode][node]
  alignas(16) T SO[NP][RC];         // odd-mode columns of S[0]: SO[node][m] = S[0][node][NP/2 + m], rows
                                    // 16-byte aligned so that output pairs (2q, 2q+1) are aligned 8-byte
                                    // constants also when NP/2 is odd (even k)
  alignas(16) T MS[4][NP][RP];      // M^P S = (S^T M^P)^T: face arrays of directions already in eigen-space
  alignas(16) T CF[4][RP];          // face coupling coefficients along the normal (C x_ext):
                                    // 0 low/u, 1 low/u', 2 high/u, 3 high/u'  (see face_* kernels)
  alignas(16) T CH[4][4][RP];       // the same in eigen-space: CH[v][kind][m] = sum_i S[v][i][m] CF[kind][i]
  alignas(16) T lam[4][RP];         // eigenvalues
  alignas(16) T act[4][RP];         // 1 / 0: mode active (Dirichlet tables; all 1 for the full kernel)
  alignas(16) T d0[RC];             // phi_j'(0)
  alignas(16) T d1[RC];             // phi_j'(1)
  alignas(16) T P[NP][RC];          // prolongation (patch-lex fine node, coarse node)
  alignas(16) T PT[NC][RP];         // restriction = P^T
  alignas(16) T w[RC];              // int phi_i
  T gamma;                          // unit penalty 2k(k+1)*scale
};

struct FE1D;

// Per-degree launcher table exported by each kernels_k<K>.cu.
struct KernelSet {
  int k;
  cudaError_t (*upload)(const FE1D& fe);   // fill and upload the __constant__ tables
  // all launchers: prec 0 = double, 1 = float; dim 2 or 3
  // y = A x (b_minus: y = b_minus - A x); dotp != nullptr: per-CTA partials of x.y,
  // *nparts = their count (x == nullptr: size query only)
  cudaError_t (*vmult)(int dim, int prec, const void* x, void* y, const LevelGeom& g,
                       const void* b_minus, double* dotp, long long* nparts, cudaStream_t s);
  cudaError_t (*smooth)(int dim, int prec, const void* x_in, const void* b, void* x_out,
                        const LevelGeom& g, int colour, cudaStream_t s);
  // the same pass with the mixed PCG's r.z fused (partials into dotp, *nparts their count;
  // *nparts = 0: not fused, the caller forms the dot); nullptr in the Dirichlet kernel sets
  cudaError_t (*smooth_rz)(int dim, int prec, const void* x_in, const void* b, void* x_out,
                           const LevelGeom& g, int colour, const double* r, double* dotp, long long* nparts,
                           cudaStream_t s);
  cudaError_t (*additive)(int dim, int prec, const void* r, void* x, const LevelGeom& g, int colour,
                          double omega, cudaStream_t s);
  cudaError_t (*restrict_)(int dim, int prec, const void* x, const void* b, void* rc,
                           const LevelGeom& gf, const LevelGeom& gc, cudaStream_t s);
  cudaError_t (*prolong)(int dim, int prec, const void* ec, void* xf, const LevelGeom& gf,
                         const LevelGeom& gc, cudaStream_t s);
};

}  // namespace ipmg
