// Vertex-patch kernels of the ipmg library, templated on dimension D, degree
// K (via IPMG_K of the including translation unit) and precision T.
//
// One CTA processes PPC vertex patches of one colour.  Each patch is staged in
// shared memory as a patch-lexicographic tensor of (2(k+1))^d values (row pitch
// 2(k+1)+1, odd, so x-lines and y-lines are bank-conflict free), loaded and
// stored with coalesced cooperative copies of whole cell chunks.  Every
// sum-factorisation step is a "line pass": each thread owns whole 1D lines of
// the tensor along one direction, reads the line into registers, multiplies it
// by a 1D matrix whose entries are compile-time indexed __constant__ operands
// (no load instructions for the matrix), and writes the line back in place.
//
//  vmult_kernel     y = A x                      PAPER.md:112-138 (Fig. 1 patch-wise
//                   over colour-0 patches;        integration, Kronecker sum of
//                   each patch writes only its   PAPER.md:118-126, face terms of
//                   own cells -> no atomics)      eq. bilinear_form)
//  smooth_kernel    one colour of Algorithm 1,
//                   full kernel, in replacement form x_j = A_j^{-1}(b_j - C_j x_ext),
//                   algebraically identical to x_j + A_j^{-1} R_j(b - A x) because
//                   A_j = R_j A R_j^T; A_j^{-1} by fast diagonalisation
//  additive_kernel  x += omega R_j^T A_j^{-1} R_j r over one colour (r precomputed)
//  restrict_kernel  r_c = P^T (b - A x) per parent cell
//  prolong_kernel   x_f += P e_c per parent cell
#pragma once
#include "common.cuh"

#ifndef IPMG_K
#error "IPMG_K must be defined by the including translation unit"
#endif

#define IPMG_CAT2(a, b) a##b
#define IPMG_CAT(a, b) IPMG_CAT2(a, b)
// every degree lives in its own namespace: the per-TU __constant__ tables and
// the kernel template instantiations must not collide at link time
#define IPMG_KK IPMG_CAT(kdeg, IPMG_K)

namespace ipmg {
namespace IPMG_KK {

constexpr int K = IPMG_K;
constexpr int NC = K + 1;
constexpr int NP = 2 * NC;

__constant__ TabData<K, double> c_tab64;
__constant__ TabData<K, float> c_tab32;

template <typename T>
__device__ __forceinline__ const TabData<K, T>& tab();
template <>
__device__ __forceinline__ const TabData<K, double>& tab<double>() { return c_tab64; }
template <>
__device__ __forceinline__ const TabData<K, float>& tab<float>() { return c_tab32; }

// ---------------------------------------------------------------- configuration
template <int D>
struct Cfg {
  static constexpr int RP = NP + 1;                  // row pitch (odd)
  static constexpr int PL = NP * RP;                 // plane pitch
  static constexpr int TSZ = (D == 2) ? NP * RP : NP * PL;
  static constexpr int NL = (D == 2) ? NP : NP * NP; // lines per direction per patch
  static constexpr int CELL = (D == 2) ? NC * NC : NC * NC * NC;
  static constexpr int NCH = 1 << D;                 // cells per patch
  static constexpr int PATCH = NCH * CELL;
  static constexpr int NFP = NL;                     // tangential points per face
  static constexpr int PPC = (256 / NL) > 1 ? (256 / NL) : 1;
  static constexpr int LINES = PPC * NL;
  static constexpr int NT0 = ((LINES + 31) / 32) * 32;
  static constexpr int NT = NT0 > 256 ? 256 : NT0;
};

template <typename T>
__device__ __forceinline__ T fma_(T a, T b, T c) { return fma(a, b, c); }

// ---------------------------------------------------------------- 1D matrices
// Each functor: get(i, j) entry of the (NOUT x NIN) matrix applied as
// out[i] = sum_j get(i,j) in[j]; nz(i,j) structural non-zero (compile-time).
template <typename T>
struct MassP {   // block-diagonal 2-cell patch mass
  static __device__ __forceinline__ T get(int i, int j) { return tab<T>().M[i % NC][j % NC]; }
  static __device__ __forceinline__ constexpr bool nz(int i, int j) { return i / NC == j / NC; }
};
template <int V, typename T>
struct LapP {    // patch stiffness + face terms; cross-cell blocks only touch the interior face
  static __device__ __forceinline__ T get(int i, int j) { return tab<T>().LP[V][i][j]; }
  static __device__ __forceinline__ constexpr bool nz(int i, int j) {
    return (i / NC == j / NC) || i == NC - 1 || i == NC || j == NC - 1 || j == NC;
  }
};
template <int V, typename T>
struct EigT {    // S^T: out[m] = sum_i S[i][m] in[i]
  static __device__ __forceinline__ T get(int m, int i) { return tab<T>().S[V][i][m]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <int V, typename T>
struct Eig {     // S: out[i] = sum_m S[i][m] in[m]
  static __device__ __forceinline__ T get(int i, int m) { return tab<T>().S[V][i][m]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct Prol {    // P: (NP x NC)
  static __device__ __forceinline__ T get(int i, int j) { return tab<T>().P[i][j]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct ProlT {   // P^T: (NC x NP)
  static __device__ __forceinline__ T get(int j, int i) { return tab<T>().P[i][j]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};

template <int NOUT, int NIN, class A, typename T>
__device__ __forceinline__ void matvec(const T (&in)[NIN], T (&out)[NOUT]) {
#pragma unroll
  for (int i = 0; i < NOUT; ++i) {
    T acc = T(0);
#pragma unroll
    for (int j = 0; j < NIN; ++j)
      if (A::nz(i, j)) acc = fma_(A::get(i, j), in[j], acc);
    out[i] = acc;
  }
}

template <int N, typename T>
__device__ __forceinline__ void load_line(const T* p, int stride, T (&v)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = p[j * stride];
}
template <int N, typename T>
__device__ __forceinline__ void store_line(T* p, int stride, const T (&v)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) p[j * stride] = v[j];
}

// line l of direction a in a patch tensor: base offset and stride
template <int D>
__device__ __forceinline__ void line_geom(int a, int l, int& base, int& stride) {
  using C = Cfg<D>;
  if (D == 2) {
    if (a == 0) { base = l * C::RP; stride = 1; }
    else        { base = l;         stride = C::RP; }
  } else {
    const int u = l % NP, v = l / NP;
    if (a == 0)      { base = u * C::RP + v * C::PL; stride = 1; }
    else if (a == 1) { base = u + v * C::PL;         stride = C::RP; }
    else             { base = u + v * C::RP;         stride = C::PL; }
  }
}

// smem offset of node (local node l of cell q) inside a patch tensor
template <int D>
__device__ __forceinline__ int node_of_cell(int q, int l) {
  using C = Cfg<D>;
  const int l0 = l % NC, l1 = (l / NC) % NC;
  const int i0 = (q & 1) * NC + l0, i1 = ((q >> 1) & 1) * NC + l1;
  if (D == 2) return i0 + i1 * C::RP;
  const int l2 = l / (NC * NC);
  const int i2 = ((q >> 2) & 1) * NC + l2;
  return i0 + i1 * C::RP + i2 * C::PL;
}

// ---------------------------------------------------------------- patch indexing
struct PatchInfo {
  int c0[3];      // lowest cell coordinates
  int var[3];     // boundary variant per direction
  bool valid;
};

template <int D>
__device__ __forceinline__ PatchInfo patch_info(const LevelGeom& g, int colour, long long p) {
  PatchInfo pi;
  int m[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) m[a] = (a < D) ? (g.n[a] / 2 - ((colour >> a) & 1)) : 1;
  const long long np = (long long)m[0] * m[1] * m[2];
  pi.valid = p < np;
  long long r = pi.valid ? p : 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int j = (int)(r % m[a]);
    r /= m[a];
    pi.c0[a] = (a < D) ? ((colour >> a) & 1) + 2 * j : 0;
    pi.var[a] = (a < D) ? ((pi.c0[a] == 0 ? 1 : 0) | (pi.c0[a] + 2 == g.n[a] ? 2 : 0)) : 0;
  }
  return pi;
}

__host__ __device__ inline long long num_patches(const LevelGeom& g, int dim, int colour) {
  long long np = 1;
  for (int a = 0; a < dim; ++a) np *= (g.n[a] / 2 - ((colour >> a) & 1));
  return np;
}

// global element offset of cell q of patch pi
template <int D>
__device__ __forceinline__ long long patch_cell_offset(const LevelGeom& g, const PatchInfo& pi, int q) {
  using C = Cfg<D>;
  return cell_offset_cells(g, pi.c0[0] + (q & 1), pi.c0[1] + ((q >> 1) & 1),
                           D == 3 ? pi.c0[2] + ((q >> 2) & 1) : 0) * (long long)C::CELL;
}

// ---------------------------------------------------------------- cooperative copies
// X[p] <- scale * src patch cells (src == nullptr -> zeros)
template <int D, typename T>
__device__ __forceinline__ void load_patches(T* X, const T* __restrict__ src, const LevelGeom& g,
                                             const PatchInfo* pis, int npc, T scale) {
  using C = Cfg<D>;
  for (int e = threadIdx.x; e < npc * C::PATCH; e += blockDim.x) {
    const int p = e / C::PATCH, r = e % C::PATCH, q = r / C::CELL, l = r % C::CELL;
    T v = T(0);
    if (src != nullptr && pis[p].valid) v = scale * __ldg(src + patch_cell_offset<D>(g, pis[p], q) + l);
    X[p * C::TSZ + node_of_cell<D>(q, l)] = v;
  }
}

// dst patch cells <- scale * X[p]  (accumulate: dst += scale * X)
template <int D, bool ACCUM, typename T>
__device__ __forceinline__ void store_patches(T* __restrict__ dst, const T* X, const LevelGeom& g,
                                              const PatchInfo* pis, int npc, T scale) {
  using C = Cfg<D>;
  for (int e = threadIdx.x; e < npc * C::PATCH; e += blockDim.x) {
    const int p = e / C::PATCH, r = e % C::PATCH, q = r / C::CELL, l = r % C::CELL;
    if (!pis[p].valid) continue;
    T* o = dst + patch_cell_offset<D>(g, pis[p], q) + l;
    const T v = scale * X[p * C::TSZ + node_of_cell<D>(q, l)];
    if (ACCUM) *o += v; else *o = v;
  }
}

// ---------------------------------------------------------------- face terms
// Coupling of a patch to the cells across its 2d outer faces (the only part of
// the residual that reads outside the patch; PAPER.md:196-198 domain of
// dependence).  For the low face in direction a, with neighbour value u and
// normal derivative u' on the face (unit h, jump read as u- - u+, A1):
//   (C x_L)_i = M_tan [ delta_{i,0} (-gamma u + u'/2) - phi_i'(0) u / 2 ]   (i in cell 0)
// and for the high face
//   (C x_R)_i = M_tan [ delta_{i,np-1} (-gamma u - u'/2) + phi_i'(1) u / 2 ] (i in cell 1).
// sgn = +1 adds C x_ext (operator), sgn = -1 subtracts it (smoother right side).
// FU / FD: PPC x 2 sides x NFP scratch.
template <int D, typename T>
__device__ void face_terms(T* X, T* FU, T* FD, const T* __restrict__ x, const LevelGeom& g,
                           const PatchInfo* pis, int npc, T sgn) {
  using C = Cfg<D>;
  const TabData<K, T>& tb = tab<T>();
#pragma unroll 1
  for (int a = 0; a < D; ++a) {
    // (1) traces of the neighbour cells on the two outer faces of direction a
    const int b = (a == 0) ? 1 : 0;
    const int c = (a == 2) ? 1 : 2;    // second tangential direction (3D)
    int strd[3] = {1, NC, NC * NC};
    for (int e = threadIdx.x; e < npc * 2 * C::NFP; e += blockDim.x) {
      const int p = e / (2 * C::NFP), s = (e / C::NFP) & 1, t = e % C::NFP;
      const PatchInfo& pi = pis[p];
      const bool exists = pi.valid && (s == 0 ? pi.c0[a] > 0 : pi.c0[a] + 2 < g.n[a]);
      T u = T(0), du = T(0);
      if (exists) {
        const int ib = t % NP, ic = t / NP;
        int cc[3] = {pi.c0[0], pi.c0[1], pi.c0[2]};
        cc[a] = (s == 0) ? pi.c0[a] - 1 : pi.c0[a] + 2;
        cc[b] += ib / NC;
        if (D == 3) cc[c] += ic / NC;
        const long long base = cell_offset_cells(g, cc[0], cc[1], cc[2]) * C::CELL +
                               (ib % NC) * strd[b] + (D == 3 ? (ic % NC) * strd[c] : 0);
        const T* px = x + base;
        const int sa = strd[a];
        if (s == 0) {
#pragma unroll
          for (int j = 0; j < NC; ++j) du = fma_(tb.d1[j], __ldg(px + j * sa), du);
          u = __ldg(px + (NC - 1) * sa);
        } else {
#pragma unroll
          for (int j = 0; j < NC; ++j) du = fma_(tb.d0[j], __ldg(px + j * sa), du);
          u = __ldg(px);
        }
      }
      FU[e] = u;
      FD[e] = du;
    }
    __syncthreads();
    // (2) tangential mass M_tan = M^P (x M^P): line passes over the face grid
#pragma unroll 1
    for (int tdim = 0; tdim < D - 1; ++tdim) {
      const int nlines = npc * 2 * 2 * (D == 3 ? NP : 1);
      for (int e = threadIdx.x; e < nlines; e += blockDim.x) {
        const int which = e & 1;                       // 0: FU, 1: FD
        const int rest = e >> 1;
        T* arr = which ? FD : FU;
        int base, stride;
        if (D == 2) { base = rest * C::NFP; stride = 1; }
        else {
          const int ps = rest / NP, o = rest % NP;     // ps = p*2+s
          if (tdim == 0) { base = ps * C::NFP + o * NP; stride = 1; }
          else           { base = ps * C::NFP + o;      stride = NP; }
        }
        T v[NP], w[NP];
        load_line<NP>(arr + base, stride, v);
        matvec<NP, NP, MassP<T>>(v, w);
        store_line<NP>(arr + base, stride, w);
      }
      __syncthreads();
    }
    // (3) add the coupling along the lines of direction a
    for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
      const int p = e / C::NL, l = e % C::NL;
      int base, stride;
      line_geom<D>(a, l, base, stride);
      T* px = X + p * C::TSZ + base;
      const T ul = FU[(p * 2 + 0) * C::NFP + l], dl = FD[(p * 2 + 0) * C::NFP + l];
      const T uh = FU[(p * 2 + 1) * C::NFP + l], dh = FD[(p * 2 + 1) * C::NFP + l];
      const T half = T(0.5);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        T lo = -half * tb.d0[i] * ul;
        if (i == 0) lo += -tb.gamma * ul + half * dl;
        T hi = half * tb.d1[i] * uh;
        if (i == NC - 1) hi += -tb.gamma * uh - half * dh;
        px[i * stride] += sgn * lo;
        px[(NC + i) * stride] += sgn * hi;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- volume term
// X <- A_jj(unit) X  (Kronecker sum with the patch matrices)
// using T1 as scratch:   2D: y = M1 (L0 x) + L1 (M0 x)
//                        3D: y = M2 (L1 M0 x + M1 L0 x) + L2 (M1 M0 x)
template <int V, typename T>
__device__ __forceinline__ void lap_line(const T (&v)[NP], T (&w)[NP]) { matvec<NP, NP, LapP<V, T>>(v, w); }

template <typename T>
__device__ __forceinline__ void lap_line_v(int var, const T (&v)[NP], T (&w)[NP]) {
  switch (var) {
    case 0: lap_line<0>(v, w); break;
    case 1: lap_line<1>(v, w); break;
    case 2: lap_line<2>(v, w); break;
    default: lap_line<3>(v, w); break;
  }
}

template <int D, typename T>
__device__ void volume_apply(T* X, T* T1, const PatchInfo* pis, int npc) {
  using C = Cfg<D>;
  // pass over x-lines: T1 = M0 x, X = L0 x
  for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
    const int p = e / C::NL, l = e % C::NL;
    int base, stride;
    line_geom<D>(0, l, base, stride);
    T v[NP], m[NP], w[NP];
    load_line<NP>(X + p * C::TSZ + base, stride, v);
    matvec<NP, NP, MassP<T>>(v, m);
    lap_line_v(pis[p].var[0], v, w);
    store_line<NP>(T1 + p * C::TSZ + base, stride, m);
    store_line<NP>(X + p * C::TSZ + base, stride, w);
  }
  __syncthreads();
  if (D == 2) {
    for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
      const int p = e / C::NL, l = e % C::NL;
      int base, stride;
      line_geom<D>(1, l, base, stride);
      T m[NP], lx[NP], y[NP], t[NP];
      load_line<NP>(T1 + p * C::TSZ + base, stride, m);
      load_line<NP>(X + p * C::TSZ + base, stride, lx);
      matvec<NP, NP, MassP<T>>(lx, y);
      lap_line_v(pis[p].var[1], m, t);
#pragma unroll
      for (int i = 0; i < NP; ++i) y[i] += t[i];
      store_line<NP>(X + p * C::TSZ + base, stride, y);
    }
    __syncthreads();
  } else {
    // y-lines: X <- L1 m0 + M1 l0 ; T1 <- M1 m0
    for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
      const int p = e / C::NL, l = e % C::NL;
      int base, stride;
      line_geom<D>(1, l, base, stride);
      T m[NP], lx[NP], y[NP], t[NP];
      load_line<NP>(T1 + p * C::TSZ + base, stride, m);
      load_line<NP>(X + p * C::TSZ + base, stride, lx);
      matvec<NP, NP, MassP<T>>(lx, y);
      lap_line_v(pis[p].var[1], m, t);
#pragma unroll
      for (int i = 0; i < NP; ++i) y[i] += t[i];
      store_line<NP>(X + p * C::TSZ + base, stride, y);
      matvec<NP, NP, MassP<T>>(m, t);
      store_line<NP>(T1 + p * C::TSZ + base, stride, t);
    }
    __syncthreads();
    // z-lines: X <- M2 X + L2 T1
    for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
      const int p = e / C::NL, l = e % C::NL;
      int base, stride;
      line_geom<D>(2, l, base, stride);
      T a[NP], bb[NP], y[NP], t[NP];
      load_line<NP>(X + p * C::TSZ + base, stride, a);
      load_line<NP>(T1 + p * C::TSZ + base, stride, bb);
      matvec<NP, NP, MassP<T>>(a, y);
      lap_line_v(pis[p].var[2], bb, t);
#pragma unroll
      for (int i = 0; i < NP; ++i) y[i] += t[i];
      store_line<NP>(X + p * C::TSZ + base, stride, y);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- fast diagonalisation
// X <- A_jj(unit)^{-1} X = (x S_a) (sum_a Lambda_a)^{-1} (x S_a^T) X
// (eq. inverse2d / inverse3d / fast_inverse)
template <int V, typename T>
__device__ __forceinline__ void eigT_line(const T (&v)[NP], T (&w)[NP]) { matvec<NP, NP, EigT<V, T>>(v, w); }
template <int V, typename T>
__device__ __forceinline__ void eig_line(const T (&v)[NP], T (&w)[NP]) { matvec<NP, NP, Eig<V, T>>(v, w); }

template <typename T>
__device__ __forceinline__ void eigT_line_v(int var, const T (&v)[NP], T (&w)[NP]) {
  switch (var) {
    case 0: eigT_line<0>(v, w); break;
    case 1: eigT_line<1>(v, w); break;
    case 2: eigT_line<2>(v, w); break;
    default: eigT_line<3>(v, w); break;
  }
}
template <typename T>
__device__ __forceinline__ void eig_line_v(int var, const T (&v)[NP], T (&w)[NP]) {
  switch (var) {
    case 0: eig_line<0>(v, w); break;
    case 1: eig_line<1>(v, w); break;
    case 2: eig_line<2>(v, w); break;
    default: eig_line<3>(v, w); break;
  }
}

template <int D, bool FORWARD, typename T>
__device__ __forceinline__ void eig_pass(T* X, int a, const PatchInfo* pis, int npc) {
  using C = Cfg<D>;
  for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
    const int p = e / C::NL, l = e % C::NL;
    int base, stride;
    line_geom<D>(a, l, base, stride);
    T v[NP], w[NP];
    load_line<NP>(X + p * C::TSZ + base, stride, v);
    if (FORWARD) eigT_line_v(pis[p].var[a], v, w);
    else eig_line_v(pis[p].var[a], v, w);
    store_line<NP>(X + p * C::TSZ + base, stride, w);
  }
  __syncthreads();
}

template <int D, typename T>
__device__ void fast_diag(T* X, const PatchInfo* pis, int npc) {
  using C = Cfg<D>;
  const TabData<K, T>& tb = tab<T>();
  constexpr int LAST = D - 1;
#pragma unroll 1
  for (int a = 0; a < LAST; ++a) eig_pass<D, true>(X, a, pis, npc);
  // last direction: S^T, divide by the eigenvalue sums, S -- in registers
  for (int e = threadIdx.x; e < npc * C::NL; e += blockDim.x) {
    const int p = e / C::NL, l = e % C::NL;
    int base, stride;
    line_geom<D>(LAST, l, base, stride);
    const PatchInfo& pi = pis[p];
    T lsum = tb.lam[pi.var[0]][l % NP];
    if (D == 3) lsum += tb.lam[pi.var[1]][l / NP];
    T v[NP], w[NP];
    load_line<NP>(X + p * C::TSZ + base, stride, v);
    eigT_line_v(pi.var[LAST], v, w);
#pragma unroll
    for (int m = 0; m < NP; ++m) w[m] = w[m] / (lsum + tb.lam[pi.var[LAST]][m]);
    eig_line_v(pi.var[LAST], w, v);
    store_line<NP>(X + p * C::TSZ + base, stride, v);
  }
  __syncthreads();
#pragma unroll 1
  for (int a = LAST - 1; a >= 0; --a) eig_pass<D, false>(X, a, pis, npc);
}

// ---------------------------------------------------------------- kernels
template <int D, typename T>
__device__ __forceinline__ void setup_patches(PatchInfo* pis, const LevelGeom& g, int colour, long long patch0, int npc) {
  if (threadIdx.x < npc) pis[threadIdx.x] = patch_info<D>(g, colour, patch0 + threadIdx.x);
  __syncthreads();
}

// y = hs * A x   or, with bminus != nullptr, y = bminus - hs * A x
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D>::NT) vmult_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                           const T* __restrict__ bminus, LevelGeom g) {
  using C = Cfg<D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* T1 = X + C::PPC * C::TSZ;
  T* FU = T1 + C::PPC * C::TSZ;
  T* FD = FU + C::PPC * 2 * C::NFP;
  __shared__ PatchInfo pis[C::PPC];
  const long long patch0 = (long long)blockIdx.x * C::PPC;
  setup_patches<D, T>(pis, g, 0, patch0, C::PPC);
  load_patches<D>(X, x, g, pis, C::PPC, T(1));
  __syncthreads();
  volume_apply<D>(X, T1, pis, C::PPC);
  face_terms<D>(X, FU, FD, x, g, pis, C::PPC, T(1));
  const T hs = T(g.hs);
  if (bminus == nullptr) {
    store_patches<D, false>(y, X, g, pis, C::PPC, hs);
  } else {
    for (int e = threadIdx.x; e < C::PPC * C::PATCH; e += blockDim.x) {
      const int p = e / C::PATCH, r = e % C::PATCH, q = r / C::CELL, l = r % C::CELL;
      if (!pis[p].valid) continue;
      const long long o = patch_cell_offset<D>(g, pis[p], q) + l;
      y[o] = __ldg(bminus + o) - hs * X[p * C::TSZ + node_of_cell<D>(q, l)];
    }
  }
}

// one colour of the multiplicative full-kernel smoother (replacement form):
// x_out_j = A_jj^{-1} (b_j - C_j x_in) for every patch j of the colour;
// extra CTAs copy the cells the colour does not cover.
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D>::NT) smooth_kernel(const T* __restrict__ x_in, const T* __restrict__ b,
                                                            T* __restrict__ x_out, LevelGeom g, int colour,
                                                            int n_patch_ctas) {
  using C = Cfg<D>;
  if ((int)blockIdx.x >= n_patch_ctas) {
    // copy role: boundary layers c_a in {0, n_a-1} of every shifted direction a
    long long idx = (long long)(blockIdx.x - n_patch_ctas) * blockDim.x + threadIdx.x;
    const long long stride_all = (long long)(gridDim.x - n_patch_ctas) * blockDim.x;
    for (int a = 0; a < D; ++a) {
      if (!((colour >> a) & 1)) continue;
      long long layer = 1;
      for (int bb = 0; bb < D; ++bb) if (bb != a) layer *= g.n[bb];
      const long long total = 2 * layer * C::CELL;
      for (long long e = idx; e < total; e += stride_all) {
        const long long cell = e / C::CELL;
        const int l = (int)(e % C::CELL);
        const int side = (int)(cell / layer);
        long long rem = cell % layer;
        int cc[3] = {0, 0, 0};
        for (int bb = 0; bb < D; ++bb) {
          if (bb == a) continue;
          cc[bb] = (int)(rem % g.n[bb]);
          rem /= g.n[bb];
        }
        cc[a] = side ? g.n[a] - 1 : 0;
        const long long o = cell_offset_cells(g, cc[0], cc[1], cc[2]) * C::CELL + l;
        x_out[o] = x_in ? __ldg(x_in + o) : T(0);
      }
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* FU = X + C::PPC * C::TSZ;
  T* FD = FU + C::PPC * 2 * C::NFP;
  __shared__ PatchInfo pis[C::PPC];
  const long long patch0 = (long long)blockIdx.x * C::PPC;
  setup_patches<D, T>(pis, g, colour, patch0, C::PPC);
  load_patches<D>(X, b, g, pis, C::PPC, T(g.hinv));
  __syncthreads();
  if (x_in != nullptr) face_terms<D>(X, FU, FD, x_in, g, pis, C::PPC, T(-1));
  fast_diag<D>(X, pis, C::PPC);
  store_patches<D, false>(x_out, X, g, pis, C::PPC, T(1));
}

// additive Schwarz over one colour: x_j += omega A_jj^{-1} r_j
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D>::NT) additive_kernel(const T* __restrict__ r, T* __restrict__ x,
                                                              LevelGeom g, int colour, T omega) {
  using C = Cfg<D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  __shared__ PatchInfo pis[C::PPC];
  const long long patch0 = (long long)blockIdx.x * C::PPC;
  setup_patches<D, T>(pis, g, colour, patch0, C::PPC);
  load_patches<D>(X, r, g, pis, C::PPC, T(g.hinv));
  __syncthreads();
  fast_diag<D>(X, pis, C::PPC);
  store_patches<D, true>(x, X, g, pis, C::PPC, omega);
}

// r_c = P^T (b - hs A x) per parent cell (colour-0 patch); x == nullptr -> P^T b
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D>::NT) restrict_kernel(const T* __restrict__ x, const T* __restrict__ b,
                                                              T* __restrict__ rc, LevelGeom gf, LevelGeom gc) {
  using C = Cfg<D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* T1 = X + C::PPC * C::TSZ;
  T* FU = T1 + C::PPC * C::TSZ;
  T* FD = FU + C::PPC * 2 * C::NFP;
  __shared__ PatchInfo pis[C::PPC];
  const long long patch0 = (long long)blockIdx.x * C::PPC;
  setup_patches<D, T>(pis, gf, 0, patch0, C::PPC);
  const T hs = T(gf.hs);
  if (x != nullptr) {
    load_patches<D>(X, x, gf, pis, C::PPC, T(1));
    __syncthreads();
    volume_apply<D>(X, T1, pis, C::PPC);
    face_terms<D>(X, FU, FD, x, gf, pis, C::PPC, T(1));
    for (int e = threadIdx.x; e < C::PPC * C::PATCH; e += blockDim.x) {
      const int p = e / C::PATCH, r = e % C::PATCH, q = r / C::CELL, l = r % C::CELL;
      const int node = p * C::TSZ + node_of_cell<D>(q, l);
      T bv = T(0);
      if (pis[p].valid) bv = __ldg(b + patch_cell_offset<D>(gf, pis[p], q) + l);
      X[node] = bv - hs * X[node];
    }
  } else {
    load_patches<D>(X, b, gf, pis, C::PPC, T(1));
  }
  __syncthreads();
  // P^T along x (all NL lines), then y (lines with i0 < NC), then z (i0,i1 < NC)
#pragma unroll 1
  for (int a = 0; a < D; ++a) {
    const int nl = (D == 2) ? (a == 0 ? NP : NC) : (a == 0 ? NP * NP : (a == 1 ? NC * NP : NC * NC));
    for (int e = threadIdx.x; e < C::PPC * nl; e += blockDim.x) {
      const int p = e / nl, li = e % nl;
      int l;   // line id in line_geom numbering
      if (D == 2) l = li;
      else if (a == 0) l = li;                          // (i1, i2) all
      else if (a == 1) l = (li % NC) + NP * (li / NC);  // (i0 < NC, i2)
      else l = (li % NC) + NP * (li / NC);              // (i0 < NC, i1 < NC)
      int base, stride;
      line_geom<D>(a, l, base, stride);
      T v[NP], w[NC];
      load_line<NP>(X + p * C::TSZ + base, stride, v);
      matvec<NC, NP, ProlT<T>>(v, w);
      store_line<NC>(X + p * C::TSZ + base, stride, w);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < C::PPC * C::CELL; e += blockDim.x) {
    const int p = e / C::CELL, l = e % C::CELL;
    if (!pis[p].valid) continue;
    const PatchInfo& pi = pis[p];
    const long long o = cell_offset_cells(gc, pi.c0[0] >> 1, pi.c0[1] >> 1, D == 3 ? pi.c0[2] >> 1 : 0) * C::CELL + l;
    rc[o] = X[p * C::TSZ + node_of_cell<D>(0, l)];
  }
}

// x_f += P e_c per parent cell
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D>::NT) prolong_kernel(const T* __restrict__ ec, T* __restrict__ xf,
                                                             LevelGeom gf, LevelGeom gc) {
  using C = Cfg<D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  __shared__ PatchInfo pis[C::PPC];
  const long long patch0 = (long long)blockIdx.x * C::PPC;
  setup_patches<D, T>(pis, gf, 0, patch0, C::PPC);
  for (int e = threadIdx.x; e < C::PPC * C::CELL; e += blockDim.x) {
    const int p = e / C::CELL, l = e % C::CELL;
    const PatchInfo& pi = pis[p];
    T v = T(0);
    if (pi.valid)
      v = __ldg(ec + cell_offset_cells(gc, pi.c0[0] >> 1, pi.c0[1] >> 1, D == 3 ? pi.c0[2] >> 1 : 0) * C::CELL + l);
    X[p * C::TSZ + node_of_cell<D>(0, l)] = v;
  }
  __syncthreads();
  // expand the last direction first so that the lines of earlier directions exist
#pragma unroll 1
  for (int a = D - 1; a >= 0; --a) {
    const int nl = (D == 2) ? (a == 1 ? NC : NP) : (a == 2 ? NC * NC : (a == 1 ? NC * NP : NP * NP));
    for (int e = threadIdx.x; e < C::PPC * nl; e += blockDim.x) {
      const int p = e / nl, li = e % nl;
      int l;
      if (D == 2) l = li;
      else if (a == 0) l = li;
      else l = (li % NC) + NP * (li / NC);
      int base, stride;
      line_geom<D>(a, l, base, stride);
      T v[NC], w[NP];
      load_line<NC>(X + p * C::TSZ + base, stride, v);
      matvec<NP, NC, Prol<T>>(v, w);
      store_line<NP>(X + p * C::TSZ + base, stride, w);
    }
    __syncthreads();
  }
  store_patches<D, true>(xf, X, gf, pis, C::PPC, T(1));
}

// ---------------------------------------------------------------- host launchers
template <int D, typename T>
constexpr size_t smem_bytes(int ntensors, bool faces) {
  using C = Cfg<D>;
  return sizeof(T) * ((size_t)ntensors * C::PPC * C::TSZ + (faces ? 4 * (size_t)C::PPC * C::NFP : 0));
}

template <typename F>
inline cudaError_t set_smem(F* f, size_t bytes) {
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int D, typename T>
cudaError_t launch_vmult(const void* x, void* y, const LevelGeom& g, const void* bm, cudaStream_t s) {
  using C = Cfg<D>;
  const long long np = num_patches(g, D, 0);
  const unsigned grid = (unsigned)((np + C::PPC - 1) / C::PPC);
  const size_t sm = smem_bytes<D, T>(2, true);
  cudaError_t e = set_smem(vmult_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  vmult_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)x, (T*)y, (const T*)bm, g);
  return cudaGetLastError();
}

template <int D, typename T>
cudaError_t launch_smooth(const void* xi, const void* b, void* xo, const LevelGeom& g, int colour, cudaStream_t s) {
  using C = Cfg<D>;
  const long long np = num_patches(g, D, colour);
  const int patch_ctas = (int)((np + C::PPC - 1) / C::PPC);
  int copy_ctas = 0;
  if (colour != 0) {
    long long cells = 0;
    for (int a = 0; a < D; ++a) {
      if (!((colour >> a) & 1)) continue;
      long long layer = 1;
      for (int bb = 0; bb < D; ++bb) if (bb != a) layer *= g.n[bb];
      cells += 2 * layer;
    }
    long long elems = cells * C::CELL;
    copy_ctas = (int)((elems + C::NT * 4 - 1) / (C::NT * 4));
    if (copy_ctas < 1) copy_ctas = 1;
    if (copy_ctas > 4 * 148) copy_ctas = 4 * 148;
  }
  const size_t sm = smem_bytes<D, T>(1, true);
  cudaError_t e = set_smem(smooth_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  if (patch_ctas + copy_ctas == 0) return cudaSuccess;
  smooth_kernel<D, T><<<patch_ctas + copy_ctas, C::NT, sm, s>>>((const T*)xi, (const T*)b, (T*)xo, g, colour,
                                                                  patch_ctas);
  return cudaGetLastError();
}

template <int D, typename T>
cudaError_t launch_additive(const void* r, void* x, const LevelGeom& g, int colour, double omega, cudaStream_t s) {
  using C = Cfg<D>;
  const long long np = num_patches(g, D, colour);
  const int grid = (int)((np + C::PPC - 1) / C::PPC);
  if (grid == 0) return cudaSuccess;
  const size_t sm = smem_bytes<D, T>(1, false);
  cudaError_t e = set_smem(additive_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  additive_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)r, (T*)x, g, colour, (T)omega);
  return cudaGetLastError();
}

template <int D, typename T>
cudaError_t launch_restrict(const void* x, const void* b, void* rc, const LevelGeom& gf, const LevelGeom& gc,
                            cudaStream_t s) {
  using C = Cfg<D>;
  const long long np = num_patches(gf, D, 0);
  const unsigned grid = (unsigned)((np + C::PPC - 1) / C::PPC);
  const size_t sm = smem_bytes<D, T>(2, true);
  cudaError_t e = set_smem(restrict_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  restrict_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)x, (const T*)b, (T*)rc, gf, gc);
  return cudaGetLastError();
}

template <int D, typename T>
cudaError_t launch_prolong(const void* ec, void* xf, const LevelGeom& gf, const LevelGeom& gc, cudaStream_t s) {
  using C = Cfg<D>;
  const long long np = num_patches(gf, D, 0);
  const unsigned grid = (unsigned)((np + C::PPC - 1) / C::PPC);
  const size_t sm = smem_bytes<D, T>(1, false);
  cudaError_t e = set_smem(prolong_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  prolong_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)ec, (T*)xf, gf, gc);
  return cudaGetLastError();
}

// runtime (dim, prec) dispatch
#define IPMG_DISPATCH(dim, prec, FN, ...)                                  \
  ((dim) == 2 ? ((prec) == 0 ? FN<2, double>(__VA_ARGS__) : FN<2, float>(__VA_ARGS__)) \
              : ((prec) == 0 ? FN<3, double>(__VA_ARGS__) : FN<3, float>(__VA_ARGS__)))

inline cudaError_t upload(const void* t64, const void* t32, size_t b64, size_t b32) {
  if (b64 != sizeof(TabData<K, double>) || b32 != sizeof(TabData<K, float>)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemcpyToSymbol(c_tab64, t64, b64);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_tab32, t32, b32);
}
inline cudaError_t vmult(int dim, int prec, const void* x, void* y, const LevelGeom& g, const void* bm, cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_vmult, x, y, g, bm, s);
}
inline cudaError_t smooth(int dim, int prec, const void* xi, const void* b, void* xo, const LevelGeom& g, int c,
                          cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_smooth, xi, b, xo, g, c, s);
}
inline cudaError_t additive(int dim, int prec, const void* r, void* x, const LevelGeom& g, int c, double om,
                            cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_additive, r, x, g, c, om, s);
}
inline cudaError_t restrict_(int dim, int prec, const void* x, const void* b, void* rc, const LevelGeom& gf,
                             const LevelGeom& gc, cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_restrict, x, b, rc, gf, gc, s);
}
inline cudaError_t prolong(int dim, int prec, const void* ec, void* xf, const LevelGeom& gf, const LevelGeom& gc,
                           cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_prolong, ec, xf, gf, gc, s);
}

}  // namespace IPMG_KK
}  // namespace ipmg

extern "C++" ipmg::KernelSet IPMG_CAT(ipmg_kernel_set_k, IPMG_K)() {
  ipmg::KernelSet ks;
  ks.k = IPMG_K;
  ks.upload = ipmg::IPMG_KK::upload;
  ks.tab_bytes64 = sizeof(ipmg::TabData<IPMG_K, double>);
  ks.tab_bytes32 = sizeof(ipmg::TabData<IPMG_K, float>);
  ks.vmult = ipmg::IPMG_KK::vmult;
  ks.smooth = ipmg::IPMG_KK::smooth;
  ks.additive = ipmg::IPMG_KK::additive;
  ks.restrict_ = ipmg::IPMG_KK::restrict_;
  ks.prolong = ipmg::IPMG_KK::prolong;
  return ks;
}
