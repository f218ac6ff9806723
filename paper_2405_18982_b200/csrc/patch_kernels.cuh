// Vertex-patch kernels of the ipmg library, templated on dimension D, degree
// K (via IPMG_K of the including translation unit) and precision T.
//
// One CTA processes PPC vertex patches of one colour.  Each patch is staged in
// shared memory as a patch-lexicographic tensor of (2(k+1))^d values (odd row
// pitch; plane and patch pitches padded by a compile-time search that minimises the
// bank conflicts of the line passes -- the face-trace loads and stores still conflict,
// ncu counts in profiles/), loaded and stored with
// coalesced (vectorised where the cell size allows) cooperative copies of
// whole cell chunks.  Every sum-factorisation step is a "line pass": a thread
// owns R whole 1D lines of one patch along one direction (R = 2 in fp32, 1 in
// fp64), reads them into registers, multiplies them by a 1D matrix whose
// entries are compile-time-indexed __constant__ data (one uniform-register
// load LDCU.128 feeds 4R FMAs), and writes the lines back in place.
//
//  vmult_kernel     y = A x over colour-0 patches   PAPER.md:112-138 (Fig. 1 patch-wise
//                   (each patch writes only its      integration), Kronecker sum of
//                   own cells -> no atomics)         PAPER.md:118-126, face terms of
//                                                    eq. bilinear_form
//  smooth_kernel    one colour of Algorithm 1, full kernel, replacement form
//                   x_j = A_j^{-1}(b_j - C_j x_ext), algebraically identical to
//                   x_j + A_j^{-1} R_j (b - A x) because A_j = R_j A R_j^T
//                   (PAPER.md:183-199, 242-257); A_j^{-1} by fast diagonalisation
//
//  additive_kernel  x += omega R_j^T A_j^{-1} R_j r over one colour (r precomputed)
//  restrict_kernel  r_c = P^T (b - A x) per parent cell
//  prolong_kernel   x_f += P e_c per parent cell
#pragma once
#include "common.cuh"
#include "fe1d.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <mutex>
#include <utility>
#include <vector>

#ifndef IPMG_K
#error "IPMG_K must be defined by the including translation unit"
#endif

#define IPMG_CAT2(a, b) a##b
#define IPMG_CAT(a, b) IPMG_CAT2(a, b)
// every degree lives in its own namespace: the per-TU __constant__ tables and
// the kernel template instantiations must not collide at link time
// The Dirichlet-kernel translation units (kernels_dir_k<K>.cu, IPMG_DIRICHLET = 1)
// fill the same table layout with the Dirichlet tables (LP <- LPR, S <- SD,
// lam <- lamD, act <- actD) in their own constant bank (64 KB per module).
#ifndef IPMG_DIRICHLET
#define IPMG_DIRICHLET 0
#endif
#if IPMG_DIRICHLET
#define IPMG_KK IPMG_CAT(kdir, IPMG_K)
#else
#define IPMG_KK IPMG_CAT(kdeg, IPMG_K)
#endif

namespace ipmg {
namespace IPMG_KK {

constexpr int K = IPMG_K;
constexpr bool kDir = IPMG_DIRICHLET != 0;
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
constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// bank multiplicity of one warp-wide access whose per-thread word offsets are
// base(u) (4-byte words for fp32; 8-byte words for fp64, served per half warp)
template <typename T, class F>
constexpr int bank_cost(F base, int nthreads) {
  int worst = 1;
  if (sizeof(T) == 4) {
    for (int b = 0; b < 32; ++b) {
      int c = 0;
      for (int u = 0; u < 32 && u < nthreads; ++u) c += ((base(u) % 32 + 32) % 32 == b);
      worst = c > worst ? c : worst;
    }
  } else {
    for (int h = 0; h < 2; ++h)
      for (int b = 0; b < 16; ++b) {
        int c = 0;
        for (int u = 16 * h; u < 16 * h + 16 && u < nthreads; ++u) c += ((base(u) % 16 + 16) % 16 == b);
        worst = c > worst ? c : worst;
      }
  }
  return worst;
}

template <int D, typename T>
struct Cfg {
  // lines per thread: fp32 2 for k <= 3, 1 for k >= 4 (C3 sweep: 3D k=4/5 smoother
  // +10 %, 2D k=7 solve 30.4 -> 29.2 ms); fp64 1
#ifndef IPMG_R64
#define IPMG_R64 0   // lines per thread of the fp64 kernels (0: as measured -- 2 for 3D k=7, else 1)
#endif
  // fp64: 3D k=7 operator 1.96 -> 1.68 ms with 2 lines per thread (and 1 patch per CTA);
  // slower for k = 2, 4, 5, 6, equal for k = 3 (tools/gpu_ab_vmult.sh)
  static constexpr int R64 = IPMG_R64 > 0 ? IPMG_R64 : ((D == 3 && NC == 8) ? 2 : 1);
#ifdef IPMG_R32
  static constexpr int R = sizeof(T) == 4 ? IPMG_R32 : R64;
#else
  static constexpr int R = (sizeof(T) == 4 && NC <= 4) ? 2 : (sizeof(T) == 8 ? R64 : 1);
#endif
  static constexpr int RP = NP + 1;                           // row pitch (odd)
  static constexpr int NL = (D == 2) ? NP : NP * NP;          // lines per direction per patch
  static constexpr int G = NL / R;                            // line groups per patch
  static constexpr int CELL = ipow(NC, D);
  static constexpr int NCH = 1 << D;                          // cells per patch
  static constexpr int PATCH = NCH * CELL;
  static constexpr int NFP = NL;                              // tangential points per face
  static constexpr int NNB = 2 * D * (1 << (D - 1));          // face-neighbour cells per patch
#ifndef IPMG_GROUPS_TARGET
#define IPMG_GROUPS_TARGET 32
#endif
  // line groups per CTA: 1 warp (measured best for k >= 3; 2 warps for fp32 with
  // R = 1); 4 warps for k <= 2,
  // whose tiny patches otherwise leave a CTA with too little work (C3 sweep: 3D
  // k=2 smoother step 10.4 -> 12.7 GDoF/s)
#ifndef IPMG_GT64
#define IPMG_GT64 IPMG_GROUPS_TARGET
#endif
  static constexpr int GT = NC <= 3 ? 4 * IPMG_GROUPS_TARGET
                                    : ((sizeof(T) == 4 && R == 1) ? 2 * IPMG_GROUPS_TARGET
                                                                  : (sizeof(T) == 8 ? IPMG_GT64 : IPMG_GROUPS_TARGET));
#ifndef IPMG_PPC3
#define IPMG_PPC3 0   // > 0: patches per CTA in 3D (experiments)
#endif
#ifndef IPMG_PPC3_NC
#define IPMG_PPC3_NC 0   // restrict IPMG_PPC3 to this NC (0: all)
#endif
#ifndef IPMG_PPC3_64
#define IPMG_PPC3_64 0   // > 0: patches per CTA of every 3D fp64 kernel (experiments); 0: as measured
#endif
  // 3D fp64 kernels (the CG operator): 2 patches per CTA for k = 4 (measured,
  // tools/gpu_ab_vmult.sh: 3D k=4 fp64 operator 3.20 -> 3.03 ms; neutral or slower for
  // k = 2, 3, 5, 6; 3 patches slower everywhere; k = 7 takes 2 lines per thread instead)
  static constexpr int PPC = (D == 3 && sizeof(T) == 8 && IPMG_PPC3_64 > 0) ? IPMG_PPC3_64
                           : (D == 3 && sizeof(T) == 8 && IPMG_PPC3_64 == 0 && NC == 5) ? 2
                           : (D == 3 && IPMG_PPC3 > 0 && (IPMG_PPC3_NC == 0 || IPMG_PPC3_NC == NC))
                                 ? IPMG_PPC3
                                 : ((GT / G) > 1 ? (GT / G) : 1);   // patches per CTA
  static constexpr int GROUPS = PPC * G;
  static constexpr int NT = (((GROUPS + 31) / 32) * 32) > 1024 ? 1024 : ((GROUPS + 31) / 32) * 32;

  // line base offset of group g (first line) of patch p for direction a
  static constexpr int line_base(int a, int p, int g, int pl, int tsz) {
    return (D == 2) ? (p * tsz + (a == 0 ? g * RP : g))
                    : (p * tsz + (a == 0 ? (g % NP) * RP + (g / NP) * pl
                                         : a == 1 ? (g % NP) + (g / NP) * pl : (g % NP) + (g / NP) * RP));
  }
  static constexpr int cost(int pl, int tsz) {
    int c = 0;
    for (int a = 0; a < D; ++a) {
      struct B {
        int a, pl, tsz;
        constexpr int operator()(int u) const { return line_base(a, u / G, u % G, pl, tsz); }
      };
      const int w = bank_cost<T>(B{a, pl, tsz}, GROUPS < NT ? GROUPS : NT);
      c = c > w ? c : w;
    }
    return c;
  }
  static constexpr int pick_pl() {
    if (D == 2) return NP * RP;
    int best = NP * RP, bc = 1 << 30;
    for (int pad = 0; pad < 32; ++pad) {
      const int pl = NP * RP + pad;
      const int c = cost(pl, NP * pl + 0);
      if (c < bc) { bc = c; best = pl; }
    }
    return best;
  }
  static constexpr int PL = pick_pl();                         // plane pitch
  static constexpr int pick_tsz() {
    const int base = (D == 2) ? NP * RP : NP * PL;
    int best = base, bc = 1 << 30;
    for (int pad = 0; pad < 32; ++pad) {
      const int c = cost(PL, base + pad);
      if (c < bc) { bc = c; best = base + pad; }
    }
    return best;
  }
  static constexpr int TSZ = pick_tsz();                       // patch pitch
  // face arrays (F): 2D one padded line per array; 3D an NP x NP grid with
  // odd row pitch FROW, array pitch FARR chosen so that the transform lines of
  // neighbouring arrays fall into disjoint banks
  static constexpr int FROW = NP + 1;
  static constexpr int pick_farr() {
    if (D == 2) return NP + 1;
    int best = NP * FROW, bc = 1 << 30;
    for (int pad = 0; pad < 64; ++pad) {
      const int fa = NP * FROW + pad;
      struct B0 { int fa; constexpr int operator()(int u) const { return (u / NP) * fa + (u % NP) * (NP + 1); } };
      struct B1 { int fa; constexpr int operator()(int u) const { return (u / NP) * fa + (u % NP); } };
      const int c0 = bank_cost<T>(B0{fa}, 32), c1 = bank_cost<T>(B1{fa}, 32);
      const int c = c0 > c1 ? c0 : c1;
      if (c < bc) { bc = c; best = fa; }
    }
    return best;
  }
  static constexpr int FARR = pick_farr();
  // face scratch per patch, padded so that the face-injection reads of the
  // patches sharing a warp (lane u -> patch u / G, line u % G) hit distinct banks
  static constexpr int fpos_c(int t) { return D == 2 ? t : (t % NP) + (t / NP) * FROW; }
  static constexpr int pick_fsz() {
    const int base = 4 * D * FARR;
    int best = base, bc = 1 << 30;
    for (int pad = 0; pad < 32; ++pad) {
      struct B { int fs; constexpr int operator()(int u) const { return (u / G) * fs + fpos_c(u % G); } };
      const int c = bank_cost<T>(B{base + pad}, 32);
      if (c < bc) { bc = c; best = base + pad; }
    }
    return best;
  }
  static constexpr int FSZ = pick_fsz();
  // neighbour-cell staging (cp.async prefetch at kernel start): one slot per
  // face-neighbour cell, slot pitch SP a multiple of 16 bytes with SP/VE odd so
  // that the 16-byte row reads of neighbouring slots hit different banks
  static constexpr int VE = 16 / (int)sizeof(T);
  static constexpr int SP0 = ((CELL + VE - 1) / VE) * VE;
  static constexpr int SP = ((SP0 / VE) % 2 == 0) ? SP0 + VE : SP0;
  static constexpr int NBS = PPC * NNB * SP;                   // staging elements per CTA
#ifdef IPMG_STAGE
  static constexpr bool STAGE = (size_t)NBS * sizeof(T) <= 48 * 1024;
#else
  static constexpr bool STAGE = false;   // measured: the occupancy loss outweighs the prefetch
#endif
  static constexpr int CPB = (CELL * (int)sizeof(T)) % 16 == 0 ? 16 : ((CELL * (int)sizeof(T)) % 8 == 0 ? 8 : 4);
  // minimum resident CTAs per SM requested from ptxas (register cap), per (dim, precision)
#ifndef IPMG_SMOOTH_MINB_2F
#define IPMG_SMOOTH_MINB_2F 0
#endif
#ifndef IPMG_SMOOTH_MINB_3F
#define IPMG_SMOOTH_MINB_3F 0
#endif
#ifndef IPMG_VMULT_MINB_2D
#define IPMG_VMULT_MINB_2D 0
#endif
  static constexpr int MINB_SMOOTH = sizeof(T) == 4 ? (D == 2 ? IPMG_SMOOTH_MINB_2F : IPMG_SMOOTH_MINB_3F) : 0;
  static constexpr int MINB_VMULT = (sizeof(T) == 8 && D == 2) ? IPMG_VMULT_MINB_2D : 0;   // 0: no request
};

template <typename T>
__device__ __forceinline__ T fma_(T a, T b, T c) { return fma(a, b, c); }

// interior patches (variant 0, the overwhelming majority) take the path with
// compile-time constant operands; boundary patches the register-indexed one
#ifdef IPMG_TIMING_FAST_ONLY   // timing experiment only: wrong on boundary patches
#define IPMG_VAR_SPLIT(var, FAST, SLOW) \
  { (void)(var); FAST; }
#else
#define IPMG_VAR_SPLIT(var, FAST, SLOW) \
  if (kFastOnly || (var) == 0) { FAST; } else { const int v_ = (var); SLOW; }
#endif
// functions instantiated for CTAs whose patches are all interior shadow this with
// a template parameter of the same name (the run-time variant paths disappear)
constexpr bool kFastOnly = false;
// reciprocal of a positive eigenvalue sum: MUFU approximation (fp32: 1 ulp);
// fp64: approximation refined by two Newton steps (full precision)
__device__ __forceinline__ float rcp_(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ double rcp_(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

// ---------------------------------------------------------------- 1D matrices
// get(i, j): entry of the (NOUT x NIN) matrix applied as out[i] = sum_j get(i,j) in[j];
// nz(i,j): structural non-zero.  The products are evaluated as outer products
// (column j times in[j] into all accumulators -- the order the compiler picks
// for ILP), so every functor reads a COLUMN of its matrix contiguously.
template <typename T>
struct MassP {   // block-diagonal 2-cell patch mass
  static __device__ __forceinline__ T get(int i, int j) {   // symmetric; explicit zero off the cell blocks
    return (i / NC == j / NC) ? tab<T>().M[j % NC][i % NC] : T(0);
  }
  static __device__ __forceinline__ constexpr bool nz(int i, int j) { return i / NC == j / NC; }
};
template <int V, typename T>
struct LapP {    // patch stiffness + face terms; cross-cell blocks only touch the interior face
  static __device__ __forceinline__ T get(int i, int j) { return tab<T>().LP[V][j][i]; }   // symmetric
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
  static __device__ __forceinline__ T get(int i, int m) { return tab<T>().ST[V][m][i]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
// Interior variant: S = [S_even | S_odd] with S_even[np-1-i][m] = S_even[i][m],
// S_odd[np-1-i][m] = -S_odd[i][m] (reflection symmetry of the interior patch
// problem, modes ordered by fe1d.cpp).  Half-size products:
//   S^T v:  even modes <- S_e^T (v_i + v_{np-1-i}),  odd modes <- S_o^T (v_i - v_{np-1-i})
//   S w:    E = S_e w_e, O = S_o w_o;  out_i = E_i + O_i,  out_{np-1-i} = E_i - O_i   (i < np/2)
template <typename T>
struct EvenT {   // (S_e^T)[m][i] = S[0][i][m],      m, i < np/2
  static __device__ __forceinline__ T get(int m, int i) { return tab<T>().S[0][i][m]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct OddT {    // (S_o^T)[m][i] = S[0][i][np/2+m]
#ifndef IPMG_ODD_ALIGNED
#define IPMG_ODD_ALIGNED 1
#endif
#if IPMG_ODD_ALIGNED
  // aligned copy: with S[0][i][NP/2 + m] the pairs straddle 8-byte boundaries for odd
  // NP/2 and cost one UMOV per constant (3D k=4: ~20 per line pass)
  static __device__ __forceinline__ T get(int m, int i) { return tab<T>().SO[i][m]; }
#else
  static __device__ __forceinline__ T get(int m, int i) { return tab<T>().S[0][i][NP / 2 + m]; }
#endif
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct EvenB {   // S_e[i][m] = ST[0][m][i]
  static __device__ __forceinline__ T get(int i, int m) { return tab<T>().ST[0][m][i]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct OddB {    // S_o[i][m] = ST[0][np/2+m][i]
  static __device__ __forceinline__ T get(int i, int m) { return tab<T>().ST[0][NP / 2 + m][i]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <int NOUT, int NIN, class A, int R, typename T>
__device__ __forceinline__ void mv(const T (&in)[R][NIN], T (&out)[R][NOUT], const A& mat);
template <int NOUT, int NIN, class A, int R>
__device__ __forceinline__ void mv(const float (&in)[R][NIN], float (&out)[R][NOUT], const A& mat);

template <int R, typename T>
__device__ __forceinline__ void eigT_eo(const T (&in)[R][NP], T (&out)[R][NP]) {
  constexpr int H = NP / 2;
  T e[R][H], o[R][H], we[R][H], wo[R][H];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int i = 0; i < H; ++i) {
      e[r][i] = in[r][i] + in[r][NP - 1 - i];
      o[r][i] = in[r][i] - in[r][NP - 1 - i];
    }
  mv<H, H, EvenT<T>, R>(e, we, EvenT<T>{});
  mv<H, H, OddT<T>, R>(o, wo, OddT<T>{});
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < H; ++m) {
      out[r][m] = we[r][m];
      out[r][H + m] = wo[r][m];
    }
}
template <int R, typename T>
__device__ __forceinline__ void eig_eo(const T (&in)[R][NP], T (&out)[R][NP]) {
  constexpr int H = NP / 2;
  T ie[R][H], io[R][H], E[R][H], O[R][H];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < H; ++m) {
      ie[r][m] = in[r][m];
      io[r][m] = in[r][H + m];
    }
  mv<H, H, EvenB<T>, R>(ie, E, EvenB<T>{});
  mv<H, H, OddB<T>, R>(io, O, OddB<T>{});
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int i = 0; i < H; ++i) {
      out[r][i] = E[r][i] + O[r][i];
      out[r][NP - 1 - i] = E[r][i] - O[r][i];
    }
}

// runtime-variant versions (boundary patches): entries are loaded with a
// register-indexed constant load instead of a uniform-register operand
template <typename T>
struct LapRT {
  int v;
  __device__ __forceinline__ T get(int i, int j) const { return tab<T>().LP[v][j][i]; }
  static __device__ __forceinline__ constexpr bool nz(int i, int j) { return LapP<0, T>::nz(i, j); }
};
template <typename T>
struct EigTRT {
  int v;
  __device__ __forceinline__ T get(int m, int i) const { return tab<T>().S[v][i][m]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct EigRT {
  int v;
  __device__ __forceinline__ T get(int i, int m) const { return tab<T>().ST[v][m][i]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct SMtRT {
  int v;
  __device__ __forceinline__ T get(int m, int i) const { return tab<T>().MS[v][i][m]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};

template <typename T>
struct Prol {    // P: (NP x NC)
  static __device__ __forceinline__ T get(int i, int j) { return tab<T>().PT[j][i]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <typename T>
struct ProlT {   // P^T: (NC x NP)
  static __device__ __forceinline__ T get(int j, int i) { return tab<T>().P[i][j]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};

// out[r][i] = sum_j A(i,j) in[r][j] for R lines sharing every matrix entry
template <int NOUT, int NIN, class A, int R, typename T>
__device__ __forceinline__ void mv(const T (&in)[R][NIN], T (&out)[R][NOUT], const A& mat = A{}) {
#pragma unroll
  for (int i = 0; i < NOUT; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) out[r][i] = T(0);
#pragma unroll
  for (int j = 0; j < NIN; ++j)
#pragma unroll
    for (int i = 0; i < NOUT; ++i)
      if (A::nz(i, j)) {
        const T a = mat.get(i, j);
#pragma unroll
        for (int r = 0; r < R; ++r) out[r][i] = fma_(a, in[r][j], out[r][i]);
      }
}
// out[r][i] += sum_j A(i,j) in[r][j]
template <int NOUT, int NIN, class A, int R, typename T>
__device__ __forceinline__ void mv_acc(const T (&in)[R][NIN], T (&out)[R][NOUT], const A& mat = A{}) {
#pragma unroll
  for (int j = 0; j < NIN; ++j)
#pragma unroll
    for (int i = 0; i < NOUT; ++i)
      if (A::nz(i, j)) {
        const T a = mat.get(i, j);
#pragma unroll
        for (int r = 0; r < R; ++r) out[r][i] = fma_(a, in[r][j], out[r][i]);
      }
}

// ---- fp32: packed FFMA2 (fma.rn.f32x2, sm_100).  Outputs are accumulated in
// pairs (i, i+1) from a column pair of the matrix (one 64-bit uniform-register
// constant) times a broadcast input: half the FMA instructions of the scalar
// form -- the smoother is issue-bound, so this is the main fp32 lever.
#ifndef IPMG_FFMA2_BUILTIN
#define IPMG_FFMA2_BUILTIN 1
#endif
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
#if IPMG_FFMA2_BUILTIN
  // the sm_100 builtin: the compiler sees the operation, so broadcast inputs
  // become the .F32 operand form instead of MOV/LOP3 register-pair packing
  return __ffma2_rn(a, b, c);
#endif
  unsigned long long ra, rb, rc, rd;
  ra = (unsigned long long)__float_as_uint(a.x) | ((unsigned long long)__float_as_uint(a.y) << 32);
  rb = (unsigned long long)__float_as_uint(b.x) | ((unsigned long long)__float_as_uint(b.y) << 32);
  rc = (unsigned long long)__float_as_uint(c.x) | ((unsigned long long)__float_as_uint(c.y) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return make_float2(__uint_as_float((unsigned)rd), __uint_as_float((unsigned)(rd >> 32)));
}
template <int NOUT, int NIN, class A, int R, bool ACC>
__device__ __forceinline__ void mv2(const float (&in)[R][NIN], float (&out)[R][NOUT], const A& mat) {
  constexpr int NPR = NOUT / 2;
  float2 acc[R][NPR > 0 ? NPR : 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q < NPR; ++q) acc[r][q] = ACC ? make_float2(out[r][2 * q], out[r][2 * q + 1]) : make_float2(0.f, 0.f);
  float tail[R];
#pragma unroll
  for (int r = 0; r < R; ++r) tail[r] = (ACC && (NOUT & 1)) ? out[r][NOUT - 1] : 0.f;
#pragma unroll
  for (int j = 0; j < NIN; ++j) {
#pragma unroll
    for (int q = 0; q < NPR; ++q)
      if (A::nz(2 * q, j) || A::nz(2 * q + 1, j)) {
        const float2 a = make_float2(mat.get(2 * q, j), mat.get(2 * q + 1, j));
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][q] = ffma2(a, make_float2(in[r][j], in[r][j]), acc[r][q]);
      }
    if ((NOUT & 1) && A::nz(NOUT - 1, j)) {
      const float a = mat.get(NOUT - 1, j);
#pragma unroll
      for (int r = 0; r < R; ++r) tail[r] = fmaf(a, in[r][j], tail[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int q = 0; q < NPR; ++q) {
      out[r][2 * q] = acc[r][q].x;
      out[r][2 * q + 1] = acc[r][q].y;
    }
    if (NOUT & 1) out[r][NOUT - 1] = tail[r];
  }
}
template <int NOUT, int NIN, class A, int R>
__device__ __forceinline__ void mv(const float (&in)[R][NIN], float (&out)[R][NOUT], const A& mat = A{}) {
  mv2<NOUT, NIN, A, R, false>(in, out, mat);
}
template <int NOUT, int NIN, class A, int R>
__device__ __forceinline__ void mv_acc(const float (&in)[R][NIN], float (&out)[R][NOUT], const A& mat = A{}) {
  mv2<NOUT, NIN, A, R, true>(in, out, mat);
}

template <int N, int R, typename T>
__device__ __forceinline__ void load_lines(const T* p, int gap, int stride, T (&v)[R][N]) {
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < N; ++j) v[r][j] = p[r * gap + j * stride];
}
template <int N, int R, typename T>
__device__ __forceinline__ void store_lines(T* p, int gap, int stride, const T (&v)[R][N]) {
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < N; ++j) p[r * gap + j * stride] = v[r][j];
}

// line geometry: first line of group g in direction a; lines of a group are
// `gap` apart (line l and l + G), elements `stride` apart
template <int D, typename T>
__device__ __forceinline__ void group_geom(int a, int g, int& base, int& gap, int& stride) {
  using C = Cfg<D, T>;
  constexpr int G = C::G;
  if (D == 2) {
    if (a == 0) { base = g * C::RP; gap = G * C::RP; stride = 1; }
    else        { base = g;         gap = G;         stride = C::RP; }
  } else {
    // line index l = u + NP * v ; l + G with G a multiple of NP/R ...: compute both explicitly
    const int u = g % NP, v = g / NP;
    const int l2 = g + G, u2 = l2 % NP, v2 = l2 / NP;
    if (a == 0)      { base = u * C::RP + v * C::PL; gap = (u2 * C::RP + v2 * C::PL) - base; stride = 1; }
    else if (a == 1) { base = u + v * C::PL;         gap = (u2 + v2 * C::PL) - base;          stride = C::RP; }
    else             { base = u + v * C::RP;         gap = (u2 + v2 * C::RP) - base;          stride = C::PL; }
  }
}

// smem offset of node (local node l of cell q) inside a patch tensor
template <int D, typename T>
__device__ __forceinline__ int node_of_cell(int q, int l) {
  using C = Cfg<D, T>;
  const int l0 = l % NC, l1 = (l / NC) % NC;
  const int i0 = (q & 1) * NC + l0, i1 = ((q >> 1) & 1) * NC + l1;
  if (D == 2) return i0 + i1 * C::RP;
  const int l2 = l / (NC * NC);
  const int i2 = ((q >> 2) & 1) * NC + l2;
  return i0 + i1 * C::RP + i2 * C::PL;
}

// ---------------------------------------------------------------- patch indexing
template <int D>
struct PInfo {
  long long coff[1 << D];                 // element offset of every patch cell (ghost cells: outside 0..n)
  long long nb[2 * D][1 << (D - 1)];      // neighbour cell across face (a, side), NO_NB: none
  int var[3];                             // boundary variant per direction (global position)
  int valid;
  int own;                                // bit s: the cells with slowest-axis bit s are local (written)
  int c0[3];                              // lowest patch cell, local coordinates
};

// patches of a colour along the slowest axis S of a slab:
// unshifted: local lowest cells 0, 2, .., n-2; shifted: -1, 1, .., n-1 without
// the ones that would leave the global domain (-1 at zoff = 0, n-1 at the top)
__host__ __device__ inline int slab_patches(const LevelGeom& g, int S, int shifted) {
  if (!shifted) return g.n[S] / 2;
  return g.n[S] / 2 + 1 - (g.zoff == 0 ? 1 : 0) - (g.zoff + g.n[S] == g.nglob ? 1 : 0);
}
__host__ __device__ inline int slab_first(const LevelGeom& g, int shifted) {
  return shifted ? (g.zoff == 0 ? 1 : -1) : 0;
}

// patch block along the slowest axis of this CTA under the launch's selection
template <int D>
__device__ __forceinline__ int slab_block(const LevelGeom& g) {
  const int b = D == 3 ? (int)blockIdx.z : (int)blockIdx.y;
  return g.zsel == 0 ? b : (g.zsel == 1 ? b + 1 : (b == 0 ? 0 : g.znb - 1));
}
// block count of a selection out of n blocks along the slowest axis
__host__ __device__ inline int slab_sel_count(int n, int zsel) {
  return zsel == 0 ? n : (zsel == 1 ? (n > 2 ? n - 2 : 0) : (n < 2 ? n : 2));
}

__host__ __device__ inline long long num_patches(const LevelGeom& g, int dim, int colour) {
  long long np = 1;
  for (int a = 0; a < dim - 1; ++a) np *= (g.n[a] / 2 - ((colour >> a) & 1));
  return np * slab_patches(g, dim - 1, (colour >> (dim - 1)) & 1);
}

// Patch lattice coordinates of a CTA ("block" (bx, by, bz) of the colour's
// patch grid: x-blocks of PPC patches, patch row j1, patch plane j2) and the
// item decomposition of its setup: item 0 = patch info, 1..NCH = patch cells,
// then the NNB face-neighbour cells.  Boundary variants and neighbour existence
// along the slowest axis use GLOBAL coordinates; patches straddling the slab
// boundary (shifted colours) are computed by both ranks, each writing only its
// own cells (`own`).
template <int D>
struct PatchPos {
  int c0[3];
  bool valid;
};
template <int D, typename T>
__device__ __forceinline__ PatchPos<D> patch_pos(const LevelGeom& g, int colour, int bx, int by, int bz, int p) {
  using C = Cfg<D, T>;
  constexpr int S = D - 1;
  PatchPos<D> pp;
  const int m0 = g.n[0] / 2 - (colour & 1);
  const int c0s = slab_first(g, (colour >> S) & 1) + 2 * (D == 3 ? bz : by);
  const int j0 = bx * C::PPC + p;
  pp.valid = j0 < m0;
  pp.c0[0] = (colour & 1) + 2 * (pp.valid ? j0 : 0);
  pp.c0[1] = (D == 3) ? ((colour >> 1) & 1) + 2 * by : c0s;
  pp.c0[2] = (D == 3) ? c0s : 0;
  return pp;
}
// element offset of cell item it >= 1 (patch cell or face neighbour), NO_NB if absent
template <int D, typename T>
__device__ __forceinline__ long long item_offset(const LevelGeom& g, const PatchPos<D>& pp, int it) {
  using C = Cfg<D, T>;
  constexpr int S = D - 1;
  const int c0x = pp.c0[0], c0y = pp.c0[1], c0z = pp.c0[2];
  if (it <= C::NCH) {
    const int q = it - 1;
    return cell_offset_cells(g, c0x + (q & 1), c0y + ((q >> 1) & 1), c0z + ((q >> 2) & 1)) * (long long)C::CELL;
  }
  const int k2 = it - 1 - C::NCH;                 // (a, side, t)
  constexpr int PER = 1 << (D - 1);
  const int fs = k2 / PER, t = k2 % PER, a = fs >> 1, s = fs & 1;
  // neighbour across face (a, s): shift -1 / +2 along a; tangential bits of t
  const int sa = s == 0 ? -1 : 2;
  const int tb = t & 1, tcb = (t >> 1) & 1;
  const int cx = c0x + (a == 0 ? sa : tb);
  const int cy = c0y + (a == 1 ? sa : (a == 0 ? tb : tcb));
  const int cz = c0z + (D == 3 ? (a == 2 ? sa : tcb) : 0);
  const int ca = a == 0 ? cx : (a == 1 ? cy : cz);
  const bool ex = pp.valid && (a == S ? (g.zoff + ca >= 0 && g.zoff + ca < g.nglob)
                                      : (ca >= 0 && ca < (a == 0 ? g.n[0] : g.n[1])));   // a < S here
  return ex ? cell_offset_cells(g, cx, cy, cz) * (long long)C::CELL : NO_NB;
}

// fills PInfo of the CTA's patches; one thread per (patch, item)
template <int D, typename T>
__device__ __forceinline__ void setup_patches(PInfo<D>* pis, const LevelGeom& g, int colour, int bx, int by, int bz) {
  using C = Cfg<D, T>;
  constexpr int S = D - 1;
  constexpr int ITEMS = 1 + C::NCH + C::NNB;
  for (int e = threadIdx.x; e < C::PPC * ITEMS; e += blockDim.x) {
    const int p = e / ITEMS, it = e % ITEMS;
    const PatchPos<D> pp = patch_pos<D, T>(g, colour, bx, by, bz, p);
    PInfo<D>& pi = pis[p];
    if (it == 0) {
      const int c0x = pp.c0[0], c0y = pp.c0[1], c0s = pp.c0[S];
      pi.valid = pp.valid;
      pi.c0[0] = pp.c0[0];
      pi.c0[1] = pp.c0[1];
      pi.c0[2] = pp.c0[2];
      pi.own = (c0s >= 0 ? 1 : 0) | (c0s + 1 < g.n[S] ? 2 : 0);
      const int gs = g.zoff + c0s;
      const int vs = (gs == 0 ? 1 : 0) | (gs + 2 == g.nglob ? 2 : 0);
      pi.var[0] = (c0x == 0 ? 1 : 0) | (c0x + 2 == g.n[0] ? 2 : 0);
      pi.var[1] = (D == 3) ? ((c0y == 0 ? 1 : 0) | (c0y + 2 == g.n[1] ? 2 : 0)) : vs;
      pi.var[2] = (D == 3) ? vs : 0;
    } else if (it <= C::NCH) {
      pi.coff[it - 1] = item_offset<D, T>(g, pp, it);
    } else {
      const int k2 = it - 1 - C::NCH;
      constexpr int PER = 1 << (D - 1);
      pi.nb[k2 / PER][k2 % PER] = item_offset<D, T>(g, pp, it);
    }
  }
  __syncthreads();
}
template <int D, typename T>
__device__ __forceinline__ void setup_patches(PInfo<D>* pis, const LevelGeom& g, int colour) {
  const int bS = slab_block<D>(g);
  setup_patches<D, T>(pis, g, colour, (int)blockIdx.x, D == 3 ? (int)blockIdx.y : bS, D == 3 ? bS : 0);
}

// L2 prefetch of the patch cells of src (TMA bulk prefetch, one instruction per
// cell; the range is widened to 16-byte granularity).  Issued right after the
// setup so that the HBM reads of the patch's own rows overlap the face-trace
// phase instead of following it (the kernels are long-scoreboard bound).
#ifndef IPMG_PREFETCH
#define IPMG_PREFETCH 0   // measured: -5% (2D k=7), neutral in 3D
#endif
template <int D, typename T>
__device__ __forceinline__ void prefetch_cells(const T* src, const PInfo<D>* pis, int npc) {
#if IPMG_PREFETCH
  using C = Cfg<D, T>;
  if (src == nullptr) return;
  for (int e = threadIdx.x; e < npc * C::NCH; e += blockDim.x) {
    const PInfo<D>& pi = pis[e / C::NCH];
    if (!pi.valid) continue;
    const unsigned long long a = (unsigned long long)(src + pi.coff[e % C::NCH]);
    const unsigned long long a0 = a & ~15ull, a1 = (a + C::CELL * sizeof(T) + 15) & ~15ull;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
  }
#endif
}

// ---------------------------------------------------------------- cooperative copies
template <typename T, int V> struct VecT;
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<double, 1> { using type = double; };

// Copies between global cell chunks and the padded patch tensor walk the patch
// in ROW-major order (a warp covers consecutive patch rows; a row is 2 cell-row
// segments of NC contiguous global values), with a vector width V that divides
// NC: global accesses are fully used 16-byte sectors and the shared-memory side
// has at most a 2-way bank conflict.
template <typename T>
constexpr int row_vec() {
  return sizeof(T) == 4 ? (NC % 4 == 0 ? 4 : (NC % 2 == 0 ? 2 : 1)) : (NC % 2 == 0 ? 2 : 1);
}
template <typename VT, typename T>
__device__ __forceinline__ T vget(const VT& v, int i) { return reinterpret_cast<const T*>(&v)[i]; }

// unit u of a patch -> (cell q, local offset l0 in the cell, patch-tensor node)
template <int D, typename T>
__device__ __forceinline__ void copy_unit(int u, int& q, int& l0, int& node) {
  using C = Cfg<D, T>;
  constexpr int V = row_vec<T>();
  constexpr int CPR = NP / V;                 // chunks per patch row
  const int h = u % CPR, row = u / CPR;       // row = i1 (2D) or i1 + NP i2 (3D)
  const int i0 = h * V, i1 = row % NP, i2 = (D == 3) ? row / NP : 0;
  q = (i0 / NC) + 2 * (i1 / NC) + 4 * (i2 / NC);
  l0 = (i0 % NC) + NC * (i1 % NC) + NC * NC * (i2 % NC);
  node = i0 + i1 * C::RP + i2 * C::PL;
}

// Calls f(p, q, l0, node) for every copy unit of the CTA's patches.  When
// NT is a multiple of the units per patch (the usual case), a thread keeps one
// unit of the patch geometry and only walks the patches.
template <int D, typename T, class Fn>
__device__ __forceinline__ void for_units(int npc, Fn&& f) {
  using C = Cfg<D, T>;
  constexpr int UPP = C::PATCH / row_vec<T>();
  if (C::NT % UPP == 0) {
    int q, l0, node;
    copy_unit<D, T>(threadIdx.x % UPP, q, l0, node);
#pragma unroll
    for (int p = threadIdx.x / UPP; p < C::PPC; p += C::NT / UPP)
      if (p < npc) f(p, q, l0, node);
  } else {
    for (int u = threadIdx.x; u < npc * UPP; u += blockDim.x) {
      int q, l0, node;
      copy_unit<D, T>(u % UPP, q, l0, node);
      f(u / UPP, q, l0, node);
    }
  }
}

// X[p] <- scale * src patch cells (src == nullptr -> zeros)
template <int D, typename T>
__device__ __forceinline__ void load_patches(T* X, const T* __restrict__ src, const PInfo<D>* pis, int npc, T scale) {
  using C = Cfg<D, T>;
  constexpr int V = row_vec<T>();
  using VT = typename VecT<T, V>::type;
  for_units<D, T>(npc, [&](int p, int q, int l0, int node) {
    VT val;
    if (src != nullptr && pis[p].valid) val = __ldg(reinterpret_cast<const VT*>(src + pis[p].coff[q] + l0));
    else val = VT{};
    T* xp = X + p * C::TSZ + node;
#pragma unroll
    for (int v = 0; v < V; ++v) xp[v] = scale * vget<VT, T>(val, v);
  });
}

// dst patch cells <- scale * X[p]  (MODE 1: dst += scale * X;  MODE 2: dst = bm - scale * X)
template <int D, int MODE, typename T>
__device__ __forceinline__ void store_patches(T* __restrict__ dst, const T* X, const PInfo<D>* pis, int npc, T scale,
                                              const T* __restrict__ bm = nullptr) {
  using C = Cfg<D, T>;
  constexpr int V = row_vec<T>();
  using VT = typename VecT<T, V>::type;
  for_units<D, T>(npc, [&](int p, int q, int l0, int node) {
    if (!pis[p].valid) return;
    const T* xp = X + p * C::TSZ + node;
    VT val;
    T* vp = reinterpret_cast<T*>(&val);
#pragma unroll
    for (int v = 0; v < V; ++v) vp[v] = scale * xp[v];
    VT* o = reinterpret_cast<VT*>(dst + pis[p].coff[q] + l0);
    if (MODE == 1) {            // accumulate
      VT old = *o;
#pragma unroll
      for (int v = 0; v < V; ++v) vp[v] += reinterpret_cast<const T*>(&old)[v];
    } else if (MODE == 2) {     // bm - scale X
      VT bb = __ldg(reinterpret_cast<const VT*>(bm + pis[p].coff[q] + l0));
#pragma unroll
      for (int v = 0; v < V; ++v) vp[v] = reinterpret_cast<const T*>(&bb)[v] - vp[v];
    }
    *o = val;
  });
}

// ---------------------------------------------------------------- face terms
// Coupling of a patch to the cells across its 2d outer faces -- the only part
// of the residual that reads outside the patch (domain of
// dependence).  With the neighbour's trace u and normal derivative u' on a face
// of direction a (unit h; jump read as u- - u+, reading A1), the coupling is
//   C x_ext = sum_{a, side} CF_{side,u}(i_a) (x)_{b != a} M_b  U  +  CF_{side,u'}(i_a) (x)_{b != a} M_b  U'
// with, on the low face (cell 0 of the patch), CF_u(i) = -phi_i'(0)/2 - gamma delta_{i0},
// CF_u'(i) = delta_{i0}/2, and on the high face (cell 1) CF_u(i) = phi_i'(1)/2 -
// gamma delta_{i,np-1}, CF_u'(i) = -delta_{i,np-1}/2.
// The traces are computed once per patch into F (all faces), transformed along
// their tangential directions (face_transform) and then injected as rank-one
// updates with compile-time coefficients CF(i_a) inside the line pass of
// direction a (no separate face pass, no atomics).
//
// F layout per patch: [family a][side s][kind u/u'][NFP], NFP tangential points
// (first tangential direction fastest).
template <int D>
__device__ __forceinline__ int fidx(int p, int a, int s, int kind) {
  return ((p * D + a) * 2 + s) * 2 + kind;
}
// element offset of face array (a, s, kind) of patch p (patch pitch FSZ)
template <int D, typename T>
__device__ __forceinline__ int fofs(int p, int a, int s, int kind) {
  using C = Cfg<D, T>;
  return p * C::FSZ + ((a * 2 + s) * 2 + kind) * C::FARR;
}

// position of tangential point t inside a face array
template <int D, typename T>
__device__ __forceinline__ int fpos(int t) {
  using C = Cfg<D, T>;
  return (D == 2) ? t : (t % NP) + (t / NP) * C::FROW;
}

// ---- neighbour staging: cp.async copies of every face-neighbour cell of the
// CTA's patches into shared memory, issued right after setup so that the
// loads overlap the first line passes (consumed only by the last pass).
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (BYTES == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int D, typename T>
__device__ __forceinline__ void stage_neighbors(T* NB, const T* __restrict__ x, const PInfo<D>* pis, int npc) {
  using C = Cfg<D, T>;
  constexpr int EPC = C::CPB / (int)sizeof(T);            // elements per copy
  constexpr int UPC = C::CELL / EPC;                       // copies per cell
  for (int e = threadIdx.x; e < npc * C::NNB * UPC; e += blockDim.x) {
    const int slot = e / UPC, c = e % UPC, p = slot / C::NNB, k = slot % C::NNB;
    const long long nb = pis[p].nb[k >> (D - 1)][k & ((1 << (D - 1)) - 1)];
    if (nb != NO_NB) cp_async<C::CPB>(NB + slot * C::SP + c * EPC, x + nb + c * EPC);
  }
  cp_async_commit();
}

// Traces of the neighbour cells: one work unit computes NC face points (the
// points of one neighbour cell sharing the second tangential index).  It reads
// the NC cell rows that carry them (row = NC contiguous values; for normal
// directions x and y the rows form one contiguous slab) -- from the staged copy
// in shared memory, or from global memory -- and forms u = x(face node) and
// u' = sum_j phi_j'(face) x_j (unit h).
// Transform mode of family a along tangential direction b (the direction the
// family is injected in is a itself, see face_inject): smoother: b < a ->
// S_b^T M (b already in eigen-space), b > a -> M; operator: b < a -> M (the
// mass the earlier pass applied to the volume term), b > a -> none.
// 0 none, 1 mass, 2 S^T M
#ifndef IPMG_SMOOTHER_EIGEN_FACES
#define IPMG_SMOOTHER_EIGEN_FACES 0
#endif
template <bool SMOOTHER>
__host__ __device__ constexpr int face_mode(int a, int b) {
#if IPMG_SMOOTHER_EIGEN_FACES
  return SMOOTHER ? (b < a ? 2 : 1) : (b < a ? 1 : 0);
#else
  // smoother: every face family is kept in physical space (tangential cell masses
  // only) and injected into the right-hand side in the first pass
  return SMOOTHER ? 1 : (b < a ? 1 : 0);
#endif
}
__host__ __device__ constexpr int first_tan(int a) { return a == 0 ? 1 : 0; }
__host__ __device__ constexpr int second_tan(int a) { return a == 2 ? 1 : 2; }

template <typename T>
struct MassC {   // cell mass (NC x NC)
  static __device__ __forceinline__ T get(int i, int j) { return tab<T>().M[j][i]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};
template <int NOUT, int NIN, class A, int R, typename T>
__device__ __forceinline__ void mv(const T (&in)[R][NIN], T (&out)[R][NOUT], const A& mat);
template <int NOUT, int NIN, class A, int R>
__device__ __forceinline__ void mv(const float (&in)[R][NIN], float (&out)[R][NOUT], const A& mat);

template <int D, int A, bool STAGED, bool SMOOTHER, typename T>
__device__ __forceinline__ void trace_unit(T* F, const T* __restrict__ x, const T* NB, const PInfo<D>& pi, int p,
                                           int s, int h, int ic) {
  using C = Cfg<D, T>;
  const TabData<K, T>& tb = tab<T>();
  constexpr int V = row_vec<T>();
  using VT = typename VecT<T, V>::type;
  const int tc = h + ((D == 3 && ic >= NC) ? 2 : 0);
  const long long nb = pi.nb[2 * A + s][tc];
  T u[NC], du[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) u[i] = du[i] = T(0);
  if (nb != NO_NB) {
    // rows: A=0 -> row lb = x_{., lb, lc}; A=1 -> row j = x_{., j, lc}; A=2 -> row j = x_{., lc, j}
    const int lc = ic % NC;
    const int off = (D == 3 ? (A == 2 ? NC * lc : NC * NC * lc) : 0);
    const T* base = STAGED ? NB + (p * C::NNB + (2 * A + s) * (1 << (D - 1)) + tc) * C::SP + off : x + nb + off;
    constexpr int RS = (A == 2) ? NC * NC : NC;       // row stride
    const int jf = (s == 0) ? NC - 1 : 0;             // face node along the normal
#pragma unroll
    for (int rr = 0; rr < NC; ++rr) {
      T row[NC];
#pragma unroll
      for (int c = 0; c < NC / V; ++c) {
        const VT val = STAGED ? reinterpret_cast<const VT*>(base + rr * RS)[c]
                              : __ldg(reinterpret_cast<const VT*>(base + rr * RS) + c);
#pragma unroll
        for (int v = 0; v < V; ++v) row[c * V + v] = vget<VT, T>(val, v);
      }
      if (A == 0) {                                   // row rr is face point lb = rr
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < NC; ++j) acc = fma_(s == 0 ? tb.d1[j] : tb.d0[j], row[j], acc);
        du[rr] = acc;
        u[rr] = (s == 0) ? row[NC - 1] : row[0];
      } else {                                        // row rr is normal index j = rr
        const T dj = (s == 0) ? tb.d1[rr] : tb.d0[rr];
#pragma unroll
        for (int lb = 0; lb < NC; ++lb) du[lb] = fma_(dj, row[lb], du[lb]);
        if (rr == jf) {
#pragma unroll
          for (int lb = 0; lb < NC; ++lb) u[lb] = row[lb];
        }
      }
    }
  }
  if (face_mode<SMOOTHER>(A, first_tan(A)) == 1) {
    // block-diagonal tangential mass along the first tangential direction, in registers
    T in2[2][NC], out2[2][NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      in2[0][i] = u[i];
      in2[1][i] = du[i];
    }
    mv<NC, NC, MassC<T>, 2>(in2, out2, MassC<T>{});
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      u[i] = out2[0][i];
      du[i] = out2[1][i];
    }
  }
  T* fu = F + fofs<D, T>(p, A, s, 0);
  T* fd = F + fofs<D, T>(p, A, s, 1);
#pragma unroll
  for (int lb = 0; lb < NC; ++lb) {
    const int pos = fpos<D, T>(h * NC + lb + NP * ic);
    fu[pos] = u[lb];
    fd[pos] = du[lb];
  }
}

// Split trace unit (two threads per unit, partner lanes u and u ^ 1): thread
// `half` loads the neighbour rows rr = half*CH + i (i < CH) only, so each thread
// keeps half the rows in flight (the unsplit unit holds all NC rows: 128
// registers in fp64 at k = 7) and the lanes that the unsplit phase leaves idle
// (2D: 8 units per patch for 16 line groups) share the load latency.  The
// partial (u, u') vectors are completed with lane shuffles, both partners apply
// the tangential mass to the full vectors, and each writes its half.
template <int D, int A, bool SMOOTHER, typename T>
__device__ __forceinline__ void trace_unit_split(T* F, const T* __restrict__ x, const PInfo<D>& pi, int p, int s,
                                                 int h, int ic, int half, bool act) {
  const TabData<K, T>& tb = tab<T>();
  constexpr int V = row_vec<T>();
  using VT = typename VecT<T, V>::type;
  constexpr int CH = (NC + 1) / 2;
  const int tc = h + ((D == 3 && ic >= NC) ? 2 : 0);
  const long long nb = act ? pi.nb[2 * A + s][tc] : NO_NB;
  // A = 0: own entries rr = half*CH + i in ou/od[i]; A != 0: partial sums over own rows (all lb)
  T ou[NC], od[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) ou[i] = od[i] = T(0);
  if (nb != NO_NB) {
    const int lc = ic % NC;
    const int off = (D == 3 ? (A == 2 ? NC * lc : NC * NC * lc) : 0);
    const T* base = x + nb + off;
    constexpr int RS = (A == 2) ? NC * NC : NC;
    const int jf = (s == 0) ? NC - 1 : 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int rr = half * CH + i;
      if (rr >= NC) break;
      T row[NC];
#pragma unroll
      for (int c = 0; c < NC / V; ++c) {
        const VT val = __ldg(reinterpret_cast<const VT*>(base + rr * RS) + c);
#pragma unroll
        for (int v = 0; v < V; ++v) row[c * V + v] = vget<VT, T>(val, v);
      }
      if (A == 0) {
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < NC; ++j) acc = fma_(s == 0 ? tb.d1[j] : tb.d0[j], row[j], acc);
        od[i] = acc;
        ou[i] = (s == 0) ? row[NC - 1] : row[0];
      } else {
        const T dj = (s == 0) ? tb.d1[rr] : tb.d0[rr];
#pragma unroll
        for (int lb = 0; lb < NC; ++lb) od[lb] = fma_(dj, row[lb], od[lb]);
        if (rr == jf) {
#pragma unroll
          for (int lb = 0; lb < NC; ++lb) ou[lb] = row[lb];
        }
      }
    }
  }
  // the partner pair only: units of different face families diverge
  const unsigned pm = 3u << ((threadIdx.x & 31) & ~1u);
  T u[NC], du[NC];
  if (A == 0) {   // full vectors: lower half from thread 0, upper from thread 1
    T pu[CH], pd[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      pu[i] = __shfl_xor_sync(pm, ou[i], 1);
      pd[i] = __shfl_xor_sync(pm, od[i], 1);
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      u[i] = half ? pu[i] : ou[i];
      du[i] = half ? pd[i] : od[i];
      if (CH + i < NC) {
        u[CH + i] = half ? ou[i] : pu[i];
        du[CH + i] = half ? od[i] : pd[i];
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      u[i] = ou[i] + __shfl_xor_sync(pm, ou[i], 1);
      du[i] = od[i] + __shfl_xor_sync(pm, od[i], 1);
    }
  }
  if (face_mode<SMOOTHER>(A, first_tan(A)) == 1) {
    T in2[2][NC], out2[2][NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      in2[0][i] = u[i];
      in2[1][i] = du[i];
    }
    mv<NC, NC, MassC<T>, 2>(in2, out2, MassC<T>{});
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      u[i] = out2[0][i];
      du[i] = out2[1][i];
    }
  }
  if (!act) return;
  T* fu = F + fofs<D, T>(p, A, s, 0);
  T* fd = F + fofs<D, T>(p, A, s, 1);
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int lb = half * CH + i;
    if (lb >= NC) break;
    const int pos = fpos<D, T>(h * NC + lb + NP * ic);
    fu[pos] = half ? u[CH + i < NC ? CH + i : 0] : u[i];
    fd[pos] = half ? du[CH + i < NC ? CH + i : 0] : du[i];
  }
}

#ifndef IPMG_TRACE_SPLIT
#define IPMG_TRACE_SPLIT 2   // 0 never, 1 always (where the pairs fit one pass), 2 fp64 only
#endif
// threads the trace phase occupies when it is a single pass (0: several passes)
template <int D, typename T>
__host__ __device__ constexpr int trace_threads() {
  using C = Cfg<D, T>;
  constexpr int units = C::PPC * D * 2 * 2 * (D == 3 ? NP : 1);
  constexpr bool split = (IPMG_TRACE_SPLIT == 1 || (IPMG_TRACE_SPLIT == 2 && sizeof(T) == 8)) && !C::STAGE &&
                         2 * units <= C::NT;
  return split ? 2 * units : (units <= C::NT ? units : 0);
}

template <int D, bool STAGED, bool SMOOTHER, typename T>
__device__ __forceinline__ void face_traces(T* F, const T* __restrict__ x, const T* NB, const PInfo<D>* pis, int npc) {
  constexpr int NIC = (D == 3) ? NP : 1;
  constexpr int UPF = 2 * 2 * NIC;                    // units per face family: side x half x ic
  using C = Cfg<D, T>;
  // measured (2D k=7): fp64 operator 0.587 -> 0.497 ms (152 -> 80 registers);
  // the fp32 smoother colour pass 0.265 -> 0.271 ms, so fp32 keeps one thread per unit
  if (!STAGED && trace_threads<D, T>() == 2 * C::PPC * D * UPF) {   // one pass, two threads per unit
    const int e = threadIdx.x >> 1, half = threadIdx.x & 1;
    const bool act = e < npc * D * UPF;
    const int p = act ? e / (D * UPF) : 0, r = e % (D * UPF), a = r / UPF, w = r % UPF;
    const int s = w & 1, h = (w >> 1) & 1, ic = w >> 2;
    if (a == 0) trace_unit_split<D, 0, SMOOTHER>(F, x, pis[p], p, s, h, ic, half, act);
    else if (a == 1) trace_unit_split<D, 1, SMOOTHER>(F, x, pis[p], p, s, h, ic, half, act);
    else trace_unit_split<D, (D == 3 ? 2 : 1), SMOOTHER>(F, x, pis[p], p, s, h, ic, half, act);
    return;
  }
  for (int e = threadIdx.x; e < npc * D * UPF; e += blockDim.x) {
    const int p = e / (D * UPF), r = e % (D * UPF), a = r / UPF, w = r % UPF;
    const int s = w & 1, h = (w >> 1) & 1, ic = w >> 2;
    if (a == 0) trace_unit<D, 0, STAGED, SMOOTHER>(F, x, NB, pis[p], p, s, h, ic);
    else if (a == 1) trace_unit<D, 1, STAGED, SMOOTHER>(F, x, NB, pis[p], p, s, h, ic);
    else trace_unit<D, (D == 3 ? 2 : 1), STAGED, SMOOTHER>(F, x, NB, pis[p], p, s, h, ic);
  }
}

// Face traces of all families (+ tangential transforms) and this thread's rows
// of the first line pass (rows()).  When the trace phase is one pass that leaves
// threads without a unit (2D fp32 k=7: 32 units for 64 threads), those threads
// issue their row loads before the barrier, so the row latency of the idle warp
// overlaps the trace loads instead of waiting at the barrier (IPMG_ROWS_IDLE).
// Measured (tools/ab_kernels.py): fp32 2D k=7 operator 0.303 -> 0.267 ms, residual +
// restriction 0.324 -> 0.291, 3D k=7 0.121 -> 0.095; the smoother loses (2D k=7 colour
// pass 0.265 -> 0.280: 56 -> 68 registers), so it keeps the rows after the barrier.
#ifndef IPMG_ROWS_IDLE
#define IPMG_ROWS_IDLE 1
#endif
#ifndef IPMG_ROWS_IDLE_SMOOTH
#define IPMG_ROWS_IDLE_SMOOTH 0
#endif
template <int D, bool SMOOTHER, typename T>
__device__ __forceinline__ void faces_prepare(T* F, const T* __restrict__ x, const T* NB, const PInfo<D>* pis, int npc);
template <int D, bool SMOOTHER, typename T>
__device__ __forceinline__ void face_transform(T* F, const PInfo<D>* pis, int npc);
template <int D, bool SMOOTHER, typename T, class Rows>
__device__ __forceinline__ void faces_and_rows(T* F, const T* __restrict__ x, const T* NB, const PInfo<D>* pis,
                                               int npc, Rows&& rows) {
  using C = Cfg<D, T>;
  constexpr int TT = trace_threads<D, T>();
  if ((SMOOTHER ? IPMG_ROWS_IDLE_SMOOTH : IPMG_ROWS_IDLE) && !C::STAGE && TT > 0 && TT < C::NT) {
    if ((int)threadIdx.x < TT) face_traces<D, false, SMOOTHER>(F, x, NB, pis, npc);
    else rows();
    __syncthreads();
    face_transform<D, SMOOTHER>(F, pis, npc);
    if ((int)threadIdx.x < TT) rows();
  } else {
    faces_prepare<D, SMOOTHER>(F, x, NB, pis, npc);
    rows();
  }
}

// traces + tangential transforms of all face families, with the staging wait
template <int D, bool SMOOTHER, typename T>
__device__ __forceinline__ void faces_prepare(T* F, const T* __restrict__ x, const T* NB, const PInfo<D>* pis, int npc);

// Tangential transform of the face arrays of family a along tangential
// direction b (see the mode rule below).
template <int V, typename T>
struct SMtM {
  static __device__ __forceinline__ T get(int m, int i) { return tab<T>().MS[V][i][m]; }
  static __device__ __forceinline__ constexpr bool nz(int, int) { return true; }
};

// one face-array line (non-inlined so that the loop around it cannot hoist the
// matrix constants into registers)
template <typename T>
__device__ __noinline__ void face_line(T* base, int stride, int mode, int var) {
  T v[1][NP], w[1][NP];
  load_lines<NP, 1>(base, 0, stride, v);
  if (mode == 1) mv<NP, NP, MassP<T>, 1>(v, w);
  else { IPMG_VAR_SPLIT(var, (mv<NP, NP, SMtM<0, T>, 1>(v, w)), (mv<NP, NP, SMtRT<T>, 1>(v, w, SMtRT<T>{v_}))); }
  store_lines<NP, 1>(base, 0, stride, w);
}

template <int D, bool SMOOTHER, typename T>
__device__ __forceinline__ void face_transform(T* F, const PInfo<D>* pis, int npc) {
  using C = Cfg<D, T>;
  // first tangential direction: only the S^T M transforms are left (mass was fused)
  constexpr bool any1 = SMOOTHER && IPMG_SMOOTHER_EIGEN_FACES;   // S^T M transforms along the first tangential
  if (any1) {
    const int nl = (D == 2) ? 1 : NP;             // lines per array
#pragma unroll 1
    for (int e = threadIdx.x; e < npc * D * 4 * nl; e += blockDim.x) {
      const int o = e % nl, arr = e / nl;         // arr = fidx(p, a, s, kind)
      const int a = (arr / 4) % D, p = arr / (4 * D);
      if (face_mode<SMOOTHER>(a, first_tan(a)) != 2) continue;
      T* base = F + p * C::FSZ + (arr % (4 * D)) * C::FARR + (D == 2 ? 0 : o * C::FROW);
      face_line<T>(base, 1, 2, pis[p].var[first_tan(a)]);
    }
    __syncthreads();
  }
#ifndef IPMG_FACE_LINE_INLINE
#define IPMG_FACE_LINE_INLINE 1
#endif
  if (D == 3 && IPMG_FACE_LINE_INLINE && !any1 && C::PPC * D * 4 * NP <= C::NT) {
    // one pass (a line per thread): the tangential mass inline, no call; modes are
    // 0 (skip) or 1 (block-diagonal mass, compile-time constants) here
    const int e = threadIdx.x;
    if (e < npc * D * 4 * NP) {
      const int o = e % NP, arr = e / NP;
      const int a = (arr / 4) % D, p = arr / (4 * D);
      if (face_mode<SMOOTHER>(a, second_tan(a)) == 1) {
        T* base = F + p * C::FSZ + (arr % (4 * D)) * C::FARR + o;
        T v[1][NP], w[1][NP];
        load_lines<NP, 1>(base, 0, C::FROW, v);
        mv<NP, NP, MassP<T>, 1>(v, w);
        store_lines<NP, 1>(base, 0, C::FROW, w);
      }
    }
    __syncthreads();
  } else if (D == 3) {                            // second tangential direction
#pragma unroll 1
    for (int e = threadIdx.x; e < npc * D * 4 * NP; e += blockDim.x) {
      const int o = e % NP, arr = e / NP;
      const int a = (arr / 4) % D, p = arr / (4 * D);
      const int b = second_tan(a);
      const int mode = face_mode<SMOOTHER>(a, b);
      if (mode == 0) continue;
      T* base = F + p * C::FSZ + (arr % (4 * D)) * C::FARR + o;
      face_line<T>(base, C::FROW, mode, pis[p].var[b]);
    }
    __syncthreads();
  }
}

template <int D, bool SMOOTHER, typename T>
__device__ __forceinline__ void faces_prepare(T* F, const T* __restrict__ x, const T* NB, const PInfo<D>* pis,
                                              int npc) {
  using C = Cfg<D, T>;
  if (C::STAGE) {
    cp_async_wait_all();
    __syncthreads();
    face_traces<D, true, SMOOTHER>(F, x, NB, pis, npc);
  } else {
    face_traces<D, false, SMOOTHER>(F, x, NB, pis, npc);
  }
  __syncthreads();
  face_transform<D, SMOOTHER>(F, pis, npc);
}

// y[r][i] += SGN * sum_{side,kind} CF_{side,kind}(i) G_{side,kind}[t(line r)]:
// the coupling of face family a, added in the line pass of direction a (the
// line's tangential point is t = line index l)
template <int D, int SGN, int R, typename T>
__device__ __forceinline__ void face_inject(T (&y)[R][NP], const T* F, int p, int a, int g) {
  using C = Cfg<D, T>;
  const TabData<K, T>& tb = tab<T>();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int pos = fpos<D, T>(g + r * C::G);
    const T ul = F[fofs<D, T>(p, a, 0, 0) + pos], dl = F[fofs<D, T>(p, a, 0, 1) + pos];
    const T uh = F[fofs<D, T>(p, a, 1, 0) + pos], dh = F[fofs<D, T>(p, a, 1, 1) + pos];
    const T sg = T(SGN);
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      T lo = tb.CF[0][i] * ul;
      if (i == 0) lo = fma_(tb.CF[1][i], dl, lo);
      y[r][i] = fma_(sg, lo, y[r][i]);
      T hi = tb.CF[2][NC + i] * uh;
      if (i == NC - 1) hi = fma_(tb.CF[3][NC + i], dh, hi);
      y[r][NC + i] = fma_(sg, hi, y[r][NC + i]);
    }
  }
}

// Smoother: coupling of the face families a >= 1 subtracted from the right-hand
// side rows of the first (x) pass, in physical space: row (i1[, i2]) gets
// - sum_{side,kind} CF_{side,kind}(i_a) F_{a,side,kind}[x-index j, other tangential index].
// Only the side containing i_a contributes (CF_u is zero on the other cell), and
// the u' kind only on the outermost row.
template <int D, int R, typename T>
__device__ __forceinline__ void face_inject_rows(T (&y)[R][NP], const T* F, int p, int g) {
  using C = Cfg<D, T>;
  const TabData<K, T>& tb = tab<T>();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int l = g + r * C::G;
    const int i1 = (D == 2) ? l : l % NP, i2 = (D == 3) ? l / NP : 0;
#pragma unroll
    for (int a = 1; a < D; ++a) {
      const int ia = a == 1 ? i1 : i2;
      const int s = ia < NC ? 0 : 1;
      const T cu = tb.CF[2 * s][ia], cd = tb.CF[2 * s + 1][ia];
      const int other = (D == 3) ? (a == 1 ? i2 : i1) : 0;       // second tangential index
      const T* fu = F + fofs<D, T>(p, a, s, 0) + other * C::FROW;
      const T* fd = F + fofs<D, T>(p, a, s, 1) + other * C::FROW;
      if (cd != T(0)) {
#pragma unroll
        for (int j = 0; j < NP; ++j) y[r][j] = fma_(-cd, fd[j], fma_(-cu, fu[j], y[r][j]));
      } else {
#pragma unroll
        for (int j = 0; j < NP; ++j) y[r][j] = fma_(-cu, fu[j], y[r][j]);
      }
    }
  }
}

// ---------------------------------------------------------------- line-pass driver
// calls f(p, g, base, gap, stride) for the group of R lines of direction a owned
// by this thread.  Exactly one group per thread (NT >= GROUPS): a loop here
// would let the compiler hoist the loop-invariant matrix constants out of it
// into ~NP^2 ordinary registers.
template <int D, typename T, class Fn>
__device__ __forceinline__ void for_groups(int a, int npc, Fn&& f) {
  using C = Cfg<D, T>;
  static_assert(C::NT >= C::GROUPS, "one line group per thread");
  const int u = threadIdx.x;
  if (u < npc * C::G) {
    const int p = u / C::G, g = u % C::G;
    int base, gap, stride;
    group_geom<D, T>(a, g, base, gap, stride);
    f(p, g, p * C::TSZ + base, gap, stride);
  }
}

// ---------------------------------------------------------------- direct global rows
// The first line pass (x-lines = patch rows) reads its rows straight from
// global memory and the last x-pass writes them straight back: a patch row is
// two cell-row segments of NC contiguous values, so these are full-sector
// vector accesses and no separate global<->shared copy phase is needed.
// Row l: 2D l = i1; 3D l = i1 + NP i2.
template <int D>
__device__ __forceinline__ void row_cells(int l, int& qlo, int& r0) {
  const int i1 = l % NP, i2 = (D == 3) ? l / NP : 0;
  qlo = 2 * (i1 / NC) + 4 * (i2 / NC);
  r0 = NC * (i1 % NC) + NC * NC * (i2 % NC);
}

template <typename T, int V>
__device__ __forceinline__ void load_seg(const T* __restrict__ src, T scale, T* out) {
  using VT = typename VecT<T, V>::type;
#pragma unroll
  for (int c = 0; c < NC / V; ++c) {
    const VT val = __ldg(reinterpret_cast<const VT*>(src) + c);
#pragma unroll
    for (int v = 0; v < V; ++v) out[c * V + v] = scale * vget<VT, T>(val, v);
  }
}
// MODE 0: dst = scale*v; 1: dst += scale*v; 2: dst = bm - scale*v
template <int MODE, typename T, int V>
__device__ __forceinline__ void store_seg(T* __restrict__ dst, const T* __restrict__ bm, T scale, const T* in) {
  using VT = typename VecT<T, V>::type;
#pragma unroll
  for (int c = 0; c < NC / V; ++c) {
    VT val;
    T* vp = reinterpret_cast<T*>(&val);
#pragma unroll
    for (int v = 0; v < V; ++v) vp[v] = scale * in[c * V + v];
    VT* o = reinterpret_cast<VT*>(dst) + c;
    if (MODE == 1) {
      const VT old = *o;
#pragma unroll
      for (int v = 0; v < V; ++v) vp[v] += reinterpret_cast<const T*>(&old)[v];
    } else if (MODE == 2) {
      const VT bb = __ldg(reinterpret_cast<const VT*>(bm) + c);
#pragma unroll
      for (int v = 0; v < V; ++v) vp[v] = reinterpret_cast<const T*>(&bb)[v] - vp[v];
    }
    *o = val;
  }
}

// rows g + r G (r < R) of patch pi from global (zeros if src == nullptr / invalid)
template <int D, int R, typename T>
__device__ __forceinline__ void load_rows(const T* __restrict__ src, const PInfo<D>& pi, int g, T scale,
                                          T (&v)[R][NP]) {
  using C = Cfg<D, T>;
  constexpr int V = row_vec<T>();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (src != nullptr && pi.valid) {
      int qlo, r0;
      row_cells<D>(g + r * C::G, qlo, r0);
      load_seg<T, V>(src + pi.coff[qlo] + r0, scale, &v[r][0]);
      load_seg<T, V>(src + pi.coff[qlo + 1] + r0, scale, &v[r][NC]);
    } else {
#pragma unroll
      for (int j = 0; j < NP; ++j) v[r][j] = T(0);
    }
  }
}
template <int D, int MODE, int R, typename T>
__device__ __forceinline__ void store_rows(T* __restrict__ dst, const T* __restrict__ bm, const PInfo<D>& pi, int g,
                                           T scale, const T (&v)[R][NP]) {
  using C = Cfg<D, T>;
  constexpr int V = row_vec<T>();
  if (!pi.valid) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int qlo, r0;
    row_cells<D>(g + r * C::G, qlo, r0);
    if (!((pi.own >> ((qlo >> (D - 1)) & 1)) & 1)) continue;   // ghost cells of a straddling patch
    store_seg<MODE, T, V>(dst + pi.coff[qlo] + r0, bm ? bm + pi.coff[qlo] + r0 : nullptr, scale, &v[r][0]);
    store_seg<MODE, T, V>(dst + pi.coff[qlo + 1] + r0, bm ? bm + pi.coff[qlo + 1] + r0 : nullptr, scale, &v[r][NC]);
  }
}
// lines of the LAST direction (2D: columns i0 = l; 3D: z-lines (i0, i1) = l) straight to global:
// element j of a line -> cell q(l, j), in-cell offset; per store instruction the
// warp's consecutive lines are consecutive addresses (coalesced)
template <int D, int MODE, int R, typename T>
__device__ __forceinline__ double store_last_lines(T* __restrict__ dst, const T* __restrict__ bm, const PInfo<D>& pi,
                                                   int g, T scale, const T (&v)[R][NP],
                                                   const T* __restrict__ xdot = nullptr) {
  using C = Cfg<D, T>;
  double dot = 0.0;   // sum xdot[o] * stored value (the fused p.q of CG), when xdot != nullptr
  if (!pi.valid) return dot;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int l = g + r * C::G;
    const int i0 = l % NP, i1 = (D == 3) ? l / NP : 0;
    const int qb = (i0 / NC) + (D == 3 ? 2 * (i1 / NC) : 0);           // cell bits of the other directions
    const int ob = (i0 % NC) + (D == 3 ? NC * (i1 % NC) : 0);
    constexpr int QS = (D == 2) ? 2 : 4, SS = (D == 2) ? NC : NC * NC;  // cell step / in-cell stride along the line
    const long long o_lo = pi.coff[qb] + ob, o_hi = pi.coff[qb + QS] + ob;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const long long o = (j < NC ? o_lo : o_hi) + (long long)(j % NC) * SS;
      T val = scale * v[r][j];
      if (MODE == 1) val += dst[o];
      else if (MODE == 2) val = __ldg(bm + o) - val;
      dst[o] = val;
      if (xdot != nullptr) dot = fma((double)__ldg(xdot + o), (double)val, dot);
    }
  }
  return dot;
}

// ---------------------------------------------------------------- volume term
// y = A_jj(unit) x + C x_ext (Kronecker sum with the patch matrices,
// PAPER.md:118-126, plus the face coupling injected in the last pass)
//   2D: y = M1 (L0 x) + L1 (M0 x)                         + C x_ext
//   3D: y = M2 (L1 M0 x + M1 L0 x) + L2 (M1 M0 x)         + C x_ext
// vol_pre: all passes but the last (x-rows come in registers); vol_last: the
// last pass, lines handed to out(p, g, base, gap, stride, y).  X, T1: smem.
template <int D, bool FACES, typename T>
__device__ void vol_pre(T (&xr)[Cfg<D, T>::R][NP], T* X, T* T1, const T* F, const PInfo<D>* pis, int npc) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  for_groups<D, T>(0, npc, [&](int p, int g, int base, int gap, int stride) {
    T w[R][NP];
    mv<NP, NP, MassP<T>, R>(xr, w);
    store_lines<NP, R>(T1 + base, gap, stride, w);
    IPMG_VAR_SPLIT(pis[p].var[0], (mv<NP, NP, LapP<0, T>, R>(xr, w)), (mv<NP, NP, LapRT<T>, R>(xr, w, LapRT<T>{v_})));
    if (FACES) face_inject<D, 1, R>(w, F, p, 0, g);
    store_lines<NP, R>(X + base, gap, stride, w);
  });
  __syncthreads();
  if (D == 3) {
    // y-lines: X <- L1 m0 + M1 l0 (+ y-face coupling) ; T1 <- M1 m0
    for_groups<D, T>(1, npc, [&](int p, int g, int base, int gap, int stride) {
      T m[R][NP], lx[R][NP], y[R][NP];
      load_lines<NP, R>(T1 + base, gap, stride, m);
      load_lines<NP, R>(X + base, gap, stride, lx);
      mv<NP, NP, MassP<T>, R>(lx, y);
      IPMG_VAR_SPLIT(pis[p].var[1], (mv_acc<NP, NP, LapP<0, T>, R>(m, y)), (mv_acc<NP, NP, LapRT<T>, R>(m, y, LapRT<T>{v_})));
      if (FACES) face_inject<D, 1, R>(y, F, p, 1, g);
      store_lines<NP, R>(X + base, gap, stride, y);
      mv<NP, NP, MassP<T>, R>(m, y);
      store_lines<NP, R>(T1 + base, gap, stride, y);
    });
    __syncthreads();
  }
}
template <int D, bool FACES, typename T, class Out>
__device__ void vol_last(T* X, T* T1, const T* F, const PInfo<D>* pis, int npc, Out&& out) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  constexpr int LAST = D - 1;
  for_groups<D, T>(LAST, npc, [&](int p, int g, int base, int gap, int stride) {
    T a[R][NP], bb[R][NP], y[R][NP];
    load_lines<NP, R>(X + base, gap, stride, a);
    mv<NP, NP, MassP<T>, R>(a, y);
#if IPMG_VOL_ORDER
    // a is dead before bb is loaded: two line arrays live instead of three
    // (fp64 2D k=7 vmult: 152 registers, 18 % occupancy)
    asm volatile("" ::: "memory");
#endif
    load_lines<NP, R>(T1 + base, gap, stride, bb);
    IPMG_VAR_SPLIT(pis[p].var[LAST], (mv_acc<NP, NP, LapP<0, T>, R>(bb, y)),
                   (mv_acc<NP, NP, LapRT<T>, R>(bb, y, LapRT<T>{v_})));
    if (FACES) face_inject<D, 1, R>(y, F, p, LAST, g);
    out(p, g, base, gap, stride, y);
  });
}

// ---------------------------------------------------------------- fast diagonalisation
// x = A_jj(unit)^{-1} (rhs - C x_ext) = (x S_a) (sum_a Lambda_a)^{-1} (x S_a^T) (rhs - C x_ext)
// (eq. inverse2d / inverse3d / fast_inverse).  The face
// coupling of face family a is subtracted in the forward pass of direction a,
// with the face arrays transformed into the matching (eigen-)space.
template <int R, typename T, bool kFastOnly = false>
__device__ __forceinline__ void fwd_line(const T (&v)[R][NP], T (&w)[R][NP], int var) {
  IPMG_VAR_SPLIT(var, (eigT_eo<R>(v, w)), (mv<NP, NP, EigTRT<T>, R>(v, w, EigTRT<T>{v_})));
}
template <int R, typename T, bool kFastOnly = false>
__device__ __forceinline__ void bwd_line(const T (&v)[R][NP], T (&w)[R][NP], int var) {
  IPMG_VAR_SPLIT(var, (eig_eo<R>(v, w)), (mv<NP, NP, EigRT<T>, R>(v, w, EigRT<T>{v_})));
}

// S^T, scale by 1/(lsum + lambda_m), S on R lines of the last direction (variant V)
template <int V, int R, typename T>
__device__ __forceinline__ void fd_last(T (&v)[R][NP], T (&w)[R][NP], const T (&lsum)[R], const T (&lact)[R]) {
  static_assert(V == 0, "fast path is the interior variant");
  const TabData<K, T>& tb = tab<T>();
  eigT_eo<R>(v, w);
#pragma unroll
  for (int m = 0; m < NP; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (kDir) w[r][m] *= (lact[r] * tb.act[0][m]) * rcp_(lsum[r] + tb.lam[0][m]);   // exact 0 when inactive
      else w[r][m] *= rcp_(lsum[r] + tb.lam[0][m]);
    }
  eig_eo<R>(w, v);
}
template <int R, typename T>
__device__ __forceinline__ void fd_last_rt(T (&v)[R][NP], T (&w)[R][NP], const T (&lsum)[R], const T (&lact)[R],
                                           int var) {
  const TabData<K, T>& tb = tab<T>();
  mv<NP, NP, EigTRT<T>, R>(v, w, EigTRT<T>{var});
#pragma unroll
  for (int m = 0; m < NP; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (kDir) w[r][m] *= (lact[r] * tb.act[var][m]) * rcp_(lsum[r] + tb.lam[var][m]);
      else w[r][m] *= rcp_(lsum[r] + tb.lam[var][m]);
    }
  mv<NP, NP, EigRT<T>, R>(w, v, EigRT<T>{var});
}

// forward passes of all directions but the last (x-rows from registers);
// face family a is subtracted before the S_a^T of its own pass
template <int D, bool FACES, typename T, bool kFastOnly = false>
__device__ void fd_pre(T (&xr)[Cfg<D, T>::R][NP], T* X, const T* F, const PInfo<D>* pis, int npc) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  for_groups<D, T>(0, npc, [&](int p, int g, int base, int gap, int stride) {
    T w[R][NP];
    if (FACES) face_inject<D, -1, R>(xr, F, p, 0, g);
    if (FACES && !IPMG_SMOOTHER_EIGEN_FACES) face_inject_rows<D, R>(xr, F, p, g);
    fwd_line<R, T, kFastOnly>(xr, w, pis[p].var[0]);
    store_lines<NP, R>(X + base, gap, stride, w);
  });
  __syncthreads();
  if (D == 3) {
    for_groups<D, T>(1, npc, [&](int p, int g, int base, int gap, int stride) {
      T v[R][NP], w[R][NP];
      load_lines<NP, R>(X + base, gap, stride, v);
      if (FACES && IPMG_SMOOTHER_EIGEN_FACES) face_inject<D, -1, R>(v, F, p, 1, g);
      fwd_line<R, T, kFastOnly>(v, w, pis[p].var[1]);
      store_lines<NP, R>(X + base, gap, stride, w);
    });
    __syncthreads();
  }
}
// last direction (faces, S^T, eigenvalue division, S), then the backward
// passes; the x-rows of the result are handed to out(p, g, rows)
template <int D, bool FACES, typename T, bool kFastOnly = false, class Out>
__device__ void fd_post(T* X, const T* F, const PInfo<D>* pis, int npc, Out&& out) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  constexpr int LAST = D - 1;
  const TabData<K, T>& tb = tab<T>();
  for_groups<D, T>(LAST, npc, [&](int p, int g, int base, int gap, int stride) {
    const PInfo<D>& pi = pis[p];
    T lsum[R], lact[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int l = g + r * C::G;           // line id: (m0) in 2D, (m0 + NP m1) in 3D
      lsum[r] = tb.lam[kFastOnly ? 0 : pi.var[0]][l % NP];
      if (D == 3) lsum[r] += tb.lam[kFastOnly ? 0 : pi.var[1]][l / NP];
      lact[r] = T(1);
      if (kDir) {   // Dirichlet: a line through an inactive mode of another direction is zero
        lact[r] = tb.act[pi.var[0]][l % NP];
        if (D == 3) lact[r] *= tb.act[pi.var[1]][l / NP];
      }
    }
    T v[R][NP], w[R][NP];
    load_lines<NP, R>(X + base, gap, stride, v);
    if (FACES && IPMG_SMOOTHER_EIGEN_FACES) face_inject<D, -1, R>(v, F, p, LAST, g);
    IPMG_VAR_SPLIT(pi.var[LAST], (fd_last<0, R>(v, w, lsum, lact)), (fd_last_rt<R>(v, w, lsum, lact, v_)));
    store_lines<NP, R>(X + base, gap, stride, v);
  });
  __syncthreads();
  if (D == 3) {
    for_groups<D, T>(1, npc, [&](int p, int, int base, int gap, int stride) {
      T v[R][NP], w[R][NP];
      load_lines<NP, R>(X + base, gap, stride, v);
      bwd_line<R, T, kFastOnly>(v, w, pis[p].var[1]);
      store_lines<NP, R>(X + base, gap, stride, w);
    });
    __syncthreads();
  }
  for_groups<D, T>(0, npc, [&](int p, int g, int base, int gap, int stride) {
    T v[R][NP], w[R][NP];
    load_lines<NP, R>(X + base, gap, stride, v);
    bwd_line<R, T, kFastOnly>(v, w, pis[p].var[0]);
    out(p, g, w);
  });
}

// ---------------------------------------------------------------- kernels
// ---- b staged by TMA bulk copies (IPMG_TMA_B): one elected thread arms an
// mbarrier with the byte count and issues one cp.async.bulk per patch cell right
// after the setup, so the HBM reads of b overlap the face-trace phase without
// holding registers; the first pass then reads its rows from shared memory.
#ifndef IPMG_TMA_B
#define IPMG_TMA_B 0   // measured: slower (2D k=7 colour pass 0.265 -> 0.329 ms), see DESIGN.md 4.7
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned phase) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(m)), "r"(phase)
                 : "memory");
}
template <int D, typename T>
struct Stage {
  using C = Cfg<D, T>;
  static constexpr bool ALIGNED = (C::CELL * (int)sizeof(T)) % 16 == 0;      // every cell 16-byte aligned
  static constexpr int SPB = ALIGNED ? C::CELL : ((C::CELL * (int)sizeof(T) + 31) / 16 + 1) * 16 / (int)sizeof(T);
  static constexpr int ELEMS = C::PPC * C::NCH * SPB;                        // staging elements per CTA
};
// thread 0: arm the barrier and copy the patch cells of src (valid patches) into BS;
// boff[p*NCH+q]: element offset of the cell inside its slot (16-byte widening)
template <int D, typename T>
__device__ __forceinline__ void stage_cells(T* BS, int* boff, const T* __restrict__ src, const PInfo<D>* pis,
                                            unsigned long long* mbar) {
  using C = Cfg<D, T>;
  using St = Stage<D, T>;
  if (threadIdx.x != 0) return;
  unsigned total = 0;
  for (int p = 0; p < C::PPC; ++p)
    if (pis[p].valid)
      for (int q = 0; q < C::NCH; ++q) {
        const unsigned long long a = (unsigned long long)(src + pis[p].coff[q]);
        const unsigned long long a0 = a & ~15ull, a1 = (a + C::CELL * sizeof(T) + 15) & ~15ull;
        total += (unsigned)(a1 - a0);
      }
  mbar_expect_tx(mbar, total);
  for (int p = 0; p < C::PPC; ++p) {
    if (!pis[p].valid) continue;
    for (int q = 0; q < C::NCH; ++q) {
      const unsigned long long a = (unsigned long long)(src + pis[p].coff[q]);
      const unsigned long long a0 = a & ~15ull, a1 = (a + C::CELL * sizeof(T) + 15) & ~15ull;
      boff[p * C::NCH + q] = (int)((a - a0) / sizeof(T));
      bulk_g2s(BS + (p * C::NCH + q) * St::SPB, (const void*)a0, (unsigned)(a1 - a0), mbar);
    }
  }
}
// rows of this thread's x-pass line group from the staged cells
template <int D, typename T>
__device__ __forceinline__ void my_rows_staged(const T* BS, const int* boff, const PInfo<D>* pis, int npc, T scale,
                                               T (&v)[Cfg<D, T>::R][NP]) {
  using C = Cfg<D, T>;
  using St = Stage<D, T>;
  const int u = threadIdx.x;
  if (u >= npc * C::G) return;
  const int p = u / C::G, g = u % C::G;
#pragma unroll
  for (int r = 0; r < C::R; ++r) {
    if (!pis[p].valid) {
#pragma unroll
      for (int j = 0; j < NP; ++j) v[r][j] = T(0);
      continue;
    }
    int qlo, r0;
    row_cells<D>(g + r * C::G, qlo, r0);
    const T* s0 = BS + (p * C::NCH + qlo) * St::SPB + r0 + (St::ALIGNED ? 0 : boff[p * C::NCH + qlo]);
    const T* s1 = BS + (p * C::NCH + qlo + 1) * St::SPB + r0 + (St::ALIGNED ? 0 : boff[p * C::NCH + qlo + 1]);
    constexpr int V = St::ALIGNED ? row_vec<T>() : 1;
    using VT = typename VecT<T, V>::type;
#pragma unroll
    for (int c = 0; c < NC / V; ++c) {
      const VT a = reinterpret_cast<const VT*>(s0)[c], b = reinterpret_cast<const VT*>(s1)[c];
#pragma unroll
      for (int w = 0; w < V; ++w) {
        v[r][c * V + w] = scale * vget<VT, T>(a, w);
        v[r][NC + c * V + w] = scale * vget<VT, T>(b, w);
      }
    }
  }
}

// rows of this thread's line group (x-pass) loaded from global into registers
template <int D, typename T>
__device__ __forceinline__ void my_rows(const T* __restrict__ src, const PInfo<D>* pis, int npc, T scale,
                                        T (&v)[Cfg<D, T>::R][NP]) {
  using C = Cfg<D, T>;
  const int u = threadIdx.x;
  if (u < npc * C::G) load_rows<D, C::R>(src, pis[u / C::G], u % C::G, scale, v);
}

// y = hs * A x   or, with bminus != nullptr, y = bminus - hs * A x
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D, T>::NT, Cfg<D, T>::MINB_VMULT) vmult_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                              const T* __restrict__ bminus, LevelGeom g,
                                                              double* __restrict__ dot_partial) {
  using C = Cfg<D, T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* T1 = X + C::PPC * C::TSZ;
  T* F = T1 + C::PPC * C::TSZ;   // PPC * FSZ face scratch
  T* NB = F + C::PPC * C::FSZ;   // neighbour staging (C::STAGE)
  __shared__ PInfo<D> pis[C::PPC];
  setup_patches<D, T>(pis, g, 0);
  prefetch_cells<D>(x, pis, C::PPC);
  if (C::STAGE) stage_neighbors<D>(NB, x, pis, C::PPC);
  T xr[C::R][NP];
#ifdef IPMG_ROWS_EARLY
  my_rows<D>(x, pis, C::PPC, T(1), xr);        // in flight while the traces load
#endif
#ifndef IPMG_ROWS_EARLY
  faces_and_rows<D, false>(F, x, NB, pis, C::PPC, [&] { my_rows<D>(x, pis, C::PPC, T(1), xr); });
#else
  faces_prepare<D, false>(F, x, NB, pis, C::PPC);
#endif
  vol_pre<D, true>(xr, X, T1, F, pis, C::PPC);
  const T hs = T(g.hs);
  double dot = 0.0;
  const T* xd = dot_partial ? x : nullptr;
  if (bminus == nullptr)
    vol_last<D, true>(X, T1, F, pis, C::PPC, [&](int p, int gg, int, int, int, const T (&yy)[C::R][NP]) {
      dot += store_last_lines<D, 0, C::R>(y, (const T*)nullptr, pis[p], gg, hs, yy, xd);
    });
  else
    vol_last<D, true>(X, T1, F, pis, C::PPC, [&](int p, int gg, int, int, int, const T (&yy)[C::R][NP]) {
      dot += store_last_lines<D, 2, C::R>(y, bminus, pis[p], gg, hs, yy, xd);
    });
  if (dot_partial != nullptr) {
    // fused x.y (the p.q of CG): deterministic block partial, fixed tree
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    __shared__ double wsum[C::NT / 32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < C::NT / 32; ++w) t += wsum[w];
      const long long bS = slab_block<D>(g);   // full-grid index, also under a split launch
      dot_partial[blockIdx.x + (long long)gridDim.x * (D == 3 ? blockIdx.y + (long long)gridDim.y * bS : bS)] = t;
    }
  }
}

// one colour of the multiplicative full-kernel smoother (replacement form):
// x_out_j = A_jj^{-1} (b_j - C_j x_in) for every patch j of the colour;
// extra CTAs copy the cells the colour does not cover.
// cells a shifted colour does not cover (boundary layers c_a in {0, n_a-1} of
// every shifted direction a) are copied x_out = x_in (zero if x_in == nullptr)
template <int D, typename T>
__device__ __forceinline__ void copy_uncovered_part(const T* __restrict__ x_in, T* __restrict__ x_out, const LevelGeom& g,
                                                    int colour, long long idx0, long long stride0) {
  using C = Cfg<D, T>;
  // 32-bit index math (a boundary layer pair has < 2^31 values)
  const unsigned idx = (unsigned)idx0, stride_all = (unsigned)stride0;
#pragma unroll 1
  for (int a = 0; a < D; ++a) {
    if (!((colour >> a) & 1)) continue;
    // the other directions b0 < b1 (b1 only in 3D)
    const unsigned n0 = (unsigned)(a == 0 ? g.n[1] : g.n[0]), n1 = D == 3 ? (unsigned)(a == 2 ? g.n[1] : g.n[2]) : 1u;
    const unsigned layer = n0 * n1;
    // slowest axis of a slab: only the layers on the global domain boundary are uncovered
    const int s_first = (a == D - 1 && g.zoff != 0) ? 1 : 0;
    const int s_last = (a == D - 1 && g.zoff + g.n[D - 1] != g.nglob) ? 0 : 1;
    if (s_last < s_first) continue;
    const unsigned total = (unsigned)(s_last - s_first + 1) * layer * (unsigned)C::CELL;
    for (unsigned e = idx; e < total; e += stride_all) {
      const unsigned cell = e / (unsigned)C::CELL, l = e % (unsigned)C::CELL;
      const unsigned side = (unsigned)s_first + cell / layer, rem = cell % layer;
      const int na = a == 0 ? g.n[0] : (a == 1 ? g.n[1] : g.n[2]);
      const int ca = side ? na - 1 : 0, u = (int)(rem % n0), v = D == 3 ? (int)(rem / n0) : 0;
      // (a, b0, b1) = (0, 1, 2), (1, 0, 2), (2, 0, 1)
      const int cx = a == 0 ? ca : u;
      const int cy = a == 1 ? ca : (a == 0 ? u : v);
      const int cz = D == 3 ? (a == 2 ? ca : v) : 0;
      const long long o = cell_offset_cells(g, cx, cy, cz) * C::CELL + l;
      x_out[o] = x_in ? __ldg(x_in + o) : T(0);
    }
  }
}
template <int D, typename T>
__global__ void copy_uncovered_kernel(const T* __restrict__ x_in, T* __restrict__ x_out, LevelGeom g, int colour) {
  copy_uncovered_part<D, T>(x_in, x_out, g, colour, (long long)blockIdx.x * blockDim.x + threadIdx.x,
                            (long long)gridDim.x * blockDim.x);
}

// one colour of the multiplicative full-kernel smoother (replacement form):
// x_out_j = A_jj^{-1} (b_j - C_j x_in) for every patch j of the colour.
// (Measured alternatives: a persistent grid of resident CTAs
// with an L2 prefetch of the next block, cp.async staging of the neighbour
// cells, loading the b rows before the traces -- all slower.)
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D, T>::NT, Cfg<D, T>::MINB_SMOOTH)
    smooth_kernel(const T* __restrict__ x_in, const T* __restrict__ b, T* __restrict__ x_out, LevelGeom g, int colour,
                  int nbx) {
  using C = Cfg<D, T>;
  if ((int)blockIdx.x >= nbx) {   // the extra column of CTAs copies the cells the colour does not cover
    const long long q = blockIdx.y + (long long)gridDim.y * blockIdx.z;
    copy_uncovered_part<D, T>(x_in, x_out, g, colour, q * blockDim.x + threadIdx.x,
                              (long long)gridDim.y * gridDim.z * blockDim.x);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* F = X + C::PPC * C::TSZ;
  T* NB = F + C::PPC * C::FSZ;   // neighbour staging (C::STAGE)
  __shared__ PInfo<D> pis[C::PPC];
#if IPMG_TMA_B
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ int boff[C::PPC * C::NCH];
  T* BS = reinterpret_cast<T*>((reinterpret_cast<unsigned long long>(NB + (C::STAGE ? C::NBS : 0)) + 15) & ~15ull);
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
#endif
  setup_patches<D, T>(pis, g, colour);
#if IPMG_TMA_B
  stage_cells<D, T>(BS, boff, b, pis, &mbar);
#else
  prefetch_cells<D>(b, pis, C::PPC);
#endif
  if (x_in != nullptr && C::STAGE) stage_neighbors<D>(NB, x_in, pis, C::PPC);   // lands during fd_pre
  T br[C::R][NP];
#if IPMG_TMA_B
#define IPMG_MY_B_ROWS()                                  \
  do {                                                    \
    mbar_wait(&mbar, 0);                                  \
    my_rows_staged<D>(BS, boff, pis, C::PPC, T(g.hinv), br); \
  } while (0)
#else
#define IPMG_MY_B_ROWS() my_rows<D>(b, pis, C::PPC, T(g.hinv), br)
#endif
#ifdef IPMG_ROWS_EARLY
  my_rows<D>(b, pis, C::PPC, T(g.hinv), br);    // in flight while the traces load
#endif
  auto out = [&](int p, int gg, const T (&w)[C::R][NP]) {
    store_rows<D, 0, C::R>(x_out, (const T*)nullptr, pis[p], gg, T(1), w);
  };
#ifndef IPMG_FAST_BODY
#define IPMG_FAST_BODY 2   // 0 off, 1 always, 2 per (dim, degree) as measured
#endif
  // CTAs whose patches are all interior (variant 0 in every direction; the vast
  // majority) run a copy of the passes without the run-time variant branches
  // (invalid padding patches are never stored, so they do not matter).  Measured
  // smoothing step, fb off -> on (tools/ab_kernels.py): 3D k=4 15.42 -> 14.77 ms,
  // k=5 2.92 -> 2.87; 2D k=5 0.698 -> 0.665, k=3/6/7 -0.7..-1.1 %; slower for 3D
  // k=1,2,3,6,7 (+1..6 %: the doubled code) and 2D k=1,2 (+6..10 %); 2D k=4 neutral
  constexpr bool fast_on = IPMG_FAST_BODY == 1 ||
                           (IPMG_FAST_BODY == 2 && ((D == 2 && (K == 3 || K >= 5)) || (D == 3 && (K == 4 || K == 5))));
  bool allint = fast_on;
#pragma unroll
  for (int p = 0; p < C::PPC; ++p)
    if (pis[p].valid && (pis[p].var[0] | pis[p].var[1] | pis[p].var[2])) allint = false;
  if (allint && x_in != nullptr) {
#if IPMG_TMA_B || defined(IPMG_ROWS_EARLY)
    faces_prepare<D, true>(F, x_in, NB, pis, C::PPC);
    IPMG_MY_B_ROWS();
#else
    faces_and_rows<D, true>(F, x_in, NB, pis, C::PPC, [&] { IPMG_MY_B_ROWS(); });
#endif
    fd_pre<D, true, T, true>(br, X, F, pis, C::PPC);
    fd_post<D, true, T, true>(X, F, pis, C::PPC, out);
  } else if (allint) {
    IPMG_MY_B_ROWS();
    fd_pre<D, false, T, true>(br, X, F, pis, C::PPC);
    fd_post<D, false, T, true>(X, F, pis, C::PPC, out);
  } else if (x_in != nullptr) {
#if IPMG_TMA_B || defined(IPMG_ROWS_EARLY)
    faces_prepare<D, true>(F, x_in, NB, pis, C::PPC);
#ifndef IPMG_ROWS_EARLY   // measured: loading the rows after the traces keeps registers low
    IPMG_MY_B_ROWS();
#endif
#else
    faces_and_rows<D, true>(F, x_in, NB, pis, C::PPC, [&] { IPMG_MY_B_ROWS(); });
#endif
    fd_pre<D, true>(br, X, F, pis, C::PPC);
    fd_post<D, true>(X, F, pis, C::PPC, out);
  } else {
#ifndef IPMG_ROWS_EARLY
    IPMG_MY_B_ROWS();
#endif
    fd_pre<D, false>(br, X, F, pis, C::PPC);
    fd_post<D, false>(X, F, pis, C::PPC, out);
  }
#undef IPMG_MY_B_ROWS
}

// additive Schwarz over one colour: x_j += omega A_jj^{-1} r_j
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D, T>::NT) additive_kernel(const T* __restrict__ r, T* __restrict__ x,
                                                                 LevelGeom g, int colour, T omega) {
  using C = Cfg<D, T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  __shared__ PInfo<D> pis[C::PPC];
  setup_patches<D, T>(pis, g, colour);
  T rr[C::R][NP];
  my_rows<D>(r, pis, C::PPC, T(g.hinv), rr);
  fd_pre<D, false>(rr, X, X, pis, C::PPC);
  fd_post<D, false>(X, X, pis, C::PPC, [&](int p, int gg, const T (&w)[C::R][NP]) {
    store_rows<D, 1, C::R>(x, (const T*)nullptr, pis[p], gg, omega, w);
  });
}

// scale * src gathered along the lines of the LAST direction (the vol_last layout)
template <int D, int R, typename T>
__device__ __forceinline__ void gather_last_lines(const T* __restrict__ src, const PInfo<D>& pi, int g, T scale,
                                                  T (&v)[R][NP]) {
  using C = Cfg<D, T>;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int l = g + r * C::G;
    const int i0 = l % NP, i1 = (D == 3) ? l / NP : 0;
    const int qb = (i0 / NC) + (D == 3 ? 2 * (i1 / NC) : 0);
    const int ob = (i0 % NC) + (D == 3 ? NC * (i1 % NC) : 0);
    constexpr int QS = (D == 2) ? 2 : 4, SS = (D == 2) ? NC : NC * NC;
#pragma unroll
    for (int j = 0; j < NP; ++j)
      v[r][j] = pi.valid ? scale * __ldg(src + (j < NC ? pi.coff[qb] : pi.coff[qb + QS]) + ob + (j % NC) * SS) : T(0);
  }
}

// parent (coarse) cell of the colour-0 patch with lowest fine cell c0 (local):
// along the slowest axis through the global index, so that a replicated coarse
// level (gc.zoff = 0, full size) and a distributed one (gc.zoff = gf.zoff / 2)
// are both addressed correctly
template <int D>
__device__ __forceinline__ long long coarse_cell(const LevelGeom& gf, const LevelGeom& gc, const int (&c0)[3]) {
  constexpr int S = D - 1;
  const int cs = ((gf.zoff + c0[S]) >> 1) - gc.zoff;
  return D == 3 ? cell_offset_cells(gc, c0[0] >> 1, c0[1] >> 1, cs) : cell_offset_cells(gc, c0[0] >> 1, cs, 0);
}

// r_c = P^T (b - hs A x) per parent cell (colour-0 patch); x == nullptr -> P^T b.
// The residual is formed in registers on the lines of the operator's LAST pass
// (b gathered along them, coalesced across the warp) and contracted with P^T
// along that direction before it ever reaches shared memory; the remaining
// directions contract the NC-wide slab (3D: y, then x), and the x-lines write
// whole coarse-cell rows to global memory.
#ifndef IPMG_RESTRICT_MINB
#define IPMG_RESTRICT_MINB 0
#endif
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D, T>::NT, IPMG_RESTRICT_MINB) restrict_kernel(const T* __restrict__ x, const T* __restrict__ b,
                                                                 T* __restrict__ rc, LevelGeom gf, LevelGeom gc) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  constexpr int LAST = D - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* T1 = X + C::PPC * C::TSZ;
  T* F = T1 + C::PPC * C::TSZ;   // PPC * FSZ face scratch
  T* NB = F + C::PPC * C::FSZ;   // neighbour staging (C::STAGE)
  __shared__ PInfo<D> pis[C::PPC];
  setup_patches<D, T>(pis, gf, 0);
  prefetch_cells<D>(b, pis, C::PPC);
  const T hs = T(gf.hs);
  // last direction: r = b - hs (A x) on the line, then P^T along it (NC outputs)
  auto last = [&](int p, int g, int base, int gap, int stride, const T (&yy)[R][NP]) {
    T r[R][NP], w[R][NC];
    gather_last_lines<D, R>(b, pis[p], g, T(1), r);
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int j = 0; j < NP; ++j) r[q][j] = fma_(-hs, yy[q][j], r[q][j]);
    mv<NC, NP, ProlT<T>, R>(r, w);
    store_lines<NC, R>(X + base, gap, stride, w);
  };
  if (x != nullptr) {
    if (C::STAGE) stage_neighbors<D>(NB, x, pis, C::PPC);
    T xr[R][NP];
    faces_and_rows<D, false>(F, x, NB, pis, C::PPC, [&] { my_rows<D>(x, pis, C::PPC, T(1), xr); });
    vol_pre<D, true>(xr, X, T1, F, pis, C::PPC);
    vol_last<D, true>(X, T1, F, pis, C::PPC, last);
  } else {
    T zero[R][NP];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int j = 0; j < NP; ++j) zero[q][j] = T(0);
    for_groups<D, T>(LAST, C::PPC, [&](int p, int g, int base, int gap, int stride) { last(p, g, base, gap, stride, zero); });
  }
  __syncthreads();
  if (D == 3) {   // y-lines (i0, i2 < NC): P^T along y
    for_groups<D, T>(1, C::PPC, [&](int, int g, int base, int gap, int stride) {
      T v[R][NP], w[R][NC];
      load_lines<NP, R>(X + base, gap, stride, v);
      mv<NC, NP, ProlT<T>, R>(v, w);
#pragma unroll
      for (int q = 0; q < R; ++q)
        if ((g + q * C::G) / NP < NC) {
#pragma unroll
          for (int j = 0; j < NC; ++j) X[base + q * gap + j * stride] = w[q][j];
        }
    });
    __syncthreads();
  }
  // x-lines (i1[, i2] < NC): P^T along x, one coarse-cell row straight to global
  for_groups<D, T>(0, C::PPC, [&](int p, int g, int base, int gap, int stride) {
    T v[R][NP], w[R][NC];
    load_lines<NP, R>(X + base, gap, stride, v);
    mv<NC, NP, ProlT<T>, R>(v, w);
    const PInfo<D>& pi = pis[p];
    if (!pi.valid) return;
    const long long cc = coarse_cell<D>(gf, gc, pi.c0) * C::CELL;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int l = g + q * C::G;
      const int i1 = l % NP, i2 = (D == 3) ? l / NP : 0;
      if (i1 < NC && i2 < NC) store_seg<0, T, row_vec<T>()>(rc + cc + NC * i1 + NC * NC * i2, (const T*)nullptr, T(1), &w[q][0]);
    }
  });
}

// x_f += P e_c per parent cell (colour-0 patch).  Expansion order (measured,
// tools/ab_kernels.py): 2D expands the columns first, reading the coarse values
// along y straight from global (coalesced across the warp), and adds the x
// expansion into the fine rows with vector read-modify-writes (2D k=7 0.131 ->
// 0.104 ms); 3D reads whole coarse-cell rows, expands x, y, and adds the z
// expansion line-wise into the fine cells (3D k=4 0.91 -> 0.52 ms).
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D, T>::NT) prolong_kernel(const T* __restrict__ ec, T* __restrict__ xf,
                                                                LevelGeom gf, LevelGeom gc) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  __shared__ PInfo<D> pis[C::PPC];
  setup_patches<D, T>(pis, gf, 0);
  if (D == 2) {
    // columns (i0 < NC) of the coarse cell, P along y
    for_groups<D, T>(1, C::PPC, [&](int p, int g, int base, int gap, int stride) {
      const PInfo<D>& pi = pis[p];
      const long long cc = pi.valid ? coarse_cell<D>(gf, gc, pi.c0) * C::CELL : 0;
      T v[R][NC], w[R][NP];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i0 = g + q * C::G;
        const bool act = pi.valid && i0 < NC;
#pragma unroll
        for (int j = 0; j < NC; ++j) v[q][j] = act ? __ldg(ec + cc + i0 + NC * j) : T(0);
      }
      mv<NP, NC, Prol<T>, R>(v, w);
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (g + q * C::G < NC) {
#pragma unroll
          for (int j = 0; j < NP; ++j) X[base + q * gap + j * stride] = w[q][j];
        }
    });
    __syncthreads();
    // x expansion, added straight into the fine rows
    for_groups<D, T>(0, C::PPC, [&](int p, int g, int base, int gap, int stride) {
      T v[R][NC], w[R][NP];
      load_lines<NC, R>(X + base, gap, stride, v);
      mv<NP, NC, Prol<T>, R>(v, w);
      store_rows<D, 1, R>(xf, (const T*)nullptr, pis[p], g, T(1), w);
    });
  } else {
    // x-lines (i1, i2 < NC): one coarse-cell row from global, P along x
    for_groups<D, T>(0, C::PPC, [&](int p, int g, int base, int gap, int stride) {
      const PInfo<D>& pi = pis[p];
      const long long cc = pi.valid ? coarse_cell<D>(gf, gc, pi.c0) * C::CELL : 0;
      T v[R][NC], w[R][NP];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int l = g + q * C::G;
        const int i1 = l % NP, i2 = l / NP;
        if (pi.valid && i1 < NC && i2 < NC) load_seg<T, row_vec<T>()>(ec + cc + NC * i1 + NC * NC * i2, T(1), &v[q][0]);
        else {
#pragma unroll
          for (int j = 0; j < NC; ++j) v[q][j] = T(0);
        }
      }
      mv<NP, NC, Prol<T>, R>(v, w);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int l = g + q * C::G;
        if (l % NP < NC && l / NP < NC) {
#pragma unroll
          for (int j = 0; j < NP; ++j) X[base + q * gap + j * stride] = w[q][j];
        }
      }
    });
    __syncthreads();
    // y-lines (i0, i2 < NC): P along y
    for_groups<D, T>(1, C::PPC, [&](int, int g, int base, int gap, int stride) {
      T v[R][NC], w[R][NP];
      load_lines<NC, R>(X + base, gap, stride, v);
      mv<NP, NC, Prol<T>, R>(v, w);
#pragma unroll
      for (int q = 0; q < R; ++q)
        if ((g + q * C::G) / NP < NC) {
#pragma unroll
          for (int j = 0; j < NP; ++j) X[base + q * gap + j * stride] = w[q][j];
        }
    });
    __syncthreads();
    // z-lines: P along z, added into the fine cells
    for_groups<D, T>(2, C::PPC, [&](int p, int g, int base, int gap, int stride) {
      T v[R][NC], w[R][NP];
      load_lines<NC, R>(X + base, gap, stride, v);
      mv<NP, NC, Prol<T>, R>(v, w);
      store_last_lines<D, 1, R>(xf, (const T*)nullptr, pis[p], g, T(1), w);
    });
  }
}

// ---------------------------------------------------------------- host side
template <int D, typename T>
constexpr size_t smem_bytes(int ntensors, bool faces) {
  using C = Cfg<D, T>;
  return sizeof(T) * ((size_t)ntensors * C::PPC * C::TSZ +
                      (faces ? (size_t)C::PPC * C::FSZ + (C::STAGE ? (size_t)C::NBS : 0) : 0));
}

// cudaFuncSetAttribute once per (kernel, device, size): it is a host API call
// that would otherwise be paid on every launch of the V-cycle
template <typename F>
inline cudaError_t set_smem(F* f, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, long long>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const long long key = ((long long)dev << 40) | (long long)bytes;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == (const void*)f && d.second == key) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.emplace_back((const void*)f, key);
  return e;
}

// grid over the colour's patch lattice: (x-blocks of PPC patches, j1, j2)
template <int D, typename T>
inline dim3 patch_grid(LevelGeom& g, int colour) {   // also sets g.znb (full count along the slowest axis)
  using C = Cfg<D, T>;
  const int m0 = g.n[0] / 2 - (colour & 1);
  int m1 = (D == 3) ? g.n[1] / 2 - ((colour >> 1) & 1) : slab_patches(g, 1, (colour >> 1) & 1);
  int m2 = (D == 3) ? slab_patches(g, 2, (colour >> 2) & 1) : 1;
  int& mS = D == 3 ? m2 : m1;
  mS = mS > 0 ? mS : 0;
  g.znb = mS;
  mS = slab_sel_count(mS, g.zsel);
  return dim3((unsigned)((m0 + C::PPC - 1) / C::PPC), (unsigned)(m1 > 0 ? m1 : 0), (unsigned)(m2 > 0 ? m2 : 0));
}

#if !IPMG_DIRICHLET
#include "smooth_pair3.cuh"
#include "op3.cuh"
// 3D fp64 operator through the staged kernel (op3.cuh): bit k of IPMG_OP3_DEGREES enables
// degree k (as measured); IPMG_OP3=0/1 in the environment forces it off / on (A/B runs)
#ifndef IPMG_OP3_DEGREES
#define IPMG_OP3_DEGREES 0x7c   // k = 2..6 (tools/gpu_deg_ab.sh: k = 7 slower, 2.30 vs 1.68 ms)
#endif
inline bool op3_enabled() {
  static const int env = [] {
    const char* e = std::getenv("IPMG_OP3");
    return e ? std::atoi(e) : -1;
  }();
  return env >= 0 ? env != 0 : ((IPMG_OP3_DEGREES >> K) & 1) != 0;
}
inline bool op3_applies(const LevelGeom& g) {
  return op3_enabled() && g.grouped && g.n[0] >= 2 && g.n[1] >= 2 && g.n[2] >= 2 && (g.n[0] % 2) == 0 &&
         (g.n[1] % 2) == 0;
}
inline pair3::Deltas pair3_deltas(const LevelGeom& g, int colour);
// the copies are widened to 16-byte granularity: x 16-byte aligned, and an even cell count
// (the widened copy of the last cell ends inside the vector; ghost layers hold an even count)
template <typename T>
inline cudaError_t launch_op3(const void* x, void* y, const LevelGeom& g, const void* bm, double* dotp,
                              long long* nparts, cudaStream_t s) {
  LevelGeom gg = g;
  const int gx = g.n[0] / 2, gy = g.n[1] / 2;
  int gz = slab_patches(g, 2, 0);
  gz = gz > 0 ? gz : 0;
  gg.znb = gz;
  gz = slab_sel_count(gz, g.zsel);
  if (nparts) *nparts = (long long)gx * gy * gg.znb;   // full grid
  if (x == nullptr) return cudaSuccess;               // size query
  if ((reinterpret_cast<unsigned long long>(x) & 15) != 0 || (g.ncells % (16 / (long long)sizeof(T))) != 0)
    return cudaErrorNotReady;
  cudaError_t e = set_smem(op3::op3_kernel<T, 0>, op3::Lay<T>::SMEM);
  if (e != cudaSuccess) return e;
  if ((long long)gx * gy * gz == 0) return cudaSuccess;
  constexpr int TY = op3::TY;
  const dim3 grid((unsigned)gx, (unsigned)(TY * gz), (unsigned)((gy + TY - 1) / TY));
  op3::op3_kernel<T, 0><<<grid, op3::NT, op3::Lay<T>::SMEM, s>>>((const T*)x, (T*)y, (const T*)bm, gg, gx, gy,
                                                                pair3_deltas(g, 0), dotp, gg);
  return cudaGetLastError();
}
#endif

template <int D, typename T>
cudaError_t launch_vmult(const void* x, void* y, const LevelGeom& g, const void* bm, double* dotp, long long* nparts,
                         cudaStream_t s) {
  using C = Cfg<D, T>;
#if !IPMG_DIRICHLET
#ifndef IPMG_OP3_VMULT32
#define IPMG_OP3_VMULT32 0x70   // degrees whose fp32 operator also takes op3 (tools/gpu_deg_key.sh, C3 sizes:
                                // k = 4 0.830 -> 0.711, k = 5 0.608 -> 0.561, k = 6 0.656 -> 0.586 ms;
                                // k = 3 slower, 0.601 -> 0.642)
#endif
  if constexpr (D == 3) {
    if (op3_applies(g) && (sizeof(T) == 8 || ((IPMG_OP3_VMULT32 >> K) & 1))) {
      const cudaError_t e = launch_op3<T>(x, y, g, bm, dotp, nparts, s);
      if (e != cudaErrorNotReady) return e;
    }
  }
#endif
  LevelGeom gg = g;
  const dim3 grid = patch_grid<D, T>(gg, 0);
  if (nparts) *nparts = (long long)grid.x * (D == 3 ? (long long)grid.y * gg.znb : gg.znb);   // full grid
  if (x == nullptr) return cudaSuccess;   // size query
  const size_t sm = smem_bytes<D, T>(2, true);
  cudaError_t e = set_smem(vmult_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  if (grid.x * grid.y * grid.z == 0) return cudaSuccess;
  vmult_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)x, (T*)y, (const T*)bm, gg, dotp);
  return cudaGetLastError();
}

#if !IPMG_DIRICHLET
// 3D fp32 colour passes through the patch-pair kernel (smooth_pair3.cuh): bit k of
// IPMG_PAIR3_DEGREES enables degree k (as measured); IPMG_PAIR3=0/1 in the
// environment forces it off / on for every degree (A/B runs)
#ifndef IPMG_PAIR3_DEGREES
#define IPMG_PAIR3_DEGREES 0x54   // k = 2, 4, 6 (tools/gpu_deg_ab.sh: k = 3, 5, 7 slower)
#endif
#ifndef IPMG_PAIR3_NPAIR
#define IPMG_PAIR3_NPAIR 1
#endif
inline bool pair3_enabled() {
  static const int env = [] {
    const char* e = std::getenv("IPMG_PAIR3");
    return e ? std::atoi(e) : -1;
  }();
  return env >= 0 ? env != 0 : ((IPMG_PAIR3_DEGREES >> K) & 1) != 0;
}
// Thread -> line tables of the y and z passes: the lines of every pass, sorted by the
// bank of their first element, are dealt round robin to the half warps, so a half
// warp holds distinct banks whenever no bank class has more lines than there are
// half warps (64-bit accesses are served per half warp).
inline cudaError_t pair3_upload_tables() {
  using namespace pair3;
  static unsigned tab[3][2][NTMAX];
  auto fill = [&](auto npc) {
    constexpr int NPAIR = decltype(npc)::value;
    constexpr int NT = PC<NPAIR>::NT, HW = NT / 16;
    for (int d = 0; d < 2; ++d) {
      std::vector<std::pair<int, int>> items;   // (bank, line id)
      for (int q = 0; q < NPAIR; ++q)
        for (int v = 0; v < NP; ++v)
          for (int u = 0; u < NP; ++u) {
            const int base = q * TSZ + u + (d == 0 ? S2 : S1) * v;
            items.emplace_back(base % 16, q * NL + u + NP * v);
          }
      std::stable_sort(items.begin(), items.end(),
                       [](const std::pair<int, int>& a, const std::pair<int, int>& b) { return a.first < b.first; });
      for (int t = 0; t < NTMAX; ++t) tab[NPAIR - 1][d][t] = 0xffffffffu;
      for (int k = 0; k < (int)items.size(); ++k) {
        const int id = items[k].second, q = id / NL, l = id % NL, u = l % NP, v = l / NP;
        const unsigned ofs = (unsigned)(q * TSZ + u + (d == 0 ? S2 : S1) * v);
        tab[NPAIR - 1][d][16 * (k % HW) + k / HW] =
            d == 0 ? ofs : (ofs | (unsigned)u << 16 | (unsigned)v << 20 | (unsigned)q << 24);
      }
    }
  };
  fill(std::integral_constant<int, 1>{});
  fill(std::integral_constant<int, 2>{});
  fill(std::integral_constant<int, 3>{});
  return cudaMemcpyToSymbol(pair3::g_lines, tab, sizeof(tab));
}
// cell-index deltas of a launch in the parent-grouped layout: a cell (c0 + d) of a patch
// whose lowest cell c0 has the colour's parities lies at cell(c0) + delta(d)
inline pair3::Deltas pair3_deltas(const LevelGeom& g, int colour) {
  pair3::Deltas d{};
  const int PX = g.n[0] / 2, PY = g.n[1] / 2;
  const int par[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
  auto delta = [&](int dx, int dy, int dz) {
    const int dd[3] = {dx, dy, dz};
    int f[3], r[3];
    for (int a = 0; a < 3; ++a) {
      const int v = par[a] + dd[a];
      f[a] = v >= 0 ? v / 2 : -((1 - v) / 2);   // floor(v / 2)
      r[a] = v - 2 * f[a];
    }
    return 8 * (f[0] + PX * (f[1] + PY * f[2])) + (r[0] - par[0]) + 2 * (r[1] - par[1]) + 4 * (r[2] - par[2]);
  };
  for (int q = 0; q < 8; ++q) d.pc[q] = delta(q & 1, (q >> 1) & 1, (q >> 2) & 1);
  for (int k = 0; k < pair3::NNB; ++k) {
    const int a = k >> 3, sd = (k >> 2) & 1, tc = k & 3;
    const int sa = sd == 0 ? -1 : 2, t0 = tc & 1, t1 = (tc >> 1) & 1;
    d.nb[k] = a == 0 ? delta(sa, t0, t1) : (a == 1 ? delta(t0, sa, t1) : delta(t0, t1, sa));
  }
  return d;
}
template <int NPAIR>
cudaError_t launch_smooth_pair3(const void* xi, const void* b, void* xo, const LevelGeom& g, int colour, cudaStream_t s,
                                const double* rdot = nullptr, double* dotp = nullptr, long long* nparts = nullptr) {
  using C = pair3::PC<NPAIR>;
  LevelGeom gg = g;
  const int m0 = g.n[0] / 2 - (colour & 1);
  const int m1 = g.n[1] / 2 - ((colour >> 1) & 1);
  int m2 = slab_patches(g, 2, (colour >> 2) & 1);
  m2 = m2 > 0 ? m2 : 0;
  gg.znb = m2;
  m2 = slab_sel_count(m2, g.zsel);
  const int gx = (m0 + C::NPAT - 1) / C::NPAT, gy = m1 > 0 ? m1 : 0, gz = m2;
  if ((long long)gx * gy * gz == 0) return cudaErrorNotReady;   // empty patch lattice: the caller copies
  cudaError_t e = dotp ? set_smem(pair3::smooth_pair3_kernel<NPAIR, true, true>, C::SMEM)
                       : (xi ? set_smem(pair3::smooth_pair3_kernel<NPAIR, false, true>, C::SMEM)
                             : set_smem(pair3::smooth_pair3_kernel<NPAIR, false, false>, C::XB));
  if (e != cudaSuccess) return e;
  constexpr int TY = pair3::TY;
  const dim3 grid((unsigned)(gx + (colour != 0 && g.zsel != 2 ? 1 : 0)), (unsigned)(TY * gz), (unsigned)((gy + TY - 1) / TY));
  if (nparts) *nparts = (long long)gx * gy * gg.znb;   // fused r.z partials (full lattice)
  // a zero-start pass (xi == nullptr) has no neighbour staging and no face arrays: X only
  if (dotp)
    pair3::smooth_pair3_kernel<NPAIR, true, true><<<grid, C::NT, C::SMEM, s>>>(
        (const float*)xi, (const float*)b, (float*)xo, gg, colour, gx, gy, pair3_deltas(g, colour), rdot, dotp);
  else if (xi)
    pair3::smooth_pair3_kernel<NPAIR, false, true><<<grid, C::NT, C::SMEM, s>>>(
        (const float*)xi, (const float*)b, (float*)xo, gg, colour, gx, gy, pair3_deltas(g, colour), nullptr, nullptr);
  else
    pair3::smooth_pair3_kernel<NPAIR, false, false><<<grid, C::NT, C::XB, s>>>(
        (const float*)xi, (const float*)b, (float*)xo, gg, colour, gx, gy, pair3_deltas(g, colour), nullptr, nullptr);
  return cudaGetLastError();
}
#endif

template <int D, typename T>
cudaError_t launch_smooth(const void* xi, const void* b, void* xo, const LevelGeom& g, int colour, cudaStream_t s) {
  using C = Cfg<D, T>;
#if !IPMG_DIRICHLET
  // the pair kernel's TMA copies need a 16-byte aligned x_in whose cell range ends on a
  // 16-byte boundary (the copies are widened to 16-byte granularity)
#ifndef IPMG_PAIR3_ZERO
#define IPMG_PAIR3_ZERO 0x10   // degrees whose zero-start passes (x_in == nullptr) also take the pair
                               // kernel (its FACES = false instantiation, 56 registers, X-only shared
                               // memory): 3D k=4 colour 0 from zero 0.839 -> 0.774 ms
#endif
  if (D == 3 && sizeof(T) == 4 && (xi != nullptr || ((IPMG_PAIR3_ZERO >> K) & 1)) && pair3_enabled() && g.grouped &&
      g.n[0] >= 2 && g.n[1] >= 2 && g.n[2] >= 2 &&
      (reinterpret_cast<unsigned long long>(xi) & 15) == 0 && (g.ncells % 4) == 0 &&
      (reinterpret_cast<unsigned long long>(xo) & 3) == 0) {
    const cudaError_t e = launch_smooth_pair3<IPMG_PAIR3_NPAIR>(xi, b, xo, g, colour, s);
    if (e != cudaErrorNotReady) return e;
  }
#endif
  LevelGeom gg = g;
  const dim3 grid = patch_grid<D, T>(gg, colour);
  // no neighbour staging (and less shared memory, more CTAs) when x_in == 0
  const size_t stg = IPMG_TMA_B ? sizeof(T) * (size_t)Stage<D, T>::ELEMS + 16 : 0;   // + alignment slack
  const size_t sm = (xi ? smem_bytes<D, T>(1, true) : smem_bytes<D, T>(1, false) + sizeof(T) * C::PPC * C::FSZ) + stg;
  cudaError_t e = set_smem(smooth_kernel<D, T>, smem_bytes<D, T>(1, true) + stg);
  if (e != cudaSuccess) return e;
  if (grid.x * grid.y * grid.z > 0) {
    // shifted colours: one extra column of CTAs copies the uncovered boundary layers
    const dim3 g2(grid.x + (colour != 0 && g.zsel != 2 ? 1 : 0), grid.y, grid.z);
    smooth_kernel<D, T><<<g2, C::NT, sm, s>>>((const T*)xi, (const T*)b, (T*)xo, gg, colour, (int)grid.x);
    return cudaGetLastError();
  }
  if (colour != 0 && g.zsel != 2) {   // empty patch lattice (tiny level / no interior blocks): copy only
    long long cells = 0;
    for (int a = 0; a < D; ++a) {
      if (!((colour >> a) & 1)) continue;
      long long layer = 1;
      for (int bb = 0; bb < D; ++bb) if (bb != a) layer *= g.n[bb];
      cells += 2 * layer;
    }
    const long long elems = cells * C::CELL;
    long long blocks = (elems + 255) / 256;
    if (blocks > 4 * 148) blocks = 4 * 148;
    if (blocks < 1) blocks = 1;
    copy_uncovered_kernel<D, T><<<(unsigned)blocks, 256, 0, s>>>((const T*)xi, (T*)xo, gg, colour);
    e = cudaGetLastError();
  }
  return e;
}

template <int D, typename T>
cudaError_t launch_additive(const void* r, void* x, const LevelGeom& g, int colour, double omega, cudaStream_t s) {
  using C = Cfg<D, T>;
  LevelGeom gg = g;
  const dim3 grid = patch_grid<D, T>(gg, colour);
  if (grid.x * grid.y * grid.z == 0) return cudaSuccess;
  const size_t sm = smem_bytes<D, T>(1, false);
  cudaError_t e = set_smem(additive_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  additive_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)r, (T*)x, gg, colour, (T)omega);
  return cudaGetLastError();
}

template <int D, typename T>
cudaError_t launch_restrict(const void* x, const void* b, void* rc, const LevelGeom& gf, const LevelGeom& gc,
                            cudaStream_t s) {
  using C = Cfg<D, T>;
#if !IPMG_DIRICHLET
#ifndef IPMG_OP3_RESTRICT
#define IPMG_OP3_RESTRICT 1   // 1: the residual + restriction through the staged operator (op3, MODE 1)
#endif
#ifndef IPMG_OP3_RESTRICT32_DEGREES
#define IPMG_OP3_RESTRICT32_DEGREES 0x78   // fp32: k = 3..6 (tools/gpu_deg_restrict.sh: k = 2 3 % slower,
                                           // k = 4 0.95 -> 0.71 ms); fp64: every op3 degree (all faster)
#endif
  if constexpr (D == 3) {
    if (IPMG_OP3_RESTRICT && x != nullptr && op3_applies(gf) &&
        (sizeof(T) == 8 || ((IPMG_OP3_RESTRICT32_DEGREES >> K) & 1)) && (reinterpret_cast<unsigned long long>(x) & 15) == 0 &&
        (gf.ncells % (16 / (long long)sizeof(T))) == 0) {
      LevelGeom gg = gf;
      const int gx = gf.n[0] / 2, gy = gf.n[1] / 2;
      int gz = slab_patches(gf, 2, 0);
      gz = gz > 0 ? gz : 0;
      gg.znb = gz;
      gz = slab_sel_count(gz, gf.zsel);
      if ((long long)gx * gy * gz == 0) return cudaSuccess;
      cudaError_t e = set_smem(op3::op3_kernel<T, 1>, op3::Lay<T>::SMEM);
      if (e != cudaSuccess) return e;
      constexpr int TY = op3::TY;
      const dim3 grid((unsigned)gx, (unsigned)(TY * gz), (unsigned)((gy + TY - 1) / TY));
      op3::op3_kernel<T, 1><<<grid, op3::NT, op3::Lay<T>::SMEM, s>>>((const T*)x, (T*)rc, (const T*)b, gg, gx, gy,
                                                                    pair3_deltas(gf, 0), nullptr, gc);
      return cudaGetLastError();
    }
  }
#endif
  LevelGeom gg = gf;
  const dim3 grid = patch_grid<D, T>(gg, 0);
  if (grid.x * grid.y * grid.z == 0) return cudaSuccess;
  const size_t sm = smem_bytes<D, T>(2, true);
  cudaError_t e = set_smem(restrict_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  restrict_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)x, (const T*)b, (T*)rc, gg, gc);
  return cudaGetLastError();
}

template <int D, typename T>
cudaError_t launch_prolong(const void* ec, void* xf, const LevelGeom& gf, const LevelGeom& gc, cudaStream_t s) {
  using C = Cfg<D, T>;
  LevelGeom gg = gf;
  const dim3 grid = patch_grid<D, T>(gg, 0);
  if (grid.x * grid.y * grid.z == 0) return cudaSuccess;
  const size_t sm = smem_bytes<D, T>(1, false);
  cudaError_t e = set_smem(prolong_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  prolong_kernel<D, T><<<grid, C::NT, sm, s>>>((const T*)ec, (T*)xf, gg, gc);
  return cudaGetLastError();
}

#if IPMG_DIRICHLET
// ---------------------------------------------------------------- Dirichlet kernel (NEXT-1)
// One colour of Algorithm 1 with the Dirichlet kernel (reading
// A20): per patch j, r = hinv b - A~ x_patch with A~ the patch operator without
// its mesh-interior outer faces (only the patch's own cells are read -- the
// domain of dependence of the continuous method), delta = A_jj^{-1} r on V_j
// (outer nodes at mesh-interior faces dropped: inactive modes of the padded
// eigenbasis), x_out = x_in + delta on the patch cells.  The extra CTA column
// copies the cells the colour does not cover.
template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D, T>::NT)
    smooth_dir_kernel(const T* __restrict__ x_in, const T* __restrict__ b, T* __restrict__ x_out, LevelGeom g,
                      int colour, int nbx) {
  using C = Cfg<D, T>;
  constexpr int R = C::R;
  if ((int)blockIdx.x >= nbx) {
    const long long q = blockIdx.y + (long long)gridDim.y * blockIdx.z;
    copy_uncovered_part<D, T>(x_in, x_out, g, colour, q * blockDim.x + threadIdx.x,
                              (long long)gridDim.y * gridDim.z * blockDim.x);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* T1 = X + C::PPC * C::TSZ;
  __shared__ PInfo<D> pis[C::PPC];
  setup_patches<D, T>(pis, g, colour);
  T xr[R][NP];
  my_rows<D>(x_in, pis, C::PPC, T(1), xr);   // zeros when x_in == nullptr
  vol_pre<D, false>(xr, X, T1, (const T*)nullptr, pis, C::PPC);
  const T hinv = T(g.hinv);
  vol_last<D, false>(X, T1, (const T*)nullptr, pis, C::PPC,
                     [&](int p, int gg, int base, int gap, int stride, const T (&yy)[R][NP]) {
                       T rr[R][NP];
                       gather_last_lines<D, R>(b, pis[p], gg, hinv, rr);
#pragma unroll
                       for (int r = 0; r < R; ++r)
#pragma unroll
                         for (int j = 0; j < NP; ++j) rr[r][j] -= yy[r][j];
                       store_lines<NP, R>(X + base, gap, stride, rr);
                     });
  __syncthreads();
  T r0[R][NP];
  for_groups<D, T>(0, C::PPC, [&](int, int, int base, int gap, int stride) { load_lines<NP, R>(X + base, gap, stride, r0); });
  fd_pre<D, false>(r0, X, (const T*)nullptr, pis, C::PPC);
  if (x_in != nullptr)
    fd_post<D, false>(X, (const T*)nullptr, pis, C::PPC, [&](int p, int gg, const T (&w)[R][NP]) {
      store_rows<D, 2, R>(x_out, x_in, pis[p], gg, T(-1), w);   // x_in + delta
    });
  else
    fd_post<D, false>(X, (const T*)nullptr, pis, C::PPC, [&](int p, int gg, const T (&w)[R][NP]) {
      store_rows<D, 0, R>(x_out, (const T*)nullptr, pis[p], gg, T(1), w);
    });
}

template <int D, typename T>
cudaError_t launch_smooth_dir(const void* xi, const void* b, void* xo, const LevelGeom& g, int colour, cudaStream_t s) {
  using C = Cfg<D, T>;
  LevelGeom gg = g;
  const dim3 grid = patch_grid<D, T>(gg, colour);
  const size_t sm = smem_bytes<D, T>(2, false);
  cudaError_t e = set_smem(smooth_dir_kernel<D, T>, sm);
  if (e != cudaSuccess) return e;
  if (grid.x * grid.y * grid.z > 0) {
    const dim3 g2(grid.x + (colour != 0 && g.zsel != 2 ? 1 : 0), grid.y, grid.z);
    smooth_dir_kernel<D, T><<<g2, C::NT, sm, s>>>((const T*)xi, (const T*)b, (T*)xo, gg, colour, (int)grid.x);
    return cudaGetLastError();
  }
  if (colour != 0 && g.zsel != 2) {
    copy_uncovered_kernel<D, T><<<4 * 148, 256, 0, s>>>((const T*)xi, (T*)xo, gg, colour);
    e = cudaGetLastError();
  }
  return e;
}
#endif

// runtime (dim, prec) dispatch
#define IPMG_DISPATCH(dim, prec, FN, ...)                                               \
  ((dim) == 2 ? ((prec) == 0 ? FN<2, double>(__VA_ARGS__) : FN<2, float>(__VA_ARGS__)) \
              : ((prec) == 0 ? FN<3, double>(__VA_ARGS__) : FN<3, float>(__VA_ARGS__)))

// host copy of the tables in the exact device layout
template <typename T>
void fill_tab(TabData<K, T>& t, const FE1D& fe) {
  std::memset(&t, 0, sizeof(t));
  for (int i = 0; i < NC; ++i)
    for (int j = 0; j < NC; ++j) t.M[i][j] = (T)fe.M[i * NC + j];
  for (int v = 0; v < 4; ++v) {
    // Dirichlet TUs: residual operator without the mesh-interior outer faces and
    // the padded local eigenbasis with its activity flags (fe1d.cpp, reading A20)
    const std::vector<double>& LPv = kDir ? fe.LPR[v] : fe.LP[v];
    const std::vector<double>& Sv = kDir ? fe.SD[v] : fe.S[v];
    for (int i = 0; i < NP; ++i)
      for (int j = 0; j < NP; ++j) {
        t.LP[v][i][j] = (T)LPv[i * NP + j];
        t.S[v][i][j] = (T)Sv[i * NP + j];
        t.ST[v][j][i] = (T)Sv[i * NP + j];
        if (v == 0 && j >= NP / 2) t.SO[i][j - NP / 2] = (T)Sv[i * NP + j];
      }
    for (int i = 0; i < NP; ++i) {
      t.lam[v][i] = (T)(kDir ? fe.lamD[v][i] : fe.lam[v][i]);
      t.act[v][i] = (T)(kDir ? fe.actD[v][i] : 1.0);
    }
  }
  for (int v = 0; v < 4; ++v)
    for (int i = 0; i < NP; ++i)
      for (int m = 0; m < NP; ++m) {
        double acc = 0.0;   // (M^P S)[i][m] = sum_j M^P[i][j] S[j][m] = ((S^T M^P)^T)[i][m]
        for (int j = 0; j < NP; ++j) acc += fe.MP[i * NP + j] * fe.S[v][j * NP + m];
        t.MS[v][i][m] = (T)acc;
      }
  for (int i = 0; i < NP; ++i) {   // face coupling coefficients (C x_ext), see face_* kernels
    t.CF[0][i] = (T)(i < NC ? -0.5 * fe.d0[i] - (i == 0 ? fe.gamma : 0.0) : 0.0);
    t.CF[1][i] = (T)(i == 0 ? 0.5 : 0.0);
    t.CF[2][i] = (T)(i >= NC ? 0.5 * fe.d1[i - NC] - (i == NP - 1 ? fe.gamma : 0.0) : 0.0);
    t.CF[3][i] = (T)(i == NP - 1 ? -0.5 : 0.0);
  }
  for (int v = 0; v < 4; ++v)
    for (int kd = 0; kd < 4; ++kd)
      for (int m = 0; m < NP; ++m) {
        double acc = 0.0;   // CH[v][kd][m] = sum_i S[v][i][m] CF[kd][i]
        for (int i = 0; i < NP; ++i) {
          const double cf = kd == 0 ? (i < NC ? -0.5 * fe.d0[i] - (i == 0 ? fe.gamma : 0.0) : 0.0)
                          : kd == 1 ? (i == 0 ? 0.5 : 0.0)
                          : kd == 2 ? (i >= NC ? 0.5 * fe.d1[i - NC] - (i == NP - 1 ? fe.gamma : 0.0) : 0.0)
                                    : (i == NP - 1 ? -0.5 : 0.0);
          acc += fe.S[v][i * NP + m] * cf;
        }
        t.CH[v][kd][m] = (T)acc;
      }
  for (int i = 0; i < NC; ++i) {
    t.d0[i] = (T)fe.d0[i];
    t.d1[i] = (T)fe.d1[i];
    t.w[i] = (T)fe.w[i];
  }
  for (int i = 0; i < NP; ++i)
    for (int j = 0; j < NC; ++j) {
      t.P[i][j] = (T)fe.P[i * NC + j];
      t.PT[j][i] = (T)fe.P[i * NC + j];
    }
  t.gamma = (T)fe.gamma;
}

inline cudaError_t upload(const FE1D& fe) {
  if (fe.k != K) return cudaErrorInvalidValue;
  static TabData<K, double> t64;
  static TabData<K, float> t32;
  fill_tab(t64, fe);
  fill_tab(t32, fe);
  cudaError_t e = cudaMemcpyToSymbol(c_tab64, &t64, sizeof(t64));
  if (e != cudaSuccess) return e;
#if !IPMG_DIRICHLET
  e = pair3_upload_tables();
  if (e != cudaSuccess) return e;
#endif
  return cudaMemcpyToSymbol(c_tab32, &t32, sizeof(t32));
}
#if IPMG_DIRICHLET
inline cudaError_t smooth_dir(int dim, int prec, const void* xi, const void* b, void* xo, const LevelGeom& g, int c,
                              cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_smooth_dir, xi, b, xo, g, c, s);
}
#else
inline cudaError_t vmult(int dim, int prec, const void* x, void* y, const LevelGeom& g, const void* bm, double* dotp,
                         long long* nparts, cudaStream_t s) {
  return IPMG_DISPATCH(dim, prec, launch_vmult, x, y, g, bm, dotp, nparts, s);
}
// Colour pass with the r.z of the mixed PCG fused in (3D fp32 colour 0 through the pair
// kernel: every dof is stored by exactly one patch): partials of sum r_i x_out_i into dotp,
// *nparts = their count; any other case runs the plain pass and sets *nparts = 0.
inline cudaError_t smooth_rz(int dim, int prec, const void* xi, const void* b, void* xo, const LevelGeom& g, int c,
                             const double* r, double* dotp, long long* nparts, cudaStream_t s) {
  *nparts = 0;
#if !IPMG_DIRICHLET
  if (dim == 3 && prec == 1 && c == 0 && xi != nullptr && pair3_enabled() && g.grouped && g.n[0] >= 2 &&
      g.n[1] >= 2 && g.n[2] >= 2 && (reinterpret_cast<unsigned long long>(xi) & 15) == 0 && (g.ncells % 4) == 0 &&
      (reinterpret_cast<unsigned long long>(xo) & 3) == 0) {
    const cudaError_t e = launch_smooth_pair3<IPMG_PAIR3_NPAIR>(xi, b, xo, g, c, s, r, dotp, nparts);
    if (e != cudaErrorNotReady) return e;
    *nparts = 0;
  }
#endif
  return IPMG_DISPATCH(dim, prec, launch_smooth, xi, b, xo, g, c, s);
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
#endif

}  // namespace IPMG_KK
}  // namespace ipmg

#if IPMG_DIRICHLET
// Dirichlet-kernel set: only the table upload and the smoother colour pass
extern "C++" ipmg::KernelSet IPMG_CAT(ipmg_kernel_set_dir_k, IPMG_K)() {
  ipmg::KernelSet ks{};
  ks.k = IPMG_K;
  ks.upload = ipmg::IPMG_KK::upload;
  ks.smooth = ipmg::IPMG_KK::smooth_dir;
  return ks;
}
#else
extern "C++" ipmg::KernelSet IPMG_CAT(ipmg_kernel_set_k, IPMG_K)() {
  ipmg::KernelSet ks;
  ks.k = IPMG_K;
  ks.upload = ipmg::IPMG_KK::upload;
  ks.vmult = ipmg::IPMG_KK::vmult;
  ks.smooth = ipmg::IPMG_KK::smooth;
  ks.smooth_rz = ipmg::IPMG_KK::smooth_rz;
  ks.additive = ipmg::IPMG_KK::additive;
  ks.restrict_ = ipmg::IPMG_KK::restrict_;
  ks.prolong = ipmg::IPMG_KK::prolong;
  return ks;
}
#endif
