// 3D fp64 operator apply, one colour-0 vertex patch per CTA, staged (included by
// patch_kernels.cuh inside namespace ipmg::kdeg<K> after smooth_pair3.cuh; full kernel only).
//
// Same operator as vmult_kernel<3, double> (Fig. 1 patch-wise
// integration; Kronecker sum of the patch matrices PAPER.md:118-126; face terms of the
// SIPG bilinear form PAPER.md:90-95): for every colour-0 patch j (the colour-0 patches
// tile the mesh, so each writes only its own cells -- no atomics)
//     y_j = h^{d-2} (A_jj x_j + C_j x_ext)      (or b_j - that, for a residual),
//   A_jj x = M2 (L1 M0 x + M1 L0 x) + L2 (M1 M0 x)   (patch-local 1D mass M, stiffness +
//   face terms L, boundary variants per direction), C_j x_ext from the traces of the 24
//   face-neighbour cells.  What differs from vmult_kernel is how it reaches the data
//   (ncu of vmult_kernel<3,double> at k = 4: 27 % of the stall samples long_sb -- the
//   neighbour traces and the x rows were read straight from global memory by dependent
//   loads, 5.8 k warp instructions per patch):
//
//  * the patch's own 8 cells and its 24 face-neighbour cells are copied into shared
//    memory with 16-byte cp.async at the start (one warp per cell, lanes on consecutive
//    chunks, the copy widened to the 16-byte boundaries around the cell: 63 chunks per
//    1000-byte cell); the line tensors X, T1 alias the neighbour copies once the traces
//    are formed;
//  * trace units (family a, side s, tangential cell h, second tangential index ic) read a
//    5x5 block of a staged neighbour cell and form u (face value) and u' (normal
//    derivative) at NC face points; the tangential masses the operator needs are applied
//    where the sum factorisation does not apply them anyway: the x-normal family is
//    injected into L0 x in the x pass (M1, M2 follow), the y-normal family into the y
//    pass (needs M along x), the z-normal family into the z pass (needs M along x and y);
//  * y- and z-lines are dealt to threads by the bank-sorted tables of the pair smoother
//    (same strides, same 8-byte elements);
//  * the z pass writes the result straight to global memory and forms the fused x.y of
//    CG from the staged x.
#if !IPMG_DIRICHLET
namespace op3 {
#ifndef IPMG_OP3_STAGE_OWN
#define IPMG_OP3_STAGE_OWN 0   // 1: the own cells are staged with the neighbours (x pass reads shared memory):
                               // 42 KB, 5 CTAs/SM, 3D k=4 128^3 operator 2.50 ms; 0: x rows from global, 6 CTAs/SM, 2.41 ms
#endif
constexpr int NL = NP * NP;
constexpr int CELL = NC * NC * NC;
constexpr int S1 = NP + 1, S2 = NP * S1, TSZ = NP * S2;   // line tensor strides (as pair3)
constexpr int FROW = NP;                                    // face array: t1 fastest, t2 rows
constexpr int FARR = NP * FROW + 1;                         // array pitch (odd)
constexpr int NNB = 24;
// a staged cell: the copy covers the cell from the 16-byte boundary at or below its start
// to the one at or above its end: ceil((CELL sizeof(T) + 16 - sizeof(T)) / 16) chunks at most
template <typename T>
struct Lay {
  static constexpr int EPC = 16 / (int)sizeof(T);                                // elements per chunk
  static constexpr int CHUNKS = ((int)sizeof(T) * CELL + 16 - (int)sizeof(T) + 15) / 16;
  static constexpr int SLOT = EPC * CHUNKS;                                       // elements per slot
  static constexpr size_t NBB = sizeof(T) * (size_t)NNB * SLOT;
  static constexpr size_t XB = sizeof(T) * 2 * (size_t)TSZ;                      // X and T1 (alias the slots)
  static constexpr size_t OWNB = IPMG_OP3_STAGE_OWN ? sizeof(T) * 8 * (size_t)SLOT : 0;
  static constexpr size_t FB = sizeof(T) * 12 * (size_t)FARR;
  static constexpr size_t SMEM = NBB + OWNB + FB;
  static_assert(XB <= NBB, "op3: X, T1 alias the neighbour slots");
};
constexpr int NT = (((NL > 12 * NP ? NL : 12 * NP) + 31) / 32) * 32;   // a line / trace unit per thread
static_assert(NT <= pair3::NTMAX, "line tables");
constexpr int NSTAGE = NNB + (IPMG_OP3_STAGE_OWN ? 8 : 0);  // staged cells

__device__ __forceinline__ int farr(int a, int s, int kind) { return ((a * 2 + s) * 2 + kind) * FARR; }
// elements between a staged cell's slot start and the cell (x is 16-byte aligned)
template <typename T>
__device__ __forceinline__ int soff(long long cell) { return (int)((cell * CELL) & (long long)(Lay<T>::EPC - 1)); }

// Trace unit of family A (compile-time: one code path per family, no selects):
// u[lb] = x(face node), du[lb] = sum_j phi_j'(face) x_j of the neighbour across face
// (A, s) at the NC face points lb along t1 in t1-cell h, second tangential index ic;
// families 1 and 2 get the cell mass along t1 (= x) applied.
template <int A, typename T>
__device__ __forceinline__ void trace_unit(T* F, const T* c, bool exists, int s, int h, int ic) {
  const TabData<K, T>& tb = tab<T>();
  const int lc = ic % NC;
  T u[NC], du[NC];
  if (exists) {
    // element (normal j, point lb) of the 5x5 block at c + PS * lb + NS * j + TS * lc
    constexpr int PS = A == 0 ? NC : 1;            // point stride (t1 = y for A = 0, x otherwise)
    constexpr int NS = A == 0 ? 1 : (A == 1 ? NC : NC * NC);
    constexpr int TS = A == 2 ? NC : NC * NC;      // second tangential (t2 = z, z, y)
    const T* b0 = c + TS * lc;
    T v[NC][NC];   // [point][normal]
#pragma unroll
    for (int lb = 0; lb < NC; ++lb)
#pragma unroll
      for (int j = 0; j < NC; ++j) v[lb][j] = b0[PS * lb + NS * j];
#pragma unroll
    for (int lb = 0; lb < NC; ++lb) {
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < NC; ++j) acc = fma_(s == 0 ? tb.d1[j] : tb.d0[j], v[lb][j], acc);
      du[lb] = acc;
      u[lb] = s == 0 ? v[lb][NC - 1] : v[lb][0];   // face node: the neighbour's last (low side) / first node
    }
  } else {
#pragma unroll
    for (int lb = 0; lb < NC; ++lb) u[lb] = du[lb] = T(0);
  }
  T* fu = F + farr(A, s, 0) + h * NC + FROW * ic;
  T* fd = F + farr(A, s, 1) + h * NC + FROW * ic;
  if (A == 0) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      fu[i] = u[i];
      fd[i] = du[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      T mu = T(0), md = T(0);
#pragma unroll
      for (int lb = 0; lb < NC; ++lb) {
        mu = fma_(tb.M[lb][i], u[lb], mu);
        md = fma_(tb.M[lb][i], du[lb], md);
      }
      fu[i] = mu;
      fd[i] = md;
    }
  }
}

// second tangential mass (along y) of the z-normal family: line e of 40 = (side, kind, x index o)
template <typename T>
__device__ __forceinline__ void t2_mass(T* F, int e) {
  const int o = e % NP, sk = e / NP;   // sk = side * 2 + kind
  T* base = F + farr(2, sk >> 1, sk & 1) + o;
  T v[1][NP], w[1][NP];
  load_lines<NP, 1>(base, 0, FROW, v);
  mv<NP, NP, MassP<T>, 1>(v, w);
  store_lines<NP, 1>(base, 0, FROW, w);
}

#ifndef IPMG_OP3_T2HALF
#define IPMG_OP3_T2HALF 1   // 1: the y mass of the z-normal family as half-line units on the idle threads
#endif
// one cell block (NC entries) of a t2_mass line: unit e of 8 NP = (side, kind, x index o, cell c)
template <typename T>
__device__ __forceinline__ void t2_mass_half(T* F, int e) {
  const TabData<K, T>& tb = tab<T>();
  const int c = e & 1, o = (e >> 1) % NP, sk = (e >> 1) / NP;
  T* base = F + farr(2, sk >> 1, sk & 1) + o + FROW * NC * c;
  T v[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) v[j] = base[FROW * j];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    T acc = T(0);
#pragma unroll
    for (int j = 0; j < NC; ++j) acc = fma_(tb.M[j][i], v[j], acc);
    base[FROW * i] = acc;
  }
}

// injection of face family a at tangential position pos into a line along a (operator sign +)
template <typename T>
__device__ __forceinline__ void inject(T (&y)[1][NP], const T* F, int a, int pos) {
  const TabData<K, T>& tb = tab<T>();
  const T ul = F[farr(a, 0, 0) + pos], dl = F[farr(a, 0, 1) + pos];
  const T uh = F[farr(a, 1, 0) + pos], dh = F[farr(a, 1, 1) + pos];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    T lo = tb.CF[0][i] * ul;
    if (i == 0) lo = fma_(tb.CF[1][i], dl, lo);
    y[0][i] += lo;
    T hi = tb.CF[2][NC + i] * uh;
    if (i == NC - 1) hi = fma_(tb.CF[3][NC + i], dh, hi);
    y[0][NC + i] += hi;
  }
}

template <bool FAST, typename T>
__device__ __forceinline__ void lap(const T (&v)[1][NP], T (&w)[1][NP], int var) {
  if (FAST) mv<NP, NP, LapP<0, T>, 1>(v, w);
  else if (var == 0) mv<NP, NP, LapP<0, T>, 1>(v, w);
  else mv<NP, NP, LapRT<T>, 1>(v, w, LapRT<T>{var});
}
template <bool FAST, typename T>
__device__ __forceinline__ void lap_acc(const T (&v)[1][NP], T (&w)[1][NP], int var) {
  if (FAST) mv_acc<NP, NP, LapP<0, T>, 1>(v, w);
  else if (var == 0) mv_acc<NP, NP, LapP<0, T>, 1>(v, w);
  else mv_acc<NP, NP, LapRT<T>, 1>(v, w, LapRT<T>{var});
}

struct PatchInfo {
  int base, var[3], own;
};

// MODE 0: y = hs A x (or bm - hs A x) stored, fused x.y returned; MODE 1 (restriction):
// r = b - hs A x formed on the z-lines and contracted with P^T along z in place (the
// kernel then contracts y and x and writes the coarse cell)
template <bool FAST, int MODE, typename T>
__device__ __forceinline__ double op3_body(const T* __restrict__ x, T* __restrict__ y, const T* __restrict__ bm,
                                           const LevelGeom& g, const PatchInfo& P, const pair3::Deltas& dl, T* X,
                                           T* T1, const T* OWN, T* F, bool dot) {
  using LY = Lay<T>;
  // half-line units need idle threads; fp32 only (tools/gpu_deg_key.sh: fp32 restriction k = 4
  // 0.711 -> 0.687 ms, k = 5, 6 -2 to -3 %; the fp64 operator 1 to 7 % slower with them)
  constexpr bool HALF = IPMG_OP3_T2HALF && NT > NL && sizeof(T) == 4;
  const int t = threadIdx.x;
  // ---- x pass: T1 = M0 x, X = L0 x + x-normal family; the z-normal family's y mass on idle threads
  if (t < NL) {
    const int i1 = t % NP, i2 = t / NP;
    const int qlo = 2 * (i1 / NC) + 4 * (i2 / NC), r0 = NC * (i1 % NC) + NC * NC * (i2 % NC);
    T v[1][NP], w[1][NP];
#if IPMG_OP3_STAGE_OWN
    const T* s0 = OWN + qlo * LY::SLOT + soff<T>(P.base + dl.pc[qlo]) + r0;
    const T* s1 = OWN + (qlo + 1) * LY::SLOT + soff<T>(P.base + dl.pc[qlo + 1]) + r0;
#else
    const T* s0 = x + (long long)(P.base + dl.pc[qlo]) * CELL + r0;
    const T* s1 = x + (long long)(P.base + dl.pc[qlo + 1]) * CELL + r0;
#endif
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      v[0][j] = s0[j];
      v[0][NC + j] = s1[j];
    }
    mv<NP, NP, MassP<T>, 1>(v, w);
    store_lines<NP, 1>(T1 + S1 * i1 + S2 * i2, 0, 1, w);
    lap<FAST>(v, w, P.var[0]);
    inject(w, F, 0, i1 + FROW * i2);
    store_lines<NP, 1>(X + S1 * i1 + S2 * i2, 0, 1, w);
  } else if (HALF) {
    // the z-normal family's y mass as (line, cell) half-line units dealt over the threads
    // without an x-line (k = 4: 80 units on 28 threads, at most 3 each)
    for (int e = t - NL; e < 8 * NP; e += (HALF ? NT - NL : 1)) t2_mass_half(F, e);
  } else if (t - NL < 4 * NP) {
    t2_mass(F, t - NL);
  }
  // (whole lines) the lines the idle threads do not cover go to the first threads
  if (!HALF && NT - NL < 4 * NP && t < 4 * NP - (NT - NL)) t2_mass(F, NT - NL + t);
  __syncthreads();
  // ---- y pass: X = M1 X + L1 T1 + y-normal family, T1 = M1 T1
  const unsigned ly = __ldg(&pair3::g_lines[0][0][t]);
  if (ly != 0xffffffffu) {
    const int base = (int)ly, i0 = base % S2, i2 = base / S2;
    T m[1][NP], lx[1][NP], w[1][NP];
    load_lines<NP, 1>(T1 + base, 0, S1, m);
    load_lines<NP, 1>(X + base, 0, S1, lx);
    mv<NP, NP, MassP<T>, 1>(lx, w);
    lap_acc<FAST>(m, w, P.var[1]);
    inject(w, F, 1, i0 + FROW * i2);
    store_lines<NP, 1>(X + base, 0, S1, w);
    mv<NP, NP, MassP<T>, 1>(m, w);
    store_lines<NP, 1>(T1 + base, 0, S1, w);
  }
  __syncthreads();
  // ---- z pass: hs (M2 X + L2 T1 + z-normal family)
  double dacc = 0.0;
  const unsigned lz = __ldg(&pair3::g_lines[0][1][t]);
  if (lz != 0xffffffffu) {
    const int base = (int)(lz & 0xffff), i0 = (lz >> 16) & 0xf, i1 = (lz >> 20) & 0xf;
    T a[1][NP], bb[1][NP], w[1][NP];
    load_lines<NP, 1>(X + base, 0, S2, a);
    mv<NP, NP, MassP<T>, 1>(a, w);
    load_lines<NP, 1>(T1 + base, 0, S2, bb);
    lap_acc<FAST>(bb, w, P.var[2]);
    inject(w, F, 2, i0 + FROW * i1);
    const T hs = T(g.hs);
    const int qb = (i0 / NC) + 2 * (i1 / NC), ob = (i0 % NC) + NC * (i1 % NC);
    if (MODE == 1) {
      // residual on the z-line (b gathered along it), then P^T along z into the line's
      // first NC entries (only this thread touches the line in this phase)
      T r[1][NP], rc[1][NC];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const T* bo = bm + ((long long)P.base + dl.pc[qb + 4 * c]) * CELL + ob;
#pragma unroll
        for (int j = 0; j < NC; ++j) r[0][c * NC + j] = fma_(-hs, w[0][c * NC + j], __ldg(bo + NC * NC * j));
      }
      mv<NC, NP, ProlT<T>, 1>(r, rc);
#pragma unroll
      for (int j = 0; j < NC; ++j) X[base + j * S2] = rc[0][j];
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (!((P.own >> c) & 1)) continue;   // ghost cells of a straddling patch
        const long long cell = (long long)P.base + dl.pc[qb + 4 * c];
        T* yo = y + cell * CELL + ob;
#if IPMG_OP3_STAGE_OWN
        const T* xo = OWN + (qb + 4 * c) * LY::SLOT + soff<T>(cell) + ob;
#else
        const T* xo = x + cell * CELL + ob;
#endif
        const T* bo = bm ? bm + cell * CELL + ob : nullptr;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          T val = hs * w[0][c * NC + j];
          if (bo) val = __ldg(bo + NC * NC * j) - val;
          yo[NC * NC * j] = val;
          if (dot) dacc = fma((double)xo[NC * NC * j], (double)val, dacc);
        }
      }
    }
  }
  return dacc;
}

#ifndef IPMG_OP3_TY
#define IPMG_OP3_TY 8   // rows per traversal tile (as pair3: z-face neighbours stay in L2)
#endif
constexpr int TY = IPMG_OP3_TY;

// MODE 0: the operator (y = hs A x, or bm - hs A x; fused x.y partials when dot_partial).
// MODE 1: the restriction r_c = P^T (bm - hs A x) of the patch (= parent cell) into rc on
// the coarse level gc (restrict_kernel's contract).
template <typename T, int MODE>
__global__ void __launch_bounds__(NT) op3_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                 const T* __restrict__ bm, LevelGeom g, int gx, int gy,
                                                 const __grid_constant__ pair3::Deltas dl,
                                                 double* __restrict__ dot_partial, LevelGeom gc) {
  using LY = Lay<T>;
  // grid (gx, TY * gz, ceil(gy / TY)): tiles of TY patch rows, as the pair smoother
  const int bxi = blockIdx.x, byi = (int)blockIdx.z * TY + (int)(blockIdx.y % TY), jz = (int)(blockIdx.y / TY);
  if (byi >= gy) return;   // the last tile's missing rows (no partial: see the launcher)
  const int bzi = g.zsel == 0 ? jz : (g.zsel == 1 ? jz + 1 : (jz == 0 ? 0 : g.znb - 1));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* NBs = reinterpret_cast<T*>(smem_raw);
  T* X = NBs;   // X, T1 alias the neighbour slots (dead after the trace units)
  T* T1 = NBs + TSZ;
  T* OWN = NBs + NNB * LY::SLOT;   // the own cells follow the neighbour slots (slot 24 + q)
  T* F = reinterpret_cast<T*>(smem_raw + LY::NBB + LY::OWNB);
  const int t = threadIdx.x;
  // patch data in registers (every thread: no barrier, no shared table)
  PatchInfo P;
  const int c0x = 2 * bxi, c0y = 2 * byi, c0z = 2 * bzi;   // colour 0: slab_first = 0
  {
    P.base = (int)cell_offset_cells(g, c0x, c0y, c0z);
    const int gs = g.zoff + c0z;
    P.own = (c0z >= 0 ? 1 : 0) | (c0z + 1 < g.n[2] ? 2 : 0);
    P.var[0] = (c0x == 0 ? 1 : 0) | (c0x + 2 == g.n[0] ? 2 : 0);
    P.var[1] = (c0y == 0 ? 1 : 0) | (c0y + 2 == g.n[1] ? 2 : 0);
    P.var[2] = (gs == 0 ? 1 : 0) | (gs + 2 == g.nglob ? 2 : 0);
  }
  // staging: entry e < 24 the face neighbour k = e (absent across the domain boundary),
  // e >= 24 the own cell q = e - 24, in slot e; a warp per entry.  Lane i of warp w first
  // forms the source of entry w + NW i (one cell-index load each, in parallel), the copy
  // loop takes them by shuffle.
  {
    const int lane = t & 31, w = t >> 5;
    constexpr int NW = NT / 32, PER = (NSTAGE + NW - 1) / NW;
    static_assert(PER <= 32, "op3 staging");
    // an absent neighbour (face on the domain boundary) copies the patch's own first cell
    // instead (never read: its trace units see exists = false) -- no branch in the copy loop
    unsigned long long my = 0ull;   // 16-byte aligned source
    {
      const int e = w + NW * lane;
      int cell = P.base + dl.pc[0];
      if (lane < PER && e < NSTAGE) {
        if (e < NNB) {
          const int va = e < 8 ? P.var[0] : (e < 16 ? P.var[1] : P.var[2]);
          if (!((va >> ((e >> 2) & 1)) & 1)) cell = P.base + dl.nb[e];
        } else {
          cell = P.base + dl.pc[e - NNB];
        }
      }
      my = reinterpret_cast<unsigned long long>(x + (long long)cell * CELL) & ~15ull;
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (w + NW * i >= NSTAGE) break;
      const unsigned long long src = __shfl_sync(0xffffffffu, my, i);
      T* dst = NBs + (w + NW * i) * LY::SLOT;
      // chunks c0 + lane; lanes past the end repeat chunk CHUNKS - 1 (the same bytes): no branch
#pragma unroll
      for (int c0 = 0; c0 < LY::CHUNKS; c0 += 32) {
        const int c = c0 + lane < LY::CHUNKS ? c0 + lane : LY::CHUNKS - 1;
        cp_async<16>(dst + LY::EPC * c, reinterpret_cast<const void*>(src + 16ull * c));
      }
    }
    cp_async_commit();
  }
  cp_async_wait_all();
  __syncthreads();
  // trace units: family a = u / 40, (side, t1 cell, second tangential index) within
  if (t < 12 * NP) {
    const int a = t / (4 * NP), r = t % (4 * NP);
    const int ic = r % NP, h = (r / NP) & 1, s = r / (2 * NP);
    const int tc = h + ((ic >= NC) ? 2 : 0);
    const int k = (2 * a + s) * 4 + tc;
    const int va = a == 0 ? P.var[0] : (a == 1 ? P.var[1] : P.var[2]);
    const bool ex = !((va >> s) & 1);
    const T* c = NBs + k * LY::SLOT + (ex ? soff<T>(P.base + dl.nb[k]) : 0);
    if (a == 0) trace_unit<0>(F, c, ex, s, h, ic);
    else if (a == 1) trace_unit<1>(F, c, ex, s, h, ic);
    else trace_unit<2>(F, c, ex, s, h, ic);
  }
  __syncthreads();
  const bool fast = (P.var[0] | P.var[1] | P.var[2]) == 0;
  const bool dot = MODE == 0 && dot_partial != nullptr;
  double d = fast ? op3_body<true, MODE>(x, y, bm, g, P, dl, X, T1, (const T*)OWN, F, dot)
                  : op3_body<false, MODE>(x, y, bm, g, P, dl, X, T1, (const T*)OWN, F, dot);
  if (MODE == 1) {
    // P^T along y on the lines (i0, i2 < NC) of the z-contracted slab, in place
    __syncthreads();
    if (t < NP * NC) {
      const int i0 = t % NP, i2 = t / NP;
      T v[1][NP], w[1][NC];
      load_lines<NP, 1>(X + i0 + S2 * i2, 0, S1, v);
      mv<NC, NP, ProlT<T>, 1>(v, w);
#pragma unroll
      for (int j = 0; j < NC; ++j) X[i0 + S2 * i2 + S1 * j] = w[0][j];
    }
    __syncthreads();
    // P^T along x on the lines (i1, i2 < NC): one coarse-cell row each, straight to global
    if (t < NC * NC) {
      const int i1 = t % NC, i2 = t / NC;
      T v[1][NP], w[1][NC];
      load_lines<NP, 1>(X + S1 * i1 + S2 * i2, 0, 1, v);
      mv<NC, NP, ProlT<T>, 1>(v, w);
      const int c0[3] = {c0x, c0y, c0z};
      T* dst = y + coarse_cell<3>(g, gc, c0) * CELL + NC * i1 + NC * NC * i2;
#pragma unroll
      for (int j = 0; j < NC; ++j) dst[j] = w[0][j];
    }
    return;
  }
  if (dot) {
    // fused x.y of CG: deterministic CTA partial (fixed tree), full-grid index
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    __shared__ double wsum[NT / 32];
    if ((t & 31) == 0) wsum[t >> 5] = d;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += wsum[w];
      dot_partial[bxi + (long long)gx * (byi + (long long)gy * bzi)] = s;
    }
  }
}
}  // namespace op3
#endif
