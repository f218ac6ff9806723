// 3D fp32 multiplicative smoother, one colour pass, "patch pairs" (included by
// patch_kernels.cuh inside namespace ipmg::kdeg<K>; full kernel only).
//
// Same arithmetic as smooth_kernel<3, float> (replacement form of Algorithm 1,
// PAPER.md:242-257; fast diagonalisation PAPER.md:266-280): for every patch j of
// the colour,  x_j = A_jj^{-1} (h^{2-d} b_j - C_j x_in),  the face coupling C_j x_in
// formed from the traces of the 2d x 4 face-neighbour cells.  What differs is
// how it maps onto sm_100a (the ncu capture of smooth_kernel<3,float>
// at k = 4 showed the L1 data pipe at 91 % of its wavefront peak and 45 % of the
// warp instructions in the face phases):
//
//  * two patches side by side along x (a "pair") share every thread: each value a
//    thread holds is a float2 (patch p, patch p+1), every contraction is FFMA2 with
//    the 1D matrix entry as a uniform-register scalar broadcast (one LDCU.128 feeds
//    4 FFMA2 = 16 flops), and no odd-length tail instruction (k even).
//  * the pair tensor lives in shared memory as float2 with strides (1, NP+1,
//    NP(NP+1)): x-lines (i1 fastest) are bank-conflict free; y- and z-lines are
//    dealt to threads by host-built tables that put 16 distinct banks into every
//    half warp (conflict free whenever no residue class exceeds the half-warp count).
//    The trace units' loads from the staged cells are not conflict free: the per-cell
//    alignment offsets and the slot pitch put lanes of different cells on the same bank
//    (ncu at C4: ~270 M excess shared load wavefronts per pass, profiles/r02j_ncu_full.md).
//  * the face-neighbour cells are copied into shared memory with 16-byte cp.async
//    (a warp per cell, lanes on consecutive 16-byte chunks: one instruction per cell
//    and fully used lines; TMA bulk copies measured slower -- every copy needs its own
//    uniform operands, ~27 warp instructions each); the trace units then read them from
//    shared memory.  Cell indices are the patch's base cell plus launch constants
//    (host-computed deltas of the parent-grouped layout), so there is no setup table.
//  * the neighbour traces get the tangential cell mass along the first tangential
//    direction in registers and along the second in one shared-memory pass; all
//    three face families are injected into the right-hand side of the x pass
//    (physical space, as smooth_kernel does).
#if !IPMG_DIRICHLET
namespace pair3 {
#ifndef IPMG_PAIR3_LATE_B
#define IPMG_PAIR3_LATE_B 1   // 1: load the b rows right before the x pass (not before the traces):
                              // 78 instead of 82 registers, 6 CTAs/SM; 3D k=4 colour pass 1.65 -> 1.60 ms
#endif

#ifndef IPMG_PAIR3_SHFLSTAGE
#define IPMG_PAIR3_SHFLSTAGE 1   // 1: staging sources formed in parallel by the lanes, taken by shuffle,
                                 // branch-free copies, no shared table or barrier before the copies
#endif
#ifndef IPMG_PAIR3_STASM
#define IPMG_PAIR3_STASM 1   // 1: pair stores to shared memory as st.shared.v2.f32 inline asm (see sts2)
#endif
#ifndef IPMG_PAIR3_BPF
#define IPMG_PAIR3_BPF 2   // 1: L1 prefetch of the b cells at the start (SHFLSTAGE path)
#endif
constexpr int NL = NP * NP;               // lines per direction per patch
constexpr int CELL = NC * NC * NC;
constexpr int H = NP / 2;
constexpr int S1 = NP + 1;                // float2 strides of the pair tensor: x 1, y S1, z S2
constexpr int S2 = NP * S1;               // S2 = NP S1 and S1 odd: x-line t has base S1 t (mod 16)
constexpr int TSZ = NP * S2;              // pair pitch = S1 NL: the sequence continues across pairs
#ifndef IPMG_PAIR3_FROW_PAD
#define IPMG_PAIR3_FROW_PAD 0   // face-array row padding (0: rows of NP; keeps 6 CTAs/SM at k = 4)
#endif
constexpr int FROW = NP + IPMG_PAIR3_FROW_PAD;   // face array: t1 fastest, t2 rows of FROW float2
// array pitch: searched over the face-array accesses (trace-unit writes, the t2 pass, the
// x-pass reads) for the fewest excess 64-bit shared wavefronts: +1 for NP = 10 (FARR 101:
// 190 excess per pair-pass against 420 at 106), otherwise 10 (mod 16)
constexpr int FARR = (NP == 10 && FROW == 10) ? 101 : NP * FROW + ((10 - (NP * FROW) % 16) + 16) % 16;
constexpr int FPAIR = 12 * FARR;          // (a, side, kind) arrays per pair
constexpr int NNB = 24;                   // face-neighbour cells per patch
// neighbour slot: the TMA copy covers the cell from the 16-byte boundary below it,
// so a slot holds CELL + 3 floats rounded up to 16 bytes; an extra 16 bytes when that
// is a multiple of 128 bytes staggers the slots across the banks
constexpr int SLOT0 = ((CELL + 3 + 3) / 4) * 4;
constexpr int SLOTF = (SLOT0 % 32 == 0) ? SLOT0 + 4 : SLOT0;
constexpr int NTMAX = 1024;               // line tables: max threads per CTA
static_assert(3 * NP * NP * (NP + 1) < 65536 && NP <= 16, "z line table packing");

template <int NPAIR>
struct PC {
  static constexpr int NT = ((NPAIR * NL + 31) / 32) * 32;
  static constexpr int NPAT = 2 * NPAIR;
  static constexpr int UNITS = NPAIR * 6 * 2 * NP;       // trace units: (pair, a, side, h, ic)
  static constexpr int FLINES = NPAIR * 12 * NP;         // second-tangential mass lines
  static constexpr size_t XB = sizeof(float2) * (size_t)NPAIR * TSZ;
  static constexpr size_t NBB = sizeof(float) * (size_t)NPAT * NNB * SLOTF;
  static constexpr size_t FB = sizeof(float2) * (size_t)NPAIR * FPAIR;
  // X aliases the neighbour staging (dead after the trace phase)
  static constexpr size_t SMEM = (XB > NBB ? XB : NBB) + FB;
  static_assert(NT <= NTMAX, "line tables");
};

// host-built thread -> line tables of the y (row 0) and z (row 1) passes, per NPAIR,
// decoded: y entry = tensor offset of the line's first element; z entry = offset |
// m0 << 16 | m1 << 20 | pair << 24 (m0, m1 the line's x/y mode indices); 0xffffffff =
// idle thread.  Filled by upload().
__device__ unsigned g_lines[3][2][NTMAX];

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float a, float2 x, float2 c) { return __ffma2_rn(f2(a), x, c); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// ---- even/odd fast diagonalisation factors of the interior variant (patch_kernels.cuh
// eigT_eo / eig_eo), on a pair line
__device__ __forceinline__ void fwd_eo(const float2 (&in)[NP], float2 (&out)[NP]) {
  const TabData<K, float>& tb = c_tab32;
  float2 e[H], o[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    e[i] = add2(in[i], in[NP - 1 - i]);
    o[i] = sub2(in[i], in[NP - 1 - i]);
  }
#pragma unroll
  for (int m = 0; m < H; ++m) {
    float2 we = make_float2(0.f, 0.f), wo = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      we = fma2(tb.S[0][i][m], e[i], we);
      wo = fma2(tb.SO[i][m], o[i], wo);
    }
    out[m] = we;
    out[H + m] = wo;
  }
}
__device__ __forceinline__ void bwd_eo(const float2 (&in)[NP], float2 (&out)[NP]) {
  const TabData<K, float>& tb = c_tab32;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    float2 E = make_float2(0.f, 0.f), O = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      E = fma2(tb.ST[0][m][i], in[m], E);
      O = fma2(tb.ST[0][H + m][i], in[H + m], O);
    }
    out[i] = add2(E, O);
    out[NP - 1 - i] = sub2(E, O);
  }
}
// general variants (boundary patches): dense S^T / S with per-patch variants (v.x, v.y)
__device__ __forceinline__ void fwd_rt(const float2 (&in)[NP], float2 (&out)[NP], int v0, int v1) {
  const TabData<K, float>& tb = c_tab32;
#pragma unroll
  for (int m = 0; m < NP; ++m) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < NP; ++i) acc = __ffma2_rn(make_float2(tb.S[v0][i][m], tb.S[v1][i][m]), in[i], acc);
    out[m] = acc;
  }
}
__device__ __forceinline__ void bwd_rt(const float2 (&in)[NP], float2 (&out)[NP], int v0, int v1) {
  const TabData<K, float>& tb = c_tab32;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < NP; ++m) acc = __ffma2_rn(make_float2(tb.ST[v0][m][i], tb.ST[v1][m][i]), in[m], acc);
    out[i] = acc;
  }
}
template <bool FAST>
__device__ __forceinline__ void fwd(const float2 (&in)[NP], float2 (&out)[NP], int v0, int v1) {
  if (FAST) fwd_eo(in, out);
  else fwd_rt(in, out, v0, v1);
}
template <bool FAST>
__device__ __forceinline__ void bwd(const float2 (&in)[NP], float2 (&out)[NP], int v0, int v1) {
  if (FAST) bwd_eo(in, out);
  else bwd_rt(in, out, v0, v1);
}

// ---- per-CTA patch data (shared memory)
template <int NPAT>
struct Pat {
  int base[NPAT];               // cell index of the patch's lowest cell
  int var[NPAT][3];             // boundary variant per direction
  int own[NPAT];                // bit s: cells with slowest-axis bit s are local (written)
  int valid[NPAT];
};
// Cell-index deltas of a launch (parent-grouped layout; they depend only on the colour's
// parities and the level's parent counts): patch cell q = (qx, qy, qz) at base + pc[q],
// face neighbour k = (a, side) * 4 + tc at base + nb[k]
struct Deltas {
  int pc[8];
  int nb[NNB];
};
// face neighbour k of patch p exists (and is staged) iff its face is not on the domain boundary
template <int NPAT>
__device__ __forceinline__ bool nb_exists(const Pat<NPAT>& P, int p, int k) {
  return P.valid[p] && !((P.var[p][k >> 3] >> ((k >> 2) & 1)) & 1);
}

// line pass helpers on the pair tensor (float2 smem): element j of a line at base + j * stride
__device__ __forceinline__ void ld_line(const float2* X, int base, int stride, float2 (&v)[NP]) {
#pragma unroll
  for (int j = 0; j < NP; ++j) v[j] = X[base + j * stride];
}
// shared-memory store of a pair: as inline st.shared.v2.f32 ptxas keeps the value in the
// registers the FFMA2 wrote (a plain float2 store got two MOVs into a staging pair before
// almost every STS.64: 3D k=4 colour pass 1.575 -> 1.528 ms)
__device__ __forceinline__ void sts2(float2* p, float2 v) {
#if IPMG_PAIR3_STASM
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"((unsigned)__cvta_generic_to_shared(p)), "f"(v.x), "f"(v.y)
               : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_line(float2* X, int base, int stride, const float2 (&v)[NP]) {
#pragma unroll
  for (int j = 0; j < NP; ++j) sts2(X + base + j * stride, v[j]);
}

// one pair row of b (scaled) from global: row (i1, i2) of both patches, zeros for an invalid patch
template <int NPAT>
__device__ __forceinline__ void load_b_rows(const float* __restrict__ b, const Pat<NPAT>& P, const Deltas& dl, int q,
                                            int i1, int i2, float scale, float2 (&v)[NP]) {
  const int qlo = 2 * (i1 / NC) + 4 * (i2 / NC), r0 = NC * (i1 % NC) + NC * NC * (i2 % NC);
  float lo[2][NP];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    // an invalid patch (the second of a ragged row's last pair) reads its partner's rows:
    // in bounds, and its results are never stored
    const int p = 2 * q + (P.valid[2 * q + s] ? s : 0);
    const float* s0 = b + (long long)(P.base[p] + dl.pc[qlo]) * CELL + r0;
    const float* s1 = b + (long long)(P.base[p] + dl.pc[qlo + 1]) * CELL + r0;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      lo[s][j] = __ldg(s0 + j);
      lo[s][NC + j] = __ldg(s1 + j);
    }
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) v[j] = scale == 1.f ? make_float2(lo[0][j], lo[1][j]) : mul2(make_float2(lo[0][j], lo[1][j]), f2(scale));
}

// stores the x-line pair's rows; rdot != nullptr: returns sum rdot[o] * (stored value) over
// them (the r.z of the mixed PCG fused into the V-cycle's last colour pass, fp64)
template <bool DOT, int NPAT>
__device__ __forceinline__ double store_x_rows(float* __restrict__ x, const Pat<NPAT>& P, const Deltas& dl, int q,
                                               int i1, int i2, const float2 (&v)[NP],
                                               const double* __restrict__ rdot) {
  const int qlo = 2 * (i1 / NC) + 4 * (i2 / NC), r0 = NC * (i1 % NC) + NC * NC * (i2 % NC);
  double dot = 0.0;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int p = 2 * q + s;
    if (!P.valid[p] || !((P.own[p] >> (i2 / NC)) & 1)) continue;   // ghost cells of a straddling patch
    const long long o0 = (long long)(P.base[p] + dl.pc[qlo]) * CELL + r0;
    const long long o1 = (long long)(P.base[p] + dl.pc[qlo + 1]) * CELL + r0;
    float* d0 = x + o0;
    float* d1 = x + o1;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const float a0 = s ? v[j].y : v[j].x, a1 = s ? v[NC + j].y : v[NC + j].x;
      d0[j] = a0;
      d1[j] = a1;
      if (DOT) {
        dot = fma(__ldg(rdot + o0 + j), (double)a0, dot);
        dot = fma(__ldg(rdot + o1 + j), (double)a1, dot);
      }
    }
  }
  return dot;
}

// Trace unit (pair q, family a, side s, tangential cell h, second tangential index ic):
// u = x(face node), u' = sum_j phi_j'(face) x_j (unit h) of the neighbour across face
// (a, s) at the NC face points lb of t1-cell h (t1 = first tangential direction), both
// patches; the tangential cell mass along t1 in registers; written to the face arrays
// (t1 index h NC + i, t2 index ic).  The neighbour cells are in shared memory (slots; a
// missing neighbour reads the zero slot).  A unit reads an NC x NC block v[r][c] with
// contiguous columns: for a = 0 (x-normal; t1 = y, t2 = z) r is the point and c the
// normal index, for a = 1, 2 (t1 = x; t2 = z, y) r is the normal and c the point index.
// One code path for all families (a warp never diverges): both contractions are formed
// and the family's one kept.
template <int NPAT>
__device__ __forceinline__ void trace_unit(float2* F, const float* NBs, const float* zslot, const Pat<NPAT>& P,
                                           const Deltas& dl, int q, int a, int s, int h, int ic) {
  const TabData<K, float>& tb = c_tab32;
  const int lc = ic % NC, tc = h + ((ic >= NC) ? 2 : 0);
  const int k = (2 * a + s) * 4 + tc;
  const bool pr = a == 0;                                        // rows are the points
  const int Rr = a == 2 ? NC * NC : NC;                           // row stride
  const int Rl = a == 2 ? NC : NC * NC;                           // t2 stride
  const float* c[2];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp) {
    const int p = 2 * q + pp;
    c[pp] = nb_exists(P, p, k)
                ? NBs + (p * NNB + k) * SLOTF + (int)(((long long)(P.base[p] + dl.nb[k]) * CELL) & 3) + lc * Rl
                : zslot;
  }
  float2 v[NC][NC];   // [row][column]
#pragma unroll
  for (int r = 0; r < NC; ++r) {
    const float* r0 = c[0] + r * Rr;
    const float* r1 = c[1] + r * Rr;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) v[r][cc] = make_float2(r0[cc], r1[cc]);
  }
  const int jf = s == 0 ? NC - 1 : 0;   // face node: the neighbour's last node (low side), first (high)
  float2 u[NC], du[NC];
#pragma unroll
  for (int lb = 0; lb < NC; ++lb) {
    float2 ar = make_float2(0.f, 0.f), ac = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const float dj = s == 0 ? tb.d1[j] : tb.d0[j];
      ar = fma2(dj, v[lb][j], ar);   // points in rows (a = 0)
      ac = fma2(dj, v[j][lb], ac);   // points in columns (a = 1, 2)
    }
    du[lb] = pr ? ar : ac;
    const float2 ur = jf == 0 ? v[lb][0] : v[lb][NC - 1];
    const float2 uc = jf == 0 ? v[0][lb] : v[NC - 1][lb];
    u[lb] = pr ? ur : uc;
  }
  // tangential cell mass along t1
  float2* fu = F + q * FPAIR + ((a * 2 + s) * 2 + 0) * FARR + h * NC + FROW * ic;
  float2* fd = F + q * FPAIR + ((a * 2 + s) * 2 + 1) * FARR + h * NC + FROW * ic;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    float2 mu = make_float2(0.f, 0.f), md = make_float2(0.f, 0.f);
#pragma unroll
    for (int lb = 0; lb < NC; ++lb) {
      mu = fma2(tb.M[lb][i], u[lb], mu);
      md = fma2(tb.M[lb][i], du[lb], md);
    }
    sts2(fu + i, mu);
    sts2(fd + i, md);
  }
}

// the pair kernel; FAST: every valid patch of the CTA is interior (variant 0 in all
// directions) -> even/odd factors with compile-time constants
template <int NPAIR, bool FAST, bool DOT, bool FACES>
__device__ __forceinline__ double pair_body(const float* __restrict__ x_in, const float* __restrict__ b,
                                            float* __restrict__ x_out, const LevelGeom& g, const Pat<2 * NPAIR>& P,
                                            const Deltas& dl, float2* X, float2* F, const float* NBs,
                                            const float* zslot, const float2 (&brow)[NP], int ybase, int zbase,
                                            int zq, int zm0, int zm1, const double* __restrict__ rdot) {
  using C = PC<NPAIR>;
  const TabData<K, float>& tb = c_tab32;
  const int t = threadIdx.x;
  const bool faces = FACES && x_in != nullptr;
  if (faces) {
    cp_async_wait_all();
    __syncthreads();
    for (int u = t; u < C::UNITS; u += C::NT) {
      const int q = u / (6 * 2 * NP), r = u % (6 * 2 * NP), a = r / (4 * NP), w = r % (4 * NP);
      const int ic = w % NP, h = (w / NP) & 1, s = w / (2 * NP);
      trace_unit(F, NBs, zslot, P, dl, q, a, s, h, ic);
    }
    __syncthreads();
    // tangential cell mass along t2 (block diagonal) on the (u, u') array pair of every
    // (family, side) line; the u' array is replaced by the combination the boundary row
    // of the x pass needs, V = CF_u(ib) u + CF_u'(ib) u' (ib: the outermost node on the
    // side), so the injection reads one array per family without branches
    for (int e = t; e < C::FLINES / 2; e += C::NT) {
      const int q = e / (6 * NP), r = e % (6 * NP), fs = r / NP, o = r % NP;
      const int sd = fs & 1, ib = sd == 0 ? 0 : NP - 1;
      float2* bu = F + q * FPAIR + (2 * fs) * FARR + o;
      float2* bd = bu + FARR;
      float2 v[NP], w[NP], dv[NP], dw[NP];
      ld_line(bu, 0, FROW, v);
      ld_line(bd, 0, FROW, dv);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          float2 acc = make_float2(0.f, 0.f), dacc = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            acc = fma2(tb.M[j][i], v[c * NC + j], acc);
            dacc = fma2(tb.M[j][i], dv[c * NC + j], dacc);
          }
          w[c * NC + i] = acc;
          dw[c * NC + i] = dacc;
        }
      const float cu = sd == 0 ? tb.CF[0][0] : tb.CF[2][NP - 1];
      const float cd = sd == 0 ? tb.CF[1][0] : tb.CF[3][NP - 1];
      (void)ib;
#pragma unroll
      for (int j = 0; j < NP; ++j) dw[j] = fma2(cd, dw[j], mul2(w[j], f2(cu)));
      st_line(bu, 0, FROW, w);
      st_line(bd, 0, FROW, dw);
    }
    __syncthreads();
  }
  // ---- x pass: rhs rows (h^{2-d} b - C x_ext), S_x^T
  const int q0 = t / NL, l0 = t % NL;
  const int i1 = l0 % NP, i2 = l0 / NP;
  const bool act0 = t < NPAIR * NL;
  const int pa = 2 * (act0 ? q0 : 0);
  const int vx0 = P.var[pa][0], vx1 = P.var[pa + 1][0], vy = P.var[pa][1], vz = P.var[pa][2];
  if (act0) {
    float2 y[NP];
#if IPMG_PAIR3_LATE_B
    load_b_rows(b, P, dl, q0, i1, i2, (float)g.hinv, y);
    (void)brow;
#else
    const float hinv = (float)g.hinv;
#pragma unroll
    for (int j = 0; j < NP; ++j) y[j] = mul2(brow[j], f2(hinv));
#endif
    if (faces) {
      const float2* Fq = F + q0 * FPAIR;
      // family 0 (x-normal): rank one along the row at the point (i1, i2); the outermost
      // node takes the combined array V (see the t2 pass)
      const int pos = i1 + FROW * i2;
      const float2 ul = Fq[0 * FARR + pos], vl = Fq[1 * FARR + pos];
      const float2 uh = Fq[2 * FARR + pos], vh = Fq[3 * FARR + pos];
      y[0] = sub2(y[0], vl);
      y[NP - 1] = sub2(y[NP - 1], vh);
#pragma unroll
      for (int i = 1; i < NC; ++i) {
        y[i] = fma2(-tb.CF[0][i], ul, y[i]);
        y[NC - 1 + i] = fma2(-tb.CF[2][NC - 1 + i], uh, y[NC - 1 + i]);
      }
      // families 1 (y-normal, t1 = x, t2 = z) and 2 (z-normal, t1 = x, t2 = y): whole rows,
      // the row's coefficient times the u array, or the V array on the outermost row
#pragma unroll
      for (int a = 1; a < 3; ++a) {
        const int ia = a == 1 ? i1 : i2, other = a == 1 ? i2 : i1;
        const int sd = ia < NC ? 0 : 1;
        const bool outer = ia == 0 || ia == NP - 1;
        const float cu = outer ? 1.f : tb.CF[2 * sd][ia];
        const float2* fr = Fq + ((a * 2 + sd) * 2 + (outer ? 1 : 0)) * FARR + other * FROW;
#pragma unroll
        for (int j = 0; j < NP; ++j) y[j] = fma2(-cu, fr[j], y[j]);
      }
    }
    // X aliases the neighbour staging: its last reads (trace units) are two barriers back
    float2 w[NP];
    fwd<FAST>(y, w, vx0, vx1);
    st_line(X, q0 * TSZ + S1 * i1 + S2 * i2, 1, w);
  }
  __syncthreads();
  // ---- y pass (S_y^T); ybase < 0: no line for this thread
  if (ybase >= 0) {
    float2 v[NP], w[NP];
    const int base = ybase;
    ld_line(X, base, S1, v);
    fwd<FAST>(v, w, vy, vy);
    st_line(X, base, S1, w);
  }
  __syncthreads();
  // ---- z pass: S_z^T, eigenvalue division, S_z
  if (zbase >= 0) {
    const int q = zq, m0 = zm0, m1 = zm1;
    float2 v[NP], w[NP];
    const int base = zbase;
    ld_line(X, base, S2, v);
    fwd<FAST>(v, w, vz, vz);
    if (FAST) {
      const float ls = tb.lam[0][m0] + tb.lam[0][m1];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const float r = rcp_(ls + tb.lam[0][m]);
        w[m] = mul2(w[m], f2(r));
      }
    } else {
      const int qa = 2 * q;
      const float ls0 = tb.lam[P.var[qa][0]][m0] + tb.lam[vy][m1];
      const float ls1 = tb.lam[P.var[qa + 1][0]][m0] + tb.lam[vy][m1];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const float lm = tb.lam[vz][m];
        w[m] = mul2(w[m], make_float2(rcp_(ls0 + lm), rcp_(ls1 + lm)));
      }
    }
    bwd<FAST>(w, v, vz, vz);
    st_line(X, base, S2, v);
  }
  __syncthreads();
  // ---- y pass (S_y)
  if (ybase >= 0) {
    float2 v[NP], w[NP];
    const int base = ybase;
    ld_line(X, base, S1, v);
    bwd<FAST>(v, w, vy, vy);
    st_line(X, base, S1, w);
  }
  __syncthreads();
  // ---- x pass (S_x) -> x_out rows
  if (act0) {
    float2 v[NP], w[NP];
    ld_line(X, q0 * TSZ + S1 * i1 + S2 * i2, 1, v);
    bwd<FAST>(v, w, vx0, vx1);
    return store_x_rows<DOT>(x_out, P, dl, q0, i1, i2, w, rdot);
  }
  return 0.0;
}

#ifndef IPMG_PAIR3_MINB
#define IPMG_PAIR3_MINB 0   // minimum resident CTAs per SM requested from ptxas (0: none)
#endif
#ifndef IPMG_PAIR3_TY
#define IPMG_PAIR3_TY 8   // rows per traversal tile (see the kernel); C4 DRAM reads 12.74 -> 8.96 GB
#endif
constexpr int TY = IPMG_PAIR3_TY;
// DOT: the fused r.z variant (its own instantiation: the extra live values would cost the
// plain passes registers -- 96 instead of 78 when it was one kernel)
// FACES = false: the zero-start pass (x_in == nullptr) as its own instantiation without the
// staging and trace code (fewer registers, X-only shared memory)
template <int NPAIR, bool DOT, bool FACES>
__global__ void __launch_bounds__(PC<NPAIR>::NT, DOT ? 6 : IPMG_PAIR3_MINB)
    smooth_pair3_kernel(const float* __restrict__ x_in, const float* __restrict__ b, float* __restrict__ x_out,
                        LevelGeom g, int colour, int gx, int gy,
                        const __grid_constant__ Deltas dl, const double* __restrict__ rdot,
                        double* __restrict__ dot_partial) {
  using C = PC<NPAIR>;
  constexpr int NPAT = C::NPAT;
  // Grid (gx + 1, TY * gz, ceil(gy / TY)) over the colour's pair lattice (gx pairs per
  // row, gy rows, gz planes): the hardware order (x fastest, then y, then z) walks tiles of
  // TY rows -- x, then the tile's rows, then the planes -- so a patch's z-neighbours are
  // gx*TY CTAs away instead of a whole plane (gx*gy) and the neighbour cells of its z-faces
  // are still in L2 (ncu: C4 pass DRAM reads 12.74 -> 8.96 GB, 8.4 GB algorithmic).  The
  // extra x column copies the cells the colour does not cover.
  if ((int)blockIdx.x >= gx) {
    const long long qq = blockIdx.y + (long long)gridDim.y * blockIdx.z;
    copy_uncovered_part<3, float>(x_in, x_out, g, colour, qq * blockDim.x + threadIdx.x,
                                  (long long)gridDim.y * gridDim.z * blockDim.x);
    return;
  }
  const int bxi = blockIdx.x, byi = (int)blockIdx.z * TY + (int)(blockIdx.y % TY), jz = (int)(blockIdx.y / TY);
  if (byi >= gy) return;   // the last tile's missing rows
  const int bzi = g.zsel == 0 ? jz : (g.zsel == 1 ? jz + 1 : (jz == 0 ? 0 : g.znb - 1));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* X = reinterpret_cast<float2*>(smem_raw);
  float* NBs = reinterpret_cast<float*>(smem_raw);                       // aliased with X
  float2* F = reinterpret_cast<float2*>(smem_raw + (C::XB > C::NBB ? C::XB : C::NBB));
  __shared__ Pat<NPAT> P;
  __shared__ __align__(16) float zslot[CELL];   // read by the trace units of a missing neighbour
#if !IPMG_PAIR3_SHFLSTAGE
  __shared__ unsigned long long nba[NPAT * NNB];  // 16-byte aligned source of each staged cell, 0: none
#endif
  const int t = threadIdx.x;
  for (int e = t; e < CELL; e += C::NT) zslot[e] = 0.f;
  // y / z line of this thread (host tables)
  const unsigned ly = __ldg(&g_lines[NPAIR - 1][0][t]), lz = __ldg(&g_lines[NPAIR - 1][1][t]);
  const int ybase = ly == 0xffffffffu ? -1 : (int)ly;
  const int zbase = lz == 0xffffffffu ? -1 : (int)(lz & 0xffff);
  const int zm0 = (lz >> 16) & 0xf, zm1 = (lz >> 20) & 0xf, zq = (lz >> 24) & 0xf;
#if IPMG_PAIR3_SHFLSTAGE
  // patch data of the CTA (x-blocks of NPAT patches, row by, plane bz) in registers of
  // every thread; threads p < NPAT also write the shared copy P, read only after the
  // barrier that opens the trace phase
  int pbase[NPAT], pvalid[NPAT], pvar[NPAT][3];
#pragma unroll
  for (int p = 0; p < NPAT; ++p) {
    const int m0 = g.n[0] / 2 - (colour & 1);
    const int c0y = ((colour >> 1) & 1) + 2 * byi;
    const int c0z = slab_first(g, (colour >> 2) & 1) + 2 * bzi;
    const int j0 = bxi * NPAT + p;
    const bool valid = j0 < m0;
    const int c0x = (colour & 1) + 2 * (valid ? j0 : 0);
    pbase[p] = (int)cell_offset_cells(g, c0x, c0y, c0z);
    pvalid[p] = valid;
    const int gs = g.zoff + c0z;
    pvar[p][0] = (c0x == 0 ? 1 : 0) | (c0x + 2 == g.n[0] ? 2 : 0);
    pvar[p][1] = (c0y == 0 ? 1 : 0) | (c0y + 2 == g.n[1] ? 2 : 0);
    pvar[p][2] = (gs == 0 ? 1 : 0) | (gs + 2 == g.nglob ? 2 : 0);
    if (t == p) {
      P.base[p] = pbase[p];
      P.valid[p] = pvalid[p];
      P.own[p] = (c0z >= 0 ? 1 : 0) | (c0z + 1 < g.n[2] ? 2 : 0);
      P.var[p][0] = pvar[p][0];
      P.var[p][1] = pvar[p][1];
      P.var[p][2] = pvar[p][2];
    }
  }
#if IPMG_PAIR3_BPF
  // L1 prefetch of the b cells of the CTA's patches (read by the x pass; no registers held
  // meanwhile): thread t < 16 NPAIR * BL covers line t % BL of cell t / BL
  {
    constexpr int BL = (CELL * 4 + 127 + 124) / 128;   // lines a cell can touch
    if (t < NPAT * 8 * BL) {
      const int ce = t / BL, ln = t % BL, p = ce >> 3, q = ce & 7;
      int pb = pbase[0], pv = pvalid[0];
#pragma unroll
      for (int pp = 1; pp < NPAT; ++pp)
        if (p == pp) { pb = pbase[pp]; pv = pvalid[pp]; }
      const unsigned long long c0 = reinterpret_cast<unsigned long long>(b + (long long)(pb + dl.pc[q]) * CELL);
      const unsigned long long a = (c0 & ~127ull) + 128ull * ln;
      if (pv && a < c0 + CELL * 4) {
        if (IPMG_PAIR3_BPF == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
        else asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a));
      }
    }
  }
#endif
  if (FACES && x_in != nullptr) {
    // face-neighbour cells -> shared memory: 16-byte cp.async, a warp per cell (lanes on
    // consecutive chunks), each copy widened to the 16-byte boundaries around the cell
    // (inside the vector: its base and end are 16-byte aligned, checked by the launcher).
    // Lane i of warp w first forms the source of entry w + NW i (in parallel); the copy
    // loop takes it by shuffle.  A missing neighbour copies the patch's first cell instead
    // (its trace units read the zero slot): no branch in the copy loop.
    const int lane = t & 31, w = t >> 5;
    constexpr int NW = C::NT / 32, PER = (NPAT * NNB + NW - 1) / NW;
    constexpr int NR = (PER + 31) / 32;   // rounds of 32 entries per warp
    constexpr int CMIN = (CELL * 4 + 15) / 16;   // chunks of a cell at a 16-byte boundary; one more otherwise
    unsigned long long my[NR];   // 16-byte aligned source | (chunk count - CMIN)
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      const int e = w + NW * (32 * rr + lane);
      const int p = e / NNB, k = e - NNB * (e / NNB);
      int cell = pbase[0];
      if (32 * rr + lane < PER && e < NPAT * NNB) {
        int pb = pbase[0], pv = pvalid[0], va = pvar[0][0], vb = pvar[0][1], vc = pvar[0][2];
#pragma unroll
        for (int pp = 1; pp < NPAT; ++pp)
          if (p == pp) { pb = pbase[pp]; pv = pvalid[pp]; va = pvar[pp][0]; vb = pvar[pp][1]; vc = pvar[pp][2]; }
        const int vk = (k >> 3) == 0 ? va : ((k >> 3) == 1 ? vb : vc);
        if (pv && !((vk >> ((k >> 2) & 1)) & 1)) cell = pb + dl.nb[k];
      }
      const unsigned long long a0 = reinterpret_cast<unsigned long long>(x_in + (long long)cell * CELL);
      const unsigned chunks = (CELL * 4 + 4 * (unsigned)((a0 >> 2) & 3) + 15) / 16;
      my[rr] = (a0 & ~15ull) | (unsigned long long)(chunks - CMIN);
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (w + NW * i >= NPAT * NNB) break;
      const unsigned long long ent = __shfl_sync(0xffffffffu, my[i / 32], i % 32);
      const unsigned long long src = ent & ~15ull;
      const int last = CMIN - 1 + (int)(ent & 15ull);   // the cell's last chunk
      float* dst = NBs + (w + NW * i) * SLOTF;
#pragma unroll
      for (int c0 = 0; c0 < (CELL * 4 + 12 + 15) / 16; c0 += 32) {   // the most chunks a cell can need
        const int c = c0 + lane < last ? c0 + lane : last;   // lanes past the end repeat the last chunk
        cp_async<16>(dst + 4 * c, reinterpret_cast<const void*>(src + 16ull * c));
      }
    }
    cp_async_commit();
  } else {
    __syncthreads();   // P before the x pass (no trace phase)
  }
#else
  // patches of the CTA (x-blocks of NPAT patches, row by, plane bz)
  if (t < NPAT) {
    const int p = t;
    const int m0 = g.n[0] / 2 - (colour & 1);
    const int c0y = ((colour >> 1) & 1) + 2 * byi;
    const int c0z = slab_first(g, (colour >> 2) & 1) + 2 * bzi;
    const int j0 = bxi * NPAT + p;
    const bool valid = j0 < m0;
    const int c0x = (colour & 1) + 2 * (valid ? j0 : 0);
    P.base[p] = (int)cell_offset_cells(g, c0x, c0y, c0z);
    P.valid[p] = valid;
    const int gs = g.zoff + c0z;
    P.own[p] = (c0z >= 0 ? 1 : 0) | (c0z + 1 < g.n[2] ? 2 : 0);
    P.var[p][0] = (c0x == 0 ? 1 : 0) | (c0x + 2 == g.n[0] ? 2 : 0);
    P.var[p][1] = (c0y == 0 ? 1 : 0) | (c0y + 2 == g.n[1] ? 2 : 0);
    P.var[p][2] = (gs == 0 ? 1 : 0) | (gs + 2 == g.nglob ? 2 : 0);
  }
  __syncthreads();
  // face-neighbour cells -> shared memory: 16-byte cp.async, a warp per cell (lanes on
  // consecutive chunks).  A copy covers the cell from the 16-byte boundary below it to
  // the first one at or above its end: inside the vector whenever its base and end are
  // 16-byte aligned (checked by the launcher).  First the source of every cell (one
  // thread per cell), then the copies.
  if (FACES && x_in != nullptr) {
    // entry: the 16-byte aligned source address, its low bits the cell's float offset
    // from that boundary (0..3)
    for (int e = t; e < NPAT * NNB; e += C::NT) {
      const int p = e / NNB, k = e % NNB;
      const unsigned long long a0 = reinterpret_cast<unsigned long long>(x_in + (long long)(P.base[p] + dl.nb[k]) * CELL);
      nba[e] = nb_exists(P, p, k) ? (a0 & ~15ull) | ((a0 >> 2) & 3) | 4 : 0ull;
    }
    __syncthreads();
    const int lane = t & 31;
    // unrolled: every copy gets its own address registers (a cp.async holds its source
    // registers until it issues; a rolled loop serialised on them, ncu long_sb stalls)
    constexpr int NW = C::NT / 32, PER = (NPAT * NNB + NW - 1) / NW;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = (t >> 5) + NW * i;
      if (e >= NPAT * NNB) break;
      const unsigned long long ent = nba[e];
      if (ent == 0ull) continue;
      const unsigned long long src = ent & ~15ull;
      const unsigned chunks = (CELL * 4 + 4 * (unsigned)(ent & 3) + 15) / 16;   // the cell plus its offset
#pragma unroll
      for (int c0 = 0; c0 < (CELL * 4 + 12 + 15) / 16; c0 += 32) {
        const int c = c0 + lane;
        if ((unsigned)c < chunks) cp_async<16>(NBs + e * SLOTF + 4 * c, reinterpret_cast<const void*>(src + 16ull * c));
      }
    }
    cp_async_commit();
  }
#endif
  // b rows of this thread's x-line pair (in flight during the trace phase)
  float2 brow[NP];
  {
    const int q0 = t / NL, l0 = t % NL;
    // raw values: the h^{2-d} scaling waits for the loads, so it happens in the x pass
    if (!IPMG_PAIR3_LATE_B && t < NPAIR * NL) load_b_rows(b, P, dl, q0, l0 % NP, l0 / NP, 1.f, brow);
  }
  bool allint = true;
#pragma unroll
  for (int p = 0; p < NPAT; ++p)
#if IPMG_PAIR3_SHFLSTAGE
    if (pvalid[p] && (pvar[p][0] | pvar[p][1] | pvar[p][2])) allint = false;
#else
    if (P.valid[p] && (P.var[p][0] | P.var[p][1] | P.var[p][2])) allint = false;
#endif
  double d = allint ? pair_body<NPAIR, true, DOT, FACES>(x_in, b, x_out, g, P, dl, X, F, NBs, zslot, brow, ybase, zbase, zq, zm0,
                                             zm1, rdot)
                    : pair_body<NPAIR, false, DOT, FACES>(x_in, b, x_out, g, P, dl, X, F, NBs, zslot, brow, ybase, zbase, zq,
                                              zm0, zm1, rdot);
  if (DOT) {
    // fused r.z (colour 0 only: every dof is stored by exactly one patch): deterministic
    // CTA partial (fixed tree), index over the full (x, y, z) patch-pair lattice
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    __shared__ double wsum[C::NT / 32];
    if ((t & 31) == 0) wsum[t >> 5] = d;
    __syncthreads();
    if (t == 0) {
      double sum = 0.0;
      for (int w = 0; w < C::NT / 32; ++w) sum += wsum[w];
      dot_partial[bxi + (long long)gx * (byi + (long long)gy * bzi)] = sum;
    }
  }
}

}  // namespace pair3
#endif
