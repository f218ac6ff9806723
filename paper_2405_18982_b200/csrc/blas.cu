// Degree-independent kernels: precision casts, deterministic dot products, the
// fused PCG vector updates, layout permutation, right-hand side and the coarse
// fast-diagonalisation solve.
//
// Reductions are deterministic: a fixed grid of RED_BLOCKS blocks, each
// accumulating a fixed strided subset in fp64 and reducing in shared memory
// with a fixed tree; a single-block finalize sums the partials in order.
#include "blas.cuh"

namespace ipmg {

namespace {

template <typename T>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  // warp shuffle tree, then one warp over the per-warp sums
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;   // valid in thread 0
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(RED_THREADS) dot_partial_kernel(const TA* __restrict__ a, const TB* __restrict__ b,
                                                                   long long n, double* __restrict__ partial) {
  __shared__ double sh[32];
  double s = 0.0;
  long long start = 0;
  if (sizeof(TA) == 8 && sizeof(TB) == 4 &&
      ((reinterpret_cast<unsigned long long>(a) & 15) | (reinterpret_cast<unsigned long long>(b) & 7)) == 0) {
    // r . z32 of the mixed PCG: double2 / float2 accesses
    const long long n2 = n >> 1;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const float2* b2 = reinterpret_cast<const float2*>(b);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
      const double2 u = __ldg(a2 + i);
      const float2 v = __ldg(b2 + i);
      s = fma(u.x, (double)v.x, s);
      s = fma(u.y, (double)v.y, s);
    }
    start = n2 << 1;
  }
  for (long long i = start + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s = fma((double)a[i], (double)b[i], s);
  s = block_sum<double>(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) finalize_kernel(const double* __restrict__ partial, long long np,
                                                                double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < np; i += blockDim.x) s += partial[i];
  s = block_sum<double>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

// x += alpha p ; r -= alpha q ; partial ||r||^2   with alpha = s[i_rz] / s[i_pq];
// r32 != nullptr: also r32 = (float) r (the fp32 V-cycle input).
// VEC: 16-byte (double2) accesses, two pairs per thread and iteration in flight
// (the scalar grid-stride loop kept ~30 KB per SM in flight: 5.2 TB/s under ncu)
template <bool VEC, bool DOX>
__global__ void __launch_bounds__(RED_THREADS) cg_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                             const double* __restrict__ p, const double* __restrict__ q,
                                                             long long n, const double* __restrict__ sc, int i_rz,
                                                             int i_pq, double* __restrict__ partial,
                                                             float* __restrict__ r32) {
  __shared__ double sh[32];
  const double alpha = sc[i_rz] / sc[i_pq];
  double s = 0.0;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (VEC) {
    const long long n2 = n >> 1;   // double2 pairs
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    float2* f2 = reinterpret_cast<float2*>(r32);
    for (long long i = t0; i < n2; i += 2 * nt) {
      const long long j = i + nt;
      const bool two = j < n2;
      double2 xa{}, pa{}, xb{}, pb{};
      if (DOX) { xa = x2[i]; pa = __ldg(p2 + i); }
      const double2 qa = __ldg(q2 + i), ra = r2[i];
      double2 qb, rb;
      if (two) {
        if (DOX) { xb = x2[j]; pb = __ldg(p2 + j); }
        qb = __ldg(q2 + j);
        rb = r2[j];
      }
      double2 ro;
      ro.x = fma(-alpha, qa.x, ra.x);
      ro.y = fma(-alpha, qa.y, ra.y);
      if (DOX) x2[i] = make_double2(fma(alpha, pa.x, xa.x), fma(alpha, pa.y, xa.y));
      r2[i] = ro;
      if (r32) f2[i] = make_float2((float)ro.x, (float)ro.y);
      s = fma(ro.x, ro.x, s);
      s = fma(ro.y, ro.y, s);
      if (two) {
        ro.x = fma(-alpha, qb.x, rb.x);
        ro.y = fma(-alpha, qb.y, rb.y);
        if (DOX) x2[j] = make_double2(fma(alpha, pb.x, xb.x), fma(alpha, pb.y, xb.y));
        r2[j] = ro;
        if (r32) f2[j] = make_float2((float)ro.x, (float)ro.y);
        s = fma(ro.x, ro.x, s);
        s = fma(ro.y, ro.y, s);
      }
    }
    done = n2 << 1;
  }
  for (long long i = done + t0; i < n; i += nt) {
    if (DOX) x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    if (r32) r32[i] = (float)ri;
    s = fma(ri, ri, s);
  }
  s = block_sum<double>(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// p = (double) z32 + beta p (beta = s[i_new] / s[i_old]; i_old < 0: beta = 0)
__global__ void cg_p32_kernel(double* __restrict__ p, const float* __restrict__ z, long long n,
                              const double* __restrict__ sc, int i_new, int i_old) {
  const double beta = i_old < 0 ? 0.0 : sc[i_new] / sc[i_old];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = i_old < 0 ? (double)z[i] : fma(beta, p[i], (double)z[i]);
}

// deferred CG solution update fused with the direction update (mixed precision):
// x += alpha p_old (alpha = s[i_rz] / s[i_pq], the step cg_xr_kernel took with
// DOX = false), then p = (double) z32 + beta p_old (beta = s[i_new] / s[i_rz]).
// The same fma on the same p_old as in cg_xr_kernel: x is bit-identical, and the
// x/p streams are read once instead of twice per iteration.
template <bool VEC>
__global__ void cg_xp32_kernel(double* __restrict__ x, double* __restrict__ p, const float* __restrict__ z,
                               long long n, const double* __restrict__ sc, int i_new, int i_rz, int i_pq) {
  const double alpha = sc[i_rz] / sc[i_pq], beta = sc[i_new] / sc[i_rz];
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  const long long n2 = VEC ? n >> 1 : 0;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* p2 = reinterpret_cast<double2*>(p);
  const float2* z2 = reinterpret_cast<const float2*>(z);
  for (long long i = t0; i < n2; i += 2 * nt) {   // two pairs in flight per thread
    const long long j = i + nt;
    const bool two = j < n2;
    const double2 xo = x2[i], po = p2[i];
    const float2 zz = __ldg(z2 + i);
    double2 xo2{}, po2{};
    float2 zz2{};
    if (two) { xo2 = x2[j]; po2 = p2[j]; zz2 = __ldg(z2 + j); }
    x2[i] = make_double2(fma(alpha, po.x, xo.x), fma(alpha, po.y, xo.y));
    p2[i] = make_double2(fma(beta, po.x, (double)zz.x), fma(beta, po.y, (double)zz.y));
    if (two) {
      x2[j] = make_double2(fma(alpha, po2.x, xo2.x), fma(alpha, po2.y, xo2.y));
      p2[j] = make_double2(fma(beta, po2.x, (double)zz2.x), fma(beta, po2.y, (double)zz2.y));
    }
  }
  for (long long i = (n2 << 1) + t0; i < n; i += nt) {
    const double po = p[i];
    x[i] = fma(alpha, po, x[i]);
    p[i] = fma(beta, po, (double)z[i]);
  }
}

// x += alpha p (alpha = s[i_rz] / s[i_pq]): the deferred update of the last step
__global__ void cg_x_kernel(double* __restrict__ x, const double* __restrict__ p, long long n,
                            const double* __restrict__ sc, int i_rz, int i_pq) {
  const double alpha = sc[i_rz] / sc[i_pq];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = fma(alpha, p[i], x[i]);
}

// p = z + beta p, beta = s[i_new] / s[i_old]
__global__ void cg_p_kernel(double* __restrict__ p, const double* __restrict__ z, long long n,
                            const double* __restrict__ sc, int i_new, int i_old) {
  const double beta = sc[i_new] / sc[i_old];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

// zd = (double) zf ; partial r . zd
__global__ void __launch_bounds__(RED_THREADS) cast_dot_kernel(const float* __restrict__ zf, double* __restrict__ zd,
                                                                const double* __restrict__ r, long long n,
                                                                double* __restrict__ partial) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double z = (double)zf[i];
    zd[i] = z;
    s = fma(r[i], z, s);
  }
  s = block_sum<double>(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// ---- GMRES (modified Gram-Schmidt, right preconditioning)
// w -= h[ih] * v ; partial of w . u (u == nullptr: w . w) -- one MGS step fused
// with the dot product of the next step
__global__ void __launch_bounds__(RED_THREADS) mgs_axpy_dot_kernel(double* __restrict__ w, const double* __restrict__ v,
                                                                    const double* __restrict__ u, long long n,
                                                                    const double* __restrict__ h, int ih,
                                                                    double* __restrict__ partial) {
  __shared__ double sh[32];
  const double c = h[ih];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double wi = fma(-c, v[i], w[i]);
    w[i] = wi;
    s = fma(wi, u ? u[i] : wi, s);
  }
  s = block_sum<double>(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// v = w / sqrt(nrm2[0]) ; v32 = (float) v (the next V-cycle input) when v32 != nullptr;
// nrm2 == nullptr: v = w * scale
__global__ void scale_kernel(double* __restrict__ v, const double* __restrict__ w, long long n,
                             const double* __restrict__ nrm2, double scale, float* __restrict__ v32) {
  const double f = nrm2 ? 1.0 / sqrt(nrm2[0]) : scale;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double vi = w[i] * f;
    v[i] = vi;
    if (v32) v32[i] = (float)vi;
  }
}

// x = sum_i y[i] Z[i] (i < m), fixed order
__global__ void combine_kernel(double* __restrict__ x, const double* const* __restrict__ Z, const double* __restrict__ y,
                               int m, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(y[j], Z[j][i], s);
    x[i] = s;
  }
}

template <typename TI, typename TO>
__global__ void cast_kernel(const TI* __restrict__ in, TO* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (TO)in[i];
}

// to_cellwise: out[cell_lex*cell + l] = in[lib(cell)*cell + l]; from_cellwise the inverse
template <typename T, bool TO_CW>
__global__ void permute_kernel(const T* __restrict__ in, T* __restrict__ out, LevelGeom g, int cell, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / cell;
    const int l = (int)(e % cell);
    const int cx = (int)(c % g.n[0]);
    const int cy = (int)((c / g.n[0]) % g.n[1]);
    const int cz = (int)(c / ((long long)g.n[0] * g.n[1]));
    const long long lib = cell_offset_cells(g, cx, cy, cz) * cell + l;
    if (TO_CW) out[e] = in[lib];
    else out[lib] = in[e];
  }
}

// b = scale * gx (x) gy (x) gz per cell (separable manufactured right-hand side); the
// 1D tables are over GLOBAL cells, the slab offset zoff applies to the slowest axis.
__global__ void sep_fill_kernel(double* __restrict__ b, const double* __restrict__ gx,
                                const double* __restrict__ gy, const double* __restrict__ gz, LevelGeom g,
                                int nc, int dim, double scale, long long n) {
  const int cell = dim == 3 ? nc * nc * nc : nc * nc;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / cell;
    const int l = (int)(e % cell);
    const int cx = (int)(c % g.n[0]);
    const int cy = (int)((c / g.n[0]) % g.n[1]);
    const int cz = (int)(c / ((long long)g.n[0] * g.n[1]));
    const int ix = l % nc, iy = (l / nc) % nc, iz = l / (nc * nc);
    double v = scale * gx[cx * nc + ix];
    if (dim == 3) v *= gy[cy * nc + iy] * gz[(cz + g.zoff) * nc + iz];
    else v *= gy[(cy + g.zoff) * nc + iy];
    b[cell_offset_cells(g, cx, cy, cz) * cell + l] = v;
  }
}

__global__ void pattern_fill_kernel(double* __restrict__ b, const double* __restrict__ pat, int cell, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    b[e] = pat[e % cell];
}

// Coarse solve x0 = A_0^{-1} b0 by global fast diagonalisation on level 0
// (lexicographic cells); one CTA, tensor of N0 x N1 (x N2) global nodes in smem.
template <typename T>
__global__ void coarse_fd_kernel(const T* __restrict__ b, T* __restrict__ x, CoarseDesc cd, const T* __restrict__ S0,
                                 const T* __restrict__ S1, const T* __restrict__ S2, const T* __restrict__ l0,
                                 const T* __restrict__ l1, const T* __restrict__ l2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  const int N0 = cd.N[0], N1 = cd.N[1], N2 = cd.N[2], nc = cd.nc, d = cd.dim;
  const int total = N0 * N1 * N2;
  const int cell = (d == 2) ? nc * nc : nc * nc * nc;
  const T* S[3] = {S0, S1, S2};
  const T* L[3] = {l0, l1, l2};
  // load: global node (g0,g1,g2) <- cell (g/nc), node (g%nc)
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int g0 = e % N0, g1 = (e / N0) % N1, g2 = e / (N0 * N1);
    const int c0 = g0 / nc, c1 = g1 / nc, c2 = g2 / nc;
    const int loc = (g0 % nc) + nc * ((g1 % nc) + nc * (g2 % nc));
    const long long off = ((long long)c0 + cd.n0[0] * (c1 + (long long)cd.n0[1] * c2)) * cell + loc;
    X[e] = (T)cd.scale * b[off];
  }
  __syncthreads();
  const int Ns[3] = {N0, N1, N2};
  const int strides[3] = {1, N0, N0 * N1};
  // forward S^T along each direction, divide, S back
  for (int pass = 0; pass < 2 * d + 1; ++pass) {
    if (pass == d) {
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int g0 = e % N0, g1 = (e / N0) % N1, g2 = e / (N0 * N1);
        T ls = L[0][g0] + L[1][g1];
        if (d == 3) ls += L[2][g2];
        X[e] = X[e] / ls;
      }
      __syncthreads();
      continue;
    }
    const bool fwd = pass < d;
    const int a = fwd ? pass : (2 * d - pass);
    const int N = Ns[a], st = strides[a];
    const int nlines = total / N;
    for (int li = threadIdx.x; li < nlines; li += blockDim.x) {
      // base of line li along a
      int base;
      if (a == 0) base = li * N0;
      else if (a == 1) base = (li % N0) + (li / N0) * N0 * N1;
      else base = li;
      T v[CoarseDesc::NMAX], w[CoarseDesc::NMAX];
      for (int j = 0; j < N; ++j) v[j] = X[base + j * st];
      for (int i = 0; i < N; ++i) {
        T acc = T(0);
        for (int j = 0; j < N; ++j) acc += (fwd ? S[a][j * N + i] : S[a][i * N + j]) * v[j];
        w[i] = acc;
      }
      for (int j = 0; j < N; ++j) X[base + j * st] = w[j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int g0 = e % N0, g1 = (e / N0) % N1, g2 = e / (N0 * N1);
    const int c0 = g0 / nc, c1 = g1 / nc, c2 = g2 / nc;
    const int loc = (g0 % nc) + nc * ((g1 % nc) + nc * (g2 % nc));
    const long long off = ((long long)c0 + cd.n0[0] * (c1 + (long long)cd.n0[1] * c2)) * cell + loc;
    x[off] = X[e];
  }
}

// buf = sum over ranks in rank order; the own block is buf itself, the others
// are packed (rank order, own skipped) in scratch -- deterministic and
// identical on every rank
template <typename T>
__global__ void sum_ranks_kernel(T* __restrict__ buf, const T* __restrict__ scratch, int nranks, int rank,
                                 long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    T s = T(0);
    int j = 0;
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) s += buf[i];
      else s += scratch[(long long)(j++) * n + i];
    }
    buf[i] = s;
  }
}

// out[v] = sum_r g[r * nv + v] in rank order (allgathered per-rank scalars)
__global__ void gather_sum_kernel(const double* __restrict__ g, int nranks, int nv, double* __restrict__ out) {
  const int v = threadIdx.x;
  if (v >= nv) return;
  double s = 0.0;
  for (int r = 0; r < nranks; ++r) s += g[r * nv + v];
  out[v] = s;
}

inline int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 8 * 148) g = 8 * 148;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

cudaError_t dot_partial(int prec_a, int prec_b, const void* a, const void* b, long long n, double* partial,
                        cudaStream_t s) {
  if (prec_a == 0 && prec_b == 0)
    dot_partial_kernel<double, double><<<RED_BLOCKS, RED_THREADS, 0, s>>>((const double*)a, (const double*)b, n, partial);
  else if (prec_a == 1 && prec_b == 1)
    dot_partial_kernel<float, float><<<RED_BLOCKS, RED_THREADS, 0, s>>>((const float*)a, (const float*)b, n, partial);
  else if (prec_a == 0 && prec_b == 1)
    dot_partial_kernel<double, float><<<RED_BLOCKS, RED_THREADS, 0, s>>>((const double*)a, (const float*)b, n, partial);
  else
    dot_partial_kernel<float, double><<<RED_BLOCKS, RED_THREADS, 0, s>>>((const float*)a, (const double*)b, n, partial);
  return cudaGetLastError();
}

cudaError_t finalize(const double* partial, double* out, cudaStream_t s, long long np) {
  finalize_kernel<<<1, RED_THREADS, 0, s>>>(partial, np < 0 ? RED_BLOCKS : np, out);
  return cudaGetLastError();
}

cudaError_t cg_update_p32(double* p, const float* z, long long n, const double* sc, int i_new, int i_old,
                          cudaStream_t s) {
  cg_p32_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, z, n, sc, i_new, i_old);
  return cudaGetLastError();
}

cudaError_t cg_update_xr(double* x, double* r, const double* p, const double* q, long long n, const double* sc,
                         int i_rz, int i_pq, double* partial, cudaStream_t s, float* r32) {
  const bool vec = ((reinterpret_cast<unsigned long long>(x) | reinterpret_cast<unsigned long long>(r) |
                     reinterpret_cast<unsigned long long>(p) | reinterpret_cast<unsigned long long>(q)) & 15) == 0 &&
                   (reinterpret_cast<unsigned long long>(r32) & 7) == 0;
  if (x == nullptr) {   // solution update deferred (cg_update_xp32 / cg_update_x)
    if (vec) cg_xr_kernel<true, false><<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, q, n, sc, i_rz, i_pq, partial, r32);
    else cg_xr_kernel<false, false><<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, q, n, sc, i_rz, i_pq, partial, r32);
  } else {
    if (vec) cg_xr_kernel<true, true><<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, q, n, sc, i_rz, i_pq, partial, r32);
    else cg_xr_kernel<false, true><<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, q, n, sc, i_rz, i_pq, partial, r32);
  }
  return cudaGetLastError();
}

cudaError_t cg_update_xp32(double* x, double* p, const float* z, long long n, const double* sc, int i_new, int i_rz,
                           int i_pq, cudaStream_t s) {
  const bool vec = ((reinterpret_cast<unsigned long long>(x) | reinterpret_cast<unsigned long long>(p)) & 15) == 0 &&
                   (reinterpret_cast<unsigned long long>(z) & 7) == 0;
  if (vec) cg_xp32_kernel<true><<<grid_for(n, 256), 256, 0, s>>>(x, p, z, n, sc, i_new, i_rz, i_pq);
  else cg_xp32_kernel<false><<<grid_for(n, 256), 256, 0, s>>>(x, p, z, n, sc, i_new, i_rz, i_pq);
  return cudaGetLastError();
}

cudaError_t cg_update_x(double* x, const double* p, long long n, const double* sc, int i_rz, int i_pq,
                        cudaStream_t s) {
  cg_x_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, p, n, sc, i_rz, i_pq);
  return cudaGetLastError();
}

cudaError_t cg_update_p(double* p, const double* z, long long n, const double* sc, int i_new, int i_old,
                        cudaStream_t s) {
  cg_p_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, z, n, sc, i_new, i_old);
  return cudaGetLastError();
}

cudaError_t cast_f2d_dot(const float* zf, double* zd, const double* r, long long n, double* partial, cudaStream_t s) {
  cast_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(zf, zd, r, n, partial);
  return cudaGetLastError();
}

cudaError_t cast(int prec_in, int prec_out, const void* in, void* out, long long n, cudaStream_t s) {
  if (prec_in == prec_out) return cudaMemcpyAsync(out, in, n * (prec_in == 0 ? 8 : 4), cudaMemcpyDeviceToDevice, s);
  if (prec_in == 0)
    cast_kernel<double, float><<<grid_for(n, 256), 256, 0, s>>>((const double*)in, (float*)out, n);
  else
    cast_kernel<float, double><<<grid_for(n, 256), 256, 0, s>>>((const float*)in, (double*)out, n);
  return cudaGetLastError();
}

cudaError_t permute(int prec, bool to_cellwise, const void* in, void* out, const LevelGeom& g, int cell, long long n,
                    cudaStream_t s) {
  const int grid = grid_for(n, 256);
  if (prec == 0) {
    if (to_cellwise) permute_kernel<double, true><<<grid, 256, 0, s>>>((const double*)in, (double*)out, g, cell, n);
    else permute_kernel<double, false><<<grid, 256, 0, s>>>((const double*)in, (double*)out, g, cell, n);
  } else {
    if (to_cellwise) permute_kernel<float, true><<<grid, 256, 0, s>>>((const float*)in, (float*)out, g, cell, n);
    else permute_kernel<float, false><<<grid, 256, 0, s>>>((const float*)in, (float*)out, g, cell, n);
  }
  return cudaGetLastError();
}

cudaError_t sum_ranks(int prec, void* buf, const void* scratch, int nranks, int rank, long long n, cudaStream_t s) {
  if (prec == 0)
    sum_ranks_kernel<double><<<grid_for(n, 256), 256, 0, s>>>((double*)buf, (const double*)scratch, nranks, rank, n);
  else
    sum_ranks_kernel<float><<<grid_for(n, 256), 256, 0, s>>>((float*)buf, (const float*)scratch, nranks, rank, n);
  return cudaGetLastError();
}

cudaError_t gather_sum(const double* g, int nranks, int nv, double* out, cudaStream_t s) {
  gather_sum_kernel<<<1, 32, 0, s>>>(g, nranks, nv, out);
  return cudaGetLastError();
}

cudaError_t mgs_axpy_dot(double* w, const double* v, const double* u, long long n, const double* h, int ih,
                         double* partial, cudaStream_t s) {
  mgs_axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(w, v, u, n, h, ih, partial);
  return cudaGetLastError();
}

cudaError_t scale_vec(double* v, const double* w, long long n, const double* nrm2, double scale, float* v32,
                      cudaStream_t s) {
  scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, w, n, nrm2, scale, v32);
  return cudaGetLastError();
}

cudaError_t combine(double* x, const double* const* Z, const double* y, int m, long long n, cudaStream_t s) {
  combine_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, Z, y, m, n);
  return cudaGetLastError();
}

// small results to MAPPED pinned host memory by a kernel store (PCIe posted
// writes): a cudaMemcpy D2H would queue behind bulk copies on the copy engine
// (e.g. a concurrent download of the previous solution)
__global__ void to_host_kernel(double* __restrict__ dst, const double* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}
cudaError_t to_host(double* dst_mapped, const double* src, int n, cudaStream_t s) {
  to_host_kernel<<<1, 64, 0, s>>>(dst_mapped, src, n);
  return cudaGetLastError();
}

cudaError_t sep_fill(double* b, const double* gx, const double* gy, const double* gz, const LevelGeom& g, int nc,
                     int dim, double scale, long long n, cudaStream_t s) {
  sep_fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(b, gx, gy, gz, g, nc, dim, scale, n);
  return cudaGetLastError();
}

cudaError_t pattern_fill(double* b, const double* pat, int cell, long long n, cudaStream_t s) {
  pattern_fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(b, pat, cell, n);
  return cudaGetLastError();
}

cudaError_t coarse_solve(int prec, const void* b, void* x, const CoarseDesc& cd, const void* const S[3],
                         const void* const L[3], cudaStream_t s) {
  const size_t bytes = (size_t)cd.N[0] * cd.N[1] * cd.N[2] * (prec == 0 ? 8 : 4);
  if (prec == 0) {
    cudaFuncSetAttribute(coarse_fd_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    coarse_fd_kernel<double><<<1, 256, bytes, s>>>((const double*)b, (double*)x, cd, (const double*)S[0],
                                                   (const double*)S[1], (const double*)S[2], (const double*)L[0],
                                                   (const double*)L[1], (const double*)L[2]);
  } else {
    cudaFuncSetAttribute(coarse_fd_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    coarse_fd_kernel<float><<<1, 256, bytes, s>>>((const float*)b, (float*)x, cd, (const float*)S[0],
                                                  (const float*)S[1], (const float*)S[2], (const float*)L[0],
                                                  (const float*)L[1], (const float*)L[2]);
  }
  return cudaGetLastError();
}

}  // namespace ipmg
