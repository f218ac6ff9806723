// Host launchers of the degree-independent kernels (blas.cu).
#pragma once
#include "common.cuh"

namespace ipmg {

constexpr int RED_BLOCKS = 2 * 148;   // fixed reduction grid (deterministic)
constexpr int RED_THREADS = 512;

struct CoarseDesc {
  static constexpr int NMAX = 16;     // 2 cells x 8 nodes per direction
  int dim, nc;
  int n0[3];                          // level-0 cells per direction (1 or 2)
  int N[3];                           // global nodes per direction (N[2] = 1 in 2D)
  double scale;                       // h0^(2-d)
};

cudaError_t dot_partial(int prec_a, int prec_b, const void* a, const void* b, long long n, double* partial,
                        cudaStream_t s);
cudaError_t finalize(const double* partial, double* out, cudaStream_t s, long long np = -1);
cudaError_t cg_update_xr(double* x, double* r, const double* p, const double* q, long long n, const double* sc,
                         int i_rz, int i_pq, double* partial, cudaStream_t s, float* r32 = nullptr);
cudaError_t cg_update_p32(double* p, const float* z, long long n, const double* sc, int i_new, int i_old,
                          cudaStream_t s);
// x += alpha p_old ; p = z32 + beta p_old  (alpha = sc[i_rz]/sc[i_pq], beta = sc[i_new]/sc[i_rz])
cudaError_t cg_update_xp32(double* x, double* p, const float* z, long long n, const double* sc, int i_new, int i_rz,
                           int i_pq, cudaStream_t s);
// x += alpha p  (alpha = sc[i_rz]/sc[i_pq])
cudaError_t cg_update_x(double* x, const double* p, long long n, const double* sc, int i_rz, int i_pq,
                        cudaStream_t s);
cudaError_t cg_update_p(double* p, const double* z, long long n, const double* sc, int i_new, int i_old,
                        cudaStream_t s);
cudaError_t cast_f2d_dot(const float* zf, double* zd, const double* r, long long n, double* partial, cudaStream_t s);
cudaError_t cast(int prec_in, int prec_out, const void* in, void* out, long long n, cudaStream_t s);
cudaError_t permute(int prec, bool to_cellwise, const void* in, void* out, const LevelGeom& g, int cell, long long n,
                    cudaStream_t s);
cudaError_t sum_ranks(int prec, void* buf, const void* scratch, int nranks, int rank, long long n, cudaStream_t s);
cudaError_t gather_sum(const double* g, int nranks, int nv, double* out, cudaStream_t s);
cudaError_t mgs_axpy_dot(double* w, const double* v, const double* u, long long n, const double* h, int ih,
                         double* partial, cudaStream_t s);
cudaError_t scale_vec(double* v, const double* w, long long n, const double* nrm2, double scale, float* v32,
                      cudaStream_t s);
cudaError_t combine(double* x, const double* const* Z, const double* y, int m, long long n, cudaStream_t s);
cudaError_t to_host(double* dst_mapped, const double* src, int n, cudaStream_t s);
cudaError_t pattern_fill(double* b, const double* pat, int cell, long long n, cudaStream_t s);
cudaError_t sep_fill(double* b, const double* gx, const double* gy, const double* gz, const LevelGeom& g, int nc,
                     int dim, double scale, long long n, cudaStream_t s);
cudaError_t coarse_solve(int prec, const void* b, void* x, const CoarseDesc& cd, const void* const S[3],
                         const void* const L[3], cudaStream_t s);

}  // namespace ipmg
