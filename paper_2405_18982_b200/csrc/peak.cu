// CUDA-core peak microbenchmark (measurement utility of SURVEY.md 8(d) / DESIGN.md
// "Roofline"): the ALU denominator of the smoother and operator rooflines, measured on
// the device instead of derived from unit counts.  Every thread runs NCHAIN independent
// FMA dependency chains back to back (enough independent work to cover the pipe
// latency at full occupancy); flops = 2 per FMA (4 per FFMA2).  Timed with CUDA events
// on a private stream after one warm-up launch; the result is the best of `reps`.
#include <cuda_runtime.h>

#include <algorithm>

#include "ipmg.h"

namespace {

constexpr int NCHAIN = 8;
constexpr int ITERS = 2048;
constexpr int THREADS = 256;

__global__ void __launch_bounds__(THREADS) peak_ffma2(float* out, float a, float b) {
  float2 acc[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) acc[c] = make_float2(threadIdx.x * 1e-7f + c, c * 0.5f);
  const float2 va = make_float2(a, a), vb = make_float2(b, b);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) acc[c] = __ffma2_rn(acc[c], va, vb);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += acc[c].x + acc[c].y;
  if (s == 1234.5f) out[threadIdx.x] = s;   // never true; keeps the chains live
}

__global__ void __launch_bounds__(THREADS) peak_ffma(float* out, float a, float b) {
  float acc[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) acc[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += acc[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(THREADS) peak_dfma(double* out, double a, double b) {
  double acc[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += acc[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

}  // namespace

extern "C" ipmg_status ipmg_alu_peak(int device, int kind, int reps, double* tflops) {
  if (!tflops || kind < 0 || kind > 2) return IPMG_ERR_INVALID_ARG;
  if (reps < 1) reps = 5;
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return IPMG_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return IPMG_ERR_CUDA;
  ipmg_status st = IPMG_OK;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8;            // 8 x 256 threads = 2048 threads per SM (full occupancy)
  void* buf = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaMalloc(&buf, THREADS * sizeof(double)) != cudaSuccess || cudaStreamCreate(&s) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    st = IPMG_ERR_CUDA;
  } else {
    const double fma_per_thread = double(ITERS) * NCHAIN * (kind == 0 ? 2 : 1);   // FFMA2 = 2 FMAs
    const double flops = 2.0 * fma_per_thread * blocks * THREADS;
    double best = 0.0;
    for (int r = 0; r <= reps; ++r) {   // r = 0 is the warm-up
      cudaEventRecord(e0, s);
      if (kind == 0) peak_ffma2<<<blocks, THREADS, 0, s>>>((float*)buf, 0.999f, 1e-3f);
      else if (kind == 1) peak_ffma<<<blocks, THREADS, 0, s>>>((float*)buf, 0.999f, 1e-3f);
      else peak_dfma<<<blocks, THREADS, 0, s>>>((double*)buf, 0.999, 1e-3);
      cudaEventRecord(e1, s);
      if (cudaEventSynchronize(e1) != cudaSuccess) { st = IPMG_ERR_CUDA; break; }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms > 0.f) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    *tflops = best;
    if (cudaGetLastError() != cudaSuccess) st = IPMG_ERR_CUDA;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  if (buf) cudaFree(buf);
  cudaSetDevice(prev);
  return st;
}
