// NEXT-4 prototype: the fast-diagonalisation line
// transform of the 3D k = 4 smoother, out[m] = sum_i S[i][m] in[i] on lines of NP = 10
// values, on CUDA cores (FFMA2, the pair form of smooth_pair3.cuh) vs on tensor cores
// (mma.sync m16n8k8 TF32 with the 3xTF32 split, fp32-accurate: A = A_hi + A_lo,
// D += A_hi B_hi + A_hi B_lo + A_lo B_hi).  Standalone microbenchmark: a CTA keeps a tile
// of lines in shared memory and applies the transform REPS times (ping-pong between two
// buffers, a barrier per pass -- the line pass as it sits inside the smoother), then
// writes the tile back; results checked against an fp64 host reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tc_proto tools/tc_proto.cu
//   ./tc_proto            (prints one JSON line per variant)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int NP = 10;
constexpr int REPS = 64;
constexpr int LINES = 256;   // lines per CTA tile
__constant__ float cS[NP][NP];   // S[i][m]
__constant__ float cSh[16][16], cSl[16][16];   // tf32 hi / lo of S, zero padded

// ---- CUDA cores: a thread owns 2 lines (float2 pairs), 128 threads = 256 lines
__global__ void __launch_bounds__(128) ffma2_pass(const float* __restrict__ in, float* __restrict__ out) {
  __shared__ float2 buf[2][128][NP + 1];
  const int t = threadIdx.x;
  const float* src = in + (size_t)blockIdx.x * LINES * NP;
  for (int e = t; e < LINES * NP; e += 128) {
    const int l = e / NP, j = e % NP;
    float* p = reinterpret_cast<float*>(&buf[0][l >> 1][j]);
    p[l & 1] = src[e];
  }
  __syncthreads();
  int cur = 0;
  for (int r = 0; r < REPS; ++r) {
    float2 v[NP], w[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) v[j] = buf[cur][t][j];
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < NP; ++i) acc = __ffma2_rn(make_float2(cS[i][m], cS[i][m]), v[i], acc);
      w[m] = acc;
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) buf[cur ^ 1][t][j] = w[j];
    cur ^= 1;
    __syncthreads();
  }
  float* dst = out + (size_t)blockIdx.x * LINES * NP;
  for (int e = t; e < LINES * NP; e += 128) {
    const int l = e / NP, j = e % NP;
    dst[e] = reinterpret_cast<const float*>(&buf[cur][l >> 1][j])[l & 1];
  }
}

// ---- tensor cores: mma.sync.m16n8k8 tf32, 3xTF32.  A warp owns 64 lines = 4 m-tiles of
// 16 lines; K = 16 (10 used), N = 16 (10 used) -> 2 k-steps x 2 n-tiles x 3 = 12 MMAs per tile
__device__ __forceinline__ unsigned tf32(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__global__ void __launch_bounds__(128) mma_pass(const float* __restrict__ in, float* __restrict__ out) {
  constexpr int LP = 17;   // line pitch (odd: conflict-light fragment loads)
  __shared__ float buf[2][LINES][LP];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, q = lane & 3;
  const float* src = in + (size_t)blockIdx.x * LINES * NP;
  for (int e = t; e < LINES * 16; e += 128) {
    const int l = e / 16, j = e % 16;
    buf[0][l][j] = j < NP ? src[l * NP + j] : 0.f;
    buf[1][l][j] = 0.f;
  }
  // B fragments (col-major K x N: b0 = B[k = q][n = g], b1 = B[q + 4][g]) of S hi / lo
  unsigned bh[2][2][2], bl[2][2][2];   // [kstep][ntile][reg]
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      bh[ks][nt][0] = __float_as_uint(cSh[ks * 8 + q][nt * 8 + g]);
      bh[ks][nt][1] = __float_as_uint(cSh[ks * 8 + q + 4][nt * 8 + g]);
      bl[ks][nt][0] = __float_as_uint(cSl[ks * 8 + q][nt * 8 + g]);
      bl[ks][nt][1] = __float_as_uint(cSl[ks * 8 + q + 4][nt * 8 + g]);
    }
  __syncthreads();
  int cur = 0;
  for (int r = 0; r < REPS; ++r) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int l0 = warp * 64 + mt * 16;
      float d[2][4] = {};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const float a0 = buf[cur][l0 + g][ks * 8 + q], a1 = buf[cur][l0 + g + 8][ks * 8 + q];
        const float a2 = buf[cur][l0 + g][ks * 8 + q + 4], a3 = buf[cur][l0 + g + 8][ks * 8 + q + 4];
        unsigned ah[4] = {tf32(a0), tf32(a1), tf32(a2), tf32(a3)};
        unsigned al[4] = {tf32(a0 - __uint_as_float(ah[0])), tf32(a1 - __uint_as_float(ah[1])),
                          tf32(a2 - __uint_as_float(ah[2])), tf32(a3 - __uint_as_float(ah[3]))};
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          mma_tf32(d[nt], al, bh[ks][nt][0], bh[ks][nt][1]);
          mma_tf32(d[nt], ah, bl[ks][nt][0], bl[ks][nt][1]);
          mma_tf32(d[nt], ah, bh[ks][nt][0], bh[ks][nt][1]);
        }
      }
      // D fragment: c0 = D[g][2q], c1 = D[g][2q+1], c2 = D[g+8][2q], c3 = D[g+8][2q+1]
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int m = nt * 8 + 2 * q;
        if (m < NP) {
          buf[cur ^ 1][l0 + g][m] = d[nt][0];
          buf[cur ^ 1][l0 + g + 8][m] = d[nt][2];
        }
        if (m + 1 < NP) {
          buf[cur ^ 1][l0 + g][m + 1] = d[nt][1];
          buf[cur ^ 1][l0 + g + 8][m + 1] = d[nt][3];
        }
      }
    }
    cur ^= 1;
    __syncthreads();
  }
  float* dst = out + (size_t)blockIdx.x * LINES * NP;
  for (int e = t; e < LINES * NP; e += 128) dst[e] = buf[cur][e / NP][e % NP];
}

static float tf32_host(float x) {   // round to nearest, ties away (cvt.rna)
  unsigned u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

int main() {
  const int nblk = 148 * 16;
  const size_t n = (size_t)nblk * LINES * NP;
  // an orthonormal 10x10 (DCT-II basis): powers stay bounded over REPS passes
  float S[NP][NP];
  for (int i = 0; i < NP; ++i)
    for (int m = 0; m < NP; ++m)
      S[i][m] = (float)(std::sqrt((m == 0 ? 1.0 : 2.0) / NP) * std::cos(M_PI * (i + 0.5) * m / NP));
  float Sh[16][16] = {}, Sl[16][16] = {};
  for (int i = 0; i < NP; ++i)
    for (int m = 0; m < NP; ++m) {
      Sh[i][m] = tf32_host(S[i][m]);
      Sl[i][m] = tf32_host(S[i][m] - Sh[i][m]);
    }
  cudaMemcpyToSymbol(cS, S, sizeof(S));
  cudaMemcpyToSymbol(cSh, Sh, sizeof(Sh));
  cudaMemcpyToSymbol(cSl, Sl, sizeof(Sl));
  std::vector<float> h(n);
  srand(1);
  for (auto& v : h) v = (float)rand() / RAND_MAX * 2.f - 1.f;
  // fp64 host reference for the first 64 lines after REPS passes
  std::vector<double> ref(64 * NP);
  for (int l = 0; l < 64; ++l) {
    double v[NP], w[NP];
    for (int j = 0; j < NP; ++j) v[j] = h[l * NP + j];
    for (int r = 0; r < REPS; ++r) {
      for (int m = 0; m < NP; ++m) {
        w[m] = 0;
        for (int i = 0; i < NP; ++i) w[m] += (double)S[i][m] * v[i];
      }
      for (int j = 0; j < NP; ++j) v[j] = w[j];
    }
    for (int j = 0; j < NP; ++j) ref[l * NP + j] = v[j];
  }
  float *din, *dout;
  cudaMalloc(&din, n * 4);
  cudaMalloc(&dout, n * 4);
  cudaMemcpy(din, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    auto launch = [&] {
      if (variant == 0) ffma2_pass<<<nblk, 128>>>(din, dout);
      else mma_pass<<<nblk, 128>>>(din, dout);
    };
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int it = 20;
    for (int w = 0; w < it; ++w) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    std::vector<float> o(64 * NP);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (size_t i = 0; i < o.size(); ++i) {
      err = std::fmax(err, std::fabs(o[i] - ref[i]));
      mx = std::fmax(mx, std::fabs(ref[i]));
    }
    const double lines = (double)nblk * LINES * REPS;
    printf("{\"variant\": \"%s\", \"ms\": %.4f, \"glines_per_s\": %.2f, \"useful_tflops\": %.2f, "
           "\"rel_err_after_%d_passes\": %.3g, \"err\": \"%s\"}\n",
           variant == 0 ? "ffma2_pair" : "mma_sync_3xtf32", ms, lines / (ms * 1e-3) / 1e9,
           lines * 2.0 * NP * NP / (ms * 1e-3) / 1e12, REPS, err / mx, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
