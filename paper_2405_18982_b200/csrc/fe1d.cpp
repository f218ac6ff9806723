#include <cstdlib>
// Host-side 1D FE setup; see fe1d.hpp for the paper passages each table follows.
#include "fe1d.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace ipmg {

namespace {

// Legendre P_n(x) and P_n'(x) by the three-term recurrence.
void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { p = 1.0; dp = 0.0; return; }
  for (int m = 1; m < n; ++m) {
    double p2 = ((2.0 * m + 1.0) * x * p1 - m * p0) / (m + 1.0);
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  // derivative from n (x P_n - P_{n-1}) / (x^2 - 1); only used away from +-1
  dp = n * (x * p1 - p0) / (x * x - 1.0);
}

// k+1 Gauss-Lobatto points on [0,1]: endpoints plus the roots of P_k'
// (Newton with the Legendre ODE for P_k'').  PAPER.md:601.
std::vector<double> gll(int k) {
  std::vector<double> x(k + 1);
  x[0] = -1.0;
  x[k] = 1.0;
  for (int j = 1; j < k; ++j) {
    double t = -std::cos(M_PI * j / k);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre(k, t, p, dp);
      double d2p = (2.0 * t * dp - k * (k + 1.0) * p) / (1.0 - t * t);
      double dt = dp / d2p;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[j] = t;
  }
  std::sort(x.begin(), x.end());
  for (auto& v : x) v = 0.5 * (v + 1.0);
  // exact symmetry about 1/2
  for (int j = 0; j < (k + 1) / 2; ++j) {
    double s = 0.5 * (x[j] + (1.0 - x[k - j]));
    x[j] = s;
    x[k - j] = 1.0 - s;
  }
  if (k % 2 == 0) x[k / 2] = 0.5;
  x[0] = 0.0;
  x[k] = 1.0;
  return x;
}

// n-point Gauss-Legendre rule on [0,1].
void gauss(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double p = 0, dp = 0;
    for (int it = 0; it < 100; ++it) {
      legendre(n, t, p, dp);
      double dt = p / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    legendre(n, t, p, dp);
    x[i] = 0.5 * (1.0 - t);
    w[i] = 1.0 / ((1.0 - t * t) * dp * dp);     // (2/((1-t^2)P'^2)) / 2
  }
}

// Lagrange basis on `nodes`: value and derivative of phi_j at x.
void lagrange(const std::vector<double>& nodes, double x, std::vector<double>& v,
              std::vector<double>& d) {
  const int n = (int)nodes.size();
  v.assign(n, 0.0);
  d.assign(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double den = 1.0, num = 1.0, dsum = 0.0;
    for (int m = 0; m < n; ++m) {
      if (m == j) continue;
      den *= nodes[j] - nodes[m];
      num *= x - nodes[m];
    }
    for (int a = 0; a < n; ++a) {
      if (a == j) continue;
      double pr = 1.0;
      for (int m = 0; m < n; ++m)
        if (m != j && m != a) pr *= x - nodes[m];
      dsum += pr;
    }
    v[j] = num / den;
    d[j] = dsum / den;
  }
}

// Add the SIPG terms of one face to a row-major n x n matrix.  jv/gv: trace
// value and d/dx of every basis function on the face.  For an interior face
// jv = vA - vB (jump, A left of B) and gv = (gA + gB)/2 (mean derivative);
// form gamma J_i J_j - G_j J_i - J_j G_i (reading A1).
void add_face(std::vector<double>& A, int n, const std::vector<double>& jv,
              const std::vector<double>& gv, double gamma) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      A[i * n + j] += gamma * jv[i] * jv[j] - gv[j] * jv[i] - jv[j] * gv[i];
}

// 1D SIPG matrix on `ncell` unit cells; `low_bnd` / `high_bnd`: outer faces
// are domain-boundary faces (full Nitsche terms) rather than
// interior faces whose neighbour lies outside (self-terms with weight 1/2).
// outer faces: 0 mesh-interior (the chain's side of the face, weight 1/2),
// 1 domain boundary (Nitsche, weight 1), 2 omitted
std::vector<double> sipg_chain_modes(const FE1D& fe, int ncell, int low_mode, int high_mode);
std::vector<double> sipg_chain(const FE1D& fe, int ncell, bool low_bnd, bool high_bnd) {
  return sipg_chain_modes(fe, ncell, low_bnd ? 1 : 0, high_bnd ? 1 : 0);
}
std::vector<double> sipg_chain_modes(const FE1D& fe, int ncell, int low_mode, int high_mode) {
  const bool low_bnd = low_mode == 1, high_bnd = high_mode == 1;
  const int nc = fe.nc, n = ncell * nc;
  std::vector<double> A(n * n, 0.0);
  for (int c = 0; c < ncell; ++c)
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j) A[(c * nc + i) * n + c * nc + j] += fe.K[i * nc + j];
  std::vector<double> jv(n), gv(n);
  // interior faces between cell c-1 (A) and c (B)
  for (int c = 1; c < ncell; ++c) {
    std::fill(jv.begin(), jv.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    jv[(c - 1) * nc + nc - 1] += 1.0;     // vA: right end of cell c-1
    jv[c * nc] -= 1.0;                    // -vB: left end of cell c
    for (int j = 0; j < nc; ++j) {
      gv[(c - 1) * nc + j] += 0.5 * fe.d1[j];
      gv[c * nc + j] += 0.5 * fe.d0[j];
    }
    add_face(A, n, jv, gv, fe.gamma);
  }
  // low outer face: the chain is the "B" (right) side; J = -vB, G = w * gB
  if (low_mode != 2) {
    std::fill(jv.begin(), jv.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    const double wt = low_bnd ? 1.0 : 0.5;
    jv[0] = -1.0;
    for (int j = 0; j < nc; ++j) gv[j] = wt * fe.d0[j];
    add_face(A, n, jv, gv, low_bnd ? fe.gamma_b : fe.gamma);
  }
  // high outer face: the chain is the "A" (left) side; J = vA, G = w * gA
  if (high_mode != 2) {
    std::fill(jv.begin(), jv.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    const double wt = high_bnd ? 1.0 : 0.5;
    jv[n - 1] = 1.0;
    for (int j = 0; j < nc; ++j) gv[(ncell - 1) * nc + j] = wt * fe.d1[j];
    add_face(A, n, jv, gv, high_bnd ? fe.gamma_b : fe.gamma);
  }
  return A;
}

std::vector<double> block_mass(const FE1D& fe, int ncell) {
  const int nc = fe.nc, n = ncell * nc;
  std::vector<double> M(n * n, 0.0);
  for (int c = 0; c < ncell; ++c)
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j) M[(c * nc + i) * n + c * nc + j] = fe.M[i * nc + j];
  return M;
}

}  // namespace

bool gen_eig(int n, const std::vector<double>& L, const std::vector<double>& M,
             std::vector<double>& S, std::vector<double>& lam) {
  // Cholesky M = C C^T (lower triangular C)
  std::vector<double> C(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double s = M[j * n + j];
    for (int p = 0; p < j; ++p) s -= C[j * n + p] * C[j * n + p];
    if (s <= 0.0) return false;
    C[j * n + j] = std::sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double t = M[i * n + j];
      for (int p = 0; p < j; ++p) t -= C[i * n + p] * C[j * n + p];
      C[i * n + j] = t / C[j * n + j];
    }
  }
  // Y = C^{-1} L (forward substitution on every column), A = C^{-1} Y^T
  auto fwd = [&](std::vector<double>& B) {  // B <- C^{-1} B, B row-major n x n
    for (int col = 0; col < n; ++col)
      for (int i = 0; i < n; ++i) {
        double t = B[i * n + col];
        for (int p = 0; p < i; ++p) t -= C[i * n + p] * B[p * n + col];
        B[i * n + col] = t / C[i * n + i];
      }
  };
  std::vector<double> Y = L;
  fwd(Y);
  std::vector<double> A(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A[i * n + j] = Y[j * n + i];
  fwd(A);
  for (int i = 0; i < n; ++i)  // symmetrise round-off
    for (int j = i + 1; j < n; ++j) {
      double s = 0.5 * (A[i * n + j] + A[j * n + i]);
      A[i * n + j] = A[j * n + i] = s;
    }
  // cyclic Jacobi: A = Q diag Q^T
  std::vector<double> Q(n * n, 0.0);
  for (int i = 0; i < n; ++i) Q[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[i * n + j] * A[i * n + j];
        if (i != j) off += A[i * n + j] * A[i * n + j];
      }
    if (off <= 1e-32 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = A[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        double theta = 0.5 * (A[q * n + q] - A[p * n + p]) / apq;
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < n; ++r) {  // A <- A J (columns p, q)
          double arp = A[r * n + p], arq = A[r * n + q];
          A[r * n + p] = c * arp - s * arq;
          A[r * n + q] = s * arp + c * arq;
        }
        for (int r = 0; r < n; ++r) {  // A <- J^T A (rows p, q)
          double apr = A[p * n + r], aqr = A[q * n + r];
          A[p * n + r] = c * apr - s * aqr;
          A[q * n + r] = s * apr + c * aqr;
        }
        for (int r = 0; r < n; ++r) {  // Q <- Q J
          double qrp = Q[r * n + p], qrq = Q[r * n + q];
          Q[r * n + p] = c * qrp - s * qrq;
          Q[r * n + q] = s * qrp + c * qrq;
        }
      }
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return A[a * n + a] < A[b * n + b]; });
  // S = C^{-T} Q (back substitution), columns in ascending eigenvalue order
  S.assign(n * n, 0.0);
  lam.assign(n, 0.0);
  std::vector<double> col(n);
  for (int m = 0; m < n; ++m) {
    int src = ord[m];
    lam[m] = A[src * n + src];
    for (int i = n - 1; i >= 0; --i) {
      double t = Q[i * n + src];
      for (int p = i + 1; p < n; ++p) t -= C[p * n + i] * col[p];
      col[i] = t / C[i * n + i];
    }
    int imax = 0;
    for (int i = 1; i < n; ++i)
      if (std::fabs(col[i]) > std::fabs(col[imax]) + 1e-12) imax = i;
    double sg = col[imax] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < n; ++i) S[i * n + m] = sg * col[i];
  }
  return true;
}

// Gauss-Jordan inverse of a small dense matrix (row-major); false if singular
static bool invert(int n, std::vector<double> A, std::vector<double>& Ai) {
  Ai.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) Ai[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (std::fabs(A[piv * n + c]) < 1e-300) return false;
    for (int j = 0; j < n; ++j) {
      std::swap(A[c * n + j], A[piv * n + j]);
      std::swap(Ai[c * n + j], Ai[piv * n + j]);
    }
    const double inv = 1.0 / A[c * n + c];
    for (int j = 0; j < n; ++j) {
      A[c * n + j] *= inv;
      Ai[c * n + j] *= inv;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        A[r * n + j] -= f * A[c * n + j];
        Ai[r * n + j] -= f * Ai[c * n + j];
      }
    }
  }
  return true;
}

FE1D build_fe1d(int k, double penalty_scale, int basis, int dir_width, double boundary_scale) {
  FE1D fe;
  fe.k = k;
  fe.basis = basis;
  fe.dir_width = dir_width;
  fe.nc = k + 1;
  fe.np = 2 * fe.nc;
  const int nc = fe.nc, np = fe.np;
  fe.gamma = penalty_scale * 2.0 * k * (k + 1);
  fe.gamma_b = fe.gamma * (boundary_scale > 0 ? boundary_scale : 1.0);
  fe.nodes = gll(k);
  std::vector<double> qx, qw, v, d;
  gauss(nc, qx, qw);   // exact for degree 2k (reading A3)
  fe.M.assign(nc * nc, 0.0);
  fe.K.assign(nc * nc, 0.0);
  for (int q = 0; q < nc; ++q) {
    lagrange(fe.nodes, qx[q], v, d);
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j) {
        fe.M[i * nc + j] += qw[q] * v[i] * v[j];
        fe.K[i * nc + j] += qw[q] * d[i] * d[j];
      }
  }
  fe.w.assign(nc, 0.0);
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < nc; ++j) fe.w[i] += fe.M[i * nc + j];
  lagrange(fe.nodes, 0.0, v, fe.d0);
  lagrange(fe.nodes, 1.0, v, fe.d1);
  // Hermite-type basis (clamped kernel, reading A19): the dual
  // basis of {v(0), v'(0), v(eta_1..eta_{k-3}), -v'(1), v(1)}, eta = interior Gauss
  // points.  With F[i][n] = l_i(phi_n) (functionals on the GLL Lagrange basis),
  // psi_j = sum_n T[n][j] phi_n with T = F^{-1}, i.e. T[i][j] = psi_j(xi_i); every
  // table below is the Lagrange one transformed by T (exact).
  std::vector<double> T, F;
  if (basis == 1) {
    F.assign(nc * nc, 0.0);
    std::vector<double> eta, ew;
    if (k > 3) gauss(k - 3, eta, ew);
    for (int n = 0; n < nc; ++n) {
      F[0 * nc + n] = n == 0 ? 1.0 : 0.0;
      F[1 * nc + n] = fe.d0[n];
      F[(k - 1) * nc + n] = -fe.d1[n];
      F[k * nc + n] = n == k ? 1.0 : 0.0;
    }
    for (int m = 0; m < k - 3; ++m) {
      lagrange(fe.nodes, eta[m], v, d);
      for (int n = 0; n < nc; ++n) F[(2 + m) * nc + n] = v[n];
    }
    invert(nc, F, T);
    auto tt = [&](const std::vector<double>& A) {   // T^T A T
      std::vector<double> B(nc * nc, 0.0), C(nc * nc, 0.0);
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j)
          for (int p = 0; p < nc; ++p) B[i * nc + j] += A[i * nc + p] * T[p * nc + j];
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j)
          for (int p = 0; p < nc; ++p) C[i * nc + j] += T[p * nc + i] * B[p * nc + j];
      return C;
    };
    auto tv = [&](const std::vector<double>& a) {   // T^T a
      std::vector<double> b(nc, 0.0);
      for (int j = 0; j < nc; ++j)
        for (int p = 0; p < nc; ++p) b[j] += T[p * nc + j] * a[p];
      return b;
    };
    fe.M = tt(fe.M);
    fe.K = tt(fe.K);
    fe.w = tv(fe.w);
    fe.d0 = tv(fe.d0);
    fe.d1 = tv(fe.d1);
  }
  fe.MP = block_mass(fe, 2);
  for (int var = 0; var < 4; ++var) {
    fe.LP[var] = sipg_chain(fe, 2, var & 1, var & 2);
    gen_eig(np, fe.LP[var], fe.MP, fe.S[var], fe.lam[var]);
  }
  // The interior patch problem (variant 0) is symmetric under the reflection
  // i -> np-1-i, so every eigenvector is even or odd.  Order its modes as
  // [even modes (ascending) | odd modes (ascending)] and symmetrise exactly;
  // the kernels then apply S and S^T with half-size even/odd products.
  {
    std::vector<int> ev, od;
    for (int m = 0; m < np; ++m) {
      double se = 0.0, so = 0.0;
      for (int i = 0; i < np; ++i) {
        se += std::fabs(fe.S[0][i * np + m] - fe.S[0][(np - 1 - i) * np + m]);
        so += std::fabs(fe.S[0][i * np + m] + fe.S[0][(np - 1 - i) * np + m]);
      }
      (se < so ? ev : od).push_back(m);
    }
    if ((int)ev.size() == np / 2 && (int)od.size() == np / 2) {
      std::vector<double> S2(np * np), l2(np);
      for (int k = 0; k < np; ++k) {
        const int m = k < np / 2 ? ev[k] : od[k - np / 2];
        const double sg = k < np / 2 ? 1.0 : -1.0;
        l2[k] = fe.lam[0][m];
        for (int i = 0; i < np / 2; ++i) {
          const double a = 0.5 * (fe.S[0][i * np + m] + sg * fe.S[0][(np - 1 - i) * np + m]);
          S2[i * np + k] = a;
          S2[(np - 1 - i) * np + k] = sg * a;
        }
      }
      fe.S[0] = S2;
      fe.lam[0] = l2;
      fe.even_odd = true;
    }
  }
  // ---- Dirichlet kernel tables (reading A20)
  fe.even_odd_dir = false;
  for (int var = 0; var < 4; ++var) {
    const bool lo_b = var & 1, hi_b = var & 2;
    const int wd = dir_width;   // 1 Dirichlet (Lagrange), 2 clamped (Hermite: value + derivative)
    fe.LPR[var] = sipg_chain_modes(fe, 2, lo_b ? 1 : 2, hi_b ? 1 : 2);
    std::vector<int> keep;
    for (int i = 0; i < np; ++i)
      if (!((i < wd && !lo_b) || (i >= np - wd && !hi_b))) keep.push_back(i);
    const int nk = (int)keep.size();
    std::vector<double> Lk(nk * nk), Mk(nk * nk), Sk, lk;
    for (int a = 0; a < nk; ++a)
      for (int b = 0; b < nk; ++b) {
        Lk[a * nk + b] = fe.LP[var][keep[a] * np + keep[b]];   // = LPR on kept nodes (outer terms vanish there)
        Mk[a * nk + b] = fe.MP[keep[a] * np + keep[b]];
      }
    gen_eig(nk, Lk, Mk, Sk, lk);
    std::vector<double>& S = fe.SD[var];
    S.assign(np * np, 0.0);
    fe.lamD[var].assign(np, 1.0);
    fe.actD[var].assign(np, 0.0);
    if (var == 0) {
      // reflection-symmetric: split the nk = np-2 modes into even / odd, then
      // prepend the inactive boundary pair to each half
      std::vector<int> ev, od;
      for (int m = 0; m < nk; ++m) {
        double se = 0.0, so = 0.0;
        for (int a = 0; a < nk; ++a) {
          se += std::fabs(Sk[a * nk + m] - Sk[(nk - 1 - a) * nk + m]);
          so += std::fabs(Sk[a * nk + m] + Sk[(nk - 1 - a) * nk + m]);
        }
        (se < so ? ev : od).push_back(m);
      }
      if ((int)ev.size() != nk / 2 || (int)od.size() != nk / 2) continue;
      const double r2 = std::sqrt(0.5);
      for (int h = 0; h < 2; ++h) {
        const int base = h * (np / 2);
        const double sg = h == 0 ? 1.0 : -1.0;
        for (int q = 0; q < wd; ++q) {   // inactive boundary pairs (e_q +- e_{np-1-q}) / sqrt2
          S[q * np + base + q] = r2;
          S[(np - 1 - q) * np + base + q] = sg * r2;
        }
        for (int q = 0; q < nk / 2; ++q) {
          const int m = h == 0 ? ev[q] : od[q], col = base + wd + q;
          fe.lamD[var][col] = lk[m];
          fe.actD[var][col] = 1.0;
          for (int a = 0; a < nk / 2; ++a) {   // exact symmetrisation
            const double v = 0.5 * (Sk[a * nk + m] + sg * Sk[(nk - 1 - a) * nk + m]);
            S[keep[a] * np + col] = v;
            S[keep[nk - 1 - a] * np + col] = sg * v;
          }
        }
      }
      fe.even_odd_dir = true;
    } else {
      int col = 0;
      for (int m = 0; m < nk; ++m, ++col) {
        fe.lamD[var][col] = lk[m];
        fe.actD[var][col] = 1.0;
        for (int a = 0; a < nk; ++a) S[keep[a] * np + col] = Sk[a * nk + m];
      }
      for (int i = 0; i < np; ++i)   // inactive unit modes on the dropped nodes
        if (std::find(keep.begin(), keep.end(), i) == keep.end()) S[i * np + col++] = 1.0;
    }
  }
  fe.P.assign(np * nc, 0.0);
  for (int i = 0; i < np; ++i) {
    double x = 0.5 * (fe.nodes[i % nc] + (i / nc));
    lagrange(fe.nodes, x, v, d);
    for (int j = 0; j < nc; ++j) fe.P[i * nc + j] = v[j];
  }
  if (basis == 1) {   // P_H (child c) = F P_L(child c) T
    std::vector<double> PH(np * nc, 0.0);
    for (int c = 0; c < 2; ++c)
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) {
          double acc = 0.0;
          for (int p = 0; p < nc; ++p)
            for (int q = 0; q < nc; ++q) acc += F[i * nc + p] * fe.P[(c * nc + p) * nc + q] * T[q * nc + j];
          PH[(c * nc + i) * nc + j] = acc;
        }
    fe.P = PH;
  }
  return fe;
}

std::vector<double> sin_moments(const FE1D& fe, int ncell, int c0, double h, double ell) {
  // g[c * nc + i] = int over global cell c0 + c of sin(pi x / ell) phi_i((x - x_c) / h) dx,
  // Gauss quadrature with nc + 6 points per cell (GLL Lagrange basis only)
  const int nc = fe.nc;
  std::vector<double> qx, qw, v, d;
  gauss(nc + 6, qx, qw);
  const double pi = 3.14159265358979323846;
  std::vector<double> g((size_t)ncell * nc, 0.0);
  for (int c = 0; c < ncell; ++c)
    for (size_t q = 0; q < qx.size(); ++q) {
      lagrange(fe.nodes, qx[q], v, d);
      const double f = std::sin(pi * ((c0 + c) + qx[q]) * h / ell) * qw[q] * h;
      for (int i = 0; i < nc; ++i) g[(size_t)c * nc + i] += f * v[i];
    }
  return g;
}

void global_1d(const FE1D& fe, int ncell, std::vector<double>& L, std::vector<double>& M) {
  L = sipg_chain(fe, ncell, true, true);
  M = block_mass(fe, ncell);
}

}  // namespace ipmg
