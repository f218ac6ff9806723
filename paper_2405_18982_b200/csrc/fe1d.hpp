// Host-side 1D finite-element setup for the ipmg library (layer 1 of the build).
//
// Everything the sm_100a kernels need is derived from 1D objects on the unit
// interval (h = 1); a level of size h scales the whole operator by h^(d-2)
// (mass ~ h, stiffness/penalty/derivatives ~ 1/h), so the tables are level
// independent.  Sources:
//   * GLL Lagrange basis ............ PAPER.md:599-604 (Appendix A)
//   * SIPG form, penalty ............ PAPER.md:81-100 (eq. jump_mean, bilinear_form)
//   * Kronecker cell matrices ....... PAPER.md:118-126
//   * fast diagonalisation .......... PAPER.md:259-280 (eq. inverse2d/3d, fast_inverse)
//   * canonical-embedding transfer .. PAPER.md:152
// Independent of oracle/ (different language, algorithms: Newton for the
// Legendre roots, Kronecker patch matrices, Jacobi eigen-solver).
#pragma once
#include <vector>

namespace ipmg {

struct FE1D {
  int k = 0, nc = 0, np = 0;       // degree, nodes per cell, nodes per 2-cell patch
  int basis = 0;                   // 0 GLL Lagrange, 1 Hermite-type (clamped kernel, reading A19)
  int dir_width = 1;               // nodes dropped per mesh-interior patch side: 1 Dirichlet, 2 clamped
  double gamma = 0;                // unit-h penalty 2k(k+1)*scale (reading A2)
  double gamma_b = 0;              // unit-h penalty on domain-boundary faces (reading A2: = gamma
                                   // by default; boundary_scale probes the one-sided k(k+1)/h)
  std::vector<double> nodes;       // GLL nodes on [0,1]                       (nc)
  std::vector<double> w;           // int_0^1 phi_i                             (nc)
  std::vector<double> M, K;        // unit cell mass / stiffness, row-major    (nc*nc)
  std::vector<double> d0, d1;      // phi_j'(0), phi_j'(1)                     (nc)
  // 2-cell patch matrices, variant v: bit0 = low outer face on the domain
  // boundary, bit1 = high outer face on the domain boundary.
  std::vector<double> MP;          // patch mass (block diagonal)             (np*np)
  std::vector<double> LP[4];       // patch stiffness + face terms            (np*np)
  std::vector<double> S[4];        // generalized eigenvectors, S[i*np+m] = node i, mode m
  std::vector<double> lam[4];      // eigenvalues (variant 0: even modes then odd modes, each ascending)
  bool even_odd = false;           // variant-0 modes ordered [even | odd] (always true in practice)
  std::vector<double> P;           // prolongation, P[i*nc+j] = phi_j((xi_{i%nc} + i/nc)/2)  (np*nc)
  // Dirichlet kernel (reading A20), variant v as above:
  //  LPR[v]  patch matrix WITHOUT the mesh-interior outer faces (the residual operator)
  //  SD[v]   eigenvectors of the local problem on the kept nodes (outer nodes at
  //          mesh-interior faces dropped), padded to np x np; excluded nodes get
  //          inactive modes (actD = 0).  Variant 0: [even | odd], the boundary pair
  //          (e_0 +- e_{np-1})/sqrt2 is the first mode of each half.
  std::vector<double> LPR[4], SD[4], lamD[4], actD[4];
  bool even_odd_dir = false;
};

// Build all unit tables for degree k (1..7); penalty_scale multiplies gamma;
// boundary_scale multiplies the domain-boundary penalty relative to gamma
// (<= 0: 1, i.e. gamma_b = gamma); basis 1 = Hermite-type (k >= 3); dir_width:
// reduced-space width of the Dirichlet/clamped tables.
FE1D build_fe1d(int k, double penalty_scale, int basis = 0, int dir_width = 1,
                double boundary_scale = 1.0);

// Global 1D SIPG matrix (unit h) on ncell cells with boundary faces at both ends
// and its mass; row-major (ncell*nc)^2.  Used for the coarse solve (reading A10).
void global_1d(const FE1D& fe, int ncell, std::vector<double>& L, std::vector<double>& M);

// Manufactured right-hand side (ipmg_rhs kind 1): 1D moments of sin(pi x / ell) against
// the GLL Lagrange basis on ncell cells of size h starting at global cell c0, (ncell*nc).
std::vector<double> sin_moments(const FE1D& fe, int ncell, int c0, double h, double ell);

// Generalized symmetric eigenproblem L S = M S diag(lam), S^T M S = I, lam ascending,
// sign fixed so that the largest-|.| entry of each column is positive.
// Cholesky + cyclic Jacobi.  Returns false if M is not SPD.
bool gen_eig(int n, const std::vector<double>& L, const std::vector<double>& M,
             std::vector<double>& S, std::vector<double>& lam);

}  // namespace ipmg
