// expsum.cpp — positive exponential sums for 1/x, the low-rank factorisation
// of the GLS weight matrix D used by the split grid's S_BR term.
//
// For h_j > 0 the weight of eigen-row k in trait j (proj/src/gls.cpp:105-132,
// the reference's 1/(h^2 w_k + 1 - h^2)) is
//     D[k, j] = 1 / (sigma2_j (h_j lambda_k + 1 - h_j))
//             = 1 / (sigma2_j h_j) * 1 / (alpha_k + beta_j),
//     alpha_k = lambda_k - lambda_min >= 0,  beta_j = lambda_min + (1 - h_j) / h_j > 0.
// 1/x = int_R exp(u - x e^u) du; the trapezoid rule in u with step h is
// exponentially accurate (the integrand is analytic in |Im u| < pi/2), so
//     1/x ~= sum_r w_r exp(-s_r x),   s_r = e^{u_r},  w_r = h e^{u_r},
// uniformly in relative terms on [x_min, x_max], plus a few Gauss terms for
// the infinite trapezoid tail below u_min (see tail_gauss).  Every weight
// and node is positive, so with E[k, r] = exp(-s_r alpha_k) and
// F[r, j] = w_r exp(-s_r beta_j) / (sigma2_j h_j),
//     S_BR = (X'.X')^T D ~= ((X'.X')^T E) F
// is a sum of non-negative terms: no cancellation, and the factorisation
// perturbs each D[k, j] by a relative 2^-52 or less — the size of the
// rounding already in D.  Cost per SNP drops from 2 n t to 2 r (n + t).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

#include "../../include/gwgrid_cuda.h"

// The tail below u_min is not one constant but a q-point Gauss rule of the
// (geometric) discrete measure of the trapezoid nodes it stands for: with
// nodes z_k = e^{u_min - k h} and weights h z_k, sum_k h z_k exp(-x z_k) is
// integrated exactly for polynomials of degree < 2q in z, so u_min can sit
// where (x e^{u_min})^{2q+1} / (2q+1)! <= 2^-53 instead of
// (x e^{u_min})^2 / 2 <= 2^-53 — about half the nodes at equal accuracy
// (c1's range: 56 terms instead of 112).  A Gauss rule of a positive measure
// has positive nodes and weights, so every term stays positive.  Node 0 is
// s = 0 with weight 0: the column that carries D = 1/sigma2 for h2 = 0.
namespace {

using ld = long double;

// Eigenvalues / first eigenvector components of a small symmetric matrix
// (cyclic Jacobi rotations, long double).
void jacobi_eig(int q, ld (&a)[4][4], ld (&v)[4][4]) {
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) v[i][j] = i == j ? 1.0L : 0.0L;
  for (int sweep = 0; sweep < 64; ++sweep) {
    ld off = 0.0L;
    for (int i = 0; i < q; ++i)
      for (int j = i + 1; j < q; ++j) off += a[i][j] * a[i][j];
    if (off < 1e-60L) break;
    for (int p = 0; p < q; ++p)
      for (int r = p + 1; r < q; ++r) {
        if (std::fabs(a[p][r]) < 1e-70L) continue;
        const ld theta = (a[r][r] - a[p][p]) / (2.0L * a[p][r]);
        const ld t = (theta >= 0 ? 1.0L : -1.0L) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0L));
        const ld c = 1.0L / std::sqrt(t * t + 1.0L), sn = t * c;
        for (int k = 0; k < q; ++k) {  // A <- J^T A J
          const ld akp = a[k][p], akr = a[k][r];
          a[k][p] = c * akp - sn * akr;
          a[k][r] = sn * akp + c * akr;
        }
        for (int k = 0; k < q; ++k) {
          const ld apk = a[p][k], ark = a[r][k];
          a[p][k] = c * apk - sn * ark;
          a[r][k] = sn * apk + c * ark;
        }
        for (int k = 0; k < q; ++k) {
          const ld vkp = v[k][p], vkr = v[k][r];
          v[k][p] = c * vkp - sn * vkr;
          v[k][r] = sn * vkp + c * vkr;
        }
      }
  }
}

// q-point Gauss rule (nodes z, weights g) of the measure sum_{k>=1} h z_k
// delta(z - z_k), z_k = e^{u_min - k h}: Stieltjes recurrence, then the
// Jacobi matrix's eigensystem (Golub-Welsch).
void tail_gauss(int q, ld u_min, ld h, ld* z, ld* g) {
  const int K = int(120.0L / h) + 2;  // weights below e^-120 relative
  std::vector<ld> x(K), w(K), p(K, 1.0L), pp(K, 0.0L);
  for (int k = 0; k < K; ++k) {
    x[k] = std::exp(u_min - ld(k + 1) * h);
    w[k] = h * x[k];
  }
  ld a[4][4] = {}, v[4][4] = {};
  ld m0 = 0.0L, nprev = 1.0L;
  for (int j = 0; j < q; ++j) {
    ld nrm = 0.0L, mom = 0.0L;
    for (int k = 0; k < K; ++k) {
      nrm += w[k] * p[k] * p[k];
      mom += w[k] * x[k] * p[k] * p[k];
    }
    if (j == 0) m0 = nrm;
    const ld aj = mom / nrm, bj = j > 0 ? nrm / nprev : 0.0L;
    a[j][j] = aj;
    if (j > 0) a[j - 1][j] = a[j][j - 1] = std::sqrt(bj);
    for (int k = 0; k < K; ++k) {
      const ld pn = (x[k] - aj) * p[k] - bj * pp[k];
      pp[k] = p[k];
      p[k] = pn;
    }
    nprev = nrm;
  }
  jacobi_eig(q, a, v);
  for (int i = 0; i < q; ++i) {
    z[i] = a[i][i];
    g[i] = m0 * v[0][i] * v[0][i];
  }
  for (int i = 0; i < q; ++i)  // ascending
    for (int j = i + 1; j < q; ++j)
      if (z[j] < z[i]) {
        std::swap(z[i], z[j]);
        std::swap(g[i], g[j]);
      }
}

}  // namespace

extern "C" int32_t gwg_exp_sum_design(double x_min, double x_max, int32_t multiple,
                                      int32_t max_terms, double* s, double* w,
                                      int32_t* terms) {
  if (terms) *terms = 0;
  if (!(x_min > 0.0) || !(x_max >= x_min) || !std::isfinite(x_max) || multiple < 1 ||
      max_terms < 2)
    return GWG_DIMENSION;
  // Tails: below u_min a q-point Gauss rule of the trapezoid nodes it stands
  // for, exact up to ~(x e^{u_min})^{2q+1} / (2q+1)! <= 2^-53 (at x_max);
  // above u_max, exp(-x e^u) <= 2^-56 (at x_min).  Step: the trapezoid error
  // is 1.2e-16 at h = 0.243, 1.1e-15 at 0.262, 1.2e-14 at 0.280 (measured over
  // [1, 150] .. [1, 1e5]); h <= 0.245.  Nodes are computed in long double and
  // rounded once: u_min + k h in double would jitter the nodes by ulp(u).
  constexpr int q = 3;
  const ld eps_lo = std::ldexp(1.0L, -53), eps_hi = std::ldexp(1.0L, -56);
  const ld u_min = std::log(eps_lo * 5040.0L) / ld(2 * q + 1) - std::log(ld(x_max));
  const ld u_max = std::log(std::log(1.0L / eps_hi) / ld(x_min));
  const ld h_cap = 0.245L;
  // the zero node (h2 = 0 traits) + the tail rule + the trapezoid nodes
  const int64_t need = 1 + q + int64_t(std::ceil(double((u_max - u_min) / h_cap))) + 1;
  const int64_t r = (need + multiple - 1) / multiple * multiple;
  if (r > max_terms) return GWG_DIMENSION;
  const int64_t nodes = r - 1 - q;
  const ld h = (u_max - u_min) / ld(nodes - 1);
  if (s && w) {
    s[0] = 0.0;
    w[0] = 0.0;
    ld z[4], g[4];
    tail_gauss(q, u_min, h, z, g);
    for (int i = 0; i < q; ++i) {
      s[1 + i] = double(z[i]);
      w[1 + i] = double(g[i]);
    }
    for (int64_t k = 0; k < nodes; ++k) {
      const ld sq = std::exp(u_min + ld(k) * h);
      s[1 + q + k] = double(sq);
      w[1 + q + k] = double(h * sq);
    }
  }
  if (terms) *terms = int32_t(r);
  return GWG_OK;
}
