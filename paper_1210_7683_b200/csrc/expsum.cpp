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
//     1/x ~= c0 + sum_r w_r exp(-s_r x),   s_r = e^{u_r},  w_r = h e^{u_r},
// uniformly in relative terms on [x_min, x_max].  c0 is the closed-form tail
// of the infinite trapezoid sum below u_min (exp(-s x) ~ 1 there).  Every
// weight and node is positive, so with E[k, r] = exp(-s_r alpha_k) and
// F[r, j] = w_r exp(-s_r beta_j) / (sigma2_j h_j),
//     S_BR = (X'.X')^T D ~= ((X'.X')^T E) F
// is a sum of non-negative terms: no cancellation, and the factorisation
// perturbs each D[k, j] by a relative 2^-52 or less — the size of the
// rounding already in D.  Cost per SNP drops from 2 n t to 2 r (n + t).
#include <cmath>
#include <cstdint>

#include "../../include/gwgrid_cuda.h"

extern "C" int32_t gwg_exp_sum_design(double x_min, double x_max, int32_t multiple,
                                      int32_t max_terms, double* s, double* w,
                                      int32_t* terms) {
  if (terms) *terms = 0;
  if (!(x_min > 0.0) || !(x_max >= x_min) || !std::isfinite(x_max) || multiple < 1 ||
      max_terms < 2)
    return GWG_DIMENSION;
  // Tails: the constant term stands for the nodes below u_min, exact up to
  // x^2 e^{2 u_min} / 2 <= 2^-53 (at x_max); above u_max, exp(-x e^u) <= 2^-56
  // (at x_min).  Step: the trapezoid error is 1.2e-16 at h = 0.243, 1.1e-15 at
  // 0.262, 1.2e-14 at 0.280 (measured over [1, 150] .. [1, 1e5]); h <= 0.245.
  // Nodes are computed in long double and rounded once: u_min + k h in double
  // would jitter the nodes by ulp(u) ~ 4e-15 and cost ~1e-15.
  using ld = long double;
  const ld eps_lo = std::ldexp(1.0L, -53), eps_hi = std::ldexp(1.0L, -56);
  const ld u_min = std::log(std::sqrt(2.0L * eps_lo) / ld(x_max));
  const ld u_max = std::log(std::log(1.0L / eps_hi) / ld(x_min));
  const ld h_cap = 0.245L;
  const int64_t need = int64_t(std::ceil(double((u_max - u_min) / h_cap))) + 2;  // + constant
  const int64_t r = (need + multiple - 1) / multiple * multiple;
  if (r > max_terms) return GWG_DIMENSION;
  const int64_t nodes = r - 1;
  const ld h = (u_max - u_min) / ld(nodes - 1);
  if (s && w) {
    // constant: h sum_{k >= 1} e^{u_min - k h} = h e^{u_min} / (e^h - 1)
    s[0] = 0.0;
    w[0] = double(h * std::exp(u_min) / std::expm1(h));
    for (int64_t q = 0; q < nodes; ++q) {
      const ld sq = std::exp(u_min + ld(q) * h);
      s[q + 1] = double(sq);
      w[q + 1] = double(h * sq);
    }
  }
  if (terms) *terms = int32_t(r);
  return GWG_OK;
}
