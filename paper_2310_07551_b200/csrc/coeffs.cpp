// Split coefficients used by the library (host).  Written from the paper's tables; evaluated
// from the radical forms in long double (80-bit) and rounded once to double (reading R18).
//   second order  eq:secondord: one term, eta = l!^{d-1}, l_1 = l, alpha = 1
//   Table 1: d = 2, l = (1, 2), real columns, "+" branch
//   Table 3: d >= 2, l = (1, 2, 1), eta_2 carries 2^{d-3}, "+" branch
#include <cmath>

#include "kx_internal.h"

namespace kx {

int scheme_terms(int scheme, int ell, int d, double* eta, int* inner, double* alpha) {
  if (d < 1 || (ell != 1 && ell != 2)) return 0;
  if (scheme == 1) {  // KX_ETD2RKDS: second-order split
    double f = (ell == 2) ? std::ldexp(1.0, d - 1) : 1.0;   // l!^{d-1}
    eta[0] = f;
    inner[0] = ell;
    for (int mu = 0; mu < d; ++mu) alpha[mu] = 1.0;
    return 1;
  }
  if (scheme != 2 || d < 2) return 0;
  if (d == 2) {  // Table 1, upper signs
    long double e1, e2, a11, a12, a21, a22;
    if (ell == 1) {
      const long double r = sqrtl(10.0L);
      e1 = -5.0L / 4.0L;
      e2 = 9.0L;
      a11 = 4.0L * r / 15.0L + 4.0L / 3.0L;
      a12 = -4.0L * r / 15.0L + 4.0L / 3.0L;
      a21 = 2.0L * r / 9.0L + 16.0L / 9.0L;
      a22 = -2.0L * r / 9.0L + 16.0L / 9.0L;
    } else {
      const long double r = sqrtl(33.0L);
      e1 = -4.0L / 3.0L;
      e2 = 22.0L / 3.0L;
      a11 = r / 8.0L + 9.0L / 8.0L;
      a12 = -r / 8.0L + 9.0L / 8.0L;
      a21 = 3.0L * r / 22.0L + 3.0L / 2.0L;
      a22 = -3.0L * r / 22.0L + 3.0L / 2.0L;
    }
    eta[0] = (double)e1;
    eta[1] = (double)e2;
    inner[0] = 1;
    inner[1] = 2;
    alpha[0] = (double)a11;
    alpha[1] = (double)a12;
    alpha[2] = (double)a21;
    alpha[3] = (double)a22;
    return 2;
  }
  // Table 3, upper signs
  long double e1, e2, e3, a1, a2, a3;
  const long double two = ldexpl(1.0L, d - 3);
  if (ell == 1) {
    const long double r = sqrtl(2991111.0L);
    e1 = 2243.0L / 1350.0L + 440521.0L / (675.0L * r);
    a1 = 3.0L * (5161.0L + r) / 15869.0L;
    e2 = -12544.0L / 675.0L * two;
    a2 = 45.0L / 28.0L;
    e3 = 2243.0L / 1350.0L - 440521.0L / (675.0L * r);
    a3 = 3.0L * (5161.0L - r) / 15869.0L;
  } else {
    const long double r = sqrtl(2391.0L);
    e1 = 19.0L / 27.0L + 151.0L / (27.0L * r);
    a1 = 3.0L * (121.0L + r) / 490.0L;
    e2 = -196.0L / 27.0L * two;
    a2 = 9.0L / 7.0L;
    e3 = 19.0L / 27.0L - 151.0L / (27.0L * r);
    a3 = 3.0L * (121.0L - r) / 490.0L;
  }
  eta[0] = (double)e1;
  eta[1] = (double)e2;
  eta[2] = (double)e3;
  inner[0] = 1;
  inner[1] = 2;
  inner[2] = 1;
  for (int mu = 0; mu < d; ++mu) {
    alpha[0 * d + mu] = (double)a1;
    alpha[1 * d + mu] = (double)a2;
    alpha[2 * d + mu] = (double)a3;
  }
  return 3;
}

// Table 2: complex two-term split, d >= 2, l = (1, 2), alpha independent of mu,
// eta_2 carrying 2^{d-2}.  Branch: the paper's "+ in alpha_{1,mu}", i.e. the lower
// sign of every -+/+- pair (reading R3): alpha_1 = 12/11 + 4 sqrt2/11 i for l = 1.
int scheme_terms_cplx(int ell, int d, double* eta_re, double* eta_im, int* inner, double* alpha_re,
                      double* alpha_im) {
  if (d < 2 || (ell != 1 && ell != 2)) return 0;
  const long double two = ldexpl(1.0L, d - 2);
  long double e1r, e1i, a1r, a1i, e2r, e2i, a2r, a2i;
  if (ell == 1) {
    const long double r = sqrtl(2.0L);
    e1r = 7.0L / 4.0L;
    e1i = -3.0L * r / 2.0L;
    a1r = 12.0L / 11.0L;
    a1i = 4.0L * r / 11.0L;
    e2r = two * -3.0L;
    e2i = two * 6.0L * r;
    a2r = 4.0L / 3.0L;
    a2i = 2.0L * r / 3.0L;
  } else {
    const long double r = sqrtl(3.0L);
    e1r = 2.0L / 3.0L;
    e1i = -2.0L * r / 3.0L;
    a1r = 3.0L / 4.0L;
    a1i = r / 4.0L;
    e2r = two * (-2.0L / 3.0L);
    e2i = two * 8.0L * r / 3.0L;
    a2r = 6.0L / 7.0L;
    a2i = 3.0L * r / 7.0L;
  }
  eta_re[0] = (double)e1r;
  eta_im[0] = (double)e1i;
  eta_re[1] = (double)e2r;
  eta_im[1] = (double)e2i;
  inner[0] = 1;
  inner[1] = 2;
  for (int mu = 0; mu < d; ++mu) {
    alpha_re[mu] = (double)a1r;
    alpha_im[mu] = (double)a1i;
    alpha_re[d + mu] = (double)a2r;
    alpha_im[d + mu] = (double)a2i;
  }
  return 2;
}

}  // namespace kx
