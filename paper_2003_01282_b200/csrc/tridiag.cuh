// Batched symmetric tridiagonal eigensolver core shared by rules.cu and batched.cu.
#pragma once
#include <cfloat>
#include <cmath>

namespace slq {

// sqrt(a^2 + b^2): the plain formula when neither square can overflow or underflow (the usual
// case: tridiagonal entries of L, P are O(1) .. O(1e-9)), else the library hypot.
__device__ __forceinline__ double fast_hypot(double a, double b) {
  const double m = fmax(fabs(a), fabs(b));
  if (m > 1e-150 && m < 1e150) return sqrt(fma(a, a, b * b));
  return hypot(a, b);
}

// Implicit QL on (d, e) of order m; z holds the first row of the accumulated rotations.
// Returns 0 on convergence, 1 if an eigenvalue needed more than 60 sweeps.
__device__ __forceinline__ int tridiag_ql_first_row(double* d, double* e, double* z, int m) {
  for (int l = 0; l < m; ++l) {
    int sweeps = 0;
    for (;;) {
      int mm = l;
      for (; mm < m - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= DBL_EPSILON * dd || fabs(e[mm]) < DBL_MIN) break;
      }
      if (mm == l) break;
      if (++sweeps > 60) return 1;
      // Wilkinson-type shift from the leading 2x2 block
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = fast_hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      bool deflated = false;
      for (int i = mm - 1; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        // r = hypot(f, g) and 1/r from one reciprocal square root (one long-latency sequence on the
        // rotation's dependent chain instead of a square root and a division)
        double rinv;
        const double mfg = fmax(fabs(f), fabs(g));
        if (mfg > 1e-150 && mfg < 1e150) {
          const double h2 = fma(f, f, g * g);
          rinv = rsqrt(h2);
          r = h2 * rinv;
        } else {
          r = hypot(f, g);
          rinv = r != 0.0 ? 1.0 / r : 0.0;
        }
        e[i + 1] = r;
        if (r == 0.0) {          // underflow: split the matrix here and restart
          d[i + 1] -= p;
          e[mm] = 0.0;
          deflated = true;
          break;
        }
        s = f * rinv;
        c = g * rinv;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        f = z[i + 1];
        z[i + 1] = s * z[i] + c * f;
        z[i] = c * z[i] - s * f;
      }
      if (deflated) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  return 0;
}

}  // namespace slq
