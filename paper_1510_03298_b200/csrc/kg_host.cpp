// Host-side input builders and index helpers of the C ABI (no device work):
// bspline_design (bspline.cpp:64-104), default_basis_count (bspline.cpp:20-26),
// linear_index (array.cpp:22-36).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/kronglm_b200.h"

extern "C" {

kg_status kg_bspline_design(int64_t npts, const double* pts, int64_t order, int64_t nb, double* out) {
  if (npts < 2) return KG_EINVAL;
  for (int64_t i = 1; i < npts; ++i)
    if (!(pts[i] > pts[i - 1])) return KG_EINVAL;
  if (order < 1 || nb < order) return KG_EINVAL;
  const double lo = pts[0], hi = pts[npts - 1];
  const int64_t deg = order - 1, spans = nb - order + 1;
  const double h = (hi - lo) / static_cast<double>(spans);
  // clamped knot vector: order copies of each end, uniform interior knots
  std::vector<double> t(nb + order);
  for (int64_t i = 0; i < order; ++i) t[i] = lo;
  for (int64_t i = 0; i < nb - order; ++i) t[order + i] = lo + h * static_cast<double>(i + 1);
  for (int64_t i = 0; i < order; ++i) t[nb + i] = hi;
  std::fill(out, out + npts * nb, 0.0);
  std::vector<double> N(order), L(order), R(order);
  for (int64_t row = 0; row < npts; ++row) {
    const double x = pts[row];
    int64_t s = nb - 1;
    if (x < t[nb]) {  // binary search for the knot span containing x
      int64_t a = deg, b = nb;
      while (b - a > 1) {
        const int64_t m = (a + b) / 2;
        (x < t[m] ? b : a) = m;
      }
      s = a;
    }
    // Cox-de Boor on the order nonvanishing functions of the span
    N[0] = 1.0;
    for (int64_t j = 1; j <= deg; ++j) {
      L[j] = x - t[s + 1 - j];
      R[j] = t[s + j] - x;
      double carry = 0.0;
      for (int64_t m = 0; m < j; ++m) {
        const double tmp = N[m] / (R[m + 1] + L[j - m]);
        N[m] = carry + R[m + 1] * tmp;
        carry = L[j - m] * tmp;
      }
      N[j] = carry;
    }
    for (int64_t m = 0; m <= deg; ++m) out[row + npts * (s - deg + m)] = N[m];
  }
  return KG_OK;
}

int64_t kg_default_basis_count(int64_t n, int64_t ratio) {
  if (n < 1 || ratio < 1) return -1;
  return std::max<int64_t>((n + ratio - 1) / ratio, 5);
}

int64_t kg_linear_index(int64_t d, const int64_t* idx, const int64_t* dims) {
  int64_t pos = 0;
  for (int64_t j = d - 1; j >= 0; --j) {
    if (idx[j] < 1 || idx[j] > dims[j]) return -1;
    pos = (idx[j] - 1) + dims[j] * pos;
  }
  return pos + 1;
}

}  // extern "C"
