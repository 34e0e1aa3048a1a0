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

// Gather plan of the slab pass (kronglm_b200.h).  Shared with the design
// builder (kg_solver.cu: build_slab_gather).
kg_status kg_slab_gather_plan(int64_t n, int64_t p, const double* X, int32_t* slots, int32_t* gmax, int32_t* plane) {
  constexpr int kW = 5, kG = 8;
  if (!X || !slots || !gmax || !plane || n < 4 || (n & 3) || p < kW) return KG_EINVAL;
  std::vector<int> lo(static_cast<size_t>(n), 0), len(static_cast<size_t>(n), 0);
  for (int64_t r = 0; r < n; ++r) {  // row bands by an exact-zero test
    int64_t a = p, b = 0;
    for (int64_t k = 0; k < p; ++k)
      if (X[r + n * k] != 0.0) {
        a = std::min(a, k);
        b = std::max(b, k + 1);
      }
    lo[static_cast<size_t>(r)] = a < b ? static_cast<int>(a) : 0;
    len[static_cast<size_t>(r)] = a < b ? static_cast<int>(b - a) : 0;
  }
  const int nq = static_cast<int>(n / 4), groups = static_cast<int>((p + 7) / 8);
  int PL = nq * kW + 1;
  while ((PL & 7) != 2) ++PL;
  if (PL > 0xffff) return KG_EINVAL;
  int gm = 0;
  for (int k = 0; k < groups * 8; ++k) {
    int cnt = 0;
    for (int j = 0; j < kG; ++j) slots[static_cast<size_t>(k) * kG + j] = PL - 1;  // the zero slot
    for (int q = 0; q < nq && k < p; ++q) {
      const int wlo = std::min<int>(lo[static_cast<size_t>(4 * q)], static_cast<int>(p) - kW);
      bool hit = false;
      for (int r = 4 * q; r < 4 * q + 4; ++r)
        hit = hit || (lo[static_cast<size_t>(r)] <= k && k < lo[static_cast<size_t>(r)] + len[static_cast<size_t>(r)]);
      if (!hit) continue;
      if (k < wlo || k >= wlo + kW || cnt == kG) return KG_EINVAL;
      slots[static_cast<size_t>(k) * kG + cnt++] = q * kW + (k - wlo);
    }
    gm = std::max(gm, cnt);
  }
  *gmax = gm;
  *plane = PL;
  return KG_OK;
}

kg_status kg_halo_plan(int64_t n, int64_t p, const double* X, int world, int rank, int64_t* out) {
  if (!X || !out || n < 1 || p < 1 || world < 1 || rank < 0 || rank >= world || n < world) return KG_EINVAL;
  // touched coefficient range of every rank's rows (rows without nonzeros add nothing)
  std::vector<int64_t> tlo(world, p), thi(world, 0);
  for (int r = 0; r < world; ++r) {
    const int64_t lo = n * r / world, hi = n * (r + 1) / world;
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t k = 0; k < p; ++k)
        if (X[i + n * k] != 0.0) {
          tlo[r] = std::min(tlo[r], k);
          thi[r] = std::max(thi[r], k + 1);
        }
    if (thi[r] == 0) tlo[r] = thi[r] = (r == 0 ? 0 : thi[r - 1]);
  }
  auto own_lo = [&](int r) { return r == 0 ? int64_t(0) : tlo[r]; };
  auto own_hi = [&](int r) { return r == world - 1 ? p : tlo[r + 1]; };
  bool ok = true;
  for (int r = 0; r < world; ++r) {
    if (own_lo(r) > own_hi(r)) ok = false;        // owned ranges must tile [0, p) in order
    if (tlo[r] < own_lo(r)) ok = false;           // nothing to the left of the owned range
    if (r + 1 < world && thi[r] > own_hi(r + 1)) ok = false;  // the right halo stays in the right neighbour
    if (r + 1 == world && thi[r] > p) ok = false;
  }
  const int r = rank;
  out[0] = ok ? 1 : 0;
  out[1] = own_lo(r);
  out[2] = own_hi(r);
  out[3] = tlo[r];
  out[4] = thi[r];
  out[5] = own_lo(r);                                            // L = [own_lo, t_hi(r - 1))
  out[6] = r > 0 ? std::max(own_lo(r), std::min(thi[r - 1], own_hi(r))) : own_lo(r);
  out[7] = own_hi(r);                                            // R = [own_hi, t_hi)
  out[8] = r + 1 < world ? std::max(own_hi(r), thi[r]) : own_hi(r);
  return KG_OK;
}

}  // extern "C"
