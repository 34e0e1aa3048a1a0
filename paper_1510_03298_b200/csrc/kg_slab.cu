// Modes 1 and 2 of X^T V X x fused per slab of the last mode (d = 3).
//
// With A1 = x x_3 X3 (p1 x p2 x n3, a p-side banded contraction) the n-space
// work of one prox-grad step is, for every slab k3 of the last mode,
//   A2  = A1[:, :, k3] x_2 X2          (p1 x n2)
//   eta = X1 A2                         (n1 x n2)   (h_map, design.cpp:89-102)
//   w   = v .* eta,  sum v eta^2        (inner_quadratic, inner.cpp:109-119, expanded)
//   Q2  = X1^T w                        (p1 x n2)   (g_map, design.cpp:104-116)
//   B1[:, :, k3] = Q2 x_2 X2^T          (p1 x p2)
// and S x = B1 x_3 X3^T afterwards.  One CTA owns whole slabs (persistent
// grid, slabs dealt round-robin), so B1 is written once, in ascending-row
// order, with no cross-CTA reduction, and neither A2 nor Q2 nor eta ever
// reaches HBM: the only n-sized traffic is one read of v.
//
// Every contraction is a sweep in ascending row order with a 4-wide sliding
// window held in registers (B-spline rows have <= 4 nonzeros, so a row's band
// start advances by at most a few columns per row): the window of inputs only
// loads a value when the band start advances, and the 4 output accumulators
// retire one column at a time.  In the n-space sweep (phase b) the 32 lanes of
// a warp take 32 columns of the tile (the operands in shared memory are stored
// with an odd column stride, so lanes hit distinct banks) and the warps take
// row segments; v goes straight from HBM to registers with 32-byte loads.  A
// column of X1^T whose rows straddle a segment boundary gets one partial sum
// from each side, added in row order after the sweep.
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "kg_internal.h"

namespace kg {

namespace {

constexpr int SB = 512;  // threads per CTA (one CTA per SM)

__device__ __forceinline__ void ld4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

__device__ __forceinline__ double warp_sum_s(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Rows are split into segments of R rows; within a segment the band start of
// X1 moves by at most KS - 4 columns, so a segment touches KS columns of X1 and
// every row's 4 coefficients sit at a fixed place of a KS-wide zero-padded
// vector (expanded once per design into shared memory).  A row then costs KS
// FMAs for eta and KS for the scatter, with compile-time register indices and
// no data-dependent branch.  Column groups of phases (a) / (d) are sized the
// same way for X2.
template <int R, int KS>
__global__ void __launch_bounds__(SB, 1) k_slab12(SlabArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[SB / 32];
  const int n1 = a.n1, n2 = a.n2, p1 = a.p1, p2 = a.p2, P1 = p1 + 1;
  const int CG = a.CG, NT2 = 32 * CG, SEGL = n1 / R;
  const int NG = SB / p1;  // column groups of phases (a) / (d)
  double* sA2 = sm;                                   // P1 x NT2
  double* sQ2 = sA2 + P1 * NT2;                       // P1 x NT2
  double* sPa = sQ2 + P1 * NT2;                       // SEGL x KS x NT2 segment partials
  double* sB1 = sPa + SEGL * KS * NT2;                // p1 x p2
  double* sDp = sB1 + p1 * p2;                        // NG x KS x p1 group partials of (d)
  double* sc1 = sDp + NG * KS * p1;                   // n1 x KS expanded X1 rows
  double* sc2 = sc1 + n1 * KS;                        // n2 x KS expanded X2 rows (relative to the group base)
  int* klo = reinterpret_cast<int*>(sc2 + n2 * KS);   // SEGL: first X1 column of segment s
  int* lo2 = klo + SEGL;                              // n2
  int* sk0 = lo2 + n2;                                // p1: first segment whose window holds column k
  const int tid = threadIdx.x;
  for (int s = tid; s < SEGL; s += SB) klo[s] = __ldg(a.H1.lo + s * R);
  for (int i = tid; i < n2; i += SB) lo2[i] = __ldg(a.H2.lo + i);
  __syncthreads();
  for (int k = tid; k < p1; k += SB) {
    int s0 = 0;
    while (s0 < SEGL && klo[s0] + KS <= k) ++s0;
    sk0[k] = s0;
  }
  for (int i = tid; i < n1; i += SB) {  // X1 row i at offset lo1(i) - klo(segment)
    const int l = __ldg(a.H1.lo + i), n = __ldg(a.H1.len + i), o = l - klo[i / R];
    const double* c = a.H1.coef + __ldg(a.H1.off + i);
#pragma unroll
    for (int t = 0; t < KS; ++t) {
      const int j = t - o;
      sc1[i * KS + t] = (j >= 0 && j < n) ? __ldg(c + j) : 0.0;
    }
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  const int ka = tid % p1, ga = tid / p1;
  double accE = 0.0;  // sum v eta^2 of this thread's cells
  const i64 plane = static_cast<i64>(p1) * p2;
  for (i64 u = blockIdx.x; u < a.n3; u += gridDim.x) {
    const double* A1u = a.A1 + u * plane;
    double* B1u = a.B1 + u * plane;
    const double* vu = a.v + u * static_cast<i64>(n1) * n2;
    for (int e = tid; e < p1 * p2; e += SB) sB1[e] = 0.0;
    for (int j0 = 0; j0 < n2; j0 += NT2) {
      const int nc = min(NT2, n2 - j0);
      const int per = (nc + NG - 1) / NG, c0 = ga * per, c1 = min(nc, c0 + per);
      const bool actg = ga < NG && c0 < c1;
      const int kf = actg ? lo2[j0 + c0] : 0;  // first X2 column of this group's rows
      // expanded X2 rows of this tile, relative to their group's first column
      for (int e = tid; e < nc * KS; e += SB) {
        const int c = e / KS, t = e - c * KS, i2 = j0 + c, g = c / per;
        const int o = lo2[i2] - lo2[j0 + g * per];
        const int n = __ldg(a.H2.len + i2), jj = t - o;
        sc2[i2 * KS + t] = (jj >= 0 && jj < n) ? __ldg(a.H2.coef + __ldg(a.H2.off + i2) + jj) : 0.0;
      }
      __syncthreads();
      // (a) A2[k1, c] = sum_t X2[i2, kf + t] A1[k1, kf + t]
      if (actg) {
        double wa[KS];
#pragma unroll
        for (int t = 0; t < KS; ++t) wa[t] = kf + t < p2 ? __ldg(A1u + ka + static_cast<i64>(p1) * (kf + t)) : 0.0;
        for (int c = c0; c < c1; ++c) {
          const double* cc = sc2 + (j0 + c) * KS;
          double s2 = 0.0;
#pragma unroll
          for (int t = 0; t < KS; t += 2) {
            const double2 x = *reinterpret_cast<const double2*>(cc + t);
            s2 = fma(x.x, wa[t], s2);
            s2 = fma(x.y, wa[t + 1], s2);
          }
          sA2[ka + P1 * c] = s2;
        }
      }
      __syncthreads();
      // (b) per (column group, segment): rows of the segment for column j0 + col
      for (int it = warp; it < CG * SEGL; it += SB / 32) {
        const int cg = it % CG, sg = it / CG;
        const int col = cg * 32 + lane;
        const int r0 = sg * R, kl = klo[sg];
        double win[KS], acc[KS];
        if (col < nc) {
          const double* A2c = sA2 + P1 * col;
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            win[t] = kl + t < p1 ? A2c[kl + t] : 0.0;
            acc[t] = 0.0;
          }
          const double* vc = vu + static_cast<i64>(j0 + col) * n1 + r0;
          double vn[4];
          ld4(vc, vn[0], vn[1], vn[2], vn[3]);
#pragma unroll 1
          for (int q0 = 0; q0 < R; q0 += 4) {
            const double vq[4] = {vn[0], vn[1], vn[2], vn[3]};
            if (q0 + 4 < R) ld4(vc + q0 + 4, vn[0], vn[1], vn[2], vn[3]);  // next chunk in flight
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double* cr = sc1 + (r0 + q0 + q) * KS;
              double cx[KS];
#pragma unroll
              for (int t = 0; t < KS; t += 2) {
                const double2 x = *reinterpret_cast<const double2*>(cr + t);
                cx[t] = x.x;
                cx[t + 1] = x.y;
              }
              double eta = 0.0;
#pragma unroll
              for (int t = 0; t < KS; ++t) eta = fma(cx[t], win[t], eta);
              const double w = vq[q] * eta;
              accE = fma(w, eta, accE);
#pragma unroll
              for (int t = 0; t < KS; ++t) acc[t] = fma(cx[t], w, acc[t]);
            }
          }
#pragma unroll
          for (int t = 0; t < KS; ++t) sPa[(sg * KS + t) * NT2 + col] = acc[t];
        }
      }
      __syncthreads();
      // (b2) Q2[k, c] = segment partials of column k, in segment order
      for (int k = warp; k < p1; k += SB / 32) {  // lanes over columns: conflict-free
        const int s0 = sk0[k];
        for (int c = lane; c < nc; c += 32) {
          double q = 0.0;
          for (int sg = s0; sg < SEGL && klo[sg] <= k; ++sg) q += sPa[(sg * KS + k - klo[sg]) * NT2 + c];
          sQ2[k + P1 * c] = q;
        }
      }
      __syncthreads();
      // (d) group partials of B1[k1, kf + t] = sum_c X2[i2, kf + t] Q2[k1, c]
      if (actg) {
        double wd[KS];
#pragma unroll
        for (int t = 0; t < KS; ++t) wd[t] = 0.0;
        for (int c = c0; c < c1; ++c) {
          const double* cc = sc2 + (j0 + c) * KS;
          const double q = sQ2[ka + P1 * c];
#pragma unroll
          for (int t = 0; t < KS; t += 2) {
            const double2 x = *reinterpret_cast<const double2*>(cc + t);
            wd[t] = fma(x.x, q, wd[t]);
            wd[t + 1] = fma(x.y, q, wd[t + 1]);
          }
        }
#pragma unroll
        for (int t = 0; t < KS; ++t) sDp[(ga * KS + t) * p1 + ka] = wd[t];
      }
      __syncthreads();
      // B1[k1, k2] += group partials in group order
      {
        const int kf0 = lo2[j0], kl0 = min(p2 - 1, lo2[j0 + nc - 1] + 3);
        const int ngu = min(NG, (nc + per - 1) / per);  // groups with rows
        for (int e = tid; e < p1 * (kl0 - kf0 + 1); e += SB) {
          const int k1 = e % p1, k2 = kf0 + e / p1;
          double b = sB1[k1 + p1 * k2];
          for (int g = 0; g < ngu; ++g) {
            const int t = k2 - lo2[j0 + g * per];
            if (t >= 0 && t < KS) b += sDp[(g * KS + t) * p1 + k1];
          }
          sB1[k1 + p1 * k2] = b;
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < p1 * p2; e += SB) B1u[e] = sB1[e];
    __syncthreads();  // sB1 is cleared for the next slab
  }
  // deterministic CTA sum of v eta^2
  double v = warp_sum_s(accE);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double r = lane < SB / 32 ? red[lane] : 0.0;
    r = warp_sum_s(r);
    if (lane == 0) a.partial[blockIdx.x] = r;
  }
}

struct SlabShape {
  int CG = 0, R = 0, KS = 0;
  size_t smem = 0;
};

// Largest segment length R (rows of X1 per segment) and smallest window KS for
// which every segment's band-start spread and every (a)/(d) column group's
// spread fit the window.
SlabShape slab_shape(const SlabArgs& a) {
  SlabShape best;
  if (!a.H1.hlo || !a.H2.hlo) return best;
  for (int ks : {8, 12}) {
    for (int r : {32, 16, 8}) {
      if (a.n1 % r != 0 || a.n1 / r > 64) continue;
      bool ok = true;
      for (int s = 0; s < a.n1 / r && ok; ++s) ok = a.H1.hlo[s * r + r - 1] - a.H1.hlo[s * r] + 4 <= ks;
      if (!ok) continue;
      const int segl = a.n1 / r, cg = segl >= 16 ? 1 : 2, nt2 = 32 * cg, ng = SB / a.p1;
      const int per = std::max(1, (std::min(nt2, a.n2) + ng - 1) / ng);
      for (int j0 = 0; j0 < a.n2 && ok; j0 += nt2)
        for (int g = 0; g * per < std::min(nt2, a.n2 - j0) && ok; ++g) {
          const int i0 = j0 + g * per, i1 = std::min(a.n2 - 1, std::min(j0 + nt2 - 1, i0 + per - 1));
          ok = a.H2.hlo[i1] - a.H2.hlo[i0] + 4 <= ks;
        }
      if (!ok) continue;
      SlabShape s;
      s.CG = cg;
      s.R = r;
      s.KS = ks;
      const size_t P1 = a.p1 + 1;
      s.smem = sizeof(double) * (2 * P1 * nt2 + static_cast<size_t>(segl) * ks * nt2 +
                                 static_cast<size_t>(a.p1) * a.p2 + static_cast<size_t>(ng) * ks * a.p1 +
                                 static_cast<size_t>(a.n1) * ks + static_cast<size_t>(a.n2) * ks) +
               sizeof(int) * (static_cast<size_t>(segl) + a.n2 + a.p1);
      return s;
    }
  }
  return best;
}

template <int R, int KS>
void launch_slab(const Launch& L, SlabArgs a, const SlabShape& s, int grid) {
  smem_attr(k_slab12<R, KS>, 220 * 1024);
  a.CG = s.CG;
  k_slab12<R, KS><<<grid, SB, s.smem, L.s>>>(a);
}

}  // namespace

bool slab_ok(const SlabArgs& a) {
  if (a.p1 < 1 || a.p1 > SB || a.p2 < 1 || a.n2 < 1 || a.n3 < 1) return false;
  if (a.H1.maxlen > 4 || a.H2.maxlen > 4) return false;
  const SlabShape s = slab_shape(a);
  return s.CG != 0 && s.smem <= 220 * 1024;
}

int slab_grid(const SlabArgs& a) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<int>(std::min<i64>(a.n3, nsm));
}

void slab12(const Launch& L, const SlabArgs& a) {
  const SlabShape s = slab_shape(a);
  if (!s.CG) throw Error(E_CUDA, "slab12: unsupported shape");
  const int g = slab_grid(a);
  if (s.KS == 8) {
    if (s.R == 32) launch_slab<32, 8>(L, a, s, g);
    else if (s.R == 16) launch_slab<16, 8>(L, a, s, g);
    else launch_slab<8, 8>(L, a, s, g);
  } else {
    if (s.R == 32) launch_slab<32, 12>(L, a, s, g);
    else if (s.R == 16) launch_slab<16, 12>(L, a, s, g);
    else launch_slab<8, 12>(L, a, s, g);
  }
  launched(L);
}

}  // namespace kg
