// sm_100a kernels of the GLAM fit path.
//
// Every n-array pass is HBM-bound FP64 work (banded B-spline factors give
// ~1 flop/byte, far below the FP64 ridge), so the kernels are written for
// coalesced streaming, on-chip reuse and fusion, not for tensor cores.
// Reductions are deterministic: per-CTA warp-shuffle trees written to a
// partials array, then summed in fixed order by a single CTA (no floating
// point atomics), so results are bitwise reproducible run to run.
#include <cfloat>
#include <cstdlib>
#include <climits>
#include <algorithm>

#include "kg_internal.h"

namespace kg {

namespace {

constexpr int NT = 256;            // threads per CTA for streaming kernels
constexpr double kEtaBound = 30.0;  // family.hpp:16
constexpr double kFloor = 1e-10;    // family.hpp:17

__device__ __forceinline__ double clampe(double e) { return fmin(fmax(e, -kEtaBound), kEtaBound); }
__device__ __forceinline__ double logistic(double e) { return 1.0 / (1.0 + exp(-clampe(e))); }
__device__ __forceinline__ double log1pexp(double e) { return e > 0.0 ? e + log1p(exp(-e)) : log1p(exp(e)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA reduction (fixed shuffle tree, then warp 0 over the
// per-warp partials).  Result valid in thread 0.  `sh` needs 32 doubles.
template <bool MAX>
__device__ double block_reduce(double v, double* sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = MAX ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = MAX ? -DBL_MAX : 0.0;
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    r = l < nw ? sh[l] : (MAX ? -DBL_MAX : 0.0);
    r = MAX ? warp_max(r) : warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ void record_min(i64* err, i64 cell) {
  atomicMin(reinterpret_cast<unsigned long long*>(err), static_cast<unsigned long long>(cell));
}

// score u_i (family.cpp:164-196), before the dispersion division.
__device__ __forceinline__ double score_of(int fam, double y, double a, double e) {
  const double ec = clampe(e);
  switch (fam) {
    case 0: return a * (y - e);
    case 1: return a * (y - logistic(e));
    case 2: return a * (y - exp(ec));
    default: return a * exp(-ec) * (y - exp(ec));
  }
}

// log-likelihood kernel term (family.cpp:129-162); caller skips a == 0.
__device__ __forceinline__ double ll_term(int fam, double y, double a, double e) {
  switch (fam) {
    case 0: return a * (y * e - 0.5 * e * e);
    case 1: return a * (y * e - log1pexp(e));
    case 2: return a * (y * e - exp(clampe(e)));
    default: return a * (-y * exp(-clampe(e)) - e);
  }
}

template <class F>
__device__ __forceinline__ double band_dot(const BandOp& op, i64 row, F&& at) {
  const int lo = __ldg(op.lo + row), len = __ldg(op.len + row);
  const double* c = op.coef + __ldg(op.off + row);
  double s = 0.0;
  for (int q = 0; q < len; ++q) s = fma(__ldg(c + q), at(lo + q), s);
  return s;
}

int grid_for(i64 work, int per_cta, int cap) {
  i64 g = (work + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

inline void bump(const Launch& L) {
  launched(L);
}

}  // namespace

int elem_grid(i64 n) { return grid_for(n, NT * 4, 148 * 8); }
int pgrid(i64 p) { return grid_for(p, NT, 148 * 8); }
// k_fista_update's grid (2 CTAs per SM, 4 elements per thread and trip): fewer
// per-CTA partials for the single-CTA control kernel to reduce
int ugrid(i64 p) { return grid_for(p, NT * 4, 148 * 2); }

// ------------------------------------------------------------ contraction
// Mode-k banded contraction of A (a x K x b, column-major) with the operator
// C (M x K): out[al, m, be] = sum_t C[m, lo_m + t] A[al, lo_m + t, be].  One
// output per thread along the flattened (coalesced) output index.
template <typename IX>
__global__ void __launch_bounds__(NT) k_contract(const double* __restrict__ A, double* __restrict__ out, IX a, IX K,
                                                 IX M, IX b, BandOp op, int accumulate) {
  const IX total = a * M * b;
  const IX stride = static_cast<IX>(gridDim.x) * NT;
  for (IX idx = static_cast<IX>(blockIdx.x) * NT + threadIdx.x; idx < total; idx += stride) {
    const IX al = idx % a;
    const IX t = idx / a;
    const IX m = t % M;
    const IX be = t / M;
    const double* src = A + al + a * K * be;
    const double s = band_dot(op, m, [&](int k) { return __ldg(src + static_cast<IX>(k) * a); });
    out[idx] = accumulate ? out[idx] + s : s;
  }
}

// Division by a loop-invariant divisor as multiply-high + shift (valid for
// numerators < 2^31).
// Same contraction with a 2-D launch: grid.x walks the (alpha, m) plane of
// one beta slab, grid.y (+ grid.z) the slabs; one fast division per output.
// The band loop keeps two partial sums so long G-direction bands pipeline.
__global__ void __launch_bounds__(NT) k_contract2(const double* __restrict__ A, double* __restrict__ out, uint32_t a,
                                                  uint32_t K, uint32_t M, uint32_t b, FastDiv fa, BandOp op,
                                                  int accumulate) {
  const uint32_t plane = a * M;
  const uint32_t idx = blockIdx.x * NT + threadIdx.x;
  const uint32_t be = blockIdx.y + gridDim.y * blockIdx.z;
  if (idx >= plane || be >= b) return;
  const uint32_t m = fa.div(idx);
  const uint32_t al = idx - m * a;
  const int lo = __ldg(op.lo + m), len = __ldg(op.len + m);
  const double* c = op.coef + __ldg(op.off + m);
  const double* src = A + static_cast<size_t>(be) * a * K + al + static_cast<size_t>(lo) * a;
  double s0 = 0.0, s1 = 0.0;
  int t = 0;
  for (; t + 1 < len; t += 2) {
    s0 = fma(__ldg(c + t), __ldg(src + static_cast<size_t>(t) * a), s0);
    s1 = fma(__ldg(c + t + 1), __ldg(src + static_cast<size_t>(t + 1) * a), s1);
  }
  if (t < len) s0 = fma(__ldg(c + t), __ldg(src + static_cast<size_t>(t) * a), s0);
  const double s = s0 + s1;
  double* o = out + static_cast<size_t>(be) * plane + idx;
  *o = accumulate ? *o + s : s;
}

// Row-stationary banded contraction: a thread owns one output row (alpha, m)
// for the whole launch -- its band coefficients live in registers -- and
// streams over a chunk of beta slabs.  Per output: `len` coalesced loads,
// `len` FMAs and one coalesced store.
template <int MAXB>
__global__ void __launch_bounds__(NT) k_contract_rs(const double* __restrict__ A, double* __restrict__ out,
                                                    uint32_t a, uint32_t K, uint32_t M, uint32_t b, uint32_t bch,
                                                    FastDiv fa, BandOp op, int accumulate) {
  const uint32_t pairs = a * M;
  const uint32_t pi = blockIdx.x * NT + threadIdx.x;
  if (pi >= pairs) return;
  const uint32_t m = fa.div(pi);
  const uint32_t al = pi - m * a;
  const int lo = __ldg(op.lo + m), len = __ldg(op.len + m);
  const double* cf = op.coef + __ldg(op.off + m);
  double c[MAXB];
#pragma unroll
  for (int t = 0; t < MAXB; ++t) c[t] = t < len ? __ldg(cf + t) : 0.0;
  const uint32_t b0 = blockIdx.y * bch;
  const uint32_t b1 = min(b, b0 + bch);
  const size_t in_step = static_cast<size_t>(a) * K, out_step = pairs;
  const double* src = A + al + static_cast<size_t>(a) * lo + in_step * b0;
  double* dst = out + pi + out_step * b0;
  uint32_t be = b0;
  if (MAXB <= 8) {  // QB beta slabs per pass: QB x len independent loads in flight
    constexpr int QB = 4;  // measured: 4 beats 8 on C5 (149 vs 158 us)
    for (; be + QB - 1 < b1; be += QB, src += QB * in_step, dst += QB * out_step) {
      double s[QB][2];
#pragma unroll
      for (int q = 0; q < QB; ++q) s[q][0] = s[q][1] = 0.0;
#pragma unroll
      for (int t = 0; t < MAXB; t += 2)
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const double* sq = src + q * in_step;
          if (t < len) s[q][0] = fma(c[t], __ldg(sq + static_cast<size_t>(t) * a), s[q][0]);
          if (t + 1 < len) s[q][1] = fma(c[t + 1], __ldg(sq + static_cast<size_t>(t + 1) * a), s[q][1]);
        }
#pragma unroll
      for (int q = 0; q < QB; ++q) {
        const double v = s[q][0] + s[q][1];
        double* d = dst + q * out_step;
        *d = accumulate ? *d + v : v;
      }
    }
  }
  for (; be < b1; ++be, src += in_step, dst += out_step) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int t = 0; t < MAXB; t += 2) {
      if (t < len) s0 = fma(c[t], __ldg(src + static_cast<size_t>(t) * a), s0);
      if (t + 1 < len) s1 = fma(c[t + 1], __ldg(src + static_cast<size_t>(t + 1) * a), s1);
    }
    const double s = s0 + s1;
    *dst = accumulate ? *dst + s : s;
  }
}

// Wide-window row-blocked contraction for G operators (X_j^T of B-spline
// factors, ~17-26 nonzeros per row, consecutive rows shifted by n_j / p_j):
// CTA = (group of kGB output rows, alpha block, beta block); the group's
// zero-padded kGB x kGW coefficient block sits in shared memory (broadcast
// reads), each thread loads one kGW-row input window per (alpha, beta) and
// produces kGB outputs from it, so an input element is fetched once per group
// instead of once per output row (~2.3x less L2 traffic than the
// row-stationary kernel).  Sums ascend over the window (zeros included).
template <int RB, int RW>
__global__ void __launch_bounds__(NT, RB <= 4 ? 4 : 1) k_contract_gb(const double* __restrict__ A, double* __restrict__ out, uint32_t a,
                                                    uint32_t K, uint32_t M, uint32_t b, uint32_t ab, uint32_t bspan,
                                                    const int* __restrict__ wblo, const double* __restrict__ wbcoef,
                                                    int accumulate) {
  __shared__ double cs[RB * RW];
  const uint32_t g = blockIdx.x;
  for (int i = threadIdx.x; i < RB * RW; i += NT) cs[i] = __ldg(wbcoef + static_cast<size_t>(g) * RB * RW + i);
  __syncthreads();
  // programmatic dependent launch (Launch::pdl): everything above reads design
  // constants only; the input array belongs to the kernel before this one
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t nbl = NT / ab;  // beta lanes per CTA
  const uint32_t lane_a = threadIdx.x % ab, lane_b = threadIdx.x / ab;
  const uint32_t al = blockIdx.y * ab + lane_a;
  if (lane_b >= nbl || al >= a) return;
  const int wlo = __ldg(wblo + g);
  const int nr = static_cast<int>(min(static_cast<uint32_t>(RB), M - g * RB));
  const size_t in_step = static_cast<size_t>(a) * K, out_step = static_cast<size_t>(a) * M;
  const uint32_t b0 = blockIdx.z * bspan, b1 = min(b, b0 + bspan);
  for (uint32_t be = b0 + lane_b; be < b1; be += nbl) {
    const double* src = A + al + static_cast<size_t>(a) * wlo + in_step * be;
    double* dst = out + al + static_cast<size_t>(a) * (g * RB) + out_step * be;
    if constexpr (RB <= 4) {
      double s0[RB], s1[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) s0[r] = s1[r] = 0.0;
      // stream the wide window: every loaded pair feeds all RB rows (even /
      // odd window positions into separate sums, then their sum per row)
#pragma unroll
      for (int w = 0; w < RW; w += 2) {
        const double x0 = __ldg(src + static_cast<size_t>(w) * a), x1 = __ldg(src + static_cast<size_t>(w + 1) * a);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          s0[r] = fma(cs[r * RW + w], x0, s0[r]);
          s1[r] = fma(cs[r * RW + w + 1], x1, s1[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (r < nr) {
          const double v = s0[r] + s1[r];
          double* d = dst + static_cast<size_t>(r) * a;
          *d = accumulate ? *d + v : v;
        }
      }
    } else {  // narrow window, many rows: keep the window, one row at a time
      double win[RW];
#pragma unroll
      for (int w = 0; w < RW; ++w) win[w] = __ldg(src + static_cast<size_t>(w) * a);
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (r < nr) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int w = 0; w < RW; w += 2) {
            s0 = fma(cs[r * RW + w], win[w], s0);
            s1 = fma(cs[r * RW + w + 1], win[w + 1], s1);
          }
          const double v = s0 + s1;
          double* d = dst + static_cast<size_t>(r) * a;
          *d = accumulate ? *d + v : v;
        }
      }
    }
  }
}

static bool gb_enabled() {
  static const bool on = dev_env("KG_NO_GB") == nullptr;
  return on;
}

template <int RB, int RW>
static bool launch_blk(const Launch& L, const double* A, double* out, i64 a, i64 K, i64 M, i64 b, const int* blo,
                       const double* bcoef, bool accumulate) {
  const i64 groups = (M + RB - 1) / RB;
  const i64 ab = std::min<i64>(a, NT);
  const i64 nbl = NT / ab;
  const i64 gy = (a + ab - 1) / ab;
  // beta span per CTA: about 148 x 8 CTAs in total, a multiple of the beta lanes
  i64 gz = std::max<i64>(1, (148 * 8 + groups * gy - 1) / (groups * gy));
  gz = std::min<i64>(gz, std::max<i64>(1, (b + nbl - 1) / nbl));
  i64 bspan = (b + gz - 1) / gz;
  bspan = (bspan + nbl - 1) / nbl * nbl;
  gz = (b + bspan - 1) / bspan;
  if (groups > 0x7fffffff || gy > 65535 || gz > 65535) return false;
  if (groups * gy * gz < 2 * 148) return false;  // too few CTAs to fill the GPU: the row-stationary kernel
  PdlConfig pc(dim3(static_cast<unsigned>(groups), static_cast<unsigned>(gy), static_cast<unsigned>(gz)), dim3(NT), 0, L);
  cudaLaunchKernelEx(&pc.cfg, k_contract_gb<RB, RW>, A, out, static_cast<uint32_t>(a), static_cast<uint32_t>(K),
                     static_cast<uint32_t>(M), static_cast<uint32_t>(b), static_cast<uint32_t>(ab),
                     static_cast<uint32_t>(bspan), blo, bcoef, static_cast<int>(accumulate));
  bump(L);
  return true;
}

// Row-blocked banded contraction (H operators): a thread computes kRB
// consecutive output rows m of one (alpha, beta) from their common input
// window of kRW values, loaded once (the rows of a B-spline factor overlap),
// with the dense zero-padded kRB x kRW coefficient block of the group.
__global__ void __launch_bounds__(NT) k_contract_rb(const double* __restrict__ A, double* __restrict__ out,
                                                    uint32_t a, uint32_t K, uint32_t M, uint32_t b, uint32_t bch,
                                                    FastDiv fa, BandOp op) {
  const uint32_t groups = (M + kRB - 1) / kRB, pairs = a * groups;
  const uint32_t pi = blockIdx.x * NT + threadIdx.x;
  if (pi >= pairs) return;
  const uint32_t g = fa.div(pi), al = pi - g * a;
  const int wlo = __ldg(op.blo + g);
  const double* cb = op.bcoef + static_cast<size_t>(g) * kRB * kRW;
  const uint32_t b0 = blockIdx.y * bch, b1 = min(b, b0 + bch);
  const size_t in_step = static_cast<size_t>(a) * K, out_step = static_cast<size_t>(a) * M;
  const double* src = A + al + static_cast<size_t>(a) * wlo + in_step * b0;
  double* dst = out + al + static_cast<size_t>(a) * (g * kRB) + out_step * b0;
  const int nr = static_cast<int>(min(static_cast<uint32_t>(kRB), M - g * kRB));
  for (uint32_t be = b0; be < b1; ++be, src += in_step, dst += out_step) {
    double win[kRW];
#pragma unroll
    for (int w = 0; w < kRW; ++w) win[w] = __ldg(src + static_cast<size_t>(w) * a);
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      if (r < nr) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kRW; ++w) s = fma(__ldg(cb + r * kRW + w), win[w], s);
        dst[static_cast<size_t>(r) * a] = s;
      }
    }
  }
}

static bool rb_enabled() {  // opt-in (KG_RB=1): slower than k_contract_rs on the C5 path so far
  static const bool on = dev_env("KG_RB") != nullptr && dev_env("KG_RB")[0] == '1';
  return on;
}

template <int MAXB>
static void launch_rs(const Launch& L, const double* A, double* out, i64 a, i64 K, i64 M, i64 b, const BandOp& op,
                      bool accumulate) {
  const i64 pairs = a * M;
  const i64 gx = (pairs + NT - 1) / NT;
  static const i64 cap = [] {
    const char* e = dev_env("KG_RS_BLOCKS");
    return e ? std::max<i64>(148, std::atoll(e)) : 148 * 32;
  }();
  // ~cap CTAs; each thread's beta chunk a multiple of the 4-slab pass (no scalar tail)
  i64 gy = std::max<i64>(1, (cap + gx - 1) / gx);
  gy = std::min<i64>(gy, std::min<i64>(b, 65535));
  i64 bch = (b + gy - 1) / gy;
  if (MAXB <= 8 && b >= 4) bch = (bch + 3) / 4 * 4;
  gy = (b + bch - 1) / bch;
  k_contract_rs<MAXB><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), NT, 0, L.s>>>(
      A, out, static_cast<uint32_t>(a), static_cast<uint32_t>(K), static_cast<uint32_t>(M),
      static_cast<uint32_t>(b), static_cast<uint32_t>(bch), FastDiv(static_cast<uint32_t>(a)), op, accumulate);
}

void contract(const Launch& L, const double* A, double* out, i64 a, i64 K, i64 M, i64 b, const BandOp& op,
              bool accumulate) {
  const i64 total = a * M * b;
  if (total == 0) return;
  // row-blocked kernel: H operators with a blocked copy, window inside the input
  if (op.blo && !accumulate && rb_enabled() && a >= 32 && K >= kRW && a * ((M + kRB - 1) / kRB) < (i64(1) << 31) &&
      a * K * b < (i64(1) << 31) * 4) {
    const i64 pairs = a * ((M + kRB - 1) / kRB);
    const i64 gx = (pairs + NT - 1) / NT;
    i64 gy = std::max<i64>(1, (148 * 16 + gx - 1) / gx);
    gy = std::min<i64>(gy, std::min<i64>(b, 65535));
    const i64 bch = (b + gy - 1) / gy;
    gy = (b + bch - 1) / bch;
    k_contract_rb<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), NT, 0, L.s>>>(
        A, out, static_cast<uint32_t>(a), static_cast<uint32_t>(K), static_cast<uint32_t>(M), static_cast<uint32_t>(b),
        static_cast<uint32_t>(bch), FastDiv(static_cast<uint32_t>(a)), op);
    bump(L);
    return;
  }
  // row-blocked kernels from the operators' blocked copies: G (kGB rows,
  // kGW-wide windows) and H (kHB rows, kHW-wide windows)
  if (gb_enabled() && a >= 64 && a < (i64(1) << 31) && b < (i64(1) << 31) && a * K * b < (i64(1) << 31) * 4) {
    if (op.wblo && K >= kGW && launch_blk<kGB, kGW>(L, A, out, a, K, M, b, op.wblo, op.wbcoef, accumulate)) return;
    if (op.hblo && K >= kHW && launch_blk<kHB, kHW>(L, A, out, a, K, M, b, op.hblo, op.hbcoef, accumulate)) return;
  }
  // register-hoisted row-stationary kernel for banded operators (all B-spline factors)
  if (op.maxlen <= 64 && a * M < (i64(1) << 31) && a * K * b < (i64(1) << 31) * 4 && b < (i64(1) << 31) &&
      (a * M + NT - 1) / NT < (i64(1) << 31)) {
    if (op.maxlen <= 4) launch_rs<4>(L, A, out, a, K, M, b, op, accumulate);
    else if (op.maxlen <= 8) launch_rs<8>(L, A, out, a, K, M, b, op, accumulate);
    else if (op.maxlen <= 16) launch_rs<16>(L, A, out, a, K, M, b, op, accumulate);
    else if (op.maxlen <= 24) launch_rs<24>(L, A, out, a, K, M, b, op, accumulate);
    else if (op.maxlen <= 32) launch_rs<32>(L, A, out, a, K, M, b, op, accumulate);
    else launch_rs<64>(L, A, out, a, K, M, b, op, accumulate);
    bump(L);
    return;
  }
  if (a * M < (i64(1) << 31) && a * K < (i64(1) << 31) && b < (i64(1) << 31)) {
    const i64 gx = (a * M + NT - 1) / NT;
    const i64 gy = std::min<i64>(b, 65535);
    const i64 gz = (b + gy - 1) / gy;
    if (gx < (i64(1) << 31) && gz <= 65535) {
      k_contract2<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(gz)), NT, 0,
                    L.s>>>(A, out, static_cast<uint32_t>(a), static_cast<uint32_t>(K), static_cast<uint32_t>(M),
                           static_cast<uint32_t>(b), FastDiv(static_cast<uint32_t>(a)), op, accumulate);
      bump(L);
      return;
    }
  }
  const int g = grid_for(total, NT * 2, 148 * 16);
  if (a * K * b < (i64(1) << 31) && total < (i64(1) << 31)) {
    k_contract<uint32_t><<<g, NT, 0, L.s>>>(A, out, static_cast<uint32_t>(a), static_cast<uint32_t>(K),
                                            static_cast<uint32_t>(M), static_cast<uint32_t>(b), op, accumulate);
  } else {
    k_contract<uint64_t><<<g, NT, 0, L.s>>>(A, out, a, K, M, b, op, accumulate);
  }
  bump(L);
}

// -------------------------------------------------------- fused mode-1 pass
// One CTA owns T consecutive mode-1 fibres (a contiguous chunk of n1*T cells
// of every n-array).  FISTA variant: eta = X1 P (from the shared-memory P
// tile), the weighted residual sum v (eta - z)^2, w = v eta kept in shared
// memory, then Q = X1^T w for the tile: the n-array eta is never written.
template <int VAR>
__global__ void __launch_bounds__(NT) k_fused1(FusedArgs f) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const int n1 = static_cast<int>(f.n1), p1 = static_cast<int>(f.p1);
  const i64 c0 = static_cast<i64>(blockIdx.x) * f.T;
  const int Tc = static_cast<int>(min(static_cast<i64>(f.T), f.m - c0));
  double* Ps = sm;
  double* W = sm + static_cast<i64>(p1) * f.T;
  const i64 base = c0 * n1;
  if (VAR == FV_FISTA) {
    const double* P = f.P + c0 * p1;
    for (int e = threadIdx.x; e < p1 * Tc; e += NT) Ps[e] = __ldg(P + e);
    __syncthreads();
  }
  double acc = 0.0;
  for (int e = threadIdx.x; e < n1 * Tc; e += NT) {
    const int col = e / n1;
    const int i = e - col * n1;
    double w;
    if (VAR == FV_FISTA) {
      const double* pc = Ps + col * p1;
      const double eta = band_dot(f.H, i, [&](int k) { return pc[k]; });
      const double vv = __ldg(f.v + base + e);
      const double r = eta - __ldg(f.z + base + e);
      acc = fma(vv, r * r, acc);
      w = vv * eta;
    } else if (VAR == FV_XTWZ) {
      w = __ldg(f.v + base + e) * __ldg(f.z + base + e);
    } else {
      w = score_of(f.fam, __ldg(f.y + base + e), __ldg(f.a + base + e), 0.0) / f.disp;
      if (!isfinite(w)) record_min(f.err, f.cell_base + base + e);
    }
    W[e] = w;
  }
  if (VAR == FV_FISTA) {
    const double s = block_reduce<false>(acc, red);
    if (threadIdx.x == 0) f.partial[blockIdx.x] = s;
  }
  __syncthreads();
  double* Q = f.Q + c0 * p1;
  for (int q = threadIdx.x; q < p1 * Tc; q += NT) {
    const int col = q / p1;
    const int k = q - col * p1;
    const double* wc = W + col * n1;
    Q[q] = band_dot(f.G, k, [&](int i) { return wc[i]; });
  }
}

static size_t fused_smem(const FusedArgs& f) { return static_cast<size_t>(f.p1 + f.n1) * f.T * sizeof(double); }

int fused_grid(const FusedArgs& f) { return static_cast<int>((f.m + f.T - 1) / f.T); }

void fused_mode1(const Launch& L, int variant, const FusedArgs& f) {
  const size_t sm = fused_smem(f);
  const int g = fused_grid(f);
  smem_attr(k_fused1<FV_FISTA>, 200 * 1024);
  smem_attr(k_fused1<FV_XTWZ>, 200 * 1024);
  smem_attr(k_fused1<FV_SCORE0>, 200 * 1024);
  switch (variant) {
    case FV_FISTA: k_fused1<FV_FISTA><<<g, NT, sm, L.s>>>(f); break;
    case FV_XTWZ: k_fused1<FV_XTWZ><<<g, NT, sm, L.s>>>(f); break;
    default: k_fused1<FV_SCORE0><<<g, NT, sm, L.s>>>(f); break;
  }
  bump(L);
}

// ------------------------------------------------ H-last with reductions
// eta_new = X1 P (written if HL_WRITE), plus per-CTA partials of
//   col 0: log-likelihood kernel of eta_new           (HL_LL_NEW)
//   col 1: <u, eta_new - eta_old>, u = score(eta_old)  (HL_DOT; u on the fly if HL_U_FLY)
//   col 2+j: log-likelihood at eta_old + t_j (eta_new - eta_old)  (HL_TRIALS)
// which are the Armijo / Gaussian-shortcut quantities (outer.cpp:106-144,
// outer.cpp:197-231) evaluated in the same pass that produces eta_tilde.
__global__ void __launch_bounds__(NT) k_hlast(HlastArgs h) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const int n1 = static_cast<int>(h.n1), p1 = static_cast<int>(h.p1);
  const i64 c0 = static_cast<i64>(blockIdx.x) * h.T;
  const int Tc = static_cast<int>(min(static_cast<i64>(h.T), h.m - c0));
  const i64 base = c0 * n1;
  if (h.P) {
    const double* P = h.P + c0 * p1;
    for (int e = threadIdx.x; e < p1 * Tc; e += NT) sm[e] = __ldg(P + e);
    __syncthreads();
  }
  double acc[kHlastCols];
#pragma unroll
  for (int q = 0; q < kHlastCols; ++q) acc[q] = 0.0;
  // a thread keeps one grid row when n1 divides the block: its (<= 4) band
  // coefficients live in registers, zero-padded at the end, so the sequential
  // FMA chain is band_dot's to the bit
  const bool fixed_row = h.P && (NT % n1) == 0 && h.H.maxlen <= 4;
  const int frow = threadIdx.x % n1;
  int flo = 0;
  bool fast_row = false;
  double fc[4] = {0.0, 0.0, 0.0, 0.0};
  if (fixed_row) {
    flo = __ldg(h.H.lo + frow);
    fast_row = flo <= p1 - 4;  // the 4-wide window fits in the tile row
    const int len = __ldg(h.H.len + frow);
    const double* cf = h.H.coef + __ldg(h.H.off + frow);
#pragma unroll
    for (int t = 0; t < 4; ++t) fc[t] = (t < len) ? __ldg(cf + t) : 0.0;
  }
  // the global operands of a cell are loaded one cell ahead (software pipeline)
  const bool need_y = (h.flags & (HL_LL_NEW | HL_DOT | HL_TRIALS)) != 0;
  const bool need_eo = (h.flags & (HL_DOT | HL_TRIALS)) != 0;
  double nyy = 0.0, naa = h.a_val, neo = 0.0;
  auto fetch = [&](int e) {
    if (e >= n1 * Tc) return;
    const i64 g = base + e;
    if (need_y) {
      nyy = __ldcs(h.y + g);
      if (h.a) naa = __ldcs(h.a + g);
    }
    if (need_eo) neo = __ldcs(h.eta_old + g);
  };
  fetch(threadIdx.x);
  for (int e = threadIdx.x; e < n1 * Tc; e += NT) {
    const i64 g = base + e;
    const double cyy = nyy, caa = naa, ceo = neo;
    fetch(e + NT);
    double en;
    if (fixed_row) {
      const double* pc = sm + (e / n1) * p1;
      if (fast_row) {  // zeros after the band: fma(0, p, s) == s
        const double* q = pc + flo;
        en = fma(fc[3], q[3], fma(fc[2], q[2], fma(fc[1], q[1], fma(fc[0], q[0], 0.0))));
      } else {
        en = band_dot(h.H, frow, [&](int k) { return pc[k]; });
      }
      if (h.flags & HL_WRITE) h.eta_new[g] = en;
    } else if (h.P) {
      const int col = e / n1;
      const int i = e - col * n1;
      const double* pc = sm + col * p1;
      en = band_dot(h.H, i, [&](int k) { return pc[k]; });
      if (h.flags & HL_WRITE) h.eta_new[g] = en;
    } else {
      en = __ldg(h.eta_new + g);
    }
    if (need_y) {
      const double yy = cyy, aa = caa;
      if ((h.flags & HL_LL_NEW) && aa != 0.0) {
        const double t = ll_term(h.fam, yy, aa, en);
        if (!isfinite(t)) record_min(h.err + 0, h.cell_base + g);
        acc[0] += t;
      }
      if (need_eo) {
        const double eo = ceo;
        if (h.flags & HL_DOT) {
          double u;
          if (h.flags & HL_U_FLY) {
            u = score_of(h.fam, yy, aa, eo) / h.disp;
            if (!isfinite(u)) record_min(h.err + 1, h.cell_base + g);
          } else {
            u = __ldg(h.u + g);
          }
          acc[1] = fma(u, en - eo, acc[1]);
        }
        if ((h.flags & HL_TRIALS) && aa != 0.0) {
          for (int j = 0; j < h.ntrial; ++j) {
            const double et = eo + h.t[j] * (en - eo);
            const double t = ll_term(h.fam, yy, aa, et);
            if (!isfinite(t)) record_min(h.err + 2 + j, h.cell_base + g);
            acc[2 + j] += t;
          }
        }
      }
    }
  }
  const int ncols = 2 + h.ntrial;
  for (int q = 0; q < ncols; ++q) {
    const double s = block_reduce<false>(acc[q], red);
    if (threadIdx.x == 0) h.partial[static_cast<i64>(blockIdx.x) * kHlastCols + q] = s;
  }
}

int hlast_grid(const HlastArgs& h) { return static_cast<int>((h.m + h.T - 1) / h.T); }

void hlast_mode1(const Launch& L, const HlastArgs& h) {
  smem_attr(k_hlast, 200 * 1024);
  const size_t sm = h.P ? static_cast<size_t>(h.p1) * h.T * sizeof(double) : 0;
  k_hlast<<<hlast_grid(h), NT, sm, L.s>>>(h);
  bump(L);
}

// ------------------------------------------------------- elementwise family
__global__ void __launch_bounds__(NT) k_family(FamilyArgs f) {
  __shared__ double red[32];
  double vmax = -DBL_MAX;
  auto cell = [&](i64 i, double yy, double aa, double e) {
    const double ec = clampe(e);
    double u, v, z;
    if (f.fam == 2 && f.mode != 1) {  // Poisson, exact weights: one exp(clamp(eta)) serves score, weight and z
      const double mu = exp(ec);
      u = aa * (yy - mu) / f.disp;   // score_of (family.cpp:164-196)
      v = fmax(mu, kFloor) / f.disp;
      z = aa * (yy - mu) / fmax(mu, kFloor) + e;
    } else {
      u = score_of(f.fam, yy, aa, e) / f.disp;
      if (f.mode == 1) {  // unit weights, generic working response (outer.cpp:148-155)
        v = 1.0;
        z = u / v + e;
      } else {
        double w = 1.0;
        if (f.fam == 1) {
          const double mu = logistic(e);
          w = mu * (1.0 - mu);
        } else if (f.fam == 2) {
          w = exp(ec);
        }
        v = fmax(w, kFloor) / f.disp;
        switch (f.fam) {
          case 0: z = aa * (yy - e) + e; break;
          case 1: {
            const double mu = logistic(ec);
            z = aa * (yy - mu) / fmax(mu * (1.0 - mu), kFloor) + e;
            break;
          }
          case 2: {
            const double mu = exp(ec);
            z = aa * (yy - mu) / fmax(mu, kFloor) + e;
            break;
          }
          default: {
            const double mu = exp(ec);
            z = aa * (yy - mu) / mu + e;
            break;
          }
        }
      }
    }
    if (!isfinite(u)) record_min(f.err + 0, f.cell_base + i);
    if (f.mode != 1 && !isfinite(z)) record_min(f.err + 1, f.cell_base + i);
    if (f.u) f.u[i] = u;
    f.v[i] = v;
    f.z[i] = z;
    vmax = fmax(vmax, v);
  };
  // four cells per thread and trip, their loads issued together
  const i64 G = static_cast<i64>(gridDim.x) * NT;
  for (i64 i0 = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i0 < f.n; i0 += 4 * G) {
    double yy[4], aa[4], ee[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const i64 i = i0 + k * G;
      yy[k] = aa[k] = ee[k] = 0.0;
      if (i < f.n) {
        yy[k] = __ldcs(f.y + i);
        ee[k] = __ldcs(f.eta + i);
        aa[k] = f.a ? __ldcs(f.a + i) : f.a_val;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * G < f.n) cell(i0 + k * G, yy[k], aa[k], ee[k]);
  }
  const double m = block_reduce<true>(vmax, red);
  if (threadIdx.x == 0) f.partial[blockIdx.x] = m;
}

void family_pass(const Launch& L, const FamilyArgs& f) {
  k_family<<<elem_grid(f.n), NT, 0, L.s>>>(f);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_gauss_weights(i64 n, double disp, const double* a, double* v, double* part) {
  __shared__ double red[32];
  double vmax = -DBL_MAX;
  const double w = fmax(1.0, kFloor) / disp;  // glm_weights(gaussian) (family.cpp:198-221)
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double vv = w * a[i];
    v[i] = vv;
    vmax = fmax(vmax, vv);
  }
  const double m = block_reduce<true>(vmax, red);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

void gauss_weights(const Launch& L, i64 n, double disp, const double* a, double* v, double* partial) {
  k_gauss_weights<<<elem_grid(n), NT, 0, L.s>>>(n, disp, a, v, partial);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_wss(i64 n, const double* eta, const double* v, const double* z, double* w,
                                            double* part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double e = eta[i], vv = v[i], r = e - z[i];
    acc = fma(vv, r * r, acc);
    w[i] = vv * e;
  }
  const double s = block_reduce<false>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void wss(const Launch& L, i64 n, const double* eta, const double* v, const double* z, double* w, double* partial) {
  k_wss<<<elem_grid(n), NT, 0, L.s>>>(n, eta, v, z, w, partial);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_vz(i64 n, const double* v, const double* z, double* w) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT)
    w[i] = v[i] * z[i];
}

void vz(const Launch& L, i64 n, const double* v, const double* z, double* w) {
  k_vz<<<elem_grid(n), NT, 0, L.s>>>(n, v, z, w);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_score0(i64 n, int fam, double disp, const double* y, const double* a,
                                               double* w, i64* err, i64 cell_base) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double u = score_of(fam, y[i], a[i], 0.0) / disp;
    if (!isfinite(u)) record_min(err, cell_base + i);
    w[i] = u;
  }
}

void score0(const Launch& L, i64 n, int fam, double disp, const double* y, const double* a, double* w, i64* err,
            i64 cell_base) {
  k_score0<<<elem_grid(n), NT, 0, L.s>>>(n, fam, disp, y, a, w, err, cell_base);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_validate(i64 n, int fam, const double* y, const double* a, i64* err,
                                                 i64 cell_base) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double ai = a[i];
    bool bad = !(ai >= 0.0) || !isfinite(ai);
    if (!bad && ai != 0.0) {
      const double yi = y[i];
      bad = !isfinite(yi) || (fam == 1 && (yi < 0.0 || yi > 1.0)) || (fam == 2 && yi < 0.0) ||
            (fam == 3 && !(yi > 0.0));
    }
    if (bad) record_min(err, cell_base + i);
  }
}

void validate_pass(const Launch& L, i64 n, int fam, const double* y, const double* a, i64* err, i64 cell_base) {
  k_validate<<<elem_grid(n), NT, 0, L.s>>>(n, fam, y, a, err, cell_base);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_eta_combine(i64 n, double t, const double* et, double* eta) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double e = eta[i];
    eta[i] = e + t * (et[i] - e);  // trial_eta (outer.cpp:131)
  }
}

void eta_combine(const Launch& L, i64 n, double t, const double* eta_t, double* eta) {
  k_eta_combine<<<elem_grid(n), NT, 0, L.s>>>(n, t, eta_t, eta);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_mean(i64 n, int fam, const double* eta, double* mu) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double e = eta[i];
    mu[i] = fam == 0 ? e : (fam == 1 ? logistic(e) : exp(clampe(e)));
  }
}

void mean_map(const Launch& L, i64 n, int fam, const double* eta, double* mu) {
  k_mean<<<elem_grid(n), NT, 0, L.s>>>(n, fam, eta, mu);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_fill(i64 n, double v, double* x) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) x[i] = v;
}

void fill(const Launch& L, i64 n, double v, double* x) {
  k_fill<<<elem_grid(n), NT, 0, L.s>>>(n, v, x);
  bump(L);
}

// ---------------------------------------------------------------- p-space
// The step, threshold and soft-threshold use explicitly rounded operations
// (never contracted into FMAs, as the reference computes them): at
// lambda = lambda_max the first step must land exactly on zero, which needs
// |y - delta g| <= delta lambda to be decided on separately rounded values.
__device__ __forceinline__ double soft(double z, double g) {
  const double m = __dsub_rn(fabs(z), g);
  if (m <= 0.0) return 0.0;
  return z > 0.0 ? m : -m;
}

__device__ __forceinline__ double prox1(int pen, double alpha, double gamma, double z) {
  if (pen == 0) return soft(z, gamma);
  if (pen == 1) return z * (1.0 / (1.0 + 2.0 * gamma));
  return (1.0 / (1.0 + 2.0 * alpha * gamma)) * soft(z, gamma);
}

// J pieces: l1 and squared l2 partial sums are kept separate so J is formed
// as in penalty.cpp:24-34.
__device__ __forceinline__ void jacc(double x, double& l1, double& l2) {
  l1 += fabs(x);
  l2 = fma(x, x, l2);
}

// One accelerated proximal-gradient step (inner.cpp:163-193), using
// S(y) = S(x) + omega (S(x) - S(x_prev)) with S = X^T W X (linearity of the
// map), so each iteration needs one n-array pass on the new iterate only.
__global__ void __launch_bounds__(NT) k_fista_update(const FistaCtl* __restrict__ ctl, i64 p, int pen, double alpha,
                                                     double* x, double* xp, double* Sx, double* Sxp, const double* b,
                                                     double* best, double* Sbest, double* Jpart,
                                                     double* bxpart) {
  __shared__ double red[32];
  if (ctl->done) return;  // batched host loops (sharded contexts) enqueue steps past the stop
  const double omega = ctl->omega, delta = ctl->delta, lambda = ctl->lambda, n = ctl->n, sscale = ctl->sscale;
  const int copy_best = ctl->copy_best, restart = ctl->restart;
  const double gamma = __dmul_rn(delta, lambda);
  double l1 = 0.0, l2 = 0.0, bx = 0.0;
  // the thread's elements in grid-stride order (so the partials are summed in
  // the same order), four per trip with their loads issued together
  const i64 G = static_cast<i64>(gridDim.x) * NT;
  for (i64 i0 = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i0 < p; i0 += 4 * G) {
    double lx[4], lxp[4], lsx[4], lsxp[4], lb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const i64 i = i0 + k * G;
      if (i < p) {
        lx[k] = x[i];
        lxp[k] = xp[i];
        lsx[k] = Sx[i];
        lsxp[k] = Sxp[i];
        lb[k] = b[i];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
    const i64 i = i0 + k * G;
    if (i >= p) break;
    double xi = lx[k], xpi = lxp[k], sxi = lsx[k], sxpi = lsxp[k];
    const double bi = lb[k];
    if (copy_best) {
      best[i] = xi;
      Sbest[i] = sxi;
    }
    if (restart) {
      xi = xpi = best[i];
      sxi = sxpi = Sbest[i];
    }
    const double yi = xi + omega * (xi - xpi);
    const double syi = sxi + omega * (sxi - sxpi);
    const double g = (sscale * syi - bi) / n;
    double ci = __dsub_rn(yi, __dmul_rn(delta, g));
    if (lambda > 0.0) ci = prox1(pen, alpha, gamma, ci);
    xp[i] = xi;
    x[i] = ci;
    Sxp[i] = sxi;
    jacc(ci, l1, l2);
    if (bxpart) bx = fma(bi, ci, bx);
    }
  }
  const double s1 = block_reduce<false>(l1, red);
  const double s2 = block_reduce<false>(l2, red);
  if (threadIdx.x == 0) {
    Jpart[2 * blockIdx.x] = s1;
    Jpart[2 * blockIdx.x + 1] = s2;
  }
  if (bxpart) {
    const double s3 = block_reduce<false>(bx, red);
    if (threadIdx.x == 0) bxpart[blockIdx.x] = s3;
  }
}

void fista_update(const Launch& L, const FistaCtl* ctl, i64 p, int pen, double alpha, double* x, double* xp,
                  double* Sx, double* Sxp, const double* b, double* best, double* Sbest, double* Jpart,
                  double* bxpart) {
  k_fista_update<<<ugrid(p), NT, 0, L.s>>>(ctl, p, pen, alpha, x, xp, Sx, Sxp, b, best, Sbest, Jpart, bxpart);
  bump(L);
}

// ---------------------------------------------- tensor weights (iwls = tensor)
// compute_weights tensor branch (outer.cpp:53-103): slab sums of log v over
// mode j, S[i] = sum over cells with i_j = i, for the array viewed as (a, K, b).
__global__ void __launch_bounds__(NT) k_log_slab_sums(const double* v, i64 a, i64 K, i64 b, double* S) {
  __shared__ double red[32];
  const i64 i = blockIdx.x;
  const i64 cnt = a * b;
  double s = 0.0;
  for (i64 e = threadIdx.x; e < cnt; e += NT) {
    const i64 al = e % a, be = e / a;
    s += log(v[al + a * (i + K * be)]);
  }
  const double r = block_reduce<false>(s, red);
  if (threadIdx.x == 0) S[i] = r;
}

void log_slab_sums(const Launch& L, const double* v, i64 a, i64 K, i64 b, double* S) {
  k_log_slab_sums<<<static_cast<unsigned>(K), NT, 0, L.s>>>(v, a, K, b, S);
  bump(L);
}

// f_j[i] = exp(S_j[i] / m_j - log vbar + log vbar / d), log vbar = (sum of the
// mode-0 slab sums) / n; S and f are the concatenation over modes.
__global__ void k_tensor_factors(const double* S, const i64* ext, int d, i64 n, double* f) {
  __shared__ double lvbar;
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (i64 i = 0; i < ext[0]; ++i) tot += S[i];
    lvbar = tot / static_cast<double>(n);
  }
  __syncthreads();
  i64 off = 0;
  for (int j = 0; j < d; ++j) {
    const double mj = static_cast<double>(n / ext[j]);
    for (i64 i = threadIdx.x; i < ext[j]; i += blockDim.x)
      f[off + i] = exp(S[off + i] / mj - lvbar + lvbar / static_cast<double>(d));
    off += ext[j];
  }
}

void tensor_factors(const Launch& L, const double* S, const i64* ext_dev, int d, i64 n, double* f) {
  k_tensor_factors<<<1, 256, 0, L.s>>>(S, ext_dev, d, n, f);
  bump(L);
}

// v = outer product of the factors (prod = 1, *= f_0[i_0], ..., in mode order),
// z = u / v + eta (generic working response, outer.cpp:148-155), max(v) partials.
__global__ void __launch_bounds__(NT) k_tensor_vz(i64 n, TensorExt te, const double* f, const double* u,
                                                  const double* eta, double* v, double* z, double* vmax) {
  __shared__ double red[32];
  double mx = -DBL_MAX;
  for (i64 c = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; c < n; c += static_cast<i64>(gridDim.x) * NT) {
    i64 rest = c, off = 0;
    double prod = 1.0;
    for (int j = 0; j < te.d; ++j) {
      const i64 ij = rest % te.ext[j];
      rest /= te.ext[j];
      prod *= f[off + ij];
      off += te.ext[j];
    }
    v[c] = prod;
    z[c] = u[c] / prod + eta[c];
    mx = fmax(mx, prod);
  }
  const double r = block_reduce<true>(mx, red);
  if (threadIdx.x == 0) vmax[blockIdx.x] = r;
}

void tensor_vz(const Launch& L, i64 n, const TensorExt& te, const double* f, const double* u, const double* eta,
               double* v, double* z, double* vmax) {
  k_tensor_vz<<<elem_grid(n), NT, 0, L.s>>>(n, te, f, u, eta, v, z, vmax);
  bump(L);
}

// Weighted Gram band X_m^T diag(w) X_r (GramBlocks, design.cpp:126-151): for
// band row a, entries b in [lo_a, lo_a + len_a): sum over the rows both columns
// touch, ascending, of (X_m[i, a] w[i]) X_r[i, b].
__global__ void k_wgram_band(const double* Xm, const double* Xr, i64 n, const double* w, const int* clo_m,
                             const int* clen_m, const int* clo_r, const int* clen_r, BandOp g, double* coef) {
  const int a = blockIdx.x;
  const int lo = g.lo[a], len = g.len[a];
  const i64 off = g.off[a];
  for (int t = threadIdx.x; t < len; t += blockDim.x) {
    const int b = lo + t;
    const int i0 = max(clo_m[a], clo_r[b]), i1 = min(clo_m[a] + clen_m[a], clo_r[b] + clen_r[b]);
    double s = 0.0;
    for (int i = i0; i < i1; ++i) s += Xm[i + n * a] * w[i] * Xr[i + n * static_cast<i64>(b)];
    coef[off + t] = s;
  }
}

void wgram_band(const Launch& L, const double* Xm, const double* Xr, i64 n, const double* w, const int* clo_m,
                const int* clen_m, const int* clo_r, const int* clen_r, const BandOp& g, double* coef) {
  k_wgram_band<<<static_cast<unsigned>(g.rows), 64, 0, L.s>>>(Xm, Xr, n, w, clo_m, clen_m, clo_r, clen_r, g, coef);
  bump(L);
}

// dense p x p copy of a band operator (power iteration input)
__global__ void k_band_dense(BandOp g, const double* coef, i64 p, double* G) {
  const int a = blockIdx.x;
  for (int t = threadIdx.x; t < g.len[a]; t += blockDim.x) G[a + p * static_cast<i64>(g.lo[a] + t)] = coef[g.off[a] + t];
}

void band_dense(const Launch& L, const BandOp& g, const double* coef, i64 p, double* G) {
  KG_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * p * p, L.s));
  k_band_dense<<<static_cast<unsigned>(g.rows), 64, 0, L.s>>>(g, coef, p, G);
  bump(L);
}

// per-CTA partials of sum over mask == 1 of (mu - y)^2 (mse_heldout, path.cpp:111-119)
__global__ void __launch_bounds__(NT) k_masked_sse(i64 n, const double* mu, const double* y, const double* mask,
                                                   double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT)
    if (mask[i] == 1.0) {
      const double d = mu[i] - y[i];
      s = fma(d, d, s);
    }
  const double r = block_reduce<false>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void masked_sse(const Launch& L, i64 n, const double* mu, const double* y, const double* mask, double* part) {
  k_masked_sse<<<elem_grid(n), NT, 0, L.s>>>(n, mu, y, mask, part);
  bump(L);
}

// Deviance terms of eta (SURVEY 8(d) parity protocol, family.cpp conventions:
// mu with the +-30 clamp, a = 0 cells skipped, 0 log 0 = 0), per-CTA partials.
__device__ __forceinline__ double xlogy_ratio(double y, double m) { return y == 0.0 ? 0.0 : y * log(y / m); }
__global__ void __launch_bounds__(NT) k_deviance(i64 n, int fam, const double* __restrict__ y,
                                                 const double* __restrict__ a, const double* __restrict__ eta,
                                                 double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double ai = a[i];
    if (ai == 0.0) continue;
    const double yi = y[i], e = eta[i];
    double t;
    if (fam == 0) {
      const double r = yi - e;
      t = ai * (r * r);
    } else if (fam == 1) {
      const double mu = logistic(e);
      t = 2.0 * ai * (xlogy_ratio(yi, mu) + xlogy_ratio(1.0 - yi, 1.0 - mu));
    } else if (fam == 2) {
      const double mu = exp(clampe(e));
      t = 2.0 * ai * (xlogy_ratio(yi, mu) - (yi - mu));
    } else {
      const double mu = exp(clampe(e));
      t = 2.0 * ai * (-log(yi / mu) + (yi - mu) / mu);
    }
    s += t;
  }
  const double r = block_reduce<false>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void deviance_pass(const Launch& L, i64 n, int fam, const double* y, const double* a, const double* eta,
                   double* part) {
  k_deviance<<<elem_grid(n), NT, 0, L.s>>>(n, fam, y, a, eta, part);
  bump(L);
}

// ------------------------------------------ nu = 0 (backtracking every step)
// inner.cpp:162-183: y = x + omega (x - x_prev), S y by linearity, grad =
// (s S y - b) / n; partials [<y, S y>, <b, y>] for h(y).
__global__ void __launch_bounds__(NT) k_bt_prep(i64 p, double omega, double sscale, double n, const double* x,
                                                const double* xp, const double* Sx, const double* Sxp,
                                                const double* b, double* y, double* grad, double* part) {
  __shared__ double red[32];
  double a0 = 0.0, a1 = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    const double yi = x[i] + omega * (x[i] - xp[i]);
    const double syi = Sx[i] + omega * (Sx[i] - Sxp[i]);
    y[i] = yi;
    grad[i] = (sscale * syi - b[i]) / n;
    a0 = fma(yi, syi, a0);
    a1 = fma(b[i], yi, a1);
  }
  const double r0 = block_reduce<false>(a0, red);
  const double r1 = block_reduce<false>(a1, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r0;
    part[2 * blockIdx.x + 1] = r1;
  }
}

void bt_prep(const Launch& L, i64 p, double omega, double sscale, double n, const double* x, const double* xp,
             const double* Sx, const double* Sxp, const double* b, double* y, double* grad, double* part) {
  k_bt_prep<<<pgrid(p), NT, 0, L.s>>>(p, omega, sscale, n, x, xp, Sx, Sxp, b, y, grad, part);
  bump(L);
}

// one trial: cand = prox(y - delta grad); partials [<grad, step>, |step|^2,
// l1(cand), l2(cand)] with step = cand - y.
__global__ void __launch_bounds__(NT) k_bt_trial(i64 p, double delta, double lambda, int pen, double alpha,
                                                 const double* y, const double* grad, double* cand, double* part) {
  __shared__ double red[32];
  double a0 = 0.0, a1 = 0.0, l1 = 0.0, l2 = 0.0;
  const double gamma = __dmul_rn(delta, lambda);
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    double c = __dsub_rn(y[i], __dmul_rn(delta, grad[i]));
    if (lambda > 0.0) c = prox1(pen, alpha, gamma, c);
    cand[i] = c;
    const double st = c - y[i];
    a0 = fma(grad[i], st, a0);
    a1 = fma(st, st, a1);
    jacc(c, l1, l2);
  }
  const double r0 = block_reduce<false>(a0, red);
  const double r1 = block_reduce<false>(a1, red);
  const double r2 = block_reduce<false>(l1, red);
  const double r3 = block_reduce<false>(l2, red);
  if (threadIdx.x == 0) {
    part[4 * blockIdx.x] = r0;
    part[4 * blockIdx.x + 1] = r1;
    part[4 * blockIdx.x + 2] = r2;
    part[4 * blockIdx.x + 3] = r3;
  }
}

void bt_trial(const Launch& L, i64 p, double delta, double lambda, int pen, double alpha, const double* y,
              const double* grad, double* cand, double* part) {
  k_bt_trial<<<pgrid(p), NT, 0, L.s>>>(p, delta, lambda, pen, alpha, y, grad, cand, part);
  bump(L);
}

// partials [<x, S x>, <b, x>] (h(x) = (s <x, S x> - 2 <b, x> + sum v z^2) / 2n)
__global__ void __launch_bounds__(NT) k_bt_dots(i64 p, const double* x, const double* Sx, const double* b,
                                                double* part) {
  __shared__ double red[32];
  double a0 = 0.0, a1 = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    a0 = fma(x[i], Sx[i], a0);
    a1 = fma(b[i], x[i], a1);
  }
  const double r0 = block_reduce<false>(a0, red);
  const double r1 = block_reduce<false>(a1, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r0;
    part[2 * blockIdx.x + 1] = r1;
  }
}

void bt_dots(const Launch& L, i64 p, const double* x, const double* Sx, const double* b, double* part) {
  k_bt_dots<<<pgrid(p), NT, 0, L.s>>>(p, x, Sx, b, part);
  bump(L);
}

// per-CTA partials of <a, b> (p-space)
__global__ void __launch_bounds__(NT) k_pdot(i64 p, const double* a, const double* b, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT)
    s = fma(a[i], b[i], s);
  const double r = block_reduce<false>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void pdot(const Launch& L, i64 p, const double* a, const double* b, double* part) {
  k_pdot<<<pgrid(p), NT, 0, L.s>>>(p, a, b, part);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_pnorm(i64 p, const double* x, double* Jpart) {
  __shared__ double red[32];
  double l1 = 0.0, l2 = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT)
    jacc(x[i], l1, l2);
  const double s1 = block_reduce<false>(l1, red);
  const double s2 = block_reduce<false>(l2, red);
  if (threadIdx.x == 0) {
    Jpart[2 * blockIdx.x] = s1;
    Jpart[2 * blockIdx.x + 1] = s2;
  }
}

void pnorm(const Launch& L, i64 p, int, double, const double* x, double* Jpart) {
  k_pnorm<<<pgrid(p), NT, 0, L.s>>>(p, x, Jpart);
  bump(L);
}

struct Trials {
  double t[kMaxTrials];
};

// cols per CTA: 2 * (1 + ntrial): (l1, l2) of th_t, then of each trial point.
__global__ void __launch_bounds__(NT) k_ptrials(i64 p, const double* th, const double* tht, int ntrial, Trials T,
                                                double* part) {
  __shared__ double red[32];
  double l1[1 + kMaxTrials], l2[1 + kMaxTrials];
  for (int j = 0; j <= kMaxTrials; ++j) l1[j] = l2[j] = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    const double a = th[i], b = tht[i];
    jacc(b, l1[0], l2[0]);
    for (int j = 0; j < ntrial; ++j) jacc(a + T.t[j] * (b - a), l1[1 + j], l2[1 + j]);
  }
  const int ncol = 2 * (1 + kMaxTrials);
  for (int j = 0; j <= ntrial; ++j) {
    const double s1 = block_reduce<false>(l1[j], red);
    const double s2 = block_reduce<false>(l2[j], red);
    if (threadIdx.x == 0) {
      part[static_cast<i64>(blockIdx.x) * ncol + 2 * j] = s1;
      part[static_cast<i64>(blockIdx.x) * ncol + 2 * j + 1] = s2;
    }
  }
}

void ptrials(const Launch& L, i64 p, int, double, const double* th, const double* th_t, int ntrial, const double* t,
             double* part) {
  Trials T{};
  for (int j = 0; j < ntrial && j < kMaxTrials; ++j) T.t[j] = t[j];
  k_ptrials<<<pgrid(p), NT, 0, L.s>>>(p, th, th_t, ntrial, T, part);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_ptheta(i64 p, double t, const double* tht, double* th) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    const double a = th[i];
    th[i] = a + t * (tht[i] - a);  // trial_theta (outer.cpp:130)
  }
}

void ptheta_update(const Launch& L, i64 p, double t, const double* th_t, double* th) {
  k_ptheta<<<pgrid(p), NT, 0, L.s>>>(p, t, th_t, th);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_pcopy(i64 p, const double* s, double* d0, double* d1, double* d2) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    const double v = s[i];
    if (d0) d0[i] = v;
    if (d1) d1[i] = v;
    if (d2) d2[i] = v;
  }
}

void pcopy(const Launch& L, i64 p, const double* src, double* d0, double* d1, double* d2) {
  k_pcopy<<<pgrid(p), NT, 0, L.s>>>(p, src, d0, d1, d2);
  bump(L);
}

// Halo exchange helpers of banded last-mode sharding: y += x (the left
// neighbour's partial of S(x) over the overlap), and x := 0 outside [lo, hi)
// (before the owned-slice all-gather, so the sum over ranks is exact).
__global__ void __launch_bounds__(NT) k_padd(i64 n, const double* x, double* y) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT)
    y[i] += x[i];
}

void padd(const Launch& L, i64 n, const double* x, double* y) {
  if (n <= 0) return;
  k_padd<<<pgrid(n), NT, 0, L.s>>>(n, x, y);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_pmask(i64 p, i64 lo, i64 hi, double* x) {
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT)
    if (i < lo || i >= hi) x[i] = 0.0;
}

void pmask(const Launch& L, i64 p, i64 lo, i64 hi, double* x) {
  k_pmask<<<pgrid(p), NT, 0, L.s>>>(p, lo, hi, x);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_pmaxabs(i64 p, const double* x, double* part) {
  __shared__ double red[32];
  double m = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT)
    m = fmax(m, fabs(x[i]));
  const double r = block_reduce<true>(m, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void pmaxabs(const Launch& L, i64 p, const double* x, double* part) {
  k_pmaxabs<<<pgrid(p), NT, 0, L.s>>>(p, x, part);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_gram_dots(i64 p, double w, const double* x, const double* Sx,
                                                  const double* b, double* part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    const double xi = x[i];
    acc += xi * (w * Sx[i] - 2.0 * b[i]);
  }
  const double r = block_reduce<false>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void gram_dots(const Launch& L, i64 p, double w, const double* x, const double* Sx, const double* b, double* part) {
  k_gram_dots<<<pgrid(p), NT, 0, L.s>>>(p, w, x, Sx, b, part);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_wzz(i64 n, const double* v, const double* z, double* part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    const double zi = z[i];
    acc = fma(v[i], zi * zi, acc);
  }
  const double r = block_reduce<false>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void wzz(const Launch& L, i64 n, const double* v, const double* z, double* part) {
  k_wzz<<<elem_grid(n), NT, 0, L.s>>>(n, v, z, part);
  bump(L);
}

__global__ void __launch_bounds__(NT) k_minmax(i64 n, const double* x, double* part) {
  __shared__ double red[32];
  double mn = DBL_MAX, mx = -DBL_MAX;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * NT) {
    mn = fmin(mn, x[i]);
    mx = fmax(mx, x[i]);
  }
  const double a = -block_reduce<true>(-mn, red);
  __syncthreads();
  const double b = block_reduce<true>(mx, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

void minmax(const Launch& L, i64 n, const double* x, double* part) {
  k_minmax<<<elem_grid(n), NT, 0, L.s>>>(n, x, part);
  bump(L);
}

// best := x (and S(best) := S(x)) when the last monitor left a copy pending
__global__ void __launch_bounds__(NT) k_fista_finalize(const FistaCtl* ctl, i64 p, const double* x, double* best,
                                                       const double* Sx, double* Sbest) {
  if (!ctl->copy_best) return;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    best[i] = x[i];
    Sbest[i] = Sx[i];
  }
}

void fista_finalize(const Launch& L, const FistaCtl* ctl, i64 p, const double* x, double* best, const double* Sx,
                    double* Sbest) {
  k_fista_finalize<<<pgrid(p), NT, 0, L.s>>>(ctl, p, x, best, Sx, Sbest);
  bump(L);
}

// ----------------------------------------------------------- control CTA
// Fixed-order reduction of a partials column by one CTA of 1024 threads.
constexpr int CT = 1024;

__device__ double cta_sum_col(const double* part, int nrows, int stride, int col, double* sh) {
  double s = 0.0;
  for (int r = threadIdx.x; r < nrows; r += CT) s += part[static_cast<i64>(r) * stride + col];
  s = block_reduce<false>(s, sh);
  __syncthreads();
  if (threadIdx.x == 0) sh[32] = s;
  __syncthreads();
  const double out = sh[32];
  __syncthreads();
  return out;
}

__device__ double cta_max_col(const double* part, int nrows, int stride, int col, double* sh) {
  double s = -DBL_MAX;
  for (int r = threadIdx.x; r < nrows; r += CT) s = fmax(s, part[static_cast<i64>(r) * stride + col]);
  s = block_reduce<true>(s, sh);
  __syncthreads();
  if (threadIdx.x == 0) sh[32] = s;
  __syncthreads();
  const double out = sh[32];
  __syncthreads();
  return out;
}

__device__ __forceinline__ double penalty_of(int pen, double alpha, double l1, double l2) {
  if (pen == 0) return l1;
  if (pen == 1) return l2;
  return l1 + alpha * l2;
}

// The four sums the monitor needs -- sum v eta^2 (or sum v (eta - z)^2), the
// l1 and squared-l2 parts of J and <b, x> -- in one pass: every thread reads
// its rows of all four columns, then four fixed shuffle trees and one
// fixed-order pass over the warps (deterministic, two barriers).
__device__ void cta_sums4(const double* ss_part, int n_ss, const double* J_part, int n_J, const double* bx_part,
                          int n_bx, double* sh, double out[4]) {
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r = threadIdx.x; r < n_ss; r += CT) a[0] += ss_part[r];
  for (int r = threadIdx.x; r < n_J; r += CT) {
    a[1] += J_part[2 * r];
    a[2] += J_part[2 * r + 1];
  }
  if (bx_part)
    for (int r = threadIdx.x; r < n_bx; r += CT) a[3] += bx_part[r];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = warp_sum(a[k]);
  if (l == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[4 * w + k] = a[k];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double v = sh[4 * l + k];
      v = warp_sum(v);
      if (l == 0) sh[128 + k] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = sh[128 + k];
}

// The four objective pieces of a halo-sharded FISTA step in one launch:
// out = {sum ss_part, sum J_part[2r], sum J_part[2r+1], sum bx_part} (bx 0 if null).
__global__ void __launch_bounds__(CT) k_sums4(const double* ss_part, int n_ss, const double* J_part, int n_J,
                                              const double* bx_part, int n_bx, double* out) {
  __shared__ double sh[132];
  double s4[4];
  cta_sums4(ss_part, n_ss, J_part, n_J, bx_part, n_bx, sh, s4);
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) out[k] = s4[k];
}

void sums4(const Launch& L, const double* ss_part, int n_ss, const double* J_part, int n_J, const double* bx_part,
           int n_bx, double* out) {
  k_sums4<<<1, CT, 0, L.s>>>(ss_part, n_ss, J_part, n_J, bx_part, n_bx, out);
  bump(L);
}

__global__ void __launch_bounds__(CT) k_fista_init(FistaCtl* c, const double* ss_part, int n_ss, const double* J_part,
                                                   int n_J, const double* vmax_part, int n_vmax, int bt_always,
                                                   const double* bx_part, int n_bx) {
  __shared__ double sh[33];
  double ss = cta_sum_col(ss_part, n_ss, 1, 0, sh);
  if (bx_part) ss += -2.0 * cta_sum_col(bx_part, n_bx, 1, 0, sh);  // expanded objective (FV_FISTA_EXP)
  const double l1 = cta_sum_col(J_part, n_J, 2, 0, sh);
  const double l2 = cta_sum_col(J_part, n_J, 2, 1, sh);
  const double wmax = cta_max_col(vmax_part, n_vmax, 1, 0, sh);
  if (threadIdx.x != 0) return;
  // inner_objective (inner.cpp:109-119)
  const double g0 = 0.5 * (ss + c->ss_const) / c->n + c->lambda * penalty_of(c->pen, c->alpha, l1, l2);
  c->g_prev = g0;
  c->best_g = g0;
  // lipschitz_upper (inner.cpp:53-71): wmax * sum_r prod_j rho_rj / n
  c->bad_weights = !(wmax > 0.0);
  const double lip = wmax * c->lipfac / c->n;
  c->lip = lip;
  // stepsize policy (inner.cpp:141-145)
  double delta = bt_always ? 1.0 : 1.0 / (fmax(c->nu, 1.0e-300) * lip);
  if (c->nu == 1.0) delta = 1.0 / lip;
  c->delta = delta;
  c->omega = 0.0;
  c->it = 1;
  c->momentum = 1;
  c->streak = 0;
  c->prox_steps = 0;
  c->backtracks = 0;
  c->iterations = 0;
  c->copy_best = 0;
  c->restart = 0;
  c->converged = 0;
  c->diverged = 0;
  c->done = (c->max_iters < 1) || c->bad_weights;
}

// Objective monitor, best tracking, divergence restarts and the stop rule of
// fista_solve (inner.cpp:189-229), advanced once per iteration on the device;
// sets the graph's while-condition so the loop runs without the host.
__global__ void __launch_bounds__(CT) k_fista_control(FistaCtl* c, const double* ss_part, int n_ss,
                                                      const double* J_part, int n_J,
                                                      cudaGraphConditionalHandle h, int use_handle,
                                                      const double* bx_part, int n_bx) {
  __shared__ double sh[132];
  if (c->done) return;  // batched host loops (sharded contexts) enqueue steps past the stop
  double s4[4];
  cta_sums4(ss_part, n_ss, J_part, n_J, bx_part, n_bx, sh, s4);
  double ss = s4[0];
  if (bx_part) ss += -2.0 * s4[3];  // expanded objective (FV_FISTA_EXP)
  const double l1 = s4[1], l2 = s4[2];
  if (threadIdx.x != 0) return;
  c->copy_best = 0;
  c->restart = 0;
  const i64 it = c->it;
  c->prox_steps += 1;
  c->momentum += 1;
  c->iterations = it;
  const i64 me = c->monitor_every < 1 ? 1 : c->monitor_every;
  const bool monitored = (it % me == 0) || it == c->max_iters;
  if (monitored) {
    const double g = 0.5 * (ss + c->ss_const) / c->n + c->lambda * penalty_of(c->pen, c->alpha, l1, l2);
    const bool bad = !isfinite(g);
    bool div = bad;
    if (!div && c->bt_div && g > c->g_prev) div = (++c->streak >= 3);
    if (div) {
      if (!c->bt_div) {
        c->diverged = 1;
        c->done = 1;
      } else {
        c->restart = 1;
        c->g_prev = c->best_g;
        c->delta *= 0.5;
        c->momentum = 1;
        c->streak = 0;
        c->backtracks += 1;
      }
    } else {
      if (g <= c->g_prev) c->streak = 0;
      if (g <= c->best_g) {
        c->copy_best = 1;
        c->best_g = g;
      }
      if (fabs(g - c->g_prev) / fmax(1.0, fabs(g)) < c->tol) {
        c->converged = 1;
        c->done = 1;
      }
      c->g_prev = g;
    }
  }
  if (!c->done) {
    c->it = it + 1;
    if (c->it > c->max_iters) c->done = 1;
  }
  c->omega = c->extrapolation == 0
                 ? static_cast<double>(c->momentum - 1) / static_cast<double>(c->momentum + 2)
                 : 0.0;
  if (use_handle) cudaGraphSetConditional(h, c->done ? 0u : 1u);
}

void fista_init(const Launch& L, FistaCtl* ctl, const double* ss_part, int n_ss, const double* J_part, int n_J,
                const double* vmax_part, int n_vmax, int bt_always, const double* bx_part, int n_bx) {
  k_fista_init<<<1, CT, 0, L.s>>>(ctl, ss_part, n_ss, J_part, n_J, vmax_part, n_vmax, bt_always, bx_part, n_bx);
  bump(L);
}

void fista_control(const Launch& L, FistaCtl* ctl, const double* ss_part, int n_ss, const double* J_part, int n_J,
                   cudaGraphConditionalHandle h, int use_handle, const double* bx_part, int n_bx) {
  k_fista_control<<<1, CT, 0, L.s>>>(ctl, ss_part, n_ss, J_part, n_J, h, use_handle, bx_part, n_bx);
  bump(L);
}

__global__ void k_gate(const FistaCtl* c, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, c->done ? 0u : 1u);
}

void fista_gate(const Launch& L, const FistaCtl* ctl, cudaGraphConditionalHandle h) {
  k_gate<<<1, 32, 0, L.s>>>(ctl, h);
  bump(L);
}

// One warp per column: lanes sum strided rows sequentially, then a fixed
// shuffle tree (deterministic); no block barriers.
__global__ void k_reduce_cols(const double* part, int nrows, int ncols, int op, double* out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = w; c < ncols; c += nw) {
    double r = op ? -DBL_MAX : 0.0;
    for (int i = l; i < nrows; i += 32) {
      const double v = part[static_cast<i64>(i) * ncols + c];
      r = op ? fmax(r, v) : r + v;
    }
    r = op ? warp_max(r) : warp_sum(r);
    if (l == 0) out[c] = r;
  }
}

// Many rows (the per-CTA partials of the n-space passes: up to 32K CTAs): one
// 1024-thread CTA per column, thread t sums rows t, t + 1024, ... in order,
// then a fixed shuffle tree and a fixed-order sum over the warps.
__global__ void __launch_bounds__(1024) k_reduce_cols_wide(const double* part, int nrows, int ncols, int op,
                                                           double* out) {
  __shared__ double ws[32];
  const int c = blockIdx.x, l = threadIdx.x & 31, w = threadIdx.x >> 5;
  double r = op ? -DBL_MAX : 0.0;
  for (int i = threadIdx.x; i < nrows; i += 1024) {
    const double v = part[static_cast<i64>(i) * ncols + c];
    r = op ? fmax(r, v) : r + v;
  }
  r = op ? warp_max(r) : warp_sum(r);
  if (l == 0) ws[w] = r;
  __syncthreads();
  if (w == 0) {
    r = ws[l];
    r = op ? warp_max(r) : warp_sum(r);
    if (l == 0) out[c] = r;
  }
}

void reduce_cols(const Launch& L, const double* part, int nrows, int ncols, int op, double* out) {
  if (nrows >= 4096) {
    k_reduce_cols_wide<<<ncols, 1024, 0, L.s>>>(part, nrows, ncols, op, out);
    bump(L);
    return;
  }
  const int warps = ncols < 16 ? ncols : 16;
  k_reduce_cols<<<1, 32 * warps, 0, L.s>>>(part, nrows, ncols, op, out);
  bump(L);
}

// ------------------------------------------------------ spectral radius
// Banded Gram X^T X of one factor: row a has entries for columns [glo, ghi).
__global__ void k_gram(const double* X, i64 n, i64 p, const int* clo, const int* clen, const int* glo, const int* ghi,
                       double* G) {
  const int a = blockIdx.x;
  for (int b = glo[a] + threadIdx.x; b < ghi[a]; b += blockDim.x) {
    const int lo = max(clo[a], clo[b]);
    const int hi = min(clo[a] + clen[a], clo[b] + clen[b]);
    double s = 0.0;
    for (int i = lo; i < hi; ++i) s += X[i + n * a] * X[i + n * b];
    G[a + p * static_cast<i64>(b)] = s;
  }
}

void gram(const Launch& L, const FactorDev& f, double* G, int* glo, int* ghi) {
  k_gram<<<static_cast<unsigned>(f.p), 128, 0, L.s>>>(f.X, f.n, f.p, f.G.lo, f.G.len, glo, ghi, G);
  bump(L);
}

// Power iteration (spectral.cpp:8-42), one CTA per job (blockIdx.x), every
// factor of a design in one launch.
//
// Banded path (band <= kPowerTaps, kPowerTaps <= p <= blockDim.x *
// kPowerCtaRows): each thread owns rows i = tid + blockDim.x * r with their
// Gram band in registers, padded to kPowerTaps taps on a window clamped into
// [0, p) (no predicates in the product).  Steps are taken kPowerBlock at a
// time without renormalising: a_j = G a_{j-1} from a_0 = v, each a_j staged in
// shared memory for the next product, while every thread accumulates |a_j|^2
// and a_{j-1}.a_j.  One CTA reduction (warp shuffles, then a fixed-order sum
// over warps) of those 2 kPowerBlock sums per block replays the reference's
// per-step quantities exactly in exact arithmetic:
//   norm_j = |a_j| / |a_{j-1}|,  next_j = a_{j-1}.a_j / |a_{j-1}|^2,
// and applies its stop rule step by step (two quiet Rayleigh quotients), so
// the returned value and iteration count follow the same sequence while the
// reduction latency is paid once per block.  A block whose growth over- or
// underflows is redone one step at a time.
// Generic path (wide bands, tiny or huge p): warp 0 alone, one step at a time
// on the dense band.
__global__ void __launch_bounds__(kPowerThreads) k_power(const PowerJob* jobs, double tol, i64 max_iters,
                                                         i64 sm_doubles) {
  extern __shared__ double sh[];
  const PowerJob J = jobs[blockIdx.x];
  const i64 p = J.p;
  const int tid = threadIdx.x, l = tid & 31, warp = tid >> 5;
  const bool banded = J.band <= kPowerTaps && p >= kPowerTaps && p <= static_cast<i64>(blockDim.x) * kPowerCtaRows &&
                      (kPowerBlock + 1) * p + 2 * kPowerBlock * (blockDim.x + 1) <= sm_doubles;
  double value = 0.0;
  i64 settled = 0;
  auto finish = [&](double val, i64 it, double status) {
    if (tid == 0) {
      J.out[0] = val;
      J.out[1] = static_cast<double>(it);
      J.out[2] = status;
    }
  };
  // the reference's per-step bookkeeping; true when the iteration stops
  auto step_done = [&](double next, i64 it) {
    const double change = fabs(next - value);
    value = next;
    if (change <= tol * fmax(fabs(value), 1e-300)) {
      if (++settled >= 2) {
        finish(value, it, 0.0);
        return true;
      }
    } else {
      settled = 0;
    }
    return false;
  };
  if (!banded) {
    if (warp != 0) return;
    double* v = sh;
    double* av = sh + p;
    for (i64 i = l; i < p; i += 32) v[i] = J.v0[i];
    __syncwarp();
    for (i64 it = 1; it <= max_iters; ++it) {
      double nn = 0.0, dot = 0.0;
      for (i64 i = l; i < p; i += 32) {
        double s = 0.0;
        for (int k = J.glo[i]; k < J.ghi[i]; ++k) s += J.G[i + p * k] * v[k];
        av[i] = s;
        nn += s * s;
        dot += v[i] * s;
      }
      nn = warp_allsum(nn);
      dot = warp_allsum(dot);
      const double norm = sqrt(nn);
      if (norm == 0.0) {
        finish(0.0, it, 0.0);
        return;
      }
      __syncwarp();
      for (i64 i = l; i < p; i += 32) v[i] = av[i] / norm;
      __syncwarp();
      if (step_done(dot, it)) return;
    }
    finish(value, max_iters, 1.0);
    return;
  }
  constexpr int KB = kPowerBlock;
  double* red = sh + static_cast<i64>(KB + 1) * p;  // [2 KB][blockDim.x] partials, then tot[2 KB]
  double* tot = red + 2 * KB * blockDim.x;
  double c[kPowerCtaRows][kPowerTaps];
  int base[kPowerCtaRows];
  bool own[kPowerCtaRows];
  double a[kPowerCtaRows];
#pragma unroll
  for (int r = 0; r < kPowerCtaRows; ++r) {
    const i64 i = tid + static_cast<i64>(blockDim.x) * r;
    own[r] = i < p;
    int lo = 0, hi = 0;
    if (own[r]) {
      lo = J.glo[i];
      hi = J.ghi[i];
    }
    base[r] = min(lo, static_cast<int>(p) - kPowerTaps);
#pragma unroll
    for (int t = 0; t < kPowerTaps; ++t) {
      const int col = base[r] + t;
      c[r][t] = (own[r] && col >= lo && col < hi) ? J.G[i + p * col] : 0.0;
    }
    a[r] = own[r] ? J.v0[i] : 0.0;
    if (own[r]) sh[i] = a[r];
  }
  __syncthreads();
  bool blocked = true;
  i64 it = 0;
  while (it < max_iters) {
    const int K = !blocked ? 1 : (max_iters - it < KB ? static_cast<int>(max_iters - it) : KB);
    double ssum[KB], tsum[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      ssum[j] = 0.0;
      tsum[j] = 0.0;
      if (j < K) {
        const double* ain = sh + j * p;
        double* aout = sh + (j + 1) * p;
#pragma unroll
        for (int r = 0; r < kPowerCtaRows; ++r) {
          if (own[r]) {
            const i64 i = tid + static_cast<i64>(blockDim.x) * r;
            double s = 0.0;
#pragma unroll
            for (int t = 0; t < kPowerTaps; ++t) s += c[r][t] * ain[base[r] + t];
            ssum[j] += s * s;
            tsum[j] += ain[i] * s;
            aout[i] = s;
            a[r] = s;
          }
        }
        __syncthreads();
      }
    }
    // CTA reduction of the 2 K sums through shared memory: every thread
    // stores its partials, then 16 threads per sum add 1/16 of the rows each
    // (fixed order) and a 16-lane shuffle tree finishes it.
    {
      const int nt = blockDim.x;
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        red[(2 * j) * nt + tid] = ssum[j];
        red[(2 * j + 1) * nt + tid] = tsum[j];
      }
      __syncthreads();
      // half-warps pair up on consecutive sums and 2 K is even, so a warp's
      // halves take the same trips (the shuffles need the whole warp)
      const int part = tid & 15;
      for (int q = tid >> 4; q < 2 * K; q += nt >> 4) {
        double acc = 0.0;
        for (int k = part; k < nt; k += 16) acc += red[q * nt + k];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, 16);
        if (part == 0) tot[q] = acc;
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      if (j < K) {
        ssum[j] = tot[2 * j];
        tsum[j] = tot[2 * j + 1];
      }
    }
    bool ok = true;
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < K) ok = ok && isfinite(ssum[j]) && (ssum[j] > 0.0 || j == 0);
    if (!ok && K > 1) {  // growth left the FP64 range inside the block: redo it one step at a time
      blocked = false;
      continue;
    }
    double prev = 1.0;  // a_0 is the unit-normalised v of the reference
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      if (j < K) {
        ++it;
        if (ssum[j] == 0.0) {
          finish(0.0, it, 0.0);
          return;
        }
        if (step_done(tsum[j] / prev, it)) return;
        prev = ssum[j];
      }
    }
    // the next block starts from v = a_K / |a_K| (a_K is the one left in registers)
    const double norm = sqrt(prev);
#pragma unroll
    for (int r = 0; r < kPowerCtaRows; ++r)
      if (own[r]) sh[tid + static_cast<i64>(blockDim.x) * r] = a[r] / norm;
    __syncthreads();
  }
  finish(value, max_iters, 1.0);
}

void power_iterations(const Launch& L, const PowerJob* jobs_dev, int njobs, i64 max_p, double tol, i64 max_iters) {
  if (njobs < 1) return;
  // one row per thread up to kPowerThreads rows, then up to kPowerCtaRows each
  const i64 threads = std::min<i64>(kPowerThreads, std::max<i64>(32, (max_p + 31) / 32 * 32));
  const i64 banded_p = std::min<i64>(max_p, threads * kPowerCtaRows);
  i64 need = std::max<i64>(2 * max_p, (kPowerBlock + 1) * banded_p + 2 * kPowerBlock * (threads + 1));
  need = std::min<i64>(need, 220 * 1024 / 8);
  if (2 * max_p > need) throw Error(E_INVAL, "spectral_radius: factor too large for the device power iteration");
  const size_t sm = sizeof(double) * static_cast<size_t>(need);
  if (sm > 48 * 1024) smem_attr(k_power, static_cast<int>(sm));
  k_power<<<njobs, static_cast<unsigned>(threads), sm, L.s>>>(jobs_dev, tol, max_iters, need);
  bump(L);
}

// Nonzero count of each model's coefficient vector (kronglm_py.cpp's
// "nonzero" key): blockIdx.y = model, integer atomics (order-free, exact).
__global__ void __launch_bounds__(256) k_count_nz(const double* __restrict__ c, i64 p,
                                                  unsigned long long* __restrict__ out) {
  const double* row = c + static_cast<i64>(blockIdx.y) * p;
  unsigned n = 0;
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * blockDim.x)
    n += __ldg(row + i) != 0.0 ? 1u : 0u;
  n = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(out + blockIdx.y, static_cast<unsigned long long>(n));
}

void count_nonzero(const Launch& L, const double* coefs, i64 p, i64 models, unsigned long long* out) {
  const i64 bx = std::min<i64>((p + 255) / 256, 64);
  k_count_nz<<<dim3(static_cast<unsigned>(bx), static_cast<unsigned>(models)), 256, 0, L.s>>>(coefs, p, out);
  launched(L);
}

}  // namespace kg
