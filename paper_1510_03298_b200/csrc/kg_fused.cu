// Bulk-async (TMA engine) pipelined kernels of the GLAM fit path.
//
//  * k_fused_tma: the mode-1 fused pass.  A persistent CTA walks tiles of T
//    consecutive mode-1 fibres; every tile is a contiguous chunk of each
//    n-array, so its v, z (and the p1 x T slice of the H-partial P) arrive by
//    one cp.async.bulk each into a double-buffered shared-memory stage,
//    completion tracked by an mbarrier.  While tile i is computed, tile i+1 is
//    in flight.  Threads are row-stationary: a thread keeps one X1 row band in
//    registers and sweeps its share of the tile's fibres, so no band metadata
//    is re-read per cell.
//  * k_contract_tiled: one banded mode-k contraction.  A CTA owns an
//    (alpha block x m block x beta) output tile, stages the union of the input
//    rows its band touches in shared memory, then every warp produces whole
//    coalesced output rows.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <vector>

#include "kg_internal.h"

namespace kg {

namespace {

constexpr int NT = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < (blockDim.x >> 5) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Stages n doubles of src into the shared buffer `base` (which has one spare
// double): the buffer view starts at base + shift so that it has the same
// 16-byte phase as src; the misaligned head and odd tail element are copied
// by the calling thread, the rest by the bulk-copy engine.
__device__ __forceinline__ int stage_shift(const double* src) {
  return (reinterpret_cast<uintptr_t>(src) & 15) ? 1 : 0;
}

struct Chunk {
  i64 head, body;
};

__device__ __forceinline__ Chunk chunk_of(const double* src, i64 n) {
  Chunk c;
  c.head = stage_shift(src) ? 1 : 0;
  if (c.head > n) c.head = n;
  c.body = n - c.head;
  c.body -= c.body & 1;
  return c;
}

// manual head/tail stores; must precede the producer's arrive
__device__ __forceinline__ unsigned stage_manual(double* base, const double* src, i64 n) {
  double* dst = base + stage_shift(src);
  const Chunk c = chunk_of(src, n);
  if (c.head) dst[0] = src[0];
  if (c.head + c.body < n) dst[n - 1] = src[n - 1];
  return static_cast<unsigned>(c.body * 8);
}

__device__ __forceinline__ void stage_bulk(double* base, const double* src, i64 n, unsigned long long* bar) {
  double* dst = base + stage_shift(src);
  const Chunk c = chunk_of(src, n);
  if (c.body > 0) bulk_g2s(dst + c.head, src + c.head, static_cast<unsigned>(c.body * 8), bar);
}

__device__ __forceinline__ double score0_of(int fam, double y, double a) {
  switch (fam) {
    case 0: return a * y;
    case 1: return a * (y - 0.5);
    case 2: return a * (y - 1.0);
    default: return a * (y - 1.0);
  }
}

}  // namespace

// --------------------------------------------------------------- fused pass
constexpr int kMaxStages = 4;
struct FusedPlan {
  int T;        // fibres per tile
  int stage;    // doubles per stage
  int offP, offA, offB;  // stage-relative offsets (doubles) of P, stream A (v|y), stream B (z|a)
  int nst;      // pipeline depth (stages in flight) of the register-hoisted kernel
};

template <int VAR>
__global__ void __launch_bounds__(NT) k_fused_tma(FusedArgs f, FusedPlan pl, i64 ntiles) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long bar[2];
  __shared__ double red[32];
  const int n1 = static_cast<int>(f.n1), p1 = static_cast<int>(f.p1), T = pl.T;
  const bool hasP = VAR == FV_FISTA;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const double* srcA = VAR == FV_SCORE0 ? f.y : f.v;
  const double* srcB = VAR == FV_SCORE0 ? f.a : f.z;

  auto issue = [&](i64 tile, int s) {
    const i64 c0 = tile * T;
    const i64 Tc = min(static_cast<i64>(T), f.m - c0);
    double* st = sm + static_cast<i64>(s) * pl.stage;
    unsigned bytes = 0;
    if (hasP) bytes += stage_manual(st + pl.offP, f.P + c0 * p1, p1 * Tc);
    bytes += stage_manual(st + pl.offA, srcA + c0 * n1, n1 * Tc);
    bytes += stage_manual(st + pl.offB, srcB + c0 * n1, n1 * Tc);
    fence_proxy_async();
    mbar_expect_tx(&bar[s], bytes);
    if (hasP) stage_bulk(st + pl.offP, f.P + c0 * p1, p1 * Tc, &bar[s]);
    stage_bulk(st + pl.offA, srcA + c0 * n1, n1 * Tc, &bar[s]);
    stage_bulk(st + pl.offB, srcB + c0 * n1, n1 * Tc, &bar[s]);
  };

  // row-stationary mappings (fixed per thread for the whole kernel)
  const int RA = n1 < NT ? n1 : NT, CGA = NT / RA;
  const int tid = static_cast<int>(threadIdx.x);
  const int tA = tid < RA * CGA ? tid : -1;
  const int iA0 = tA >= 0 ? tA % RA : 0, cgA = tA >= 0 ? tA / RA : 0;
  const int RB = p1 < NT ? p1 : NT, CGB = NT / RB;
  const int tB = tid < RB * CGB ? tid : -1;
  const int kB0 = tB >= 0 ? tB % RB : 0, cgB = tB >= 0 ? tB / RB : 0;

  double acc = 0.0;
  int s = 0;
  unsigned phase[2] = {0u, 0u};
  i64 tile = blockIdx.x;
  if (threadIdx.x == 0) {
    if (tile < ntiles) issue(tile, 0);
    if (tile + gridDim.x < ntiles) issue(tile + gridDim.x, 1);
  }
  for (; tile < ntiles; tile += gridDim.x) {
    const i64 c0 = tile * T;
    const int Tc = static_cast<int>(min(static_cast<i64>(T), f.m - c0));
    double* st = sm + static_cast<i64>(s) * pl.stage;
    double* Ps = st + pl.offP + (hasP ? stage_shift(f.P + c0 * p1) : 0);
    double* As = st + pl.offA + stage_shift(srcA + c0 * n1);  // v (or y); overwritten in place by w
    double* Bs = st + pl.offB + stage_shift(srcB + c0 * n1);  // z (or a)
    mbar_wait(&bar[s], phase[s]);
    phase[s] ^= 1u;
    // phase A: eta = X1 P, sum v (eta - z)^2, w = v eta   (or w = v z / score(0))
    if (tA >= 0 && f.dbg != 1) {
      for (int i = iA0; i < n1; i += RA) {
        int lo = 0, len = 0;
        double c[4] = {0.0, 0.0, 0.0, 0.0};
        const double* cf = nullptr;
        if (hasP) {
          lo = __ldg(f.H.lo + i);
          len = __ldg(f.H.len + i);
          cf = f.H.coef + __ldg(f.H.off + i);
#pragma unroll
          for (int t = 0; t < 4; ++t) c[t] = t < len ? __ldg(cf + t) : 0.0;
        }
        for (int col = cgA; col < Tc; col += CGA) {
          const int e = i + n1 * col;
          double w;
          if (VAR == FV_FISTA) {
            const double* pc = Ps + p1 * col + lo;
            double eta = 0.0;
            if (len <= 4) {
#pragma unroll
              for (int t = 0; t < 4; ++t)
                if (t < len) eta = fma(c[t], pc[t], eta);
            } else {
              for (int t = 0; t < len; ++t) eta = fma(__ldg(cf + t), pc[t], eta);
            }
            const double vv = As[e];
            const double r = eta - Bs[e];
            acc = fma(vv, r * r, acc);
            w = vv * eta;
          } else if (VAR == FV_XTWZ) {
            w = As[e] * Bs[e];
          } else {
            w = score0_of(f.fam, As[e], Bs[e]) / f.disp;
            if (!isfinite(w))
              atomicMin(reinterpret_cast<unsigned long long*>(f.err),
                        static_cast<unsigned long long>(f.cell_base + c0 * n1 + e));
          }
          As[e] = w;
        }
      }
    }
    __syncthreads();
    // phase B: Q = X1^T w for the tile's fibres; the tile's p1 x Tc outputs
    // are contiguous in Q, so consecutive threads write consecutive doubles.
    if (tB >= 0 && f.dbg == 0) {
      double* Q = f.Q + c0 * p1;
      for (int k = kB0, col = cgB; col < Tc;) {
        const int lo = __ldg(f.G.lo + k), len = __ldg(f.G.len + k);
        const double* cf = f.G.coef + __ldg(f.G.off + k);
        const double* wr = As + lo + n1 * col;
        double o0 = 0.0, o1 = 0.0;
        int t = 0;
        for (; t + 1 < len; t += 2) {
          o0 = fma(__ldg(cf + t), wr[t], o0);
          o1 = fma(__ldg(cf + t + 1), wr[t + 1], o1);
        }
        if (t < len) o0 = fma(__ldg(cf + t), wr[t], o0);
        Q[k + p1 * col] = o0 + o1;
        k += RB;
        if (k >= p1) {
          k -= p1;
          col += CGB;
        }
      }
    }
    __syncthreads();  // stage s is free again
    if (threadIdx.x == 0 && tile + 2 * static_cast<i64>(gridDim.x) < ntiles) issue(tile + 2 * gridDim.x, s);
    s ^= 1;
  }
  if (VAR == FV_FISTA) {
    const double r = block_sum(acc, red);
    if (threadIdx.x == 0) f.partial[blockIdx.x] = r;
  }
}

// Register-hoisted variant for n1 <= NT, p1 <= NT, H bands <= 4 wide and G
// bands <= MAXG wide (every cubic B-spline factor in the BASELINE configs).
// Each thread's X1 row (phase A) and X1^T row (phase B) are fixed for the
// whole persistent kernel, so their band coefficients live in registers and
// the per-cell work is a handful of shared-memory loads and FMAs.
template <int VAR, int MAXG, int BS>
__global__ void __launch_bounds__(BS) k_fused_fast(FusedArgs f, FusedPlan pl, i64 ntiles) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long bar[kMaxStages];
  __shared__ double red[32];
  const int n1 = static_cast<int>(f.n1), p1 = static_cast<int>(f.p1), T = pl.T;
  const int nst = pl.nst;
  constexpr bool hasP = VAR == FV_FISTA || VAR == FV_FISTA_EXP;
  constexpr bool hasB = VAR != FV_FISTA_EXP;
  if (threadIdx.x == 0) {
    for (int k = 0; k < nst; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const double* srcA = VAR == FV_SCORE0 ? f.y : f.v;
  const double* srcB = VAR == FV_SCORE0 ? f.a : f.z;
  auto issue = [&](i64 tile, int s) {
    const i64 c0 = tile * T;
    const i64 Tc = min(static_cast<i64>(T), f.m - c0);
    double* st = sm + static_cast<i64>(s) * pl.stage;
    unsigned bytes = 0;
    if (hasP) bytes += stage_manual(st + pl.offP, f.P + c0 * p1, p1 * Tc);
    bytes += stage_manual(st + pl.offA, srcA + c0 * n1, n1 * Tc);
    if (hasB) bytes += stage_manual(st + pl.offB, srcB + c0 * n1, n1 * Tc);
    fence_proxy_async();
    mbar_expect_tx(&bar[s], bytes);
    if (hasP) stage_bulk(st + pl.offP, f.P + c0 * p1, p1 * Tc, &bar[s]);
    stage_bulk(st + pl.offA, srcA + c0 * n1, n1 * Tc, &bar[s]);
    if (hasB) stage_bulk(st + pl.offB, srcB + c0 * n1, n1 * Tc, &bar[s]);
  };
  const int tid = static_cast<int>(threadIdx.x);
  // phase A: row i of X1, fibres cgA, cgA + CGA, ...
  const int CGA = BS / n1;
  const bool actA = tid < n1 * CGA;
  const int iA = actA ? tid % n1 : 0, cgA = actA ? tid / n1 : 0;
  int loA = 0, lenA = 0;
  double cA[4] = {0.0, 0.0, 0.0, 0.0};
  if (hasP && actA) {
    loA = __ldg(f.H.lo + iA);
    lenA = __ldg(f.H.len + iA);
    const double* cf = f.H.coef + __ldg(f.H.off + iA);
#pragma unroll
    for (int t = 0; t < 4; ++t) cA[t] = t < lenA ? __ldg(cf + t) : 0.0;
  }
  // phase B: row k of X1^T, fibres cgB, cgB + CGB, ...
  const int CGB = BS / p1;
  const bool actB = tid < p1 * CGB;
  const int kB = actB ? tid % p1 : 0, cgB = actB ? tid / p1 : 0;
  int loB = 0, lenB = 0;
  double g[MAXG];
#pragma unroll
  for (int t = 0; t < MAXG; ++t) g[t] = 0.0;
  if (actB) {
    loB = __ldg(f.G.lo + kB);
    lenB = __ldg(f.G.len + kB);
    const double* cf = f.G.coef + __ldg(f.G.off + kB);
#pragma unroll
    for (int t = 0; t < MAXG; ++t)
      if (t < lenB) g[t] = __ldg(cf + t);
  }
  __syncthreads();

  double acc = 0.0;
  int s = 0;
  unsigned phase_bits = 0u;  // bit k: parity of stage k's next completion
  i64 tile = blockIdx.x;
  if (threadIdx.x == 0)
    for (int k = 0; k < nst; ++k)
      if (tile + static_cast<i64>(k) * gridDim.x < ntiles) issue(tile + static_cast<i64>(k) * gridDim.x, k);
  for (; tile < ntiles; tile += gridDim.x) {
    const i64 c0 = tile * T;
    const int Tc = static_cast<int>(min(static_cast<i64>(T), f.m - c0));
    double* st = sm + static_cast<i64>(s) * pl.stage;
    const double* Ps = st + pl.offP + (hasP ? stage_shift(f.P + c0 * p1) : 0);
    double* As = st + pl.offA + stage_shift(srcA + c0 * n1);  // v (or y); overwritten in place by w
    const double* Bs = hasB ? st + pl.offB + stage_shift(srcB + c0 * n1) : nullptr;
    mbar_wait(&bar[s], (phase_bits >> s) & 1u);
    phase_bits ^= 1u << s;
    if (actA && f.dbg != 1) {
      auto cell = [&](int col) {
        const int e = iA + n1 * col;
        double w;
        if (VAR == FV_FISTA || VAR == FV_FISTA_EXP) {
          const double* pc = Ps + p1 * col + loA;
          double e0 = 0.0, e1 = 0.0;
          if (lenA > 0) e0 = cA[0] * pc[0];
          if (lenA > 1) e1 = cA[1] * pc[1];
          if (lenA > 2) e0 = fma(cA[2], pc[2], e0);
          if (lenA > 3) e1 = fma(cA[3], pc[3], e1);
          const double eta = e0 + e1;
          const double vv = As[e];
          w = vv * eta;
          if (VAR == FV_FISTA) {
            const double r = eta - Bs[e];
            acc = fma(vv, r * r, acc);
          } else {
            acc = fma(w, eta, acc);
          }
        } else if (VAR == FV_XTWZ) {
          w = As[e] * Bs[e];
        } else {
          w = score0_of(f.fam, As[e], Bs[e]) / f.disp;
          if (!isfinite(w))
            atomicMin(reinterpret_cast<unsigned long long*>(f.err),
                      static_cast<unsigned long long>(f.cell_base + c0 * n1 + e));
        }
        As[e] = w;
      };
      int col = cgA;
      for (; col + CGA < Tc; col += 2 * CGA) {  // two fibres per step: independent loads in flight
        cell(col);
        cell(col + CGA);
      }
      if (col < Tc) cell(col);
    }
    __syncthreads();
    if (actB && f.dbg == 0) {
      double* Q = f.Q + c0 * p1;
      for (int col = cgB; col < Tc; col += CGB) {
        const double* wr = As + loB + n1 * col;
        double o0 = 0.0, o1 = 0.0;
#pragma unroll
        for (int t = 0; t < MAXG; t += 2) {
          if (t < lenB) o0 = fma(g[t], wr[t], o0);
          if (t + 1 < lenB) o1 = fma(g[t + 1], wr[t + 1], o1);
        }
        Q[kB + p1 * col] = o0 + o1;
      }
    }
    __syncthreads();  // stage s is free again
    const i64 next = tile + static_cast<i64>(nst) * gridDim.x;
    if (threadIdx.x == 0 && next < ntiles) issue(next, s);
    s = s + 1 == nst ? 0 : s + 1;
  }
  if (VAR == FV_FISTA || VAR == FV_FISTA_EXP) {
    const double r = block_sum(acc, red);
    if (threadIdx.x == 0) f.partial[blockIdx.x] = r;
  }
}

static FusedPlan plan_for(const FusedArgs& f, int variant) {
  FusedPlan pl;
  const bool hasP = variant == FV_FISTA || variant == FV_FISTA_EXP;
  const i64 nB = variant == FV_FISTA_EXP ? 1 : 2;  // staged n-arrays per fibre
  const i64 per_col = (hasP ? f.p1 : 0) + nB * f.n1;
  static const i64 stage_kb = [] {
    const char* e = dev_env("KG_FUSED_STAGE_KB");
    const long v = e ? std::atol(e) : 48;
    return static_cast<i64>(v >= 4 && v <= 100 ? v : 48);
  }();
  static const int stages = [] {
    const char* e = dev_env("KG_FUSED_STAGES");
    const int v = e ? std::atoi(e) : 2;
    return v >= 2 && v <= kMaxStages ? v : 2;
  }();
  pl.nst = stages;
  i64 T = std::max<i64>(1, (stage_kb * 1024 / 8) / per_col);
  T = std::min<i64>(T, f.m);
  pl.T = static_cast<int>(T);
  // 16-byte aligned sub-buffers, each with one spare double for the phase shift
  auto up2 = [](i64 x) { return (x + 2) & ~i64(1); };
  pl.offP = 0;
  const i64 nP = hasP ? up2(f.p1 * T) : 0;
  pl.offA = static_cast<int>(nP);
  pl.offB = static_cast<int>(nP + up2(f.n1 * T));
  pl.stage = static_cast<int>(nP + nB * up2(f.n1 * T));
  return pl;
}

struct LcPlan {  // DMMA fused pass (k_fused_mma)
  FusedPlan pl;
  int sw = 0, wp_off = 0, mw = 0, grid = 0, bs = 256;
  size_t smem = 0;
  bool ok = false;
};
static LcPlan lc_plan(const FusedArgs& f);

int fused_tma_grid(const FusedArgs& f, int variant) {
  if (variant == FV_FISTA_EXP) {
    const LcPlan P = lc_plan(f);
    if (P.ok) return P.grid;
  }
  const FusedPlan pl = plan_for(f, variant);
  const i64 ntiles = (f.m + pl.T - 1) / pl.T;
  const size_t sm = static_cast<size_t>(pl.nst) * pl.stage * sizeof(double);
  const int per_sm = std::max<int>(1, std::min<int>(8, static_cast<int>((220 * 1024) / (sm + 2048))));
  return static_cast<int>(std::min<i64>(ntiles, 148LL * per_sm));
}

bool fused_tma_fits(const FusedArgs& f, int variant) {
  const FusedPlan pl = plan_for(f, variant);
  return static_cast<size_t>(pl.nst) * pl.stage * sizeof(double) <= 200 * 1024;
}

// Block size of the register-hoisted fused kernel (KG_FUSED_BS = 256 | 512).
static int fused_bs() {
  static const int bs = [] {
    const char* e = dev_env("KG_FUSED_BS");
    return (e && std::atoi(e) == 512) ? 512 : 256;
  }();
  return bs;
}

template <int VAR, int MG>
static void launch_fast_one(const Launch& L, const FusedArgs& f, const FusedPlan& pl, i64 ntiles, int g, size_t sm) {
  smem_attr(k_fused_fast<VAR, MG, 256>, 210 * 1024);
  smem_attr(k_fused_fast<VAR, MG, 512>, 210 * 1024);
  if (fused_bs() == 512 && f.n1 <= 512 && f.p1 <= 512)
    k_fused_fast<VAR, MG, 512><<<g, 512, sm, L.s>>>(f, pl, ntiles);
  else
    k_fused_fast<VAR, MG, 256><<<g, 256, sm, L.s>>>(f, pl, ntiles);
}

template <int VAR>
static void launch_fast_var(const Launch& L, int mg, const FusedArgs& f, const FusedPlan& pl, i64 ntiles, int g,
                            size_t sm) {
  switch (mg) {
    case 8: launch_fast_one<VAR, 8>(L, f, pl, ntiles, g, sm); break;
    case 16: launch_fast_one<VAR, 16>(L, f, pl, ntiles, g, sm); break;
    case 24: launch_fast_one<VAR, 24>(L, f, pl, ntiles, g, sm); break;
    case 32: launch_fast_one<VAR, 32>(L, f, pl, ntiles, g, sm); break;
    default: launch_fast_one<VAR, 64>(L, f, pl, ntiles, g, sm); break;
  }
}

static void launch_fast(const Launch& L, int variant, int mg, const FusedArgs& f, const FusedPlan& pl, i64 ntiles,
                        int g, size_t sm) {
  switch (variant) {
    case FV_FISTA: launch_fast_var<FV_FISTA>(L, mg, f, pl, ntiles, g, sm); break;
    case FV_FISTA_EXP: launch_fast_var<FV_FISTA_EXP>(L, mg, f, pl, ntiles, g, sm); break;
    case FV_XTWZ: launch_fast_var<FV_XTWZ>(L, mg, f, pl, ntiles, g, sm); break;
    default: launch_fast_var<FV_SCORE0>(L, mg, f, pl, ntiles, g, sm); break;
  }
}

bool fused_fast_ok(const FusedArgs& f, int variant) {
  return fused_tma_fits(f, variant) && f.n1 <= NT && f.p1 <= NT && f.H.maxlen <= 4 && f.G.maxlen <= 64;
}

// ------------------------------------------------- DMMA fused pass
// FV_FISTA_EXP with the X1^T phase on the FP64 tensor cores:
//  * phase A (as k_fused_fast): thread row i of X1, eta = X1 P for its cells,
//    w = v eta, the partial of sum w eta, and w written to a padded tile Wp
//    whose fibre stride SW is = 4 (mod 16), so that a DMMA B fragment (4
//    consecutive rows x 8 fibres) is read without bank conflicts;
//  * phase B: Q (p1 x T) = X1^T W as m8n8k4 DMMA tiles: a warp owns a group
//    of kMmaK output rows (its A fragments, the banded X1^T window of the
//    group, sit in registers) and sweeps 8-fibre column blocks, ks DMMAs per
//    block over the group's input window.  The band's zeros ride along in
//    the tile; the tensor-core work is far below the pass's HBM time.
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int KS, int BS>
__global__ void __launch_bounds__(BS) k_fused_mma(FusedArgs f, FusedPlan pl, i64 ntiles, int sw, int wp_off) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long bar[kMaxStages];
  __shared__ double red[32];
  constexpr int NW = BS / 32;
  const int n1 = static_cast<int>(f.n1), p1 = static_cast<int>(f.p1), T = pl.T;
  const int nst = pl.nst;
  double* Wp = sm + wp_off;
  if (threadIdx.x == 0) {
    for (int k = 0; k < nst; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto issue = [&](i64 tile, int s) {
    const i64 c0 = tile * T;
    const i64 Tc = min(static_cast<i64>(T), f.m - c0);
    double* st = sm + static_cast<i64>(s) * pl.stage;
    unsigned bytes = 0;
    bytes += stage_manual(st + pl.offP, f.P + c0 * p1, p1 * Tc);
    bytes += stage_manual(st + pl.offA, f.v + c0 * n1, n1 * Tc);
    fence_proxy_async();
    mbar_expect_tx(&bar[s], bytes);
    stage_bulk(st + pl.offP, f.P + c0 * p1, p1 * Tc, &bar[s]);
    stage_bulk(st + pl.offA, f.v + c0 * n1, n1 * Tc, &bar[s]);
  };
  const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
  const int CGA = BS / n1;
  const bool actA = tid < n1 * CGA;
  const int iA = actA ? tid % n1 : 0, cgA = actA ? tid / n1 : 0;
  // X1 row band as exactly 4 taps on a window clamped into [0, p1) (zeros
  // outside the band; the host guarantees p1 >= 4)
  int loA = 0;
  double cA[4] = {0.0, 0.0, 0.0, 0.0};
  if (actA) {
    const int lo = __ldg(f.H.lo + iA), len = __ldg(f.H.len + iA);
    const double* cf = f.H.coef + __ldg(f.H.off + iA);
    loA = min(lo, p1 - 4);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = loA + t - lo;
      cA[t] = (j >= 0 && j < len) ? __ldg(cf + j) : 0.0;
    }
  }
  // phase B: fragments of the warp's row group (fixed when groups divides NW)
  const int groups = f.mg.groups;
  int cur_g = -1, gbase = 0;
  double afr[KS];
  auto load_group = [&](int g) {
    cur_g = g;
    gbase = __ldg(f.mg.base + g);
#pragma unroll
    for (int s2 = 0; s2 < KS; ++s2) afr[s2] = __ldg(f.mg.afrag + (static_cast<i64>(g) * KS + s2) * 32 + lane);
  };
  const bool fixed = NW % groups == 0;
  if (fixed) load_group(warp % groups);
  __syncthreads();
  double acc = 0.0;
  int s = 0;
  unsigned phase_bits = 0u;
  i64 tile = blockIdx.x;
  if (threadIdx.x == 0)
    for (int k = 0; k < nst; ++k)
      if (tile + static_cast<i64>(k) * gridDim.x < ntiles) issue(tile + static_cast<i64>(k) * gridDim.x, k);
  for (; tile < ntiles; tile += gridDim.x) {
    const i64 c0 = tile * T;
    const int Tc = static_cast<int>(min(static_cast<i64>(T), f.m - c0));
    double* st = sm + static_cast<i64>(s) * pl.stage;
    const double* Ps = st + pl.offP + stage_shift(f.P + c0 * p1);
    const double* As = st + pl.offA + stage_shift(f.v + c0 * n1);
    mbar_wait(&bar[s], (phase_bits >> s) & 1u);
    phase_bits ^= 1u << s;
    if (actA) {
      auto cell = [&](int col) {
        const double* pc = Ps + p1 * col + loA;
        const double eta = fma(cA[1], pc[1], cA[0] * pc[0]) + fma(cA[3], pc[3], cA[2] * pc[2]);
        const double w = As[iA + n1 * col] * eta;
        acc = fma(w, eta, acc);
        Wp[iA + sw * col] = w;
      };
      int col = cgA;
      for (; col + CGA < Tc; col += 2 * CGA) {
        cell(col);
        cell(col + CGA);
      }
      if (col < Tc) cell(col);
    }
    __syncthreads();
    const int cbs = (Tc + 7) >> 3;
    auto block = [&](int g, int cb) {
      // B fragment: row (lane % 4) of the k-step, fibre 8 cb + lane / 4
      const double* wb = Wp + sw * (8 * cb + (lane >> 2)) + gbase + (lane & 3);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) dmma_884(d0, d1, afr[s2], wb[4 * s2]);
      // D fragment: row k = kMmaK g + lane / 4, fibres 8 cb + 2 (lane % 4) + {0, 1}
      const int k = kMmaK * g + (lane >> 2), colq = 8 * cb + 2 * (lane & 3);
      if (k < p1) {
        double* q = f.Q + (c0 + colq) * p1 + k;
        if (colq < Tc) q[0] = d0;
        if (colq + 1 < Tc) q[p1] = d1;
      }
    };
    if (fixed) {
      for (int cb = warp / groups; cb < cbs; cb += NW / groups) block(cur_g, cb);
    } else {
      for (int task = warp; task < groups * cbs; task += NW) {
        const int g = task % groups;
        if (g != cur_g) load_group(g);
        block(g, task / groups);
      }
    }
    __syncthreads();  // stage s and Wp are free again
    const i64 next = tile + static_cast<i64>(nst) * gridDim.x;
    if (threadIdx.x == 0 && next < ntiles) issue(next, s);
    s = s + 1 == nst ? 0 : s + 1;
  }
  const double r = block_sum(acc, red);
  if (threadIdx.x == 0) f.partial[blockIdx.x] = r;
}

static LcPlan lc_plan(const FusedArgs& f) {
  LcPlan P;
  static const bool enabled = [] {
    const char* e = dev_env("KG_FUSED_MMA");
    return e == nullptr || std::atoi(e) != 0;
  }();
  // CTA shape: threads and the shared-memory budget per CTA (measured best on B200:
  // 256 threads, 72 KB, two stages -> three CTAs per SM for C5)
  static const int bs = [] {
    const char* e = dev_env("KG_MMA_BS");
    return (e && std::atoi(e) == 512) ? 512 : 256;
  }();
  static const i64 budget_kb = [] {
    const char* e = dev_env("KG_MMA_KB");
    const long v = e ? std::atol(e) : 72;
    return static_cast<i64>(v >= 24 && v <= 210 ? v : 72);
  }();
  static const int nst = [] {
    const char* e = dev_env("KG_MMA_STAGES");
    const int v = e ? std::atoi(e) : 2;
    return v >= 2 && v <= kMaxStages ? v : 2;
  }();
  if (!enabled || f.mg.ks == 0 || f.n1 > bs || f.H.maxlen > 4 || f.p1 < 4) return P;
  P.mw = f.mg.ks;  // 8, 12 or 16 (padded on the host)
  P.bs = bs;
  P.sw = static_cast<int>((f.n1 + 15) / 16 * 16 + 4);  // >= n1, = 4 (mod 16)
  if (P.sw - 16 >= f.n1) P.sw -= 16;
  auto up2 = [](i64 x) { return (x + 2) & ~i64(1); };
  // nst stages of (P tile, v tile), then the padded w tile (whole 8-fibre blocks)
  const i64 per_fibre = nst * (f.p1 + f.n1) + P.sw;
  i64 T = (budget_kb * 1024 / 8 - 64) / per_fibre;
  if (T >= 8) T = T / 8 * 8;  // whole 8-fibre DMMA column blocks
  T = std::min<i64>(T, f.m);
  if (T < 4) return P;
  FusedPlan& pl = P.pl;
  pl.T = static_cast<int>(T);
  pl.nst = nst;
  pl.offP = 0;
  pl.offA = static_cast<int>(up2(f.p1 * T));
  pl.offB = pl.offA;
  pl.stage = static_cast<int>(up2(f.p1 * T) + up2(f.n1 * T));
  P.wp_off = nst * pl.stage;
  const i64 wcols = (T + 7) / 8 * 8;
  P.smem = sizeof(double) * static_cast<size_t>(P.wp_off + P.sw * wcols);
  const int per_sm = std::max<int>(1, static_cast<int>((226 * 1024) / (P.smem + 2048)));
  const i64 ntiles = (f.m + T - 1) / T;
  P.grid = static_cast<int>(std::min<i64>(ntiles, 148LL * std::min(per_sm, 2048 / bs)));
  P.ok = P.smem <= 210 * 1024;
  return P;
}

template <int KS>
static void launch_mma(const Launch& L, const FusedArgs& f, const LcPlan& P, i64 ntiles) {
  if (P.bs == 512) {
    smem_attr(k_fused_mma<KS, 512>, static_cast<int>(P.smem));
    k_fused_mma<KS, 512><<<P.grid, 512, P.smem, L.s>>>(f, P.pl, ntiles, P.sw, P.wp_off);
  } else {
    smem_attr(k_fused_mma<KS, 256>, static_cast<int>(P.smem));
    k_fused_mma<KS, 256><<<P.grid, 256, P.smem, L.s>>>(f, P.pl, ntiles, P.sw, P.wp_off);
  }
}

void fused_tma(const Launch& L, int variant, const FusedArgs& f) {
  if (variant == FV_FISTA_EXP) {
    const LcPlan P = lc_plan(f);
    if (P.ok) {
      const i64 nt = (f.m + P.pl.T - 1) / P.pl.T;
      switch (P.mw) {
        case 8: launch_mma<8>(L, f, P, nt); break;
        case 12: launch_mma<12>(L, f, P, nt); break;
        default: launch_mma<16>(L, f, P, nt); break;
      }
      launched(L);
      return;
    }
  }
  const FusedPlan pl = plan_for(f, variant);
  const i64 ntiles = (f.m + pl.T - 1) / pl.T;
  const size_t sm = static_cast<size_t>(pl.nst) * pl.stage * sizeof(double);
  const int g = fused_tma_grid(f, variant);
  smem_attr(k_fused_tma<FV_FISTA>, 210 * 1024);
  smem_attr(k_fused_tma<FV_XTWZ>, 210 * 1024);
  smem_attr(k_fused_tma<FV_SCORE0>, 210 * 1024);
  const bool fast = f.n1 <= NT && f.p1 <= NT && f.H.maxlen <= 4 && f.G.maxlen <= 64;
  if (fast) {
    const int mg = f.G.maxlen <= 8 ? 8 : f.G.maxlen <= 16 ? 16 : f.G.maxlen <= 24 ? 24 : f.G.maxlen <= 32 ? 32 : 64;
    launch_fast(L, variant, mg, f, pl, ntiles, g, sm);
  } else {
    if (variant == FV_FISTA_EXP) throw Error(E_CUDA, "fused_tma: FV_FISTA_EXP needs the register-hoisted kernel");
    switch (variant) {
      case FV_FISTA: k_fused_tma<FV_FISTA><<<g, NT, sm, L.s>>>(f, pl, ntiles); break;
      case FV_XTWZ: k_fused_tma<FV_XTWZ><<<g, NT, sm, L.s>>>(f, pl, ntiles); break;
      default: k_fused_tma<FV_SCORE0><<<g, NT, sm, L.s>>>(f, pl, ntiles); break;
    }
  }
  launched(L);
}

// Bandwidth reference: grid-stride 16-byte loads of two arrays.
__global__ void __launch_bounds__(NT) k_stream_read2(i64 n2, const double2* x, const double2* y, double* part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < n2; i += static_cast<i64>(gridDim.x) * NT) {
    const double2 a = __ldg(x + i), b = __ldg(y + i);
    acc = fma(a.x, b.x, fma(a.y, b.y, acc));
  }
  const double r = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

void stream_read2(const Launch& L, i64 n, const double* x, const double* y, double* partial) {
  k_stream_read2<<<148 * 8, NT, 0, L.s>>>(n / 2, reinterpret_cast<const double2*>(x),
                                          reinterpret_cast<const double2*>(y), partial);
  launched(L);
}

// ----------------------------------------------------- tiled contraction
struct CPlan {
  int AB;   // alpha block (<= 32)
  int MB;   // outputs per m block
  int G;    // m rows per warp step (32 / AB)
  int WMAX; // max staged input rows
  i64 nab, nmb, b;
};

__global__ void __launch_bounds__(NT) k_contract_tiled(const double* __restrict__ A, double* __restrict__ out, i64 a,
                                                       i64 K, i64 M, BandOp op, CPlan pl, int accumulate) {
  extern __shared__ double S[];
  __shared__ int rng[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int AB = pl.AB, G = pl.G;
  const int al = lane % AB, msub = lane / AB;
  const i64 ntiles = pl.nab * pl.nmb * pl.b;
  for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const i64 ab = tile % pl.nab;
    const i64 rest = tile / pl.nab;
    const i64 mb = rest % pl.nmb;
    const i64 be = rest / pl.nmb;
    const i64 a0 = ab * AB;
    const int ABc = static_cast<int>(min(static_cast<i64>(AB), a - a0));
    const i64 m0 = mb * pl.MB, m1 = min(M, m0 + pl.MB);
    if (threadIdx.x == 0) {
      rng[0] = INT_MAX;
      rng[1] = 0;
    }
    __syncthreads();
    int lo_min = INT_MAX, hi_max = 0;
    for (i64 m = m0 + threadIdx.x; m < m1; m += NT) {
      const int lo = __ldg(op.lo + m), len = __ldg(op.len + m);
      if (len > 0) {
        lo_min = min(lo_min, lo);
        hi_max = max(hi_max, lo + len);
      }
    }
    if (lo_min != INT_MAX) {
      atomicMin(&rng[0], lo_min);
      atomicMax(&rng[1], hi_max);
    }
    __syncthreads();
    const int r0 = rng[0] == INT_MAX ? 0 : rng[0];
    const int W = rng[0] == INT_MAX ? 0 : rng[1] - r0;
    // stage input rows [r0, r0 + W) of the alpha block
    const double* src = A + a0 + a * (r0 + K * be);
    for (int idx = threadIdx.x; idx < W * AB; idx += NT) {
      const int r = idx / AB, x = idx - r * AB;
      S[idx] = x < ABc ? __ldg(src + x + a * static_cast<i64>(r)) : 0.0;
    }
    __syncthreads();
    if (msub < G && al < ABc) {
      for (i64 m = m0 + warp * G + msub; m < m1; m += (NT / 32) * G) {
        const int lo = __ldg(op.lo + m), len = __ldg(op.len + m);
        const double* cf = op.coef + __ldg(op.off + m);
        const double* sr = S + al + AB * (lo - r0);
        double s = 0.0;
        for (int t = 0; t < len; ++t) s = fma(__ldg(cf + t), sr[AB * t], s);
        double* o = out + a0 + al + a * (m + M * be);
        *o = accumulate ? *o + s : s;
      }
    }
    __syncthreads();
  }
}

bool contract_plan(const BandOp& op, i64 a, i64 K, i64 M, CPlan& pl);

void contract_tiled(const Launch& L, const double* A, double* out, i64 a, i64 K, i64 M, i64 b, const BandOp& op,
                    bool accumulate) {
  if (a * M * b == 0) return;
  CPlan pl;
  if (!contract_plan(op, a, K, M, pl)) {  // band too wide to stage: one output per thread
    contract(L, A, out, a, K, M, b, op, accumulate);
    return;
  }
  pl.b = b;
  const i64 ntiles = pl.nab * pl.nmb * b;
  const int g = static_cast<int>(std::min<i64>(ntiles, 148LL * 8));
  const size_t sm = static_cast<size_t>(pl.AB) * pl.WMAX * sizeof(double);
  smem_attr(k_contract_tiled, 200 * 1024);
  k_contract_tiled<<<g, NT, sm, L.s>>>(A, out, a, K, M, op, pl, accumulate);
  launched(L);
}

// Chooses the m-block so that the union of the staged input rows of every
// block fits the shared-memory budget (checked exactly on the host copy of
// the band).  Cached per (operator, alpha block).
bool contract_plan(const BandOp& op, i64 a, i64 K, i64 M, CPlan& pl) {
  pl.AB = static_cast<int>(std::min<i64>(a, 32));
  pl.G = 32 / pl.AB;
  pl.nab = (a + pl.AB - 1) / pl.AB;
  const int budget = 6144 / pl.AB;  // 48 KB of staged doubles
  if (!op.hlo || !op.hlen || M != op.rows) return false;
  struct Key {
    uint64_t uid;
    int AB;
    bool operator==(const Key& o) const { return uid == o.uid && AB == o.AB; }
  };
  static std::vector<std::pair<Key, std::pair<int, int>>> cache;  // -> (MB, W)
  for (auto& e : cache)
    if (e.first == Key{op.uid, pl.AB}) {
      if (e.second.first <= 0) return false;
      pl.MB = e.second.first;
      pl.WMAX = e.second.second;
      pl.nmb = (M + pl.MB - 1) / pl.MB;
      return true;
    }
  auto window = [&](i64 MB) {
    int worst = 0;
    for (i64 m0 = 0; m0 < M; m0 += MB) {
      int lo = INT_MAX, hi = 0;
      for (i64 m = m0; m < std::min(M, m0 + MB); ++m)
        if (op.hlen[m] > 0) {
          lo = std::min(lo, op.hlo[m]);
          hi = std::max(hi, op.hlo[m] + op.hlen[m]);
        }
      if (lo != INT_MAX) worst = std::max(worst, hi - lo);
    }
    return worst;
  };
  const double slope = static_cast<double>(K) / static_cast<double>(M);
  i64 MB = static_cast<i64>((budget - op.maxlen - 2) / std::max(slope, 1e-9));
  MB = std::max<i64>(1, std::min<i64>(MB, M));
  int W = window(MB);
  while (W > budget && MB > 1) {
    MB = std::max<i64>(1, MB / 2);
    W = window(MB);
  }
  if (W > budget) {
    cache.push_back({Key{op.uid, pl.AB}, {0, 0}});
    return false;
  }
  cache.push_back({Key{op.uid, pl.AB}, {static_cast<int>(MB), std::max(W, 1)}});
  pl.MB = static_cast<int>(MB);
  pl.WMAX = std::max(W, 1);
  pl.nmb = (M + MB - 1) / MB;
  return true;
}

}  // namespace kg
