// Constant-weight (Gram) route of the FISTA iteration.
//
// With W = w I, X^T W X = w (x)_j X_j^T X_j (the reference's
// xtwx_apply_tensor with constant weight factors, design.cpp:153-177), so a
// FISTA step needs only p-space work: the elementwise update kernel
// (k_fista_update) followed by k_gram_apply, which applies the banded Gram
// product slab by slab (one CTA per slab of the last coefficient mode, the
// other modes contracted in shared memory), emits the objective partials, and
// lets the last CTA to finish (atomic ticket) reduce every partial in fixed
// order and advance the fista_solve control block on the device.
#include <cfloat>
#include <cstdlib>

#include "../../include/kronglm_b200.h"
#include "kg_async.cuh"
#include "kg_internal.h"

namespace kg {

namespace {

constexpr int NT = 256;  // p-space reduction kernels
constexpr int kPollRows = 10;  // partial / flag rows per lane: up to 320 CTAs
// default worker width of k_gauss_path: 15 worker warps + the control warp =
// 512 threads, so ptxas may give each thread 128 registers (17 warps get 96)
constexpr int kPathBS = 480;
constexpr bool kPathCW = true;  // k_gauss_path runs a control warp beside the workers
// phase timers of k_gauss_path (KG_PATH_DBG bits 128, 512, 65536); compiled
// out by default because their live state costs registers in the hot loop
constexpr bool kPathTimers = false;
constexpr int kFlagCTAs = 64;
constexpr int kFlagStride = 32;  // one 128-byte line per CTA flag
constexpr int kMonitorNap = 200;  // ns between polls of the grid-wide monitor wait  // k_gauss_path uses the flag barrier up to this many CTAs (measured: C1 gains, C2/C4 do not)

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

__device__ __forceinline__ double penalty_of(int pen, double alpha, double l1, double l2) {
  if (pen == 0) return l1;
  if (pen == 1) return l2;
  return l1 + alpha * l2;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// deterministic CTA sum, result broadcast to all threads
template <int BS = NT>
__device__ double cta_sum(double v, double* sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    double r = l < (BS >> 5) ? sh[l] : 0.0;
    r = warp_sum(r);
    if (l == 0) sh[32] = r;
  }
  __syncthreads();
  return sh[32];
}

// Three deterministic CTA sums at once (same trees as three cta_sum calls,
// one third of the barriers).  sh needs 3 * 32 + 3 doubles.
template <int BS>
__device__ void cta_sum3(double a, double b, double c, double* sh, double* out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum(c);
  __syncthreads();
  if (l == 0) {
    sh[w] = a;
    sh[32 + w] = b;
    sh[64 + w] = c;
  }
  __syncthreads();
  if (w == 0) {
    double r0 = l < (BS >> 5) ? sh[l] : 0.0;
    double r1 = l < (BS >> 5) ? sh[32 + l] : 0.0;
    double r2 = l < (BS >> 5) ? sh[64 + l] : 0.0;
    r0 = warp_sum(r0);
    r1 = warp_sum(r1);
    r2 = warp_sum(r2);
    if (l == 0) {
      sh[96] = r0;
      sh[97] = r1;
      sh[98] = r2;
    }
  }
  __syncthreads();
  out[0] = sh[96];
  out[1] = sh[97];
  out[2] = sh[98];
}

// Mode-j contraction like smem_mode with the band rows staged in shared
// memory (sc: MB x K coefficients, tap-major so that lanes on consecutive rows
// read consecutive words; slo/slen: row ranges) and the taps unrolled to MB
// with predication; the summation order is smem_mode's.
template <int BS, int MB>
__device__ __forceinline__ void smem_mode_st(const double* in, double* out, int K, int q, const FastDiv& fa,
                                             const FastDiv& fk, const double* sc, const int* slo,
                                             const int* slen) {
  const int a = static_cast<int>(fa.d);
  for (int e = threadIdx.x; e < q; e += BS) {
    const int rest = static_cast<int>(fa.div(static_cast<uint32_t>(e)));
    const int al = e - rest * a;
    const int be = static_cast<int>(fk.div(static_cast<uint32_t>(rest)));
    const int m = rest - be * K;
    const int lo = slo[m], len = slen[m];
    const double* c = sc + m;
    const double* src = in + al + a * (lo + K * be);
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < MB; ++t)
      if (t < len) s = fma(c[t * K], src[a * t], s);
    out[e] = s;
  }
}

// in-shared-memory mode-j contraction of a q-array with extents dims (all
// modes < d-1 keep their extent because G_j is square)
template <int BS>
__device__ void smem_mode(const double* in, double* out, const int* dims, int j, const BandOp& op, int q,
                          const FastDiv& fa, const FastDiv& fk) {
  const int a = static_cast<int>(fa.d);
  const int K = dims[j];
  for (int e = threadIdx.x; e < q; e += BS) {
    const int rest = static_cast<int>(fa.div(static_cast<uint32_t>(e)));
    const int al = e - rest * a;
    const int be = static_cast<int>(fk.div(static_cast<uint32_t>(rest)));
    const int m = rest - be * K;
    const int lo = __ldg(op.lo + m), len = __ldg(op.len + m);
    const double* c = op.coef + __ldg(op.off + m);
    const double* src = in + al + a * (lo + K * be);
    double s = 0.0;
    for (int t = 0; t < len; ++t) s = fma(__ldg(c + t), src[a * t], s);
    out[e] = s;
  }
}

// fista_solve setup after the initial objective g_0 (inner.cpp:132-161).
__device__ void ctl_setup(FistaCtl& c, double g, double wmax) {
  c.g_prev = g;
  c.best_g = g;
  c.bad_weights = !(wmax > 0.0);
  const double lip = wmax * c.lipfac / c.n;  // lipschitz_upper (inner.cpp:53-71)
  c.lip = lip;
  double dl = 1.0 / (fmax(c.nu, 1.0e-300) * lip);
  if (c.nu == 1.0) dl = 1.0 / lip;
  c.delta = dl;
  c.omega = 0.0;
  c.it = 1;
  c.momentum = 1;
  c.streak = 0;
  c.prox_steps = 0;
  c.backtracks = 0;
  c.iterations = 0;
  c.copy_best = 0;
  c.restart = 0;
  c.converged = 0;
  c.diverged = 0;
  c.done = (c.max_iters < 1) || c.bad_weights;
}

// One monitor / restart / stop step of fista_solve (inner.cpp:189-229) with
// the objective g of the iterate just produced.
__device__ void ctl_step(FistaCtl& c, double g) {
  const i64 it = c.it;
  c.copy_best = 0;
  c.restart = 0;
  c.prox_steps += 1;
  c.momentum += 1;
  c.iterations = it;
  const i64 me = c.monitor_every < 1 ? 1 : c.monitor_every;
  if ((it % me == 0) || it == c.max_iters) {
    bool div = !isfinite(g);
    if (!div && c.bt_div && g > c.g_prev) div = (++c.streak >= 3);
    if (div) {
      if (!c.bt_div) {
        c.diverged = 1;
        c.done = 1;
      } else {
        c.restart = 1;
        c.g_prev = c.best_g;
        c.delta *= 0.5;
        c.momentum = 1;
        c.streak = 0;
        c.backtracks += 1;
      }
    } else {
      if (g <= c.g_prev) c.streak = 0;
      if (g <= c.best_g) {
        c.copy_best = 1;
        c.best_g = g;
      }
      if (fabs(g - c.g_prev) / fmax(1.0, fabs(g)) < c.tol) {
        c.converged = 1;
        c.done = 1;
      }
      c.g_prev = g;
    }
  }
  if (!c.done) {
    c.it = it + 1;
    if (c.it > c.max_iters) c.done = 1;
  }
  c.omega = c.extrapolation == 0 ? static_cast<double>(c.momentum - 1) / static_cast<double>(c.momentum + 2) : 0.0;
}

}  // namespace

// S'(x)[:, s] = (G_{d-2..0}) sum_t G_d[s, t] x[:, t] for slab s of the last
// mode, then per-CTA partials of w<x,S'x> - 2<x,b>; the last CTA to finish
// reduces them (and the |x| partials of the preceding update kernel) in fixed
// order and runs the fista_solve monitor / control (or its setup, init mode).
// STAGED: the band of neighbour slabs of x (one contiguous range) and b's own
// slab arrive in shared memory through one bulk-async copy each, so the whole
// input is a single round trip; otherwise the loads go through L1/L2.
template <int BS, bool STAGED>
__global__ void __launch_bounds__(BS) k_gram_apply(GramStepArgs A) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[33];
  __shared__ int am_last;
  __shared__ unsigned long long bar;
  FistaCtl* c = A.ctl;
  const int q = A.q;
  const int s = blockIdx.x;
  const double* x = A.X[0];
  double* Sx = A.S[0];
  const int lo = __ldg(A.Gd.lo + s), len = __ldg(A.Gd.len + s);
  const double* gc = A.Gd.coef + __ldg(A.Gd.off + s);
  // shared layout: [u q][t0 q][t1 q] then, staged: [x band  maxlen*q + 2][b slab q + 2]
  double* u = sm;
  double* t0 = sm + q;
  double* t1 = sm + 2 * q;
  const double* xb = x + static_cast<i64>(lo) * q;  // neighbour band, contiguous
  const double* bsrc = A.b + static_cast<i64>(s) * q;
  const double* xv_s = x + static_cast<i64>(s) * q;
  const double* bv = bsrc;
  const double* xin = xb;
  if (STAGED) {
    double* xbase = sm + 3 * q;
    double* bbase = xbase + (static_cast<i64>(A.Gd.maxlen) * q + 2);
    if (threadIdx.x == 0) {
      async::mbar_init(&bar, 1);
      async::mbar_init_fence();
      unsigned bytes = async::stage_manual(xbase, xb, static_cast<i64>(len) * q);
      bytes += async::stage_manual(bbase, bsrc, q);
      async::fence_proxy_async();
      async::mbar_expect_tx(&bar, bytes);
      async::stage_bulk(xbase, xb, static_cast<i64>(len) * q, &bar);
      async::stage_bulk(bbase, bsrc, q, &bar);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    async::mbar_wait(&bar, 0);
    xin = xbase + async::stage_shift(xb);
    bv = bbase + async::stage_shift(bsrc);
    xv_s = xin + static_cast<i64>(s - lo) * q;  // own slab inside the band (s is in its Gram band)
  }
  for (int e = threadIdx.x; e < q; e += BS) {
    const double* xe = xin + e;
    double a0 = 0.0, a1 = 0.0;
    int t = 0;
    for (; t + 1 < len; t += 2) {
      a0 = fma(__ldg(gc + t), xe[static_cast<i64>(t) * q], a0);
      a1 = fma(__ldg(gc + t + 1), xe[static_cast<i64>(t + 1) * q], a1);
    }
    if (t < len) a0 = fma(__ldg(gc + t), xe[static_cast<i64>(t) * q], a0);
    u[e] = a0 + a1;
  }
  __syncthreads();
  const double* res = u;
  double* bufs[2] = {t0, t1};
  int which = 0;
  for (int j = A.d - 2; j >= 0; --j) {
    smem_mode<BS>(res, bufs[which], A.dims, j, A.G[j], q, A.fa[j], A.fk[j]);
    __syncthreads();
    res = bufs[which];
    which ^= 1;
  }
  const double w = c->sscale;
  double dots = 0.0, l1 = 0.0, l2 = 0.0;
  for (int e = threadIdx.x; e < q; e += BS) {
    const i64 idx = static_cast<i64>(s) * q + e;
    const double sv = res[e], xv = xv_s[e];
    Sx[idx] = sv;
    dots += xv * (w * sv - 2.0 * bv[e]);
    l1 += fabs(xv);
    l2 = fma(xv, xv, l2);
  }
  dots = cta_sum<BS>(dots, red);
  l1 = cta_sum<BS>(l1, red);
  l2 = cta_sum<BS>(l2, red);
  if (threadIdx.x == 0) {
    A.part[3 * s] = dots;
    A.part[3 * s + 1] = l1;
    A.part[3 * s + 2] = l2;
    __threadfence();
    const unsigned ticket = atomicAdd(A.counter, 1u);
    am_last = ticket == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // ---- last CTA: fixed-order reductions + control
  double sd = 0.0, s1 = 0.0, s2 = 0.0;
  for (int r = threadIdx.x; r < static_cast<int>(gridDim.x); r += BS) {
    sd += __ldcg(A.part + 3 * r);
    s1 += __ldcg(A.part + 3 * r + 1);
    s2 += __ldcg(A.part + 3 * r + 2);
  }
  sd = cta_sum<BS>(sd, red);
  s1 = cta_sum<BS>(s1, red);
  s2 = cta_sum<BS>(s2, red);
  if (threadIdx.x != 0) return;
  *A.counter = 0u;
  const double g = 0.5 * (sd + c->ss_const) / c->n + c->lambda * penalty_of(A.pen, A.alpha, s1, s2);
  if (A.init) {
    ctl_setup(*c, g, w);  // every weight equals w
    return;
  }
  ctl_step(*c, g);
  if (A.use_handle) cudaGraphSetConditional(A.handle, c->done ? 0u : 1u);
}

bool gram_step_fits(i64 q) { return 3 * q * static_cast<i64>(sizeof(double)) <= 200 * 1024; }

void gram_step(const Launch& L, const GramStepArgs& A) {
  smem_attr(k_gram_apply<256, true>, 210 * 1024);
  smem_attr(k_gram_apply<256, false>, 210 * 1024);
  const size_t base = 3 * static_cast<size_t>(A.q) * sizeof(double);
  const size_t staged = base + (static_cast<size_t>(A.Gd.maxlen + 1) * A.q + 4) * sizeof(double);
  if (staged <= 200 * 1024) {
    k_gram_apply<256, true><<<static_cast<unsigned>(A.pd), 256, staged, L.s>>>(A);
  } else {
    k_gram_apply<256, false><<<static_cast<unsigned>(A.pd), 256, base, L.s>>>(A);
  }
  launched(L);
}

// ------------------------------------------------------------------------
// Persistent cooperative FISTA solve on the Gram route: one launch runs the
// whole fista_solve.  CTA s keeps slab s of x, x_prev, S'x, S'x_prev, best,
// S'best and b in shared memory for the whole solve; per iteration it
//   1. applies the elementwise step to its slab and publishes x_new[:, s],
//   2. grid barrier,
//   3. bulk-copies the neighbour band of x_new (one contiguous range) and
//      computes S'(x_new)[:, s] and its objective partials,
//   4. grid barrier, then reduces all partials in fixed order and advances a
//      replicated copy of the control block (every CTA computes the same
//      state, so no third barrier is needed).
// Co-residency of all CTAs is guaranteed by the cooperative launch.
namespace {

// Sense-reversing grid barrier with GPU-scope acquire/release atomics:
// bar[0] counts arrivals, bar[1] is the generation.  The CTA barrier before
// the arrive orders every thread's writes into thread 0's release
// (cumulativity); waiters acquire the new generation.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, old;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == nb - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned cur;
      const long long t0 = clock64();
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
        if (clock64() - t0 > async::kWatchdogCycles) {
          printf("kg watchdog: grid barrier (block %d of %u, generation %u)\n", blockIdx.x, nb, g);
          __trap();
        }
      } while (cur == g);
    }
  }
  __syncthreads();
}

template <int ID, int N>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void named_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory");
}

// grid_sync's arrive + wait for one thread (the caller orders the CTA's writes
// before it, e.g. through a named barrier)
__device__ __forceinline__ void grid_arrive_wait(unsigned* bar, unsigned nb) {
  unsigned g, old;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
  if (old == nb - 1) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
  } else {
    unsigned cur;
    const long long t0 = clock64();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      if (clock64() - t0 > async::kWatchdogCycles) {
        printf("kg watchdog: grid barrier (block %d of %u, generation %u)\n", blockIdx.x, nb, g);
        __trap();
      }
    } while (cur == g);
  }
}

}  // namespace

template <int BS>
__global__ void __launch_bounds__(BS) k_fista_persist(PersistArgs P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[33];
  __shared__ FistaCtl cs;
  __shared__ unsigned long long mb;
  const GramStepArgs& A = P.g;
  const int q = A.q;
  const int s = blockIdx.x;
  const unsigned nb = gridDim.x;
  double* xs = sm;
  double* xps = xs + q;
  double* sxs = xps + q;
  double* sxps = sxs + q;
  double* bst = sxps + q;
  double* sbst = bst + q;
  double* bs = sbst + q;
  double* u = bs + q;
  double* t0 = u + q;
  double* t1 = t0 + q;
  double* band = t1 + q;  // maxlen * q + 2
  if (threadIdx.x == 0) {
    cs = *A.ctl;
    async::mbar_init(&mb, 1);
    async::mbar_init_fence();
  }
  const int lo = __ldg(A.Gd.lo + s), len = __ldg(A.Gd.len + s);
  const double* gc = A.Gd.coef + __ldg(A.Gd.off + s);
  const i64 base = static_cast<i64>(s) * q;
  for (int e = threadIdx.x; e < q; e += BS) {
    const double x0 = P.theta[base + e];
    xs[e] = x0;
    xps[e] = x0;
    bst[e] = x0;
    bs[e] = A.b[base + e];
    P.X[base + e] = x0;
  }
  __syncthreads();  // cs and the mbarrier are read by every warp
  unsigned parity = 0;
  const double w = cs.sscale;
  // S'(x_new)[:, s] into sxs from the published X, plus objective partials
  auto apply = [&]() {
    const double* xb = P.X + static_cast<i64>(lo) * q;
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const unsigned bytes = async::stage_manual(band, xb, static_cast<i64>(len) * q);
      async::fence_proxy_async();
      async::mbar_expect_tx(&mb, bytes);
      async::stage_bulk(band, xb, static_cast<i64>(len) * q, &mb);
    }
    __syncthreads();
    async::mbar_wait(&mb, parity);
    parity ^= 1u;
    const double* xin = band + async::stage_shift(xb);
    for (int e = threadIdx.x; e < q; e += BS) {
      const double* xe = xin + e;
      double a0 = 0.0, a1 = 0.0;
      int t = 0;
      for (; t + 1 < len; t += 2) {
        a0 = fma(__ldg(gc + t), xe[static_cast<i64>(t) * q], a0);
        a1 = fma(__ldg(gc + t + 1), xe[static_cast<i64>(t + 1) * q], a1);
      }
      if (t < len) a0 = fma(__ldg(gc + t), xe[static_cast<i64>(t) * q], a0);
      u[e] = a0 + a1;
    }
    __syncthreads();
    const double* res = u;
    double* bufs[2] = {t0, t1};
    int which = 0;
    for (int j = A.d - 2; j >= 0; --j) {
      smem_mode<BS>(res, bufs[which], A.dims, j, A.G[j], q, A.fa[j], A.fk[j]);
      __syncthreads();
      res = bufs[which];
      which ^= 1;
    }
    double dots = 0.0, l1 = 0.0, l2 = 0.0;
    for (int e = threadIdx.x; e < q; e += BS) {
      const double sv = res[e], xv = xs[e];
      sxs[e] = sv;
      dots += xv * (w * sv - 2.0 * bs[e]);
      l1 += fabs(xv);
      l2 = fma(xv, xv, l2);
    }
    dots = cta_sum<BS>(dots, red);
    l1 = cta_sum<BS>(l1, red);
    l2 = cta_sum<BS>(l2, red);
    if (threadIdx.x == 0) {
      P.part[3 * s] = dots;
      P.part[3 * s + 1] = l1;
      P.part[3 * s + 2] = l2;
    }
  };
  // fixed-order reduction of every CTA's partials (identical in all CTAs)
  auto objective = [&]() -> double {
    double sd = 0.0, s1 = 0.0, s2 = 0.0;
    for (int r = threadIdx.x; r < static_cast<int>(nb); r += BS) {
      sd += __ldcg(P.part + 3 * r);
      s1 += __ldcg(P.part + 3 * r + 1);
      s2 += __ldcg(P.part + 3 * r + 2);
    }
    sd = cta_sum<BS>(sd, red);
    s1 = cta_sum<BS>(s1, red);
    s2 = cta_sum<BS>(s2, red);
    return 0.5 * (sd + cs.ss_const) / cs.n + cs.lambda * penalty_of(A.pen, A.alpha, s1, s2);
  };

  grid_sync(P.bar, nb);
  apply();
  for (int e = threadIdx.x; e < q; e += BS) {
    sxps[e] = sxs[e];
    sbst[e] = sxs[e];
  }
  grid_sync(P.bar, nb);
  {
    const double g0 = objective();
    if (threadIdx.x == 0) ctl_setup(cs, g0, w);
    __syncthreads();
  }
  while (!cs.done) {
    const double omega = cs.omega, delta = cs.delta, lambda = cs.lambda, n = cs.n;
    const int restart = cs.restart, copy_best = cs.copy_best;
    const double gamma = __dmul_rn(delta, lambda);
    for (int e = threadIdx.x; e < q; e += BS) {
      if (copy_best) {
        bst[e] = xs[e];
        sbst[e] = sxs[e];
      }
      if (restart) {
        xs[e] = xps[e] = bst[e];
        sxs[e] = sxps[e] = sbst[e];
      }
      const double xi = xs[e], xpi = xps[e], sxi = sxs[e], sxpi = sxps[e];
      const double yi = xi + omega * (xi - xpi);
      const double syi = sxi + omega * (sxi - sxpi);
      const double g = (w * syi - bs[e]) / n;
      double ci = __dsub_rn(yi, __dmul_rn(delta, g));
      if (lambda > 0.0) ci = prox1(A.pen, A.alpha, gamma, ci);
      xps[e] = xi;
      xs[e] = ci;
      sxps[e] = sxi;
      P.X[base + e] = ci;
    }
    grid_sync(P.bar, nb);
    apply();
    grid_sync(P.bar, nb);
    const double g = objective();
    if (threadIdx.x == 0) ctl_step(cs, g);
    __syncthreads();
  }
  for (int e = threadIdx.x; e < q; e += BS) {
    if (cs.copy_best) {
      bst[e] = xs[e];
      sbst[e] = sxs[e];
    }
    P.best[base + e] = bst[e];
    P.Sbest[base + e] = sbst[e];
  }
  if (s == 0 && threadIdx.x == 0) *A.ctl = cs;
}

// ------------------------------------------------------------------------
// The whole Gaussian constant-weight lambda path in one cooperative launch
// (fit_path, path.cpp:47-81, with the Gaussian shortcut of outer_solve,
// outer.cpp:197-231).  Per lambda, on the device and in lockstep:
//   f_cur = -loglik(theta)/n + lambda J(theta) from the replicated
//   (<theta,b>, <theta,S'theta>, |theta|_1, |theta|_2^2);
//   fista_solve from x_0 = theta (S'(x_0) is the slab of S'theta kept in
//   shared memory, so the setup needs no pass);
//   f_new from (<best,b>, <best,S'best>, |best|) -> accept if f_new <= f_cur;
//   status / truncation / first-model failure as path.cpp:64-73;
//   the model's coefficients are written straight into the result buffer.
constexpr int kMmLD = 36;  // padded leading dimension (= 4 mod 16 doubles: conflict-free DMMA fragments)

// DMMA in-slab contraction of k_gauss_path: d = 3, both in-slab extents <= 32,
// staged bands
__host__ __device__ inline bool path_mm(const GramStepArgs& A) {
  return A.d == 3 && A.dims[0] <= 32 && A.dims[1] <= 32 && A.G[0].maxlen <= kPathTaps && A.G[1].maxlen <= kPathTaps;
}
__host__ __device__ inline int path_qb(const GramStepArgs& A) {  // size of each contraction buffer
  return path_mm(A) ? (A.q > kMmLD * 32 ? A.q : kMmLD * 32) : A.q;
}

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int BS, bool CW>
__global__ void __launch_bounds__(BS + (CW ? 32 : 0), (!CW && BS <= 256) ? 2 : 1) k_gauss_path(PersistArgs P) {
  constexpr int MB = kPathTaps;
  // CW: one extra control warp (threads BS..BS+31) runs the grid barrier, the
  // band copy and the monitor of the nu = 1 loop while the BS worker threads
  // contract; it owns no elements (tx is past every element / row range)
  const int tx = (CW && threadIdx.x >= BS) ? (1 << 30) : static_cast<int>(threadIdx.x);
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[3 * 32 + 3];
  __shared__ FistaCtl cs;
  __shared__ unsigned long long mb;
  __shared__ double tb, tst, tl1, tl2;  // replicated path state of theta
  const GramStepArgs& A = P.g;
  const int q = A.q;
  const int s = blockIdx.x;
  const unsigned nb = gridDim.x;
  double* xs = sm;
  double* xps = xs + q;
  double* sxs = xps + q;
  double* sxps = sxs + q;
  double* bst = sxps + q;
  double* sbst = bst + q;
  double* bs = sbst + q;
  double* th = bs + q;
  double* sth = th + q;
  double* xpp = sth + q;  // CW: x_{k-2} and S'x_{k-2} (the monitor decision runs two steps late)
  double* sxpp = xpp + q;
  double* bn = sxpp + q;  // b / n: the gradient is w/n S'y - b/n, one FMA per element
  // mm: the two in-slab modes of a d = 3 design (p1, p2 <= 32) run as DMMA
  // tiles over padded (ld kMmLD) buffers and dense padded Gram matrices
  const bool mm = path_mm(A) && !(P.dbg & (1024 | 1));  // needs the staged bands (dbg & 1 disables staging)
  const int qb = path_qb(A);
  double* u = bn + q;
  double* t0 = u + qb;
  double* t1 = t0 + qb;
  double* band = t1 + qb;  // maxlen * q + 2
  double* gd0 = band + static_cast<i64>(A.Gd.maxlen) * q + 2;  // mm: G_0 (kMmLD x 32), then G_1
  double* gd1 = gd0 + kMmLD * 32;
  __shared__ int2 kr[2][4];  // mm: k-step range of each 8-row block of G_0 / G_1
  __shared__ double rbuf[3 * BS];  // per-thread objective partials of compute()
  // dbg & 65536: barrier / copy-issue / copy-latency / arrive-to-band cycles (one SM clock)
  __shared__ long long tw1, tc1, tc2, dph[4];
  // Gram bands of modes 0 .. d-2 staged in shared memory (K_j x MB
  // coefficients, zero padded, then lo / len per row); mode j starts at
  // sg + MB * (dims[0] + .. + dims[j-1]) and sgi + 2 * (same)
  double* sg = band + static_cast<i64>(A.Gd.maxlen) * q + 2 + (path_mm(A) ? 2 * kMmLD * 32 : 0);
  int rows_all = 0;
  bool staged = true;
  for (int j = 0; j < A.d - 1; ++j) {
    rows_all += A.dims[j];
    staged = staged && A.G[j].maxlen <= MB && !(P.dbg & 1);
  }
  int* sgi = reinterpret_cast<int*>(sg + static_cast<i64>(rows_all) * MB);
  if (staged) {
    int r0 = 0;
    for (int j = 0; j < A.d - 1; ++j) {
      const int K = A.dims[j];
      for (int r = tx; r < K; r += BS) {
        const int ln = __ldg(A.G[j].len + r);
        const double* c = A.G[j].coef + __ldg(A.G[j].off + r);
        sgi[2 * r0 + r] = __ldg(A.G[j].lo + r);
        sgi[2 * r0 + K + r] = ln;
        for (int t = 0; t < MB; ++t) sg[static_cast<i64>(r0) * MB + t * K + r] = t < ln ? c[t] : 0.0;  // tap-major
      }
      r0 += K;
    }
  }
  if (threadIdx.x == 0) {
    async::mbar_init(&mb, 1);
    async::mbar_init_fence();
    tb = tst = tl1 = tl2 = 0.0;
    dph[0] = dph[1] = dph[2] = dph[3] = 0;
  }
  const int lo = __ldg(A.Gd.lo + s), len = __ldg(A.Gd.len + s);
  const double* gc = A.Gd.coef + __ldg(A.Gd.off + s);
  const bool hoist = len <= MB && !(P.dbg & 2);  // uniform per CTA
  double gr[MB];
#pragma unroll
  for (int t = 0; t < MB; ++t) gr[t] = (hoist && t < len) ? __ldg(gc + t) : 0.0;
  const i64 base = static_cast<i64>(s) * q;
  const i64 p = static_cast<i64>(q) * nb;
  for (int e = tx; e < q; e += BS) {
    th[e] = 0.0;  // fit_path starts from zero blocks (path.cpp:63); S'(0) = 0
    sth[e] = 0.0;
    bs[e] = A.b[base + e];
  }
  __syncthreads();  // staged bands, mbarrier and the replicated theta state are read by every warp
  if (mm) {
    // dense G_j[r, c] at gdj[r + kMmLD c] (zero outside the band and past p_j),
    // zeroed padding of u and t0 (never written below), k-step ranges
    for (int i = tx; i < 2 * kMmLD * 32; i += BS) {
      const int j = i / (kMmLD * 32), rc = i - j * (kMmLD * 32);
      const int c = rc / kMmLD, r = rc - c * kMmLD;
      const int K = A.dims[j], r0 = j == 0 ? 0 : A.dims[0];
      double v = 0.0;
      if (r < K && c < K) {
        const int lo_r = sgi[2 * r0 + r], len_r = sgi[2 * r0 + K + r];
        if (c >= lo_r && c < lo_r + len_r) v = sg[static_cast<i64>(r0) * MB + (c - lo_r) * K + r];
      }
      gd0[i] = v;
    }
    for (int i = tx; i < 2 * qb; i += BS) u[i] = 0.0;  // u and t0 are adjacent
    if (tx < 8) {
      const int j = tx >> 2, blk = tx & 3;
      const int K = A.dims[j], r0 = j == 0 ? 0 : A.dims[0];
      int kmin = 1 << 20, kmax = 0;
      for (int r = 8 * blk; r < min(8 * blk + 8, K); ++r) {
        const int lo_r = sgi[2 * r0 + r], len_r = sgi[2 * r0 + K + r];
        if (len_r > 0) {
          kmin = min(kmin, lo_r);
          kmax = max(kmax, lo_r + len_r);
        }
      }
      kr[j][blk] = kmin < kmax ? make_int2(kmin >> 2, (kmax + 3) >> 2) : make_int2(0, 0);
    }
    __syncthreads();
  }
  unsigned parity = 0;
  const FistaCtl* tmpl = A.ctl;  // configuration (lambda filled per model); written back only at exit
  const double w = tmpl->sscale, n = tmpl->n, c0 = tmpl->ss_const;
  const double wn = w / n;
  for (int e = tx; e < q; e += BS) bn[e] = bs[e] / n;  // own elements only: no barrier
  const int bt_div = tmpl->bt_div, extrapolation = tmpl->extrapolation;
  auto reduce3 = [&](double a, double b, double c, double* out) {
    if (P.dbg & 4) {
      out[0] = cta_sum<BS>(a, red);
      out[1] = cta_sum<BS>(b, red);
      out[2] = cta_sum<BS>(c, red);
    } else {
      cta_sum3<BS>(a, b, c, red, out);
    }
  };
  // bulk-async copy of the neighbour band of slabs [lo, lo + len) of xsrc
  auto issue_now = [&](const double* xsrc) {  // by one thread
    const double* xb = xsrc + static_cast<i64>(lo) * q;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const unsigned bytes = async::stage_manual(band, xb, static_cast<i64>(len) * q);
    async::fence_proxy_async();
    async::mbar_expect_tx(&mb, bytes);
    async::stage_bulk(band, xb, static_cast<i64>(len) * q, &mb);
  };
  auto issue = [&](const double* xsrc) {
    if (threadIdx.x == 0) issue_now(xsrc);
  };
  auto wait_band = [&]() {
    async::mbar_wait(&mb, parity);
    parity ^= 1u;
  };
  unsigned gen = 0;  // flag-barrier generation (same sequence in every CTA)
  // S'(x) of this slab from the staged band -> sxs; objective partials of xs -> dst
  // defer: leave the per-thread objective partials in rbuf for the control
  // warp (no CTA reduction here)
  auto compute = [&](const double* xsrc, double* dst, int sc_, int ss_, bool defer = false) {  // dst[c * sc_ + s * ss_]
    if (CW && threadIdx.x >= BS) return;  // workers only (named barrier 3)
    const double* xin = band + async::stage_shift(xsrc + static_cast<i64>(lo) * q);
    for (int e = tx; e < q; e += BS) {
      const double* xe = xin + e;
      double a0 = 0.0, a1 = 0.0;
      if (hoist) {
#pragma unroll
        for (int t = 0; t < MB; t += 2) {
          if (t < len) a0 = fma(gr[t], xe[static_cast<i64>(t) * q], a0);
          if (t + 1 < len) a1 = fma(gr[t + 1], xe[static_cast<i64>(t + 1) * q], a1);
        }
      } else {
        int t = 0;
        for (; t + 1 < len; t += 2) {
          a0 = fma(__ldg(gc + t), xe[static_cast<i64>(t) * q], a0);
          a1 = fma(__ldg(gc + t + 1), xe[static_cast<i64>(t + 1) * q], a1);
        }
        if (t < len) a0 = fma(__ldg(gc + t), xe[static_cast<i64>(t) * q], a0);
      }
      if (mm) {
        const int m = static_cast<int>(A.fa[1].div(static_cast<uint32_t>(e)));
        u[e - m * A.dims[0] + kMmLD * m] = a0 + a1;
      } else {
        u[e] = a0 + a1;
      }
    }
    named_sync<3, BS>();
    const double* res = u;
    if (mm) {
      const int wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
      const int p1 = A.dims[0], p2 = A.dims[1];
      const int n1t = (p1 + 7) >> 3, n2t = (p2 + 7) >> 3;
      // mode 1: T = U G_1^T  (T[al, m] at t0[al + kMmLD m])
      for (int tile = wp; tile < n1t * n2t; tile += BS / 32) {
        const int tj = tile / n1t, ti = tile - tj * n1t;
        const int al = 8 * ti + (ln >> 2);
        const int2 r = kr[1][tj];
        double d0 = 0.0, d1 = 0.0;
        for (int ks = r.x; ks < r.y; ++ks) {
          const int kk = 4 * ks + (ln & 3);
          dmma_884(d0, d1, u[al + kMmLD * kk], gd1[8 * tj + (ln >> 2) + kMmLD * kk]);
        }
        const int m = 8 * tj + 2 * (ln & 3);
        if (al < p1) {
          if (m < p2) t0[al + kMmLD * m] = d0;
          if (m + 1 < p2) t0[al + kMmLD * (m + 1)] = d1;
        }
      }
      named_sync<3, BS>();
      // mode 0: S = G_0 T, written unpadded (S[m, be] at t1[m + p1 be])
      for (int tile = wp; tile < n1t * n2t; tile += BS / 32) {
        const int tj = tile / n1t, ti = tile - tj * n1t;
        const int m = 8 * ti + (ln >> 2);
        const int2 r = kr[0][ti];
        double d0 = 0.0, d1 = 0.0;
        for (int ks = r.x; ks < r.y; ++ks) {
          const int kk = 4 * ks + (ln & 3);
          dmma_884(d0, d1, gd0[m + kMmLD * kk], t0[kk + kMmLD * (8 * tj + (ln >> 2))]);
        }
        const int be = 8 * tj + 2 * (ln & 3);
        if (m < p1) {
          if (be < p2) t1[m + p1 * be] = d0;
          if (be + 1 < p2) t1[m + p1 * (be + 1)] = d1;
        }
      }
      named_sync<3, BS>();
      res = t1;
    }
    int which = 0;
    int r0 = rows_all;
    for (int j = mm ? -1 : A.d - 2; j >= 0; --j) {
      double* dst2 = which ? t1 : t0;
      const int K = A.dims[j];
      r0 -= K;
      if (staged)
        smem_mode_st<BS, MB>(res, dst2, K, q, A.fa[j], A.fk[j], sg + static_cast<i64>(r0) * MB, sgi + 2 * r0,
                             sgi + 2 * r0 + K);
      else
        smem_mode<BS>(res, dst2, A.dims, j, A.G[j], q, A.fa[j], A.fk[j]);
      named_sync<3, BS>();
      res = dst2;
      which ^= 1;
    }
    double dots = 0.0, l1 = 0.0, l2 = 0.0;
    for (int e = tx; e < q; e += BS) {
      const double sv = res[e], xv = xs[e];
      sxs[e] = sv;
      dots += xv * (w * sv - 2.0 * bs[e]);
      l1 += fabs(xv);
      l2 = fma(xv, xv, l2);
    }
    // CTA partials for thread 0 only: one barrier (red / rbuf are next written
    // after the following grid barrier)
    const int wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (defer) {  // every worker writes (zeros when it owns no element): the control sums all BS
      rbuf[threadIdx.x] = dots;
      rbuf[BS + threadIdx.x] = l1;
      rbuf[2 * BS + threadIdx.x] = l2;
      return;
    }
    if (!(P.dbg & 32768)) {
      // per-thread partials to shared memory, then warp 0 sums them in a fixed
      // order (lane-strided, then the warp tree): only the threads that own
      // elements take part, and no shuffle traffic from idle warps
      const int nact = q < BS ? q : BS;
      if (static_cast<int>(threadIdx.x) < nact) {
        rbuf[threadIdx.x] = dots;
        rbuf[BS + threadIdx.x] = l1;
        rbuf[2 * BS + threadIdx.x] = l2;
      }
      named_sync<3, BS>();
      if (wp == 0) {
        double r0 = 0.0, r1 = 0.0, r2 = 0.0;
        for (int i = ln; i < nact; i += 32) {
          r0 += rbuf[i];
          r1 += rbuf[BS + i];
          r2 += rbuf[2 * BS + i];
        }
        r0 = warp_sum(r0);
        r1 = warp_sum(r1);
        r2 = warp_sum(r2);
        if (ln == 0) {
          dst[s * ss_] = r0;
          dst[sc_ + s * ss_] = r1;
          dst[2 * sc_ + s * ss_] = r2;
        }
      }
      return;
    }
    dots = warp_sum(dots);
    l1 = warp_sum(l1);
    l2 = warp_sum(l2);
    if (ln == 0) {
      red[wp] = dots;
      red[32 + wp] = l1;
      red[64 + wp] = l2;
    }
    named_sync<3, BS>();
    if (wp == 0) {
      double r0 = ln < (BS >> 5) ? red[ln] : 0.0;
      double r1 = ln < (BS >> 5) ? red[32 + ln] : 0.0;
      double r2 = ln < (BS >> 5) ? red[64 + ln] : 0.0;
      r0 = warp_sum(r0);
      r1 = warp_sum(r1);
      r2 = warp_sum(r2);
      if (ln == 0) {
        dst[s * ss_] = r0;
        dst[sc_ + s * ss_] = r1;
        dst[2 * sc_ + s * ss_] = r2;
      }
    }
  };
  // CW-loop contraction for mm designs: the last mode over the staged band
  // (two elements per pass), one CTA barrier, then warp (ti, tj) owns output
  // tile (ti, tj) of both DMMA modes; the column-block group tj (n1t warps)
  // syncs on its own named barrier between them, and the mode-0 fragments go
  // straight into S'x and the objective partial (no further pass or barrier).
  // ul1 / ul2: |x|_1 and |x|^2 partials of the thread's own elements.
  const int n1t_ = (A.dims[0] + 7) >> 3, n2t_ = (A.dims[1] + 7) >> 3;
  const bool fused = mm && hoist && n2t_ <= BS / 32 && n2t_ <= 10 && !(P.dbg & 4096);
  // direct: the neighbour band is read straight from L2 (ld.global.cg) once the
  // control warp has seen the neighbours' flags (named barrier 4), instead of
  // a bulk copy into shared memory
  const bool direct = fused;
  auto compute_fused = [&](const double* xsrc, double ul1, double ul2) {
    const double* xin = xsrc + static_cast<i64>(lo) * q;  // global (L2), see direct
    const int p1 = A.dims[0], p2 = A.dims[1];
    for (int e = tx; e < q; e += 2 * BS) {
      const int f = e + BS;
      const bool two = f < q;
      const double* xe = xin + e;
      const double* xf = xin + (two ? f : e);
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int t = 0; t < MB; t += 2) {
        if (t < len) {
          a0 = fma(gr[t], __ldcg(xe + static_cast<i64>(t) * q), a0);
          b0 = fma(gr[t], __ldcg(xf + static_cast<i64>(t) * q), b0);
        }
        if (t + 1 < len) {
          a1 = fma(gr[t + 1], __ldcg(xe + static_cast<i64>(t + 1) * q), a1);
          b1 = fma(gr[t + 1], __ldcg(xf + static_cast<i64>(t + 1) * q), b1);
        }
      }
      const int m = static_cast<int>(A.fa[1].div(static_cast<uint32_t>(e)));
      u[e - m * p1 + kMmLD * m] = a0 + a1;
      if (two) {
        const int m2 = static_cast<int>(A.fa[1].div(static_cast<uint32_t>(f)));
        u[f - m2 * p1 + kMmLD * m2] = b0 + b1;
      }
    }
    named_sync<3, BS>();
    const int wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
    // column-block groups: warp wp serves tj = wp mod n2t and the row tiles
    // ti = gi, gi + gs, ... of that block (gi = wp / n2t, gs = group size)
    constexpr int NW = BS / 32;
    const int tj = wp % n2t_, gi = wp / n2t_, gs = (NW - tj + n2t_ - 1) / n2t_;
    double dots = 0.0;
    for (int ti = gi; ti < n1t_; ti += gs) {  // mode 1: T tile (ti, tj) = U G_1^T
        const int al = 8 * ti + (ln >> 2);
        const int2 r = kr[1][tj];
        double d0 = 0.0, d1 = 0.0;
        for (int ks = r.x; ks < r.y; ++ks) {
          const int kk = 4 * ks + (ln & 3);
          dmma_884(d0, d1, u[al + kMmLD * kk], gd1[8 * tj + (ln >> 2) + kMmLD * kk]);
        }
        const int m = 8 * tj + 2 * (ln & 3);
        if (al < p1) {
          if (m < p2) t0[al + kMmLD * m] = d0;
          if (m + 1 < p2) t0[al + kMmLD * (m + 1)] = d1;
        }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(5 + tj), "r"(32 * gs) : "memory");  // column block tj of T is complete
    for (int ti = gi; ti < n1t_; ti += gs) {  // mode 0: S tile (ti, tj) = G_0 T, fragments -> S'x and the partial
        const int m = 8 * ti + (ln >> 2);
        const int2 r = kr[0][ti];
        double d0 = 0.0, d1 = 0.0;
        for (int ks = r.x; ks < r.y; ++ks) {
          const int kk = 4 * ks + (ln & 3);
          dmma_884(d0, d1, gd0[m + kMmLD * kk], t0[kk + kMmLD * (8 * tj + (ln >> 2))]);
        }
        const int be = 8 * tj + 2 * (ln & 3);
        if (m < p1) {
          if (be < p2) {
            const int e = m + p1 * be;
            sxs[e] = d0;
            dots += xs[e] * (w * d0 - 2.0 * bs[e]);
          }
          if (be + 1 < p2) {
            const int e = m + p1 * (be + 1);
            sxs[e] = d1;
            dots += xs[e] * (w * d1 - 2.0 * bs[e]);
          }
        }
    }
    rbuf[threadIdx.x] = dots;
    rbuf[BS + threadIdx.x] = ul1;
    rbuf[2 * BS + threadIdx.x] = ul2;
  };
  auto apply = [&]() {
    issue(P.X);
    __syncthreads();
    wait_band();
    compute(P.X, P.part, 1, 3);
  };
  auto gather3 = [&](double* out) {  // fixed-order sum of every CTA's 3 partials
    double a = 0.0, b = 0.0, c = 0.0;
    for (int r = tx; r < static_cast<int>(nb); r += BS) {
      a += __ldcg(P.part + 3 * r);
      b += __ldcg(P.part + 3 * r + 1);
      c += __ldcg(P.part + 3 * r + 2);
    }
    reduce3(a, b, c, out);
  };

  int stop = 0;  // 1 truncated, 2 first model failed
  // phase timers (dbg & 128): update | grid barrier | monitor gather + control | band wait | contraction
  const bool tim = kPathTimers && (P.dbg & 128) && threadIdx.x == 0 && (s == 0 || s == static_cast<int>(nb) / 2);
  long long ph[5] = {0, 0, 0, 0, 0}, tc = clock64(), nsteps = 0;
  auto mark = [&](int i) {
    if (tim) {
      const long long now = clock64();
      ph[i] += now - tc;
      tc = now;
    }
  };
  for (int t = 0; t < P.n_lambda && !stop; ++t) {
    const double lam = P.lambdas[t];
    const double j_th = penalty_of(A.pen, A.alpha, tl1, tl2);
    const double f_cur = -(tb - 0.5 * w * tst) / n + lam * j_th;
    for (int e = tx; e < q; e += BS) {
      xs[e] = xps[e] = bst[e] = th[e];
      sxs[e] = sxps[e] = sbst[e] = sth[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      cs = *tmpl;
      cs.lambda = lam;
      // inner_objective(x_0) = (w<x0,S'x0> - 2<x0,b> + sum v z^2)/(2n) + lambda J(x_0)
      const double g0 = 0.5 * (w * tst - 2.0 * tb + c0) / n + lam * j_th;
      ctl_setup(cs, g0, w);
    }
    __syncthreads();
    if (CW && !bt_div && !cs.done) {
      // nu = 1 with a control warp.  Workers: update -> arrive(1) -> wait for
      // the band (issued by the control warp once the grid barrier passed) ->
      // contract -> sync(2) for the monitor decision of step k-1.  Control warp:
      // sync(1) -> grid barrier -> band copy -> gather + ctl_step of step k-1 ->
      // arrive(2).  The decision therefore overlaps the band copy and the
      // contraction instead of preceding them; the iterates and decisions are
      // those of the single-role loop below.
      const double delta = cs.delta, gamma = __dmul_rn(delta, lam);
      const bool flagbar = nb <= kFlagCTAs && !(P.dbg & 64);
      if (threadIdx.x >= BS) {
        // control iteration k: (a) workers' x_k and the per-thread partials of
        // step k-1 are in place; (b) reduce those into this CTA's partials of
        // k-1 (four buffers by k mod 4); (c) release flag[s] = gen, which
        // publishes x_k and the partials; (d) wait for the flags of the
        // neighbour slabs this CTA's Gram band reads (the same CTAs read this
        // slab: the band is symmetric), then bulk-copy the band; (e) wait for
        // every flag of step k-1 (all partials of k-2 are published), gather
        // them and advance the replicated control block; (f) hand the decision
        // of step k-2 to the workers.  Only (d) is on the workers' critical
        // path; (e) waits on flags released a step earlier.
        const int lane = threadIdx.x & 31;
        const int nact = BS;  // rbuf entries (the deferred contractions write all of them)
        bool done = false;
        const bool ctim = kPathTimers && (P.dbg & 512) && lane == 0 && (s == 0 || s == static_cast<int>(nb) / 2);
        long long cph[4] = {0, 0, 0, 0}, cst = 0, cta_ = 0;
        auto cmark = [&](int i) {
          if (ctim) {
            const long long now = clock64();
            cph[i] += now - cta_;
            cta_ = now;
          }
        };
        // all flags in [r0_, r1_) reach g_.  A lane with several flags polls
        // them with relaxed loads (an acquire load would serialise them: one
        // L2 round trip each) and the acquire is one fence after success.
        auto poll = [&](int r0_, int r1_, unsigned g_, int nap) {
          const long long w0 = clock64();
          const bool multi = r1_ - r0_ > 32;
          for (;; __nanosleep(nap)) {
            bool mine = true;
            for (int r = r0_ + lane; r < r1_; r += 32) {
              unsigned f;
              if (multi)
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(P.flags + kFlagStride * r) : "memory");
              else
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(P.flags + kFlagStride * r) : "memory");
              mine = mine && f >= g_;
            }
            if (__all_sync(0xffffffffu, mine)) {
              if (multi) asm volatile("fence.acq_rel.gpu;" ::: "memory");
              break;
            }
            if (clock64() - w0 > async::kWatchdogCycles) {
              if (lane == 0) printf("kg watchdog: slab flags (block %d, generation %u)\n", s, g_);
              __trap();
            }
          }
        };
        for (i64 k = 1; !done; ++k) {
          double* Xk = P.X + (k & 1) * p;
          named_sync<1, BS + 32>();  // every worker's x_k (and step k-1's partials) is written
          long long w1_ = 0;
          if ((kPathTimers && (P.dbg & 65536)) && lane == 0) w1_ = *reinterpret_cast<volatile long long*>(&tw1);
          if (ctim) cta_ = clock64();
          ++cst;
          ++gen;
          if (k >= 2) {
            double r0 = 0.0, r1 = 0.0, r2 = 0.0;  // fixed order: lane-strided, then the warp tree
            for (int i = lane; i < nact; i += 32) {
              r0 += rbuf[i];
              r1 += rbuf[BS + i];
              r2 += rbuf[2 * BS + i];
            }
            r0 = warp_sum(r0);
            r1 = warp_sum(r1);
            r2 = warp_sum(r2);
            if (lane == 0) {
              double* dst = P.part + ((k - 1) % 4) * 3 * static_cast<i64>(nb);
              dst[s] = r0;
              dst[nb + s] = r1;
              dst[2 * nb + s] = r2;
            }
          }
          if (lane == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.flags + kFlagStride * s), "r"(gen) : "memory");
          cmark(0);
          poll(lo, lo + len, gen, 0);
          cmark(1);
          if ((kPathTimers && (P.dbg & 65536)) && lane == 0) {
            const long long now = clock64();
            dph[0] += now - w1_;
            tc1 = now;
          }
          if (direct)
            named_arrive<4, BS + 32>();  // the neighbours' x_k is published: workers read it from L2
          else if (lane == 0)
            issue_now(Xk);
          if ((kPathTimers && (P.dbg & 65536)) && lane == 0) {
            tc2 = clock64();
            dph[1] += tc2 - tc1;
          }
          if (k >= 3) {
            // monitor of step k-2: its partials were published with flag k-1,
            // which every CTA released about one step ago
            poll(0, static_cast<int>(nb), gen - 1, (P.dbg >> 20) ? (P.dbg >> 20) - 1 : kMonitorNap);
            const double* pp = P.part + ((k - 2) % 4) * 3 * static_cast<i64>(nb);
            double a = 0.0, b = 0.0, c = 0.0;  // objective partials of step k-2
#pragma unroll
            for (int i = 0; i < kPollRows; ++i) {
              const int r = lane + 32 * i;
              if (r < static_cast<int>(nb)) {
                a += __ldcg(pp + r);
                b += __ldcg(pp + nb + r);
                c += __ldcg(pp + 2 * nb + r);
              }
            }
            cmark(2);
            a = warp_sum(a);
            b = warp_sum(b);
            c = warp_sum(c);
            if (lane == 0) ctl_step(cs, 0.5 * (a + c0) / n + lam * penalty_of(A.pen, A.alpha, b, c));
          }
          __syncwarp();
          done = cs.done;
          cmark(3);
          named_arrive<2, BS + 32>();  // decision of step k-2 (or none at k < 3) is in cs
        }
        if (ctim && (t == 5 || t == 20))
          printf("ctl cta %d lambda %d: %lld steps, cycles/step: reduce+release %lld neighbours %lld monitor wait+gather %lld control %lld\n", s,
                 t, cst, cph[0] / cst, cph[1] / cst, cph[2] / cst, cph[3] / cst);
      } else {
        for (i64 k = 1;; ++k) {
          const double omega =
              extrapolation == 0 ? static_cast<double>(k - 1) / static_cast<double>(k + 2) : 0.0;
          double* Xk = P.X + (k & 1) * p;
          mark(4);
          double ul1 = 0.0, ul2 = 0.0;
          for (int e = tx; e < q; e += BS) {
            const double xi = xs[e], xpi = xps[e], sxi = sxs[e], sxpi = sxps[e];
            const double yi = xi + omega * (xi - xpi);
            const double syi = sxi + omega * (sxi - sxpi);
            const double g = fma(wn, syi, -bn[e]);  // = -b/n exactly at S'y = 0 (the lambda_max step)
            double ci = __dsub_rn(yi, __dmul_rn(delta, g));
            if (lam > 0.0) ci = prox1(A.pen, A.alpha, gamma, ci);
            ul1 += fabs(ci);
            ul2 = fma(ci, ci, ul2);
            xpp[e] = xpi;
            sxpp[e] = sxpi;
            xps[e] = xi;
            xs[e] = ci;
            sxps[e] = sxi;
            Xk[base + e] = ci;
          }
          mark(0);
          ++nsteps;
          if ((kPathTimers && (P.dbg & 65536)) && threadIdx.x == 0) tw1 = clock64();
          named_arrive<1, BS + 32>();
          if (direct) {
            named_sync<4, BS + 32>();
          } else {
            async::mbar_wait(&mb, parity);
            parity ^= 1u;
          }
          if ((kPathTimers && (P.dbg & 65536)) && threadIdx.x == 0) {
            const long long now = clock64();
            if (k >= 2) {
              dph[2] += now - tc2;
              dph[3] += now - tw1;
            }
          }
          mark(3);
          if (fused) {
            compute_fused(Xk, ul1, ul2);  // partials stay in rbuf for the control warp
          } else {
            compute(Xk, nullptr, 0, 0, true);
          }
          mark(4);
          named_sync<2, BS + 32>();
          mark(2);
          if (cs.copy_best) {  // best := x_{k-2} (in the x_prev_prev slot)
            for (int e = tx; e < q; e += BS) {
              bst[e] = xpp[e];
              sbst[e] = sxpp[e];
            }
          }
          if (cs.done) break;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) cs.copy_best = 0;  // applied above
      __syncthreads();
    }
    if (!CW && !bt_div) {
      // nu = 1 (no restarts): x_k depends only on earlier iterates, omega_k =
      // (k-1)/(k+2) and the fixed step, so the monitor decision of iteration
      // k-1 is taken one step late, after the single grid barrier of step k,
      // while the neighbour band of x_k is in flight.  X and the partials are
      // double-buffered by the parity of k.
      const double delta = cs.delta, gamma = __dmul_rn(delta, lam);
      for (i64 k = 1; !cs.done; ++k) {
        const double omega =
            extrapolation == 0 ? static_cast<double>(k - 1) / static_cast<double>(k + 2) : 0.0;
        double* Xk = P.X + (k & 1) * p;
        mark(4);
        for (int e = tx; e < q; e += BS) {
          const double xi = xs[e], xpi = xps[e], sxi = sxs[e], sxpi = sxps[e];
          const double yi = xi + omega * (xi - xpi);
          const double syi = sxi + omega * (sxi - sxpi);
          const double g = fma(wn, syi, -bn[e]);  // = -b/n exactly at S'y = 0 (the lambda_max step)
          double ci = __dsub_rn(yi, __dmul_rn(delta, g));
          if (lam > 0.0) ci = prox1(A.pen, A.alpha, gamma, ci);
          xps[e] = xi;
          xs[e] = ci;
          sxps[e] = sxi;
          Xk[base + e] = ci;
        }
        // arrival: all of this CTA's x_k is written (barrier), then one release of
        // the generation; warp 0 polls every CTA's flag (acquire) and, in the same
        // pass, that CTA's objective partials of step k-1 (component-major,
        // double-buffered by parity), so the grid barrier and the monitor gather
        // cost one round trip after the last arrival
        mark(0);
        ++nsteps;
        ++gen;
        const bool flagbar = nb <= kFlagCTAs && !(P.dbg & 64);  // flag barrier for small grids, atomic otherwise
        if (flagbar)
          __syncthreads();
        else
          grid_sync(P.bar, nb);
        if (threadIdx.x < 32) {
          const int lane = threadIdx.x;
          const double* pp = P.part + ((k - 1) & 1) * 3 * static_cast<i64>(nb);
          if (flagbar) {
            if (lane == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.flags + kFlagStride * s), "r"(gen) : "memory");
            const long long w0 = clock64();
            for (;;) {  // flags only: light polling while the slowest CTA finishes
              bool mine = true;
#pragma unroll
              for (int i = 0; i < kPollRows; ++i) {
                const int r = lane + 32 * i;
                if (r < static_cast<int>(nb)) {
                  unsigned f;
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(P.flags + kFlagStride * r) : "memory");
                  mine = mine && f >= gen;
                }
              }
              if (__all_sync(0xffffffffu, mine)) break;
              if (!(P.dbg & 256)) __nanosleep(20);
              if (clock64() - w0 > async::kWatchdogCycles) {
                if (lane == 0) printf("kg watchdog: flag barrier (block %d, generation %u)\n", s, gen);
                __trap();
              }
            }
          }
          if (lane == 0) mark(1);
          double a = 0.0, b = 0.0, c = 0.0;  // objective partials of step k-1 (after the barrier)
          if (k >= 2) {
#pragma unroll
            for (int i = 0; i < kPollRows; ++i) {
              const int r = lane + 32 * i;
              if (r < static_cast<int>(nb)) {
                a += __ldcg(pp + r);
                b += __ldcg(pp + nb + r);
                c += __ldcg(pp + 2 * nb + r);
              }
            }
          }
          __syncwarp();
          if (lane == 0) issue(Xk);
          if (k >= 2) {  // monitor iteration k-1: fixed-order sum (lane-ascending, then the warp tree)
            a = warp_sum(a);
            b = warp_sum(b);
            c = warp_sum(c);
            if (lane == 0) {
              const double gk = 0.5 * (a + c0) / n + lam * penalty_of(A.pen, A.alpha, b, c);
              ctl_step(cs, gk);
              if ((P.dbg & 8) && t < 2 && k < 8)
                printf("s=%d t=%d k=%lld g=%.17g done=%d\n", s, t, static_cast<long long>(k), gk, cs.done);
            }
          }
        }
        if (k >= 2) {
          __syncthreads();  // cs is read by every thread (written again only after the next barrier)
          if (cs.copy_best) {  // best := x_{k-1} (now in the x_prev slot; own elements only)
            for (int e = tx; e < q; e += BS) {
              bst[e] = xps[e];
              sbst[e] = sxps[e];
            }
          }
        }
        mark(2);
        async::mbar_wait(&mb, parity);  // always consume the copy (keeps the barrier phase)
        parity ^= 1u;
        mark(3);
        if (cs.done) break;
        compute(Xk, P.part + (k & 1) * 3 * static_cast<i64>(nb), static_cast<int>(nb), 1);
      }
      if (threadIdx.x == 0) cs.copy_best = 0;  // any pending copy was applied above
      __syncthreads();
    }
    while (!cs.done) {
      const double omega = cs.omega, delta = cs.delta;
      const int restart = cs.restart, copy_best = cs.copy_best;
      const double gamma = __dmul_rn(delta, lam);
      for (int e = tx; e < q; e += BS) {
        if (copy_best) {
          bst[e] = xs[e];
          sbst[e] = sxs[e];
        }
        if (restart) {
          xs[e] = xps[e] = bst[e];
          sxs[e] = sxps[e] = sbst[e];
        }
        const double xi = xs[e], xpi = xps[e], sxi = sxs[e], sxpi = sxps[e];
        const double yi = xi + omega * (xi - xpi);
        const double syi = sxi + omega * (sxi - sxpi);
        const double g = fma(wn, syi, -bn[e]);  // = -b/n exactly at S'y = 0 (the lambda_max step)
        double ci = __dsub_rn(yi, __dmul_rn(delta, g));
        if (lam > 0.0) ci = prox1(A.pen, A.alpha, gamma, ci);
        xps[e] = xi;
        xs[e] = ci;
        sxps[e] = sxi;
        P.X[base + e] = ci;
      }
      grid_sync(P.bar, nb);
      apply();
      grid_sync(P.bar, nb);
      double r[3];
      gather3(r);
      if (threadIdx.x == 0) ctl_step(cs, 0.5 * (r[0] + c0) / n + lam * penalty_of(A.pen, A.alpha, r[1], r[2]));
      __syncthreads();
    }
    // best := x if the last monitor left a copy pending (k_fista_finalize)
    double bb = 0.0, bsb = 0.0, bl1 = 0.0, bl2 = 0.0, tsb = 0.0;
    for (int e = tx; e < q; e += BS) {
      if (cs.copy_best) {
        bst[e] = xs[e];
        sbst[e] = sxs[e];
      }
      const double v = bst[e];
      bb += v * bs[e];
      bsb += v * sbst[e];
      bl1 += fabs(v);
      bl2 = fma(v, v, bl2);
      tsb += sth[e] * v;  // <S' theta, best> for Delta_k
    }
    double r[3];
    reduce3(bb, bsb, bl1, r);
    const double rl2 = cta_sum<BS>(bl2, red);
    const double rts = cta_sum<BS>(tsb, red);
    if (threadIdx.x == 0) {
      P.part2[5 * s] = r[0];
      P.part2[5 * s + 1] = r[1];
      P.part2[5 * s + 2] = r[2];
      P.part2[5 * s + 3] = rl2;
      P.part2[5 * s + 4] = rts;
    }
    grid_sync(P.bar, nb);
    double g4[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < 5; ++k) {
      double a = 0.0;
      for (int rr = tx; rr < static_cast<int>(nb); rr += BS) a += __ldcg(P.part2 + 5 * rr + k);
      g4[k] = cta_sum<BS>(a, red);
    }
    // Delta_k = -<u(eta), eta_t - eta>/n + lambda (J(best) - J(theta)) with
    // X^T u(eta) = b - w S' theta: <b - w S' theta, best - theta>
    const double dk = -((g4[0] - tb) - w * (g4[4] - tst)) / n +
                      lam * (penalty_of(A.pen, A.alpha, g4[2], g4[3]) - j_th);
    if (s == 0 && threadIdx.x == 0 && P.dk_out) {
      P.dk_out[2 * t] = dk;
      P.dk_out[2 * t + 1] = f_cur;
    }
    const int status = cs.converged ? KG_S_CONVERGED : (cs.diverged ? KG_S_INNER_DIVERGENCE : KG_S_MAX_ITERATIONS);
    double f = f_cur;
    if (!cs.diverged) {
      const double f_new = -(g4[0] - 0.5 * w * g4[1]) / n + lam * penalty_of(A.pen, A.alpha, g4[2], g4[3]);
      if (f_new <= f_cur) {  // outer.cpp:216-219
        for (int e = tx; e < q; e += BS) {
          th[e] = bst[e];
          sth[e] = sbst[e];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          tb = g4[0];
          tst = g4[1];
          tl1 = g4[2];
          tl2 = g4[3];
        }
        f = f_new;
      }
    }
    if (status != KG_S_CONVERGED) {
      stop = t == 0 ? 2 : 1;
      if (s == 0 && threadIdx.x == 0) {
        P.status_out[t] = status;
        P.iters_out[t] = cs.iterations;
      }
    } else {
      for (int e = tx; e < q; e += BS) P.coefs[static_cast<i64>(t) * p + base + e] = th[e];
      if (s == 0 && threadIdx.x == 0) {
        P.obj_out[t] = f;
        P.iters_out[t] = cs.iterations;
        P.status_out[t] = status;
        P.nmodels[0] = t + 1;
      }
    }
    __syncthreads();
  }
  if (s == 0 && threadIdx.x == 0) {
    P.nmodels[1] = stop;
    *A.ctl = cs;
  }
  if ((kPathTimers && (P.dbg & 65536)) && threadIdx.x == 0 && (s == 0 || s == static_cast<int>(nb) / 2) && nsteps > 0)
    printf("cta %d cycles/step: arrive->barrier done %lld, copy issue %lld, copy latency %lld, arrive->band %lld\n", s,
           dph[0] / nsteps, dph[1] / nsteps, dph[2] / nsteps, dph[3] / nsteps);
  if (tim && nsteps > 0)
    printf("k_gauss_path cta %d: %lld steps, cycles/step: update %lld barrier %lld monitor %lld band %lld contract %lld\n", s,
           nsteps, ph[0] / nsteps, ph[1] / nsteps, ph[2] / nsteps, ph[3] / nsteps, ph[4] / nsteps);
}

static size_t path_smem(const GramStepArgs& A) {
  size_t staged = 0;  // staged Gram bands of modes 0 .. d-2
  for (int j = 0; j < A.d - 1; ++j) staged += static_cast<size_t>(A.dims[j]) * (kPathTaps * sizeof(double) + 2 * sizeof(int));
  const size_t dense = path_mm(A) ? 2 * kMmLD * 32 : 0;  // padded G_0, G_1
  return (static_cast<size_t>(12 + A.Gd.maxlen) * A.q + 3 * static_cast<size_t>(path_qb(A)) + 4 + dense) *
             sizeof(double) +
         staged;
}

// KG_PATH_CW=0 drops the control warp (single-role nu = 1 loop)
static bool path_cw() {
  static const bool cw = [] {
    const char* e = dev_env("KG_PATH_CW");
    return e ? e[0] != '0' : kPathCW;
  }();
  return cw;
}

// CTA width of k_gauss_path: more threads per slab shorten each FISTA step's
// dependent chain (fewer elements per thread, more warps to hide smem and FMA
// latency); KG_PATH_BS overrides
static int path_bs() {
  static const int bs = [] {
    const char* e = dev_env("KG_PATH_BS");
    const int v = e ? std::atoi(e) : kPathBS;
    if (v == 1024 && path_cw()) return 512;  // 1024 + the control warp exceeds the CTA limit
    if (v == 480 && !path_cw()) return 512;
    return (v == 256 || v == 480 || v == 512 || v == 1024) ? v : kPathBS;
  }();
  return bs;
}

struct PathVariant {
  const void* fn;
  int threads;
};

static PathVariant path_variant(bool cw, int bs) {
  if (cw) {
    if (bs == 480) return {reinterpret_cast<const void*>(k_gauss_path<480, true>), 512};
    if (bs == 512) return {reinterpret_cast<const void*>(k_gauss_path<512, true>), 544};
    return {reinterpret_cast<const void*>(k_gauss_path<256, true>), 288};
  }
  if (bs == 1024) return {reinterpret_cast<const void*>(k_gauss_path<1024, false>), 1024};
  if (bs == 512) return {reinterpret_cast<const void*>(k_gauss_path<512, false>), 512};
  return {reinterpret_cast<const void*>(k_gauss_path<256, false>), 256};
}

// The configured variant when its grid (one CTA per slab) is co-resident,
// otherwise the narrow single-role variant (two CTAs per SM: C4's 256 slabs);
// threads == 0 when neither fits.
static PathVariant pick_variant(const GramStepArgs& A) {
  const size_t sm = path_smem(A);
  int dev = 0, nsm = 0;
  KG_CUDA(cudaGetDevice(&dev));
  KG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const PathVariant cands[2] = {path_variant(path_cw(), path_bs()), path_variant(false, 256)};
  for (const PathVariant& v : cands) {
    smem_attr(v.fn, 210 * 1024);
    int per_sm = 0;
    KG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn, v.threads, sm));
    if (static_cast<i64>(per_sm) * nsm >= A.pd) return v;
  }
  return {nullptr, 0};
}

bool gauss_path_ok(const GramStepArgs& A) {
  const size_t sm = path_smem(A);
  if (sm > 200 * 1024 || A.pd > 32 * kPollRows) return false;  // the flag barrier polls <= 320 CTAs
  return pick_variant(A).threads > 0;
}

void gauss_path(const Launch& L, const PersistArgs& P) {
  const size_t sm = path_smem(P.g);
  const PathVariant v = pick_variant(P.g);
  PersistArgs args = P;
  void* kargs[] = {&args};
  KG_CUDA(cudaLaunchCooperativeKernel(v.fn, dim3(static_cast<unsigned>(P.g.pd)), dim3(v.threads), kargs, sm, L.s));
  launched(L);
}

static size_t persist_smem(const GramStepArgs& A) {
  return (static_cast<size_t>(10 + A.Gd.maxlen) * A.q + 4) * sizeof(double);
}

bool fista_persist_ok(const GramStepArgs& A) {
  const size_t sm = persist_smem(A);
  if (sm > 200 * 1024) return false;
  smem_attr(k_fista_persist<256>, 210 * 1024);
  int per_sm = 0, dev = 0, nsm = 0;
  KG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fista_persist<256>, 256, sm));
  KG_CUDA(cudaGetDevice(&dev));
  KG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  return static_cast<i64>(per_sm) * nsm >= A.pd;
}

void fista_persist(const Launch& L, const PersistArgs& P) {
  const size_t sm = persist_smem(P.g);
  PersistArgs args = P;
  void* kargs[] = {&args};
  KG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_fista_persist<256>),
                                      dim3(static_cast<unsigned>(P.g.pd)), dim3(256), kargs, sm, L.s));
  launched(L);
}

// Gaussian constant-weight bookkeeping in p-space (outer.cpp:197-231 via
// eta = X theta): per-CTA partials of
//   0 <th,b>  1 <th,S th>  2 <bt,b>  3 <bt,S bt>  4 <b - w S th, bt - th>
//   5,6 (l1, l2) of bt   7,8 (l1, l2) of th
__global__ void __launch_bounds__(NT) k_gauss_dots(i64 p, double w, const double* th, const double* Sth,
                                                   const double* bt, const double* Sbt, const double* b,
                                                   double* part) {
  __shared__ double red[33];
  double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (i64 i = static_cast<i64>(blockIdx.x) * NT + threadIdx.x; i < p; i += static_cast<i64>(gridDim.x) * NT) {
    const double t = th[i], st = Sth[i], u = bt[i], su = Sbt[i], bb = b[i];
    a[0] += t * bb;
    a[1] += t * st;
    a[2] += u * bb;
    a[3] += u * su;
    a[4] += (bb - w * st) * (u - t);
    a[5] += fabs(u);
    a[6] = fma(u, u, a[6]);
    a[7] += fabs(t);
    a[8] = fma(t, t, a[8]);
  }
  for (int k = 0; k < 9; ++k) {
    const double r = cta_sum(a[k], red);
    if (threadIdx.x == 0) part[9 * static_cast<i64>(blockIdx.x) + k] = r;
  }
}

int gauss_dots(const Launch& L, i64 p, double w, const double* th, const double* Sth, const double* bt,
               const double* Sbt, const double* b, double* part) {
  const int g = static_cast<int>(std::min<i64>(std::max<i64>((p + 1023) / 1024, 1), 296));
  k_gauss_dots<<<g, NT, 0, L.s>>>(p, w, th, Sth, bt, Sbt, b, part);
  launched(L);
  return g;
}

}  // namespace kg
