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

#include "kg_async.cuh"
#include "kg_internal.h"

namespace kg {

namespace {

constexpr int NT = 256;  // p-space reduction kernels

__device__ __forceinline__ double soft(double z, double g) {
  const double m = fabs(z) - g;
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
  const double n = c->n, lambda = c->lambda;
  const double g = 0.5 * (sd + c->ss_const) / n + lambda * penalty_of(A.pen, A.alpha, s1, s2);
  if (A.init) {  // fista_solve setup (inner.cpp:132-161)
    c->g_prev = g;
    c->best_g = g;
    const double wmax = w;  // every weight equals w
    c->bad_weights = !(wmax > 0.0);
    const double lip = wmax * c->lipfac / n;
    c->lip = lip;
    double dl = 1.0 / (fmax(c->nu, 1.0e-300) * lip);
    if (c->nu == 1.0) dl = 1.0 / lip;
    c->delta = dl;
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
    return;
  }
  const i64 it = c->it;
  c->copy_best = 0;
  c->restart = 0;
  c->prox_steps += 1;
  c->momentum += 1;
  c->iterations = it;
  const i64 me = c->monitor_every < 1 ? 1 : c->monitor_every;
  if ((it % me == 0) || it == c->max_iters) {
    bool div = !isfinite(g);
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
  if (A.use_handle) cudaGraphSetConditional(A.handle, c->done ? 0u : 1u);
}

bool gram_step_fits(i64 q) { return 3 * q * static_cast<i64>(sizeof(double)) <= 200 * 1024; }

void gram_step(const Launch& L, const GramStepArgs& A) {
  static bool attr = false;
  if (!attr) {
    KG_CUDA(cudaFuncSetAttribute(k_gram_apply<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    KG_CUDA(cudaFuncSetAttribute(k_gram_apply<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    attr = true;
  }
  const size_t base = 3 * static_cast<size_t>(A.q) * sizeof(double);
  const size_t staged = base + (static_cast<size_t>(A.Gd.maxlen + 1) * A.q + 4) * sizeof(double);
  if (staged <= 200 * 1024) {
    k_gram_apply<256, true><<<static_cast<unsigned>(A.pd), 256, staged, L.s>>>(A);
  } else {
    k_gram_apply<256, false><<<static_cast<unsigned>(A.pd), 256, base, L.s>>>(A);
  }
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
