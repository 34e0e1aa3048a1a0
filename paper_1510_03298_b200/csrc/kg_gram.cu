// One-kernel FISTA iteration for the constant-weight (Gram) route.
//
// With W = w I, X^T W X = w (x)_j X_j^T X_j (the reference's
// xtwx_apply_tensor with constant weight factors, design.cpp:153-177), so a
// FISTA step needs only p-space work.  k_gram_step does a whole iteration in
// one launch:
//   * CTA s owns slab s of the last coefficient mode (q = p_1..p_{d-1}
//     contiguous values).  S_new[:, s] = (G_{d-1..1}) sum_t G_d[s, t] x_new[:, t],
//     so the CTA recomputes the elementwise FISTA update (inner.cpp:163-187)
//     for every neighbour slab t in the band of G_d row s on the fly;
//   * iterates rotate through three buffers (x_{l+1} overwrites x_{l-2}), so
//     the redundant neighbour updates only ever read the previous two
//     iterates, never a slab another CTA is writing;
//   * per-CTA partials of w<x,S'x> - 2<x,b>, |x|_1 and |x|_2^2 feed the
//     objective; the last CTA to finish (atomic ticket) reduces them in fixed
//     order and runs the monitor / best / restart / stop logic of
//     fista_solve (inner.cpp:195-229), then sets the graph's while-condition.
#include <cfloat>

#include "kg_internal.h"

namespace kg {

namespace {

constexpr int NT = 256;

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
__device__ double cta_sum(double v, double* sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    double r = l < (NT >> 5) ? sh[l] : 0.0;
    r = warp_sum(r);
    if (l == 0) sh[32] = r;
  }
  __syncthreads();
  return sh[32];
}

// in-shared-memory mode-j contraction of a q-array with extents dims (all
// modes < d-1 keep their extent because G_j is square)
__device__ void smem_mode(const double* in, double* out, const int* dims, int nd, int j, const BandOp& op, int q) {
  int a = 1;
  for (int i = 0; i < j; ++i) a *= dims[i];
  const int K = dims[j];
  for (int e = threadIdx.x; e < q; e += NT) {
    const int al = e % a;
    const int rest = e / a;
    const int m = rest % K;
    const int be = rest / K;
    const int lo = __ldg(op.lo + m), len = __ldg(op.len + m);
    const double* c = op.coef + __ldg(op.off + m);
    const double* src = in + al + a * (lo + K * be);
    double s = 0.0;
    for (int t = 0; t < len; ++t) s = fma(__ldg(c + t), src[a * t], s);
    out[e] = s;
  }
}

}  // namespace

__global__ void __launch_bounds__(NT) k_gram_step(GramStepArgs A) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  __shared__ int am_last;
  FistaCtl* c = A.ctl;
  const int q = A.q;
  const int s = blockIdx.x;
  const i64 it = A.init ? 0 : c->it;
  const int cur = static_cast<int>((it + 2) % 3);  // x_{it-1}
  const int prv = static_cast<int>((it + 1) % 3);  // x_{it-2}
  const int nxt = static_cast<int>(it % 3);        // x_it
  const double omega = c->omega, delta = c->delta, lambda = c->lambda, n = c->n, w = c->sscale;
  const int restart = A.init ? 0 : c->restart, copy_best = A.init ? 0 : c->copy_best;
  const double gamma = delta * lambda;
  const double* Xc = A.X[cur];
  const double* Xp = A.X[prv];
  const double* Sc = A.S[cur];
  const double* Sp = A.S[prv];

  double* u = sm;           // sum_t G_d[s,t] x_new[:, t]
  double* t0 = sm + q;      // chain scratch
  double* t1 = sm + 2 * q;
  double* xs = sm + 3 * q;  // x_new[:, s]

  auto xnew = [&](i64 idx) -> double {
    if (A.init) return Xc[idx];
    double xi, xpi, sxi, sxpi;
    if (restart) {
      xi = xpi = A.best[idx];
      sxi = sxpi = A.Sbest[idx];
    } else {
      xi = Xc[idx];
      xpi = Xp[idx];
      sxi = Sc[idx];
      sxpi = Sp[idx];
    }
    const double yi = xi + omega * (xi - xpi);
    const double syi = sxi + omega * (sxi - sxpi);
    const double g = (w * syi - A.b[idx]) / n;
    double ci = yi - delta * g;
    if (lambda > 0.0) ci = prox1(A.pen, A.alpha, gamma, ci);
    return ci;
  };

  // pending best copy from the previous monitor (owner slab only)
  if (copy_best) {
    for (int e = threadIdx.x; e < q; e += NT) {
      const i64 idx = static_cast<i64>(s) * q + e;
      A.best[idx] = Xc[idx];
      A.Sbest[idx] = Sc[idx];
    }
  }
  // restart (inner.cpp:207-216): x = x_prev = best.  This step reads best
  // instead of the cur/prv buffers, and the cur buffer becomes the next
  // step's x_prev, so the owner slab of cur is overwritten with best.
  if (restart) {
    for (int e = threadIdx.x; e < q; e += NT) {
      const i64 idx = static_cast<i64>(s) * q + e;
      A.X[cur][idx] = A.best[idx];
      A.S[cur][idx] = A.Sbest[idx];
    }
  }
  const int lo = __ldg(A.Gd.lo + s), len = __ldg(A.Gd.len + s);
  const double* gc = A.Gd.coef + __ldg(A.Gd.off + s);
  for (int e = threadIdx.x; e < q; e += NT) {
    double acc = 0.0;
    for (int t = 0; t < len; ++t) {
      const int sl = lo + t;
      const double xn = xnew(static_cast<i64>(sl) * q + e);
      acc = fma(__ldg(gc + t), xn, acc);
      if (sl == s) xs[e] = xn;
    }
    if (s < lo || s >= lo + len) xs[e] = xnew(static_cast<i64>(s) * q + e);
    u[e] = acc;
  }
  __syncthreads();
  // S'_new[:, s] = (G_{d-2} .. G_0 applied to u)
  const double* res = u;
  double* bufs[2] = {t0, t1};
  int which = 0;
  for (int j = A.d - 2; j >= 0; --j) {
    smem_mode(res, bufs[which], A.dims, A.d - 1, j, A.G[j], q);
    __syncthreads();
    res = bufs[which];
    which ^= 1;
  }
  double dots = 0.0, l1 = 0.0, l2 = 0.0;
  double* Xn = A.X[nxt];
  double* Sn = A.S[nxt];
  for (int e = threadIdx.x; e < q; e += NT) {
    const i64 idx = static_cast<i64>(s) * q + e;
    const double xv = xs[e], sv = res[e];
    Xn[idx] = xv;
    Sn[idx] = sv;
    if (A.init) {  // x_{-1} := x_0, S_{-1} := S_0, best := x_0
      A.X[2][idx] = xv;
      A.S[2][idx] = sv;
      A.best[idx] = xv;
      A.Sbest[idx] = sv;
    }
    dots += xv * (w * sv - 2.0 * A.b[idx]);
    l1 += fabs(xv);
    l2 = fma(xv, xv, l2);
  }
  dots = cta_sum(dots, red);
  l1 = cta_sum(l1, red);
  l2 = cta_sum(l2, red);
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
  // ---- last CTA: fixed-order reduction of the partials + control
  double sd = 0.0, s1 = 0.0, s2 = 0.0;
  for (int r = threadIdx.x; r < static_cast<int>(gridDim.x); r += NT) {
    sd += __ldcg(A.part + 3 * r);
    s1 += __ldcg(A.part + 3 * r + 1);
    s2 += __ldcg(A.part + 3 * r + 2);
  }
  sd = cta_sum(sd, red);
  s1 = cta_sum(s1, red);
  s2 = cta_sum(s2, red);
  if (threadIdx.x != 0) return;
  *A.counter = 0u;
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

bool gram_step_fits(i64 q) { return 4 * q * static_cast<i64>(sizeof(double)) <= 200 * 1024; }

void gram_step(const Launch& L, const GramStepArgs& A) {
  static bool attr = false;
  if (!attr) {
    KG_CUDA(cudaFuncSetAttribute(k_gram_step, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    attr = true;
  }
  const size_t sm = 4 * static_cast<size_t>(A.q) * sizeof(double);
  k_gram_step<<<static_cast<unsigned>(A.pd), NT, sm, L.s>>>(A);
  if (L.counter) ++*L.counter;
}

// x_final = X[iterations % 3]; best := x_final (and Sbest) if the last monitor left a copy pending
__global__ void k_gram_finalize(const FistaCtl* c, i64 p, GramStepArgs A) {
  const int fin = static_cast<int>(c->iterations % 3);
  if (!c->copy_best) return;
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < p;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    A.best[i] = A.X[fin][i];
    A.Sbest[i] = A.S[fin][i];
  }
}

void gram_finalize(const Launch& L, const FistaCtl* ctl, i64 p, const GramStepArgs& A) {
  k_gram_finalize<<<static_cast<unsigned>(std::min<i64>((p + 255) / 256, 1184)), 256, 0, L.s>>>(ctl, p, A);
  if (L.counter) ++*L.counter;
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
  if (L.counter) ++*L.counter;
  return g;
}

}  // namespace kg
