// Slab pass: modes 1 AND 2 of one n-space FISTA step, fused per slice of the
// last mode (d = 3, one component, FV_FISTA_EXP objective).
//
// Per FISTA step the n-space route needs S(x) = X^T diag(v) X x
// (design.cpp:118-124, xtwx_apply).  With the mode-3 H partial
// S3 = x x_3 X3 (p1 x p2 x n3) and the slice-local maps
//     eta(:, :, i3) = X1 S3(:, :, i3) X2^T,    w = v .* eta,
//     Q3(:, :, i3)  = X1^T w(:, :, i3) X2,
// S(x) = Q3 x_3 X3^T, so the only n-sized traffic of a step is one read of v
// (the p1 x n2 x n3 partials of the mode-1 route never touch HBM).
//
// Three kernels, all one persistent CTA per SM with 8 "row" warps (eta, w,
// sum v eta^2 per 4 x 2 cells, coefficient windows in registers) and 8
// "tensor" warps (U, Y -> Z, Q3; DMMA m8n8k4) pipelined over chunks of 8
// mode-2 grid rows:
//   * k_slab4 (the default; whole chunk pairs): Y by scatter/gather of the row
//     threads' window partials, v by cp.async.bulk into a shared ring, S3
//     operands straight from L2, mbarrier hand-over in chunk pairs, chunk
//     tables in shared memory, setmaxnreg per role;
//   * k_slab2 (odd chunk counts, partial last chunks): the same scatter/gather
//     with v staged through registers and the S3 tile by bulk copies;
//   * k_slab (designs without a gather table): Y = X1^T w by DMMA over the band
//     window (A fragments in registers, w through a padded shared tile), named
//     barriers.
// In all three Z += Y X2 uses Y's accumulator layout as the A layout of the
// next DMMA (the k index runs over the chunk's rows as 0,2,4,6 | 1,3,5,7) and
// Z lives in a two-tile register window that slides with the chunk's
// coefficient window; completed tiles go straight to Q3.  Every reduction has
// a fixed order.
#include <algorithm>
#include <cstdlib>

#include "kg_async.cuh"
#include "kg_internal.h"

namespace kg {

namespace {

constexpr int kSlabBS = 512;     // row warps + tensor warps
constexpr int kTeam = 256;      // threads per role

__device__ __forceinline__ double warp_sum_s(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}


__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

constexpr int kLdr = 10;  // row stride of the row-major U tile (10 doubles: conflict-free 16-byte row reads)

// named barriers (0 is __syncthreads): U ready (tensor -> row warps) and
// w ready (row -> tensor warps), one per pipeline buffer
constexpr int kDepth = 4;  // U and w buffers: the row warps may run up to kDepth chunks ahead
constexpr int kBarUReady = 1, kBarWReady = 1 + kDepth, kBarTensor = 1 + 2 * kDepth;

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ double2 ldg2_stream(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

constexpr int kWin = 5;  // coefficient window of a row quad (cubic B-splines: 4 taps, shifting by <= 1)

// KS: k-steps of the X1^T window.
template <int KS>
__global__ void __launch_bounds__(kSlabBS, 1) k_slab(SlabArgs a) {
  using namespace async;
  extern __shared__ __align__(128) double sm[];
  __shared__ double red[32];
  __shared__ unsigned long long sbar[2];     // the two S3 tiles
  const int n1 = a.n1, n2 = a.n2, p1 = a.p1, p2 = a.p2, nch = a.nch;
  const int ldS = a.ldS, ldW = a.ldW;
  const int groups = (p1 + 7) >> 3;
  const int sbuf = ldS * p2;                  // one S3 tile
  const int ubuf = kLdr * 8 * groups;         // one U tile (row-major, rows of p1 padded to the row groups)
  const int wbuf = ldW * 8;                   // one w tile
  double* Ss = sm;                            // [2][ldS x p2]
  double* Us = Ss + 2 * sbuf;                 // [kDepth][ubuf]
  double* Ws = Us + kDepth * ubuf;            // [kDepth][wbuf]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool rowrole = warp < 8;
  const i64 p12 = static_cast<i64>(p1) * p2, n12 = static_cast<i64>(n1) * n2;
  const int rounds = static_cast<int>((a.m3 - blockIdx.x + gridDim.x - 1) / gridDim.x);  // slices of this CTA
  const int qtot = rounds * nch;
  // the S3 tile of round r (p2 padded column copies by the bulk engine)
  auto issue_s = [&](int r) {
    if (r >= rounds) return;
    const unsigned bytes = static_cast<unsigned>(p1 * 8);
    mbar_expect_tx(&sbar[r & 1], bytes * p2);
    const double* src = a.S + (blockIdx.x + static_cast<i64>(r) * gridDim.x) * p12;
    double* dst = Ss + (r & 1) * sbuf;
    for (int k = 0; k < p2; ++k) bulk_g2s(dst + ldS * k, src + static_cast<i64>(p1) * k, bytes, &sbar[r & 1]);
  };
  if (tid == 0) {
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
  }
  // zero both S3 tiles (their padded rows are read by the last row group)
  for (int k = tid; k < 2 * sbuf; k += kSlabBS) Ss[k] = 0.0;
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0;
  if (rowrole) {
    // ------------------------------------------------------------ row warps
    const int nq = n1 >> 2;                    // row quads
    const bool act = tid < 4 * nq;
    const int rq = act ? tid % nq : 0, cp = act ? tid / nq : 0;
    const int r0 = 4 * rq, c0 = 2 * cp;        // rows r0 .. r0 + 3, chunk columns c0, c0 + 1
    int lo = 0;
    double C[4][kWin];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < kWin; ++t) C[r][t] = 0.0;
    if (act) {
      lo = min(__ldg(a.H1.lo + r0), p1 - kWin);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int l = __ldg(a.H1.lo + r0 + r), len = __ldg(a.H1.len + r0 + r);
        const double* cf = a.H1.coef + __ldg(a.H1.off + r0 + r);
#pragma unroll
        for (int t = 0; t < kWin; ++t) {
          const int j = lo + t - l;
          C[r][t] = (j >= 0 && j < len) ? __ldg(cf + j) : 0.0;
        }
      }
    }
    const double* ub0 = Us + lo * kLdr + c0;
    double* wb0 = Ws + r0 + ldW * c0;
    // v of chunk (round, chunk): rows r0 .. r0 + 3 of columns c0, c0 + 1 (zeros past n2)
    const double* vbase = a.v + blockIdx.x * n12 + r0;
    const i64 vstep = static_cast<i64>(gridDim.x) * n12;
    auto load_v = [&](double (&vr)[8], int r, int c) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * c + c0 + e;
        if (act && r < rounds && col < n2) {
          const double* p = vbase + r * vstep + static_cast<i64>(n1) * col;
          const double2 x = ldg2_stream(p), y = ldg2_stream(p + 2);
          vr[4 * e + 0] = x.x;
          vr[4 * e + 1] = x.y;
          vr[4 * e + 2] = y.x;
          vr[4 * e + 3] = y.y;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) vr[4 * e + k] = 0.0;
        }
      }
    };
    double vA[8], vB[8];
    int lr = 0, lc = 0;  // cursor of the next chunk to load
    auto adv = [&](int& r, int& c) {
      if (++c == nch) {
        c = 0;
        ++r;
      }
    };
    load_v(vA, lr, lc);
    adv(lr, lc);
    load_v(vB, lr, lc);
    adv(lr, lc);
    // chunk q: U(q) is ready (and the tensor warps are done with w(q - kDepth),
    // which they read before forming U(q)); w(q) -> tile q % kDepth
    auto body = [&](int q, double (&vr)[8]) {
      const int buf = q & (kDepth - 1);
      nb_sync(kBarUReady + buf, kSlabBS);
      if (act) {
        const double* u = ub0 + buf * ubuf;
        double2 uu[kWin];
#pragma unroll
        for (int t = 0; t < kWin; ++t) uu[t] = lds2(u + t * kLdr);
        double* w = wb0 + buf * wbuf;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          double wv[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            double x = C[r][0] * (c ? uu[0].y : uu[0].x);
#pragma unroll
            for (int t = 1; t < kWin; ++t) x = fma(C[r][t], c ? uu[t].y : uu[t].x, x);
            wv[r] = vr[4 * c + r] * x;
            if (r & 1) acc1 = fma(wv[r], x, acc1);
            else acc0 = fma(wv[r], x, acc0);
          }
          // quads 4 apart are 128 bytes apart: the upper half of the quad-group
          // stores its second 16 bytes first, so a quarter warp hits 8 distinct bank groups
          const bool sw = (rq >> 2) & 1;
          *reinterpret_cast<double2*>(w + ldW * c + (sw ? 2 : 0)) = sw ? make_double2(wv[2], wv[3]) : make_double2(wv[0], wv[1]);
          *reinterpret_cast<double2*>(w + ldW * c + (sw ? 0 : 2)) = sw ? make_double2(wv[0], wv[1]) : make_double2(wv[2], wv[3]);
        }
      }
      nb_arrive(kBarWReady + buf, kSlabBS);
      load_v(vr, lr, lc);  // two chunks ahead
      adv(lr, lc);
    };
    int q = 0;
    for (; q + 1 < qtot; q += 2) {
      body(q, vA);
      body(q + 1, vB);
    }
    if (q < qtot) body(q, vA);
  } else {
    // --------------------------------------------------------- tensor warps
    const int tw = warp - 8;
    const bool gact = tw < groups;            // this warp owns p1 rows 8 tw .. 8 tw + 7
    const bool leader = tid == 8 * 32;
    const int zr = 8 * tw + (lane >> 2), zq = 2 * (lane & 3);
    double* ua0 = Us + zr * kLdr + zq;        // stage A D store (buffer 0)
    int gbase = 0;
    double afr[KS];
#pragma unroll
    for (int s = 0; s < KS; ++s) afr[s] = 0.0;
    if (gact) {
      gbase = __ldg(a.g1.base + tw);
#pragma unroll
      for (int s = 0; s < KS; ++s) afr[s] = __ldg(a.g1.afrag + (tw * KS + s) * 32 + lane);
    }
    const double* wc0 = Ws + gbase + (lane & 3) + ldW * (lane >> 2);  // B fragments of Y
    // flattened chunk cursors (round, chunk)
    struct Cur {
      int r, c;
    };
    auto adv = [&](Cur& k) {
      if (++k.c == nch) {
        k.c = 0;
        ++k.r;
      }
    };
    auto at_q = [&](int q) {  // only for the few prologue positions
      Cur k{0, 0};
      for (int i = 0; i < q; ++i) adv(k);
      return k;
    };
    if (leader) {
      mbar_init_fence();
      fence_proxy_async();
      issue_s(0);
      issue_s(1);
    }
    // chunk tables, loaded one chunk ahead of use
    struct ZT { int tz; double b0, b1, b2, b3; };
    struct AT { int wz; double b0, b1; };
    auto load_z = [&](int c) {
      ZT t;
      const double* x2 = a.x2z + c * 128;
      t.tz = __ldg(a.tz + c);
      t.b0 = __ldg(x2 + lane);
      t.b1 = __ldg(x2 + 32 + lane);
      t.b2 = __ldg(x2 + 64 + lane);
      t.b3 = __ldg(x2 + 96 + lane);
      return t;
    };
    auto load_a = [&](int c) {
      AT t;
      const double* x2 = a.x2u + c * 64;
      t.wz = __ldg(a.w0 + c);
      t.b0 = __ldg(x2 + lane);
      t.b1 = __ldg(x2 + 32 + lane);
      return t;
    };
    // U of chunk (r, c) into U buffer ub
    auto stage_a = [&](const Cur& k, int ub, const AT& t) {
      if (k.c == 0) mbar_wait(&sbar[k.r & 1], static_cast<unsigned>((k.r >> 1) & 1));
      if (!gact) return;
      const double* sr = Ss + (k.r & 1) * sbuf + zr + ldS * (t.wz + (lane & 3));
      double d0 = 0.0, d1 = 0.0;
      dmma(d0, d1, sr[0], t.b0);
      dmma(d0, d1, sr[4 * ldS], t.b1);
      *reinterpret_cast<double2*>(ua0 + ub * ubuf) = make_double2(d0, d1);
    };
    Cur ka{0, 0};  // U step cursor
    for (int q = 0; q < kDepth; ++q, adv(ka)) {
      if (q < qtot) {
        stage_a(ka, q, load_a(ka.c));
        nb_arrive(kBarUReady + q, kSlabBS);
      }
    }
    nb_sync(kBarTensor, kSlabBS - 256);
    if (leader)  // a round whose last U was just formed frees its S3 tile
      for (int q = 0; q < kDepth && q < qtot; ++q)
        if (at_q(q).c == nch - 1) issue_s(at_q(q).r + 2);
    Cur kz = at_q(1);              // Z tables: q + 1
    Cur kt = ka;                   // U tables: q + kDepth + 1
    adv(kt);
    // Z window: slot 0 = tile T, slot 1 = tile T + 1 (8 columns each) of the current slice
    int T = -1;
    double z00 = 0.0, z01 = 0.0, z10 = 0.0, z11 = 0.0;
    double* qs = a.Q + blockIdx.x * p12;
    const i64 qstep = static_cast<i64>(gridDim.x) * p12;
    auto flush = [&](int k, double x0, double x1) {
      const int zc = 8 * k + zq;
      if (zr < p1 && zc < p2) qs[zr + static_cast<i64>(p1) * zc] = x0;
      if (zr < p1 && zc + 1 < p2) qs[zr + static_cast<i64>(p1) * (zc + 1)] = x1;
    };
    ZT zt = load_z(0);
    AT at = load_a(ka.c);  // ka = kDepth
    int c = 0;
    for (int q = 0; q < qtot; ++q) {
      const int buf = q & (kDepth - 1);
      const ZT zn = load_z(kz.c);   // next chunk's Z tables
      const AT an = load_a(kt.c);   // and the U tables one further
      nb_sync(kBarWReady + buf, kSlabBS);
      if (gact) {
        const double* wb = wc0 + buf * wbuf;
        double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int s = 0; s < KS; s += 4) {
#pragma unroll
          for (int h = 0; h < 4; ++h) dmma(d[h][0], d[h][1], afr[s + h], wb[4 * (s + h)]);
        }
        const double y0 = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
        const double y1 = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
        const int t0 = zt.tz & 0xffff;
        if (T < 0) T = t0;
        while (T < t0) {  // tile T is complete: later chunks start at t0 > T
          flush(T, z00, z01);
          z00 = z10;
          z01 = z11;
          z10 = z11 = 0.0;
          ++T;
        }
        dmma(z00, z01, y0, zt.b0);
        dmma(z00, z01, y1, zt.b1);
        if (zt.tz >> 16) {
          dmma(z10, z11, y0, zt.b2);
          dmma(z10, z11, y1, zt.b3);
        }
        if (c == nch - 1) {  // slice done: the live window holds its last two tiles
          flush(T, z00, z01);
          flush(T + 1, z10, z11);
          z00 = z01 = z10 = z11 = 0.0;
          T = -1;
        }
      }
      // U(q + kDepth) into the buffer of chunk q (the row warps are done with it)
      if (q + kDepth < qtot) {
        stage_a(ka, buf, at);
        nb_arrive(kBarUReady + buf, kSlabBS);
        if (ka.c == nch - 1) {  // that round's S3 tile is free once every tensor warp formed its U
          nb_sync(kBarTensor, kSlabBS - 256);
          if (leader) {
            fence_proxy_async();
            issue_s(ka.r + 2);
          }
        }
      }
      adv(ka);
      adv(kz);
      adv(kt);
      zt = zn;
      at = an;
      if (++c == nch) {
        c = 0;
        qs += qstep;
      }
    }
  }
  // per-CTA partial of sum v eta^2 (fixed order)
  double rr = warp_sum_s(acc0 + acc1);
  __syncthreads();
  if (lane == 0) red[warp] = rr;
  __syncthreads();
  if (warp == 0) {
    rr = lane < (kSlabBS >> 5) ? red[lane] : 0.0;
    rr = warp_sum_s(rr);
    if (lane == 0) a.partial[blockIdx.x] = rr;
  }
}


// k_slab2: the same pass with Y = X1^T w in scatter/gather form instead of
// DMMA over the (35% dense) band window.  A row thread already holds the
// window coefficients C[r][t] of its 4 rows, so after w it also forms the five
// window partials sum_r C[r][t] w[r] of its two columns (40 FMAs, no extra
// operands) and stores them to slots 5 quad .. 5 quad + 4 of its column pair's
// plane; a tensor-warp lane (basis function k, column pair) sums the <= 8
// slots of the quads whose rows hold k (SlabArgs::gat, ascending quads: a
// fixed order), which lands Y directly in the A-fragment layout of the Z step.
// FP64-pipe time per chunk drops from ~800 to ~620 SM-cycles and the tensor
// warps' critical path from 12 to 0 Y DMMAs.
__global__ void __launch_bounds__(kSlabBS, 1) k_slab2(SlabArgs a) {
  using namespace async;
  extern __shared__ __align__(128) double sm[];
  __shared__ double red[32];
  __shared__ unsigned long long sbar[2];     // the two S3 tiles
  // the U / partial-tile hand-over goes through mbarriers (one arrival per warp),
  // so the warps of a role do not rendezvous per chunk
  __shared__ unsigned long long ubar[kDepth], wbar[kDepth];
  const int n1 = a.n1, n2 = a.n2, p1 = a.p1, p2 = a.p2, nch = a.nch;
  const int ldS = a.ldS, PL = a.PL;
  const int groups = (p1 + 7) >> 3;
  const int sbuf = ldS * p2;                  // one S3 tile
  const int ubuf = kLdr * 8 * groups;         // one U tile
  const int pbuf = 8 * PL;                    // one partial tile: 4 column-pair planes of PL double2 slots
  double* Ss = sm;                            // [2][ldS x p2]
  double* Us = Ss + 2 * sbuf;                 // [kDepth][ubuf]
  double* Ps = Us + kDepth * ubuf;            // [kDepth][pbuf]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool rowrole = warp < 8;
  const i64 p12 = static_cast<i64>(p1) * p2, n12 = static_cast<i64>(n1) * n2;
  const int rounds = static_cast<int>((a.m3 - blockIdx.x + gridDim.x - 1) / gridDim.x);  // slices of this CTA
  const int qtot = rounds * nch;
  auto issue_s = [&](int r) {
    if (r >= rounds) return;
    const unsigned bytes = static_cast<unsigned>(p1 * 8);
    mbar_expect_tx(&sbar[r & 1], bytes * p2);
    const double* src = a.S + (blockIdx.x + static_cast<i64>(r) * gridDim.x) * p12;
    double* dst = Ss + (r & 1) * sbuf;
    for (int k = 0; k < p2; ++k) bulk_g2s(dst + ldS * k, src + static_cast<i64>(p1) * k, bytes, &sbar[r & 1]);
  };
  if (tid == 0) {
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
    for (int k = 0; k < kDepth; ++k) {
      mbar_init(&ubar[k], 8);
      mbar_init(&wbar[k], 8);
    }
    mbar_init_fence();
  }
  for (int k = tid; k < 2 * sbuf; k += kSlabBS) Ss[k] = 0.0;
  if (tid < 4 * kDepth) {  // the zero slot of every plane
    Ps[2 * (tid * PL + PL - 1)] = 0.0;
    Ps[2 * (tid * PL + PL - 1) + 1] = 0.0;
  }
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0;
  if (rowrole) {
    // ------------------------------------------------------------ row warps
    const int nq = n1 >> 2;                    // row quads
    const bool act = tid < 4 * nq;
    const int rq = act ? tid % nq : 0, cp = act ? tid / nq : 0;
    const int r0 = 4 * rq, c0 = 2 * cp;        // rows r0 .. r0 + 3, chunk columns c0, c0 + 1
    int lo = 0;
    double C[4][kWin];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < kWin; ++t) C[r][t] = 0.0;
    if (act) {
      lo = min(__ldg(a.H1.lo + r0), p1 - kWin);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int l = __ldg(a.H1.lo + r0 + r), len = __ldg(a.H1.len + r0 + r);
        const double* cf = a.H1.coef + __ldg(a.H1.off + r0 + r);
#pragma unroll
        for (int t = 0; t < kWin; ++t) {
          const int j = lo + t - l;
          C[r][t] = (j >= 0 && j < len) ? __ldg(cf + j) : 0.0;
        }
      }
    }
    const double* ub0 = Us + lo * kLdr + c0;
    double2* pb0 = reinterpret_cast<double2*>(Ps) + cp * PL + rq * kWin;
    const double* vbase = a.v + blockIdx.x * n12 + r0;
    const i64 vstep = static_cast<i64>(gridDim.x) * n12;
    auto load_v = [&](double (&vr)[8], int r, int c) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * c + c0 + e;
        if (act && r < rounds && col < n2) {
          const double* p = vbase + r * vstep + static_cast<i64>(n1) * col;
          const double2 x = ldg2_stream(p), y = ldg2_stream(p + 2);
          vr[4 * e + 0] = x.x;
          vr[4 * e + 1] = x.y;
          vr[4 * e + 2] = y.x;
          vr[4 * e + 3] = y.y;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) vr[4 * e + k] = 0.0;
        }
      }
    };
    constexpr int VS = 2;  // v register stages (more are capped by the warp's scoreboards)
    double vv[VS][8];
    int lr = 0, lc = 0;  // cursor of the next chunk to load
    auto adv = [&](int& r, int& c) {
      if (++c == nch) {
        c = 0;
        ++r;
      }
    };
    // one thread pulls the v chunks a.pf ahead into L2 (a chunk is contiguous:
    // 8 columns of n1), so the register loads VS chunks ahead find them there
    int fr = 0, fc = 0;
    auto prefetch_v = [&]() {
      if (fr < rounds) {
        const int cols = min(8, n2 - 8 * fc);
        bulk_prefetch_l2(a.v + (blockIdx.x + static_cast<i64>(fr) * gridDim.x) * n12 + static_cast<i64>(n1) * 8 * fc,
                         static_cast<unsigned>(cols * n1 * 8));
      }
      adv(fr, fc);
    };
    const bool pfl = tid == 0 && a.pf > 0;
    if (pfl)
      for (int k = 0; k < a.pf; ++k) prefetch_v();
#pragma unroll
    for (int s = 0; s < VS; ++s) {
      load_v(vv[s], lr, lc);
      adv(lr, lc);
    }
    auto body = [&](int q, double (&vr)[8]) {
      const int buf = q & (kDepth - 1);
      if (pfl) prefetch_v();
      mbar_wait(&ubar[buf], static_cast<unsigned>(q / kDepth) & 1u);
      if (act) {
        const double* u = ub0 + buf * ubuf;
        double2 uu[kWin];
#pragma unroll
        for (int t = 0; t < kWin; ++t) uu[t] = lds2(u + t * kLdr);
        double pt[2][kWin];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            double x = C[r][0] * (c ? uu[0].y : uu[0].x);
#pragma unroll
            for (int t = 1; t < kWin; ++t) x = fma(C[r][t], c ? uu[t].y : uu[t].x, x);
            const double wv = vr[4 * c + r] * x;
            if (r & 1) acc1 = fma(wv, x, acc1);
            else acc0 = fma(wv, x, acc0);
#pragma unroll
            for (int t = 0; t < kWin; ++t) pt[c][t] = r == 0 ? C[0][t] * wv : fma(C[r][t], wv, pt[c][t]);
          }
        }
        double2* P = pb0 + buf * (pbuf >> 1);
#pragma unroll
        for (int t = 0; t < kWin; ++t) P[t] = make_double2(pt[0][t], pt[1][t]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&wbar[buf]);
      load_v(vr, lr, lc);  // VS chunks ahead
      adv(lr, lc);
    };
    int q = 0;
    for (; q + VS <= qtot; q += VS) {
#pragma unroll
      for (int s = 0; s < VS; ++s) body(q + s, vv[s]);
    }
#pragma unroll
    for (int s = 0; s < VS; ++s)
      if (q + s < qtot) body(q + s, vv[s]);
  } else {
    // --------------------------------------------------------- tensor warps
    const int tw = warp - 8;
    const bool gact = tw < groups;            // this warp owns p1 rows 8 tw .. 8 tw + 7
    const bool leader = tid == 8 * 32;
    const int zr = 8 * tw + (lane >> 2), zq = 2 * (lane & 3);
    double* ua0 = Us + zr * kLdr + zq;        // stage A D store (buffer 0)
    // gather slots of basis function zr (column pair lane & 3)
    int4 gs = make_int4(0, 0, 0, 0);
    if (gact) gs = __ldg(reinterpret_cast<const int4*>(a.gat) + zr);
    else gs.x = gs.y = gs.z = gs.w = (PL - 1) | ((PL - 1) << 16);
    const int gmax = a.gmax;
    const double2* pg0 = reinterpret_cast<const double2*>(Ps) + (lane & 3) * PL;
    struct Cur {
      int r, c;
    };
    auto adv = [&](Cur& k) {
      if (++k.c == nch) {
        k.c = 0;
        ++k.r;
      }
    };
    auto at_q = [&](int q) {  // only for the few prologue positions
      Cur k{0, 0};
      for (int i = 0; i < q; ++i) adv(k);
      return k;
    };
    if (leader) {
      mbar_init_fence();
      fence_proxy_async();
      issue_s(0);
      issue_s(1);
    }
    struct ZT { int tz; double b0, b1, b2, b3; };
    struct AT { int wz; double b0, b1; };
    auto load_z = [&](int c) {
      ZT t;
      const double* x2 = a.x2z + c * 128;
      t.tz = __ldg(a.tz + c);
      t.b0 = __ldg(x2 + lane);
      t.b1 = __ldg(x2 + 32 + lane);
      t.b2 = __ldg(x2 + 64 + lane);
      t.b3 = __ldg(x2 + 96 + lane);
      return t;
    };
    auto load_a = [&](int c) {
      AT t;
      const double* x2 = a.x2u + c * 64;
      t.wz = __ldg(a.w0 + c);
      t.b0 = __ldg(x2 + lane);
      t.b1 = __ldg(x2 + 32 + lane);
      return t;
    };
    auto stage_a = [&](const Cur& k, int ub, const AT& t) {
      if (k.c == 0) mbar_wait(&sbar[k.r & 1], static_cast<unsigned>((k.r >> 1) & 1));
      if (!gact) return;
      const double* sr = Ss + (k.r & 1) * sbuf + zr + ldS * (t.wz + (lane & 3));
      double d0 = 0.0, d1 = 0.0;
      dmma(d0, d1, sr[0], t.b0);
      dmma(d0, d1, sr[4 * ldS], t.b1);
      *reinterpret_cast<double2*>(ua0 + ub * ubuf) = make_double2(d0, d1);
    };
    Cur ka{0, 0};  // U step cursor
    for (int q = 0; q < kDepth; ++q, adv(ka)) {
      if (q < qtot) {
        stage_a(ka, q, load_a(ka.c));
        __syncwarp();
        if (lane == 0) mbar_arrive(&ubar[q]);
      }
    }
    nb_sync(kBarTensor, kSlabBS - 256);
    if (leader)  // a round whose last U was just formed frees its S3 tile
      for (int q = 0; q < kDepth && q < qtot; ++q)
        if (at_q(q).c == nch - 1) issue_s(at_q(q).r + 2);
    Cur kz = at_q(1);              // Z tables: q + 1
    Cur kt = ka;                   // U tables: q + kDepth + 1
    adv(kt);
    int T = -1;
    double z00 = 0.0, z01 = 0.0, z10 = 0.0, z11 = 0.0;
    double* qs = a.Q + blockIdx.x * p12;
    const i64 qstep = static_cast<i64>(gridDim.x) * p12;
    auto flush = [&](int k, double x0, double x1) {
      const int zc = 8 * k + zq;
      if (zr < p1 && zc < p2) qs[zr + static_cast<i64>(p1) * zc] = x0;
      if (zr < p1 && zc + 1 < p2) qs[zr + static_cast<i64>(p1) * (zc + 1)] = x1;
    };
    ZT zt = load_z(0);
    AT at = load_a(ka.c);  // ka = kDepth
    int c = 0;
    for (int q = 0; q < qtot; ++q) {
      const int buf = q & (kDepth - 1);
      const ZT zn = load_z(kz.c);   // next chunk's Z tables
      const AT an = load_a(kt.c);   // and the U tables one further
      mbar_wait(&wbar[buf], static_cast<unsigned>(q / kDepth) & 1u);
      if (gact) {
        const double2* pg = pg0 + buf * (pbuf >> 1);
        // Y(zr, columns zq, zq + 1) = sum of the quads' partials, ascending quads
        double2 g0 = pg[gs.x & 0xffff], g1 = pg[static_cast<unsigned>(gs.x) >> 16];
        double2 g2 = pg[gs.y & 0xffff], g3 = pg[static_cast<unsigned>(gs.y) >> 16];
        double y0 = ((g0.x + g1.x) + g2.x) + g3.x;
        double y1 = ((g0.y + g1.y) + g2.y) + g3.y;
        if (gmax > 4) {
          g0 = pg[gs.z & 0xffff];
          g1 = pg[static_cast<unsigned>(gs.z) >> 16];
          y0 = (y0 + g0.x) + g1.x;
          y1 = (y1 + g0.y) + g1.y;
          if (gmax > 6) {
            g2 = pg[gs.w & 0xffff];
            g3 = pg[static_cast<unsigned>(gs.w) >> 16];
            y0 = (y0 + g2.x) + g3.x;
            y1 = (y1 + g2.y) + g3.y;
          }
        }
        const int t0 = zt.tz & 0xffff;
        if (T < 0) T = t0;
        while (T < t0) {  // tile T is complete: later chunks start at t0 > T
          flush(T, z00, z01);
          z00 = z10;
          z01 = z11;
          z10 = z11 = 0.0;
          ++T;
        }
        dmma(z00, z01, y0, zt.b0);
        dmma(z00, z01, y1, zt.b1);
        if (zt.tz >> 16) {
          dmma(z10, z11, y0, zt.b2);
          dmma(z10, z11, y1, zt.b3);
        }
        if (c == nch - 1) {  // slice done: the live window holds its last two tiles
          flush(T, z00, z01);
          flush(T + 1, z10, z11);
          z00 = z01 = z10 = z11 = 0.0;
          T = -1;
        }
      }
      // U(q + kDepth) into the buffer of chunk q (the row warps are done with it)
      if (q + kDepth < qtot) {
        stage_a(ka, buf, at);
        __syncwarp();
        if (lane == 0) mbar_arrive(&ubar[buf]);
        if (ka.c == nch - 1) {  // that round's S3 tile is free once every tensor warp formed its U
          nb_sync(kBarTensor, kSlabBS - 256);
          if (leader) {
            fence_proxy_async();
            issue_s(ka.r + 2);
          }
        }
      }
      adv(ka);
      adv(kz);
      adv(kt);
      zt = zn;
      at = an;
      if (++c == nch) {
        c = 0;
        qs += qstep;
      }
    }
  }
  double rr = warp_sum_s(acc0 + acc1);
  __syncthreads();
  if (lane == 0) red[warp] = rr;
  __syncthreads();
  if (warp == 0) {
    rr = lane < (kSlabBS >> 5) ? red[lane] : 0.0;
    rr = warp_sum_s(rr);
    if (lane == 0) a.partial[blockIdx.x] = rr;
  }
}

}  // namespace

// k_slab4: the scatter/gather pass with every operand stream on the engine
// that suits it (measured on B200: the register-staged v stream of k_slab2 is
// capped by the warp's scoreboards at two chunks in flight, ~32 KB per SM,
// which bounds the pass at ~140 us before any arithmetic; the issue latency of
// 16 resident warps bounds the rest):
//   * v arrives by cp.async.bulk (one 16 KB copy per chunk, contiguous in the
//     array) into a four-chunk shared ring behind mbarriers, issued by row warp
//     0 as soon as the tiles of the pair before last are read; row
//     threads read their 4 x 2 cells with swizzled 16-byte loads (the upper
//     half of each quad group takes rows 2,3 first: conflict free);
//   * the S3 operands of the U step (2 doubles per lane and chunk) come
//     straight from L2 one pair ahead, so no S3 tile, no tile barrier;
//   * chunks are handed over in pairs through mbarriers (one arrival per
//     warp); U and partial tiles have fixed strides, so all buffer offsets are
//     immediates; the X2 chunk tables sit in shared memory; the gather slots
//     are shared addresses in registers;
//   * the FP64 chains of a chunk are issued level by level (8 to 10
//     independent chains), the shared loads of a pair's gather up front;
//     setmaxnreg: tensor warpgroups 120, row warpgroups 136.
constexpr int kPLMax = 322;                 // slots per column-pair plane at n1 = 256
constexpr int kPBuf = 8 * kPLMax;           // doubles per partial tile
// U tile of k_slab4: 64 rows (p1 <= 64) of 8 doubles = four 16-byte column-pair
// units, unit u of row r stored at unit u ^ ((r >> 1) & 3).  Both access
// patterns are then conflict free: a tensor-warp quarter (rows 2q, 2q + 1, all
// four units) writes 8 distinct bank groups, and a row-warp quarter (8
// consecutive rows, one unit) reads 8 distinct bank groups.
constexpr int kUBuf = 8 * 64;
__device__ __forceinline__ unsigned u_tile_off(int row, int unit) {  // byte offset inside a U tile
  return static_cast<unsigned>(row * 64 + ((unit ^ ((row >> 1) & 3)) << 4));
}

__device__ __forceinline__ bool mbar_try_s(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_spin_s(unsigned bar, unsigned parity) {
  const long long t0 = clock64();
  while (!mbar_try_s(bar, parity)) {
    if (clock64() - t0 > async::kWatchdogCycles) {
      printf("kg watchdog: slab mbarrier wait (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x, parity);
      __trap();
    }
  }
}
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
  if (!mbar_try_s(bar, parity)) mbar_spin_s(bar, parity);
}
__device__ __forceinline__ void mbar_arrive_s(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ double2 lds2_s(unsigned addr) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(addr));
  return r;
}
__device__ __forceinline__ double lds_s(unsigned addr) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ int ldsi_s(unsigned addr) {
  int r;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sts2_s(unsigned addr, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

constexpr int kVBuf = 8 * 256;              // doubles per v chunk tile (n1 <= 256)

// G: gather slots per basis function (5, 6 or 8; cubic B-spline factors on a 4x finer grid need 5).
template <int G>
__global__ void __launch_bounds__(kSlabBS, 1) k_slab4(SlabArgs a) {
  using namespace async;
  extern __shared__ __align__(128) double sm[];
  __shared__ double red[32];
  // pair hb: U(pair) formed / its partials stored (one arrival per warp) / its v chunks landed
  __shared__ unsigned long long ubar[2], wbar[2], vbar[2];
  const int n1 = a.n1, n2 = a.n2, p1 = a.p1, p2 = a.p2, nch = a.nch;
  const int PL = a.PL;
  double* Vs = sm;                            // [kDepth][kVBuf]  v chunks (8 columns of n1)
  double* Us = Vs + kDepth * kVBuf;           // [kDepth][kUBuf]
  double* Ps = Us + kDepth * kUBuf;           // [kDepth][kPBuf]
  double* Tz = Ps + kDepth * kPBuf;           // [nch][128]  Z-step B fragments
  double* Tu = Tz + nch * 128;                // [nch][64]   U-step B fragments
  int* Ti = reinterpret_cast<int*>(Tu + nch * 64);  // [nch][2] = {tz, w0}
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const i64 p12 = static_cast<i64>(p1) * p2, n12 = static_cast<i64>(n1) * n2;
  const int rounds = static_cast<int>((a.m3 - blockIdx.x + gridDim.x - 1) / gridDim.x);  // slices of this CTA
  const int qtot = rounds * nch, np = qtot >> 1;
  const unsigned ubar0 = smem_u32(&ubar[0]), wbar0 = smem_u32(&wbar[0]), vbar0 = smem_u32(&vbar[0]);
  if (tid == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(&ubar[k], 8);
      mbar_init(&wbar[k], 8);
      mbar_init(&vbar[k], 1);
    }
    mbar_init_fence();
  }
  for (int k = tid; k < nch * 128; k += kSlabBS) Tz[k] = __ldg(a.x2z + k);
  for (int k = tid; k < nch * 64; k += kSlabBS) Tu[k] = __ldg(a.x2u + k);
  for (int k = tid; k < nch; k += kSlabBS) {
    Ti[2 * k] = __ldg(a.tz + k);
    Ti[2 * k + 1] = __ldg(a.w0 + k);
  }
  if (tid < 4 * kDepth) {  // the zero slot of every plane
    double* z = Ps + (tid >> 2) * kPBuf + 2 * ((tid & 3) * PL + PL - 1);
    z[0] = z[1] = 0.0;
  }
  __syncthreads();
  // programmatic dependent launch (Launch::pdl): the kernel after this one may
  // be scheduled as this one's CTAs retire; of this kernel's inputs only S3
  // belongs to the kernel before it (the tensor warps wait below), v and the
  // tables are older
  asm volatile("griddepcontrol.launch_dependents;");
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  if (warp < 8) {
    // ------------------------------------------------------------ row warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 136;");
    const int nq = n1 >> 2;                    // row quads
    const bool act = tid < 4 * nq;
    const int rq = act ? tid % nq : 0, cp = act ? tid / nq : 0;
    const int r0 = 4 * rq, c0 = 2 * cp;        // rows r0 .. r0 + 3, chunk columns c0, c0 + 1
    // quads 4 apart are 128 bytes apart in a v column: the upper half of each
    // group of 8 quads holds its rows in the order 2, 3, 0, 1, so that the
    // 16-byte v loads of a quarter warp hit 8 distinct bank groups
    const bool sw = (rq >> 2) & 1;
    int lo = 0;
    double C[4][kWin];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < kWin; ++t) C[r][t] = 0.0;
    if (act) {
      lo = min(__ldg(a.H1.lo + r0), p1 - kWin);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = r0 + (sw ? (r ^ 2) : r);
        const int l = __ldg(a.H1.lo + row), len = __ldg(a.H1.len + row);
        const double* cf = a.H1.coef + __ldg(a.H1.off + row);
#pragma unroll
        for (int t = 0; t < kWin; ++t) {
          const int j = lo + t - l;
          C[r][t] = (j >= 0 && j < len) ? __ldg(cf + j) : 0.0;
        }
      }
    }
    unsigned ub[kWin];  // this thread's five window rows of U tile 0 (column pair cp)
#pragma unroll
    for (int t = 0; t < kWin; ++t) ub[t] = smem_u32(Us) + u_tile_off(lo + t, cp);
    const unsigned pb0 = smem_u32(Ps) + 16u * static_cast<unsigned>(cp * PL + rq * kWin);
    const unsigned vb0 = smem_u32(Vs + r0 + n1 * c0) + (sw ? 16u : 0u);   // rows (sw ? 2,3 : 0,1) of column c0
    const unsigned vb1 = smem_u32(Vs + r0 + n1 * c0) + (sw ? 0u : 16u);   // the other two rows
    const unsigned vcol = 8u * static_cast<unsigned>(n1);
    // v stream (row warp 0): chunk pairs by bulk copy into the ring.  Pair ip + 1
    // goes into the tiles of pair ip - 1 once every row warp has arrived on that
    // pair's partial barrier (they have all read its v by then); the tensor
    // warps, which pace the pass, carry none of it.
    const i64 vchunk = static_cast<i64>(n1) * 8;
    const i64 vjump = static_cast<i64>(gridDim.x) * n12 - vchunk * (nch - 1);  // last chunk of a slice -> first of the next
    const double* vp = a.v + blockIdx.x * n12;   // next chunk to copy
    int vc = 0, vq = 0;
    const unsigned vbytes = static_cast<unsigned>(vchunk * 8);
    const unsigned vs0 = smem_u32(Vs);
    auto copy_pair = [&](unsigned hb) {          // the next two chunks into pair hb's tiles (one lane)
      if (vq >= qtot) return;
      const unsigned bar = vbar0 + 8 * hb;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * vbytes) : "memory");
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         vs0 + 8u * static_cast<unsigned>((2 * hb + j) * kVBuf)),
                     "l"(vp), "r"(vbytes), "r"(bar)
                     : "memory");
        ++vq;
        if (++vc == nch) {
          vc = 0;
          vp += vjump;
        } else {
          vp += vchunk;
        }
      }
    };
    if (tid == 0) {
      fence_proxy_async();
      copy_pair(0);
      copy_pair(1);
    }
    // chunk j of a pair: U window at uo, partials to po, v tile at byte offset vo
    auto body = [&](const int j, const unsigned uo, const unsigned po, const unsigned vo) {
      if (act) {
        double2 uu[kWin];
#pragma unroll
        for (int t = 0; t < kWin; ++t) uu[t] = lds2_s(ub[t] + uo + 8 * j * kUBuf);
        double vr[8];
        {
          const double2 x0 = lds2_s(vb0 + vo + 8 * j * kVBuf), x1 = lds2_s(vb1 + vo + 8 * j * kVBuf);
          const double2 y0 = lds2_s(vb0 + vo + 8 * j * kVBuf + vcol), y1 = lds2_s(vb1 + vo + 8 * j * kVBuf + vcol);
          vr[0] = x0.x, vr[1] = x0.y, vr[2] = x1.x, vr[3] = x1.y;
          vr[4] = y0.x, vr[5] = y0.y, vr[6] = y1.x, vr[7] = y1.y;
        }
        // level by level over the 8 cells (8 to 10 independent FP64 chains in flight)
        double x[2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r) x[c][r] = C[r][0] * (c ? uu[0].y : uu[0].x);
#pragma unroll
        for (int t = 1; t < kWin; ++t)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int r = 0; r < 4; ++r) x[c][r] = fma(C[r][t], c ? uu[t].y : uu[t].x, x[c][r]);
        double wv[2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r) wv[c][r] = vr[4 * c + r] * x[c][r];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r & 1) {
            acc1 = fma(wv[0][r], x[0][r], acc1);
            acc3 = fma(wv[1][r], x[1][r], acc3);
          } else {
            acc0 = fma(wv[0][r], x[0][r], acc0);
            acc2 = fma(wv[1][r], x[1][r], acc2);
          }
        }
        double pt[2][kWin];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int t = 0; t < kWin; ++t) pt[c][t] = C[0][t] * wv[c][0];
#pragma unroll
        for (int r = 1; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int t = 0; t < kWin; ++t) pt[c][t] = fma(C[r][t], wv[c][r], pt[c][t]);
#pragma unroll
        for (int t = 0; t < kWin; ++t) sts2_s(po + 8 * j * kPBuf + 16 * t, pt[0][t], pt[1][t]);
      }
    };
    for (int ip = 0; ip < np; ++ip) {
      const unsigned hb = static_cast<unsigned>(ip & 1), par = static_cast<unsigned>(ip >> 1) & 1u;
      mbar_wait_s(ubar0 + 8 * hb, par);
      mbar_wait_s(vbar0 + 8 * hb, par);
      const unsigned uo = hb * (16 * kUBuf), po = pb0 + hb * (16 * kPBuf), vo = hb * (16 * kVBuf);
      if (warp == 0 && ip > 0) {  // pair ip - 1 is read: pair ip + 1 into its v tiles
        mbar_wait_s(wbar0 + 8 * (hb ^ 1u), static_cast<unsigned>((ip - 1) >> 1) & 1u);
        if (lane == 0) copy_pair(hb ^ 1u);
      }
      body(0, uo, po, vo);
      body(1, uo, po, vo);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(wbar0 + 8 * hb);
    }
  } else {
    // --------------------------------------------------------- tensor warps
    asm volatile("setmaxnreg.dec.sync.aligned.u32 120;");
    const int tw = warp - 8;
    const bool gact = tw < ((p1 + 7) >> 3);   // this warp owns p1 rows 8 tw .. 8 tw + 7
    const bool leader = tid == 8 * 32;
    const int zr = 8 * tw + (lane >> 2), zq = 2 * (lane & 3);
    const bool zok = zr < p1;
    const unsigned ua0 = smem_u32(Us) + u_tile_off(zr, lane & 3);  // U store (tile 0)
    // gather slots of basis function zr as shared addresses in partial tile 0 (column pair lane & 3)
    unsigned gs[G];
    {
      int4 g4 = make_int4(0, 0, 0, 0);
      const int zs = PL - 1;
      if (gact) g4 = __ldg(reinterpret_cast<const int4*>(a.gat) + zr);
      else g4.x = g4.y = g4.z = g4.w = zs | (zs << 16);
      const unsigned pl0 = smem_u32(Ps) + 16u * static_cast<unsigned>((lane & 3) * PL);
      const int w4[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
      for (int k = 0; k < G; ++k) gs[k] = pl0 + 16u * ((static_cast<unsigned>(w4[k >> 1]) >> (16 * (k & 1))) & 0xffffu);
    }
    // U step: chunk ca of the slice at sp; S3 operands from L2, loaded one pair ahead
    const unsigned tu0 = smem_u32(Tu) + 8u * lane, tz0 = smem_u32(Tz) + 8u * lane, ti0 = smem_u32(Ti);
    int ca = 0, sleft = rounds;                  // sleft: slices left for the U step
    unsigned tup = tu0, tia = ti0 + 4;           // Tu[ca][.][lane], w0 of chunk ca
    const double* sp = a.S + blockIdx.x * p12 + zr + static_cast<i64>(p1) * (lane & 3);
    const i64 sstep = static_cast<i64>(gridDim.x) * p12;
    struct UOp { double s0, s1, b0, b1; };
    auto load_u = [&]() {                        // operands of U(ca), then advance the cursor
      UOp o{0.0, 0.0, 0.0, 0.0};
      if (gact && sleft > 0) {
        const int wz = ldsi_s(tia);
        o.b0 = lds_s(tup);
        o.b1 = lds_s(tup + 256);
        if (zok) {
          const double* s = sp + static_cast<i64>(p1) * wz;
          o.s0 = __ldg(s);
          o.s1 = __ldg(s + 4 * static_cast<i64>(p1));
        }
      }
      if (++ca == nch) {
        ca = 0;
        tup = tu0;
        tia = ti0 + 4;
        sp += sstep;
        --sleft;
      } else {
        tup += 512;
        tia += 8;
      }
      return o;
    };
    auto store_u = [&](const UOp& o, const unsigned uoff) {
      if (gact) {
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;  // two independent DMMAs
        dmma(d0, d1, o.s0, o.b0);
        dmma(e0, e1, o.s1, o.b1);
        sts2_s(ua0 + uoff, d0 + e0, d1 + e1);
      }
    };
    asm volatile("griddepcontrol.wait;" ::: "memory");  // S3 is complete and visible
    for (int hb = 0; hb < 2; ++hb) {  // U of the first two pairs
      const UOp o0 = load_u(), o1 = load_u();
      store_u(o0, hb * (16 * kUBuf));
      store_u(o1, hb * (16 * kUBuf) + 8 * kUBuf);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(ubar0 + 8 * hb);
    }
    int T = -1, c = 0;
    unsigned tzp = tz0, tiz = ti0;            // Tz[c][.][lane], tz of chunk c
    double z00 = 0.0, z01 = 0.0, z10 = 0.0, z11 = 0.0;
    double* qs = a.Q + blockIdx.x * p12 + zr + static_cast<i64>(p1) * zq;
    const i64 qstep = static_cast<i64>(gridDim.x) * p12;
    auto flush = [&](int k, double x0, double x1) {
      const int zc = 8 * k + zq;
      if (zok && zc < p2) qs[static_cast<i64>(p1) * (8 * k)] = x0;
      if (zok && zc + 1 < p2) qs[static_cast<i64>(p1) * (8 * k + 1)] = x1;
    };
    // gather + Z of a pair (its chunks 2k, 2k + 1 lie in one slice: nch is even).
    // All shared loads of both chunks are issued up front: the tensor warps are
    // bound by the latency of their dependent shared loads otherwise.
    auto body2 = [&](const unsigned po) {
      if (gact) {
        double2 g[2][G];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int k = 0; k < G; ++k) g[j][k] = lds2_s(gs[k] + po + 8 * j * kPBuf);
        int tz[2];
        double zb[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          tz[j] = ldsi_s(tiz + 8 * j);
#pragma unroll
          for (int h = 0; h < 4; ++h) zb[j][h] = lds_s(tzp + 1024 * j + 256 * h);
        }
        // Y(zr, columns zq, zq + 1) = sum of the quads' partials: pairwise, a fixed order
        double y[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          y[j][0] = (g[j][0].x + g[j][1].x) + (g[j][2].x + g[j][3].x);
          y[j][1] = (g[j][0].y + g[j][1].y) + (g[j][2].y + g[j][3].y);
          if (G > 6) {
            y[j][0] += (g[j][4].x + g[j][5].x) + (g[j][G - 2].x + g[j][G - 1].x);
            y[j][1] += (g[j][4].y + g[j][5].y) + (g[j][G - 2].y + g[j][G - 1].y);
          } else if (G > 5) {
            y[j][0] += g[j][4].x + g[j][G - 1].x;
            y[j][1] += g[j][4].y + g[j][G - 1].y;
          } else {
            y[j][0] += g[j][4].x;
            y[j][1] += g[j][4].y;
          }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int t0 = tz[j] & 0xffff;
          if (T < 0) T = t0;
          while (T < t0) {  // tile T is complete: later chunks start at t0 > T
            flush(T, z00, z01);
            z00 = z10;
            z01 = z11;
            z10 = z11 = 0.0;
            ++T;
          }
          dmma(z00, z01, y[j][0], zb[j][0]);
          dmma(z00, z01, y[j][1], zb[j][1]);
          if (tz[j] >> 16) {
            dmma(z10, z11, y[j][0], zb[j][2]);
            dmma(z10, z11, y[j][1], zb[j][3]);
          }
        }
      }
      c += 2;
      if (c == nch) {  // slice done: the live window holds its last two tiles
        if (gact) {
          flush(T, z00, z01);
          flush(T + 1, z10, z11);
          z00 = z01 = z10 = z11 = 0.0;
          T = -1;
        }
        c = 0;
        qs += qstep;
        tzp = tz0;
        tiz = ti0;
      } else {
        tzp += 2048;
        tiz += 16;
      }
    };
    for (int ip = 0; ip < np; ++ip) {
      const unsigned hb = static_cast<unsigned>(ip & 1);
      // operands of the U step of pair ip + 2 (latency hidden behind the wait and the gather)
      const UOp o0 = load_u(), o1 = load_u();
      mbar_wait_s(wbar0 + 8 * hb, static_cast<unsigned>(ip >> 1) & 1u);
      body2(hb * (16 * kPBuf));
      // U of pair ip + 2 into this pair's U tiles (every row warp has read them)
      if (ip + 2 < np) {
        store_u(o0, hb * (16 * kUBuf));
        store_u(o1, hb * (16 * kUBuf) + 8 * kUBuf);
        __syncwarp();
        if (lane == 0) mbar_arrive_s(ubar0 + 8 * hb);
      }
    }
  }
  double rr = warp_sum_s((acc0 + acc1) + (acc2 + acc3));
  __syncthreads();
  if (lane == 0) red[warp] = rr;
  __syncthreads();
  if (warp == 0) {
    rr = lane < (kSlabBS >> 5) ? red[lane] : 0.0;
    rr = warp_sum_s(rr);
    if (lane == 0) a.partial[blockIdx.x] = rr;
  }
}

// Y in scatter/gather form (k_slab2) when the design has a gather table;
// KG_SLAB_DMMA=1 (developer switch) keeps the DMMA form (k_slab).
static bool slab_gather(const SlabArgs& a) {
  static const bool dmma_y = dev_env("KG_SLAB_DMMA") != nullptr;
  return !dmma_y && a.gat && a.gmax > 0 && a.gmax <= 8 && a.PL > 0 && a.PL <= kPLMax;  // (k_slab4 also needs an even chunk count)
}

// Leading dimensions and shared-memory size of a slab plan.
static size_t slab_layout(SlabArgs& a) {
  const int p1r = (a.p1 + 15) / 16 * 16;
  a.ldS = p1r + 4;                           // = 4 (mod 16): A fragments of stage A
  a.ldU = kLdr;
  a.ldZ = 0;
  a.ldW = (a.n1 + 15) / 16 * 16 + 4;         // = 4 (mod 16): B fragments of stage C
  a.cg = 1;
  const size_t ubuf = static_cast<size_t>(kLdr) * 8 * ((a.p1 + 7) / 8);
  if (slab_gather(a)) {
    // k_slab4: v ring, fixed-stride U / partial tiles, the X2 chunk tables; k_slab2
    // (the same shapes with an odd chunk count or a partial last chunk): two S3
    // tiles, U and partial tiles with the design's strides
    const size_t k4 = kDepth * static_cast<size_t>(kVBuf + kUBuf + kPBuf) + static_cast<size_t>(a.nch) * (128 + 64 + 1);
    const size_t k2 = 2 * static_cast<size_t>(a.ldS) * a.p2 + kDepth * ubuf + kDepth * static_cast<size_t>(8) * a.PL;
    return std::max(k4, k2) * sizeof(double);
  }
  const size_t dbl = 2 * static_cast<size_t>(a.ldS) * a.p2 + kDepth * ubuf + kDepth * static_cast<size_t>(a.ldW) * 8;
  return dbl * sizeof(double);
}

bool slab_ok(const SlabArgs& a0) {
  SlabArgs a = a0;
  if (!a.x2u || !a.x2z || !a.w0 || !a.tz || a.g1.ks == 0 || !a.H1.hlo || !a.H1.hlen) return false;
  if (a.n1 > 4 * kTeam / 4 || (a.n1 & 3) || (a.p1 & 1) || a.p1 > 64 || a.p1 < kWin || a.p2 < 8 || a.p2 > 64 ||
      a.H1.maxlen > 4)
    return false;
  if (a.g1.groups != (a.p1 + 7) / 8 || a.nch < kDepth) return false;
  // every quad of grid rows reads a kWin-wide coefficient window
  for (int r0 = 0; r0 < a.n1; r0 += 4) {
    const int lo = std::min(a.H1.hlo[r0], a.p1 - kWin);
    for (int r = r0; r < r0 + 4; ++r)
      if (a.H1.hlen[r] > 0 && (a.H1.hlo[r] < lo || a.H1.hlo[r] + a.H1.hlen[r] > lo + kWin)) return false;
  }
  return slab_layout(a) <= 232448 - 1024;
}

int slab_grid(const SlabArgs& a) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<int>(std::min<i64>(a.m3, sms));
}

template <int KS>
static void launch_slab_ks(const Launch& L, const SlabArgs& a, size_t smem, int g) {
  smem_attr(k_slab<KS>, static_cast<int>(smem));
  k_slab<KS><<<g, kSlabBS, smem, L.s>>>(a);
}

void slab_pass(const Launch& L, const SlabArgs& a0) {
  SlabArgs a = a0;
  const size_t smem = slab_layout(a);
  const int g = slab_grid(a);
  if (slab_gather(a)) {
    // KG_SLAB_K2=1 (developer switch): the register-staged kernel on every shape
    static const bool k2 = dev_env("KG_SLAB_K2") != nullptr;
    const bool k4 = !k2 && !(a.nch & 1) && a.n2 == 8 * a.nch;  // whole chunk pairs
    a.pf = 0;  // the bulk-copy ring keeps enough of v in flight without an L2 prefetch
    PdlConfig pc(dim3(g), dim3(kSlabBS), smem, L);
    if (k4 && a.gmax <= 5) {
      smem_attr(k_slab4<5>, static_cast<int>(smem));
      cudaLaunchKernelEx(&pc.cfg, k_slab4<5>, a);
    } else if (k4 && a.gmax <= 6) {
      smem_attr(k_slab4<6>, static_cast<int>(smem));
      cudaLaunchKernelEx(&pc.cfg, k_slab4<6>, a);
    } else if (k4) {
      smem_attr(k_slab4<8>, static_cast<int>(smem));
      cudaLaunchKernelEx(&pc.cfg, k_slab4<8>, a);
    } else {
      a.pf = 4;
      smem_attr(k_slab2, static_cast<int>(smem));
      k_slab2<<<g, kSlabBS, smem, L.s>>>(a);
    }
  } else {
    switch (a.g1.ks) {
      case 8: launch_slab_ks<8>(L, a, smem, g); break;
      case 12: launch_slab_ks<12>(L, a, smem, g); break;
      default: launch_slab_ks<16>(L, a, smem, g); break;
    }
  }
  launched(L);
}

}  // namespace kg
