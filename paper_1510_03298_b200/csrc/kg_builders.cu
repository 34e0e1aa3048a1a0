// Input builders on the device: the callers in front of
// the fit path that turn raw data into the response array and the marginal
// designs.
//
//  * bin_scatter (bspline.cpp:106-153): points -> count array.  HBM-bound
//    (8*d bytes per point read once): persistent CTAs stream tiles of points
//    into shared memory with the bulk-copy engine; the counts are privatised
//    per CTA in shared memory (u32) when the grid fits, and flushed with one
//    FP64 atomicAdd per nonzero cell; otherwise FP64 atomics go straight to
//    the L2-resident count array.  Counts are integers, so every accumulation
//    order gives the same bits.
//  * bspline_design (bspline.cpp:64-104): one thread per grid point, the
//    Cox-de Boor recursion on the span's `order` nonvanishing functions with
//    explicitly rounded FP64 ops (no FMA contraction), so the design is
//    bit-identical to the host builder kg_bspline_design.
#include <cuda_runtime.h>

#include <cstdint>

#include "kg_async.cuh"
#include "kg_internal.h"

namespace kg {

namespace {

// floor(RN((x - lo) / width)) as the reference computes it, without the
// division in the common case: qa = t * (1/width) is within 1.5 ulp of the
// correctly rounded quotient, so when no integer lies in qa * [1 - 2^-50,
// 1 + 2^-50] both floor to the same cell; otherwise (points on or next to a
// bin edge) the correctly rounded division decides.
__device__ __forceinline__ int cell_of(double t, double w, double inv) {
  const double qa = __dmul_rn(t, inv);
  const int c0 = __double2int_rd(__dmul_rn(qa, 1.0 - 0x1p-50));
  const int c1 = __double2int_rd(__dmul_rn(qa, 1.0 + 0x1p-50));
  if (c0 == c1) return c0;
  return __double2int_rd(__ddiv_rn(t, w));
}

// Per-dimension constants held in registers for a compile-time d.
template <int D>
struct BinDims {
  static constexpr int DM = D > 0 ? D : kMaxBinDims;
  double lo[DM], hi[DM], w[DM], inv[DM];
  int bmax[DM], stride[DM];
  int d;
  __device__ __forceinline__ explicit BinDims(const BinArgs& A) {
    d = D > 0 ? D : A.d;
#pragma unroll
    for (int j = 0; j < DM; ++j) {
      lo[j] = A.lo[j];
      hi[j] = A.hi[j];
      w[j] = A.width[j];
      inv[j] = A.inv[j];
      bmax[j] = A.bmax[j];
      stride[j] = A.stride[j];
    }
  }
};

// Column-major cell of one point, or -1 when a coordinate is outside its
// bounds (bspline.cpp:129-148).  A NaN coordinate is dropped (the reference's
// cast of floor(NaN) is undefined behaviour).
template <int D>
__device__ __forceinline__ int bin_point(const BinDims<D>& B, const double* p) {
  int off = 0;
#pragma unroll
  for (int j = 0; j < BinDims<D>::DM; ++j) {
    if (D == 0 && j >= B.d) break;
    const double x = p[j];
    if (!(x >= B.lo[j] && x <= B.hi[j])) return -1;
    const int c = min(cell_of(__dsub_rn(x, B.lo[j]), B.w[j], B.inv[j]), B.bmax[j]);  // last bin closed
    off += c * B.stride[j];
  }
  return off;
}

__device__ __forceinline__ void add_dropped(unsigned long long drop, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) drop += __shfl_xor_sync(0xffffffffu, drop, o);
  if ((threadIdx.x & 31) == 0 && drop) atomicAdd(dst, drop);
}

template <bool HIST>
__device__ __forceinline__ void count(const BinArgs& A, unsigned* hist, int c, unsigned long long& drop) {
  if (c < 0) {
    ++drop;
  } else if (HIST) {
    atomicAdd(hist + c, 1u);
  } else {
    atomicAdd(A.counts + c, 1.0);
  }
}

// Persistent CTAs walk tiles of kBinTile points (tile t = blockIdx.x + k *
// gridDim.x).  Full tiles are staged into shared memory by the bulk-copy
// engine through a kBinStages-deep mbarrier ring, so the HBM stream is one
// contiguous copy per tile whatever d is; the ragged last tile is read
// directly.  HIST: counters privatised per CTA in shared memory (u32) and
// flushed with one FP64 atomic per nonzero cell; else FP64 atomics straight
// into the (L2-resident) count array.
template <int D, bool HIST>
__global__ void __launch_bounds__(kBinThreads) k_bin_staged(BinArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = D > 0 ? D : A.d;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem_raw);
  double* stage = reinterpret_cast<double*>(smem_raw + 16 * kBinStages);
  const i64 tile_dbl = static_cast<i64>(kBinTile) * d;
  unsigned* hist = reinterpret_cast<unsigned*>(stage + kBinStages * tile_dbl);
  const i64 ntiles = (A.npts + kBinTile - 1) / kBinTile;
  const i64 nfull = A.npts / kBinTile;
  const unsigned tile_bytes = static_cast<unsigned>(tile_dbl * 8);
  if (HIST)
    for (i64 c = threadIdx.x; c < A.cells; c += kBinThreads) hist[c] = 0u;
  if (threadIdx.x == 0) {
    for (int sidx = 0; sidx < kBinStages; ++sidx) async::mbar_init(bar + 2 * sidx, 1);
    async::mbar_init_fence();
    for (int sidx = 0; sidx < kBinStages; ++sidx) {
      const i64 t = blockIdx.x + static_cast<i64>(sidx) * gridDim.x;
      if (t < nfull) {
        async::mbar_expect_tx(bar + 2 * sidx, tile_bytes);
        async::bulk_g2s(stage + sidx * tile_dbl, A.pts + t * tile_dbl, tile_bytes, bar + 2 * sidx);
      }
    }
  }
  __syncthreads();
  const BinDims<D> B(A);
  unsigned long long drop = 0;
  for (i64 k = 0;; ++k) {
    const i64 t = blockIdx.x + k * gridDim.x;
    if (t >= ntiles) break;
    const int sidx = static_cast<int>(k % kBinStages);
    if (t < nfull) {
      async::mbar_wait(bar + 2 * sidx, static_cast<unsigned>((k / kBinStages) & 1));
      const double* tile = stage + sidx * tile_dbl;
#pragma unroll
      for (int q = 0; q < kBinTile / kBinThreads; ++q) {
        const int pi = threadIdx.x + q * kBinThreads;
        count<HIST>(A, hist, bin_point<D>(B, tile + static_cast<i64>(pi) * d), drop);
      }
    } else {  // ragged last tile
      for (i64 i = t * kBinTile + threadIdx.x; i < A.npts; i += kBinThreads)
        count<HIST>(A, hist, bin_point<D>(B, A.pts + i * d), drop);
    }
    __syncthreads();  // the whole CTA is done with this stage
    if (threadIdx.x == 0) {
      const i64 tn = t + static_cast<i64>(kBinStages) * gridDim.x;
      if (tn < nfull) {
        async::fence_proxy_async();
        async::mbar_expect_tx(bar + 2 * sidx, tile_bytes);
        async::bulk_g2s(stage + sidx * tile_dbl, A.pts + tn * tile_dbl, tile_bytes, bar + 2 * sidx);
      }
    }
  }
  if (HIST) {
    __syncthreads();
    for (i64 c = threadIdx.x; c < A.cells; c += kBinThreads) {
      const unsigned v = hist[c];
      if (v) atomicAdd(A.counts + c, static_cast<double>(v));
    }
  }
  add_dropped(drop, A.dropped);
}

// Fallback for point arrays that are not 16-byte aligned: direct loads.
template <int D, bool HIST>
__global__ void __launch_bounds__(kBinThreads) k_bin_direct(BinArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* hist = reinterpret_cast<unsigned*>(smem_raw);
  const int d = D > 0 ? D : A.d;
  if (HIST) {
    for (i64 c = threadIdx.x; c < A.cells; c += kBinThreads) hist[c] = 0u;
    __syncthreads();
  }
  const BinDims<D> B(A);
  unsigned long long drop = 0;
  const i64 stride = static_cast<i64>(gridDim.x) * kBinThreads;
  for (i64 i = static_cast<i64>(blockIdx.x) * kBinThreads + threadIdx.x; i < A.npts; i += stride)
    count<HIST>(A, hist, bin_point<D>(B, A.pts + i * d), drop);
  if (HIST) {
    __syncthreads();
    for (i64 c = threadIdx.x; c < A.cells; c += kBinThreads) {
      const unsigned v = hist[c];
      if (v) atomicAdd(A.counts + c, static_cast<double>(v));
    }
  }
  add_dropped(drop, A.dropped);
}

size_t bin_smem_bytes(const BinArgs& A, bool hist, bool staged) {
  size_t b = hist ? sizeof(unsigned) * static_cast<size_t>(A.cells) : 0;
  if (staged) b += 16 * kBinStages + sizeof(double) * kBinStages * static_cast<size_t>(kBinTile) * A.d;
  return b;
}

template <int D, bool HIST>
void launch_bin_t(const Launch& L, const BinArgs& A, bool staged, int n_sm) {
  const size_t shmem = bin_smem_bytes(A, HIST, staged);
  auto kern = staged ? k_bin_staged<D, HIST> : k_bin_direct<D, HIST>;
  smem_attr(kern, static_cast<int>(shmem));
  int occ = 0;
  KG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBinThreads, shmem));
  occ = std::max(occ, 1);
  const i64 need = (A.npts + kBinTile - 1) / kBinTile;
  const int grid = static_cast<int>(std::max<i64>(1, std::min<i64>(need, static_cast<i64>(n_sm) * occ)));
  kern<<<grid, kBinThreads, shmem, L.s>>>(A);
}

template <int D>
void launch_bin(const Launch& L, const BinArgs& A, bool hist, bool staged, int n_sm) {
  if (hist) launch_bin_t<D, true>(L, A, staged, n_sm);
  else launch_bin_t<D, false>(L, A, staged, n_sm);
}

// ------------------------------------------------------------ bspline_design
__global__ void k_bspline(i64 npts, const double* __restrict__ pts, int order, i64 nb,
                          const double* __restrict__ t, double* __restrict__ out, int* bad) {
  const i64 row = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= npts) return;
  const double x = pts[row];
  if (row > 0 && !(x > pts[row - 1])) atomicExch(bad, 1);  // MarginalGrid: strictly increasing
  const int deg = order - 1;
  i64 s = nb - 1;
  if (x < t[nb]) {  // find_span: largest s in [deg, nb-1] with t[s] <= x
    i64 a = deg, b = nb;
    while (b - a > 1) {
      const i64 m = (a + b) / 2;
      if (x < t[m]) b = m;
      else a = m;
    }
    s = a;
  }
  double N[kMaxOrder], Lf[kMaxOrder], Rt[kMaxOrder];
  N[0] = 1.0;
  for (int j = 1; j <= deg; ++j) {
    Lf[j] = __dsub_rn(x, t[s + 1 - j]);
    Rt[j] = __dsub_rn(t[s + j], x);
    double carry = 0.0;
    for (int m = 0; m < j; ++m) {
      const double tmp = __ddiv_rn(N[m], __dadd_rn(Rt[m + 1], Lf[j - m]));
      N[m] = __dadd_rn(carry, __dmul_rn(Rt[m + 1], tmp));
      carry = __dmul_rn(Lf[j - m], tmp);
    }
    N[j] = carry;
  }
  for (int m = 0; m <= deg; ++m) out[row + npts * (s - deg + m)] = N[m];
}

}  // namespace

void bin_scatter(const Launch& L, const BinArgs& A, int n_sm) {
  // staged: the bulk-copy engine needs 16-byte aligned tiles (kBinTile * 8 * d
  // is a multiple of 16, so an aligned base keeps every tile aligned)
  bool staged = (reinterpret_cast<uintptr_t>(A.pts) & 15) == 0 && !(A.mode & 1);
  // shared-memory counters when they fit beside the stages and there are
  // enough points per cell to amortise each CTA's flush
  const size_t budget = static_cast<size_t>(kBinSmemBytes);
  bool hist = bin_smem_bytes(A, true, staged) <= budget && A.npts >= 8 * A.cells;
  if (A.mode & 4) hist = false;
  if ((A.mode & 8) && bin_smem_bytes(A, true, staged) <= budget) hist = true;
  switch (A.d) {
    case 1: launch_bin<1>(L, A, hist, staged, n_sm); break;
    case 2: launch_bin<2>(L, A, hist, staged, n_sm); break;
    case 3: launch_bin<3>(L, A, hist, staged, n_sm); break;
    case 4: launch_bin<4>(L, A, hist, staged, n_sm); break;
    default: launch_bin<0>(L, A, hist, staged, n_sm); break;
  }
  launched(L);
}

void bspline_design_dev(const Launch& L, i64 npts, const double* pts, int order, i64 nb, const double* knots,
                        double* out, int* bad) {
  KG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * static_cast<size_t>(npts * nb), L.s));
  const int nt = 128;
  k_bspline<<<static_cast<unsigned>((npts + nt - 1) / nt), nt, 0, L.s>>>(npts, pts, order, nb, knots, out, bad);
  launched(L);
}

}  // namespace kg
