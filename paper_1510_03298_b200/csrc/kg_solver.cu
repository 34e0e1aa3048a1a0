// Host orchestration of the GLAM fit path on one B200 and the kg_* C ABI.
//
// Control structure (reference: path.cpp:47-81 -> outer.cpp:159-303 ->
// inner.cpp:121-235):
//   * fit_path / outer_solve bookkeeping runs on the host, one stream sync per
//     outer iteration (per lambda for Gaussian models);
//   * every fista_solve runs entirely on the device: one CUDA graph whose
//     conditional WHILE node repeats the iteration body
//        p-space update -> H partial chain -> fused mode-1 pass -> G tail -> control
//     until the device-side control kernel clears the condition.
// All arrays live in HBM for the whole path; nothing n-sized crosses PCIe
// after the observation upload.
#include <dlfcn.h>

#include <functional>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_set>
#include <random>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/kronglm_b200.h"
#include "kg_internal.h"

namespace kg {

// ------------------------------------------------------------ device memory
// Workspaces come from the device's stream-ordered pool (cudaMallocAsync on
// the context stream, release threshold raised in kg_ctx_create), so repeated
// fits reuse cached memory instead of paying cudaMalloc / synchronising
// cudaFree.  g_stream is the ordering stream of the current C-ABI call; a
// buffer whose stream has been destroyed is freed synchronously.
thread_local cudaStream_t g_stream = nullptr;
std::mutex g_live_mu;
std::unordered_set<cudaStream_t> g_live_streams;

static bool stream_live(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_live_mu);
  return g_live_streams.count(s) != 0;
}

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;  // stream the allocation is ordered on (nullptr: plain cudaMalloc)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) {
      if (s && stream_live(s))
        cudaFreeAsync(p, s);
      else
        cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
    s = nullptr;
  }
  void alloc(size_t b) {
    if (b <= bytes && p) return;
    release();
    s = g_stream;
    if (s)
      KG_CUDA(cudaMallocAsync(&p, b ? b : 8, s));
    else
      KG_CUDA(cudaMalloc(&p, b ? b : 8));
    bytes = b;
  }
  double* d() const { return static_cast<double*>(p); }
  i64* l() const { return static_cast<i64*>(p); }
};

static i64 prod(const std::vector<i64>& v, size_t a, size_t b) {
  i64 s = 1;
  for (size_t i = a; i < b; ++i) s *= v[i];
  return s;
}

}  // namespace kg

// ------------------------------------------------------------------- NCCL
// libnccl is opened at run time (the same soname torch loads), so the library
// has no link-time NCCL dependency and single-GPU use never touches it.
namespace kg {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // point-to-point (halo exchange of banded last-mode sharding); optional
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

static NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
      api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
      api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
      api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
      api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
      if (api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy && api.GetErrorString) api.h = h;
    }
  }
  if (!api.h) throw Error(E_NCCL, "libnccl.so.2 could not be loaded");
  return &api;
}

void smem_attr_raw(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> done;  // (device, kernel) -> bytes set
  int dev = 0;
  KG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first.first == dev && e.first.second == fn) {
      if (e.second >= bytes) return;
      KG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      e.second = bytes;
      return;
    }
  KG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.push_back({{dev, fn}, bytes});
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(E_NCCL, std::string(what) + ": " + nccl_api()->GetErrorString(r));
}
}  // namespace kg

// ------------------------------------------------------------------ context
struct kg_ctx {
  int device = 0;
  cudaStream_t s = nullptr;
  kg::i64 launches = 0;
  std::string err;
  kg::i64 err_cell = -1;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;  // sharded context (kg_ctx_create_sharded): sums over the last-mode slabs
  void* pinned = nullptr;  // small pinned staging area for scalars
  // last whole-path kernel: event-timed device ms, algorithmic bytes, FISTA steps
  double path_ms = -1.0, path_bytes = 0.0;
  kg::i64 path_steps = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t side = nullptr;  // design-time power iterations, overlapped with the observation upload
  void* stage = nullptr;        // page-locked upload ring (kStageLanes x kStageSlots x kStageChunk bytes)
  cudaEvent_t stage_ev[16] = {};
  cudaEvent_t loop_ev[2] = {nullptr, nullptr};  // pipelined host loop of sharded n-space solves
  // fork / join of the FISTA body: the control kernel runs beside the last chain step
  cudaStream_t fork = nullptr;
  cudaEvent_t fork_ev[2] = {nullptr, nullptr};
  kg::Launch L() { return {s, &launches}; }
  double* pin() { return static_cast<double*>(pinned); }
};

// Cross-rank reductions of a sharded context (no-ops on a single GPU): the
// n-space partials of every rank's slab are summed (or max-/min-reduced) in
// place on the context stream, so the replicated p-space state stays equal
// on all ranks.
namespace kg {
static void ar(kg_ctx* ctx, void* d, size_t n, ncclDataType_t t, ncclRedOp_t op) {
  if (!ctx->comm || n == 0) return;
  nccl_check(nccl_api()->AllReduce(d, d, n, t, op, ctx->comm, ctx->s), "ncclAllReduce");
}
static void ar_sum(kg_ctx* ctx, double* d, size_t n) { ar(ctx, d, n, ncclFloat64, ncclSum); }
static void ar_max(kg_ctx* ctx, double* d, size_t n) { ar(ctx, d, n, ncclFloat64, ncclMax); }
static void ar_min_i64(kg_ctx* ctx, int64_t* d, size_t n) { ar(ctx, d, n, ncclInt64, ncclMin); }
static bool sharded(const kg_ctx* ctx) { return ctx->comm != nullptr; }
}  // namespace kg

// Layout of the 4 KB pinned staging area (doubles).
namespace kg {
constexpr int PIN_SCAL = 0;    // [0, 64): reduced scalars
constexpr int PIN_ERR = 64;    // [64, 96): error words (i64)
constexpr int PIN_CTL = 128;   // FistaCtl read back
constexpr int PIN_STAGE = 256; // FistaCtl staged for upload
constexpr int PIN_CTL2 = 384;  // second FistaCtl read-back slot (pipelined host loop)
static_assert(sizeof(FistaCtl) <= 1024, "a FistaCtl must fit one pinned slot");
constexpr int ERR_FAM = 12;    // errs[12], errs[13]: family score / working response
}  // namespace kg

namespace kg {

static void sync(kg_ctx* c) { KG_CUDA(cudaStreamSynchronize(c->s)); }

// ------------------------------------------------------------------ design
struct FactorHost {
  i64 n = 0, p = 0;
  std::vector<double> X;  // column-major
};

static void build_band(const FactorHost& h, bool rows_of_x, std::vector<int>& lo, std::vector<int>& len,
                       std::vector<i64>& off, std::vector<double>& coef, int& maxlen) {
  // rows_of_x: operator = X (rows i, columns k); else operator = X^T.
  const i64 R = rows_of_x ? h.n : h.p, K = rows_of_x ? h.p : h.n;
  lo.assign(R, 0);
  len.assign(R, 0);
  off.assign(R, 0);
  coef.clear();
  maxlen = 0;
  // first / last nonzero of every operator row; the factor is column-major, so
  // the row bands of X come from one sweep down its columns (a row-wise scan
  // strides by n doubles: 10 ms for a 4096 x 256 factor)
  std::vector<i64> first(static_cast<size_t>(R), -1), last(static_cast<size_t>(R), -1);
  if (rows_of_x) {
    for (i64 k = 0; k < K; ++k) {
      const double* col = h.X.data() + h.n * k;
      for (i64 r = 0; r < R; ++r)
        if (col[r] != 0.0) {
          if (first[static_cast<size_t>(r)] < 0) first[static_cast<size_t>(r)] = k;
          last[static_cast<size_t>(r)] = k;
        }
    }
  } else {
    for (i64 r = 0; r < R; ++r) {
      const double* col = h.X.data() + h.n * r;
      for (i64 k = 0; k < K; ++k)
        if (col[k] != 0.0) {
          if (first[static_cast<size_t>(r)] < 0) first[static_cast<size_t>(r)] = k;
          last[static_cast<size_t>(r)] = k;
        }
    }
  }
  for (i64 r = 0; r < R; ++r) {
    off[r] = static_cast<i64>(coef.size());
    const i64 a = first[static_cast<size_t>(r)], b = last[static_cast<size_t>(r)];
    if (a < 0) continue;
    lo[r] = static_cast<int>(a);
    len[r] = static_cast<int>(b - a + 1);
    maxlen = std::max(maxlen, len[r]);
    for (i64 k = a; k <= b; ++k) coef.push_back(rows_of_x ? h.X[r + h.n * k] : h.X[k + h.n * r]);
  }
}

struct FactorOwn {
  FactorDev dev;
  DBuf X, hlo, hlen, hoff, hcoef, glo, glen, goff, gcoef, rblo, rbcoef, wblo, wbcoef, hblo, hbcoef;
  std::vector<int> h_lo, h_len, g_lo, g_len;  // host copies for launch planning
  DBuf mbase, mfrag;                          // X^T as DMMA fragments (fused pass)
  MmaOp mg;
};

// X^T as DMMA A fragments for the fused pass (see MmaOp).
// Small host->device copies of kg_design_create (factor bands, Gram blocks,
// power-iteration jobs) go through a page-locked arena when one is active:
// a pageable cudaMemcpyAsync synchronises the stream first, and design
// creation issues dozens of them behind its own kernels.
struct HostArena {
  char* base = nullptr;
  size_t cap = 0, off = 0;
};
static thread_local HostArena* g_arena = nullptr;
static void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (g_arena && g_arena->off + bytes <= g_arena->cap) {
    char* b = g_arena->base + g_arena->off;
    std::memcpy(b, src, bytes);
    g_arena->off += (bytes + 255) & ~size_t(255);
    KG_CUDA(cudaMemcpyAsync(dst, b, bytes, cudaMemcpyHostToDevice, st));
  } else {
    KG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  }
}

static void build_mma(const FactorHost& h, const std::vector<int>& glo, const std::vector<int>& glen, FactorOwn& f,
                      cudaStream_t st) {
  const i64 p = h.p, n = h.n;
  const int groups = static_cast<int>((p + kMmaK - 1) / kMmaK);
  int W = 0;
  std::vector<int> lo(static_cast<size_t>(groups), 0);
  for (int g = 0; g < groups; ++g) {
    int a = INT32_MAX, b = 0;
    for (i64 k = static_cast<i64>(g) * kMmaK; k < std::min<i64>(p, (g + 1) * kMmaK); ++k)
      if (glen[k] > 0) {
        a = std::min(a, glo[k]);
        b = std::max(b, glo[k] + glen[k]);
      }
    if (a == INT32_MAX) a = b = 0;
    lo[static_cast<size_t>(g)] = a;
    W = std::max(W, b - a);
  }
  // k-steps padded to the kernel's unrolled counts (8, 12, 16), zero fragments
  // past the band, so the DMMA loop carries no predicates
  const int need = (std::max(W, 1) + 3) / 4;
  const int ks = need <= 8 ? 8 : need <= 12 ? 12 : need <= 16 ? 16 : 0;
  if (ks == 0 || 4 * ks > n) return;  // window too wide or the factor too short: k_fused_fast only
  std::vector<int> base(static_cast<size_t>(groups));
  std::vector<double> frag(static_cast<size_t>(groups) * ks * 32, 0.0);
  for (int g = 0; g < groups; ++g) {
    const int b0 = static_cast<int>(std::min<i64>(lo[static_cast<size_t>(g)], n - 4 * ks));
    base[static_cast<size_t>(g)] = b0;
    for (int s2 = 0; s2 < ks; ++s2)
      for (int lane = 0; lane < 32; ++lane) {
        const i64 k = static_cast<i64>(g) * kMmaK + lane / 4;
        const int r = b0 + 4 * s2 + lane % 4;
        if (k < p && r >= glo[k] && r < glo[k] + glen[k])
          frag[(static_cast<size_t>(g) * ks + s2) * 32 + lane] = h.X[r + n * k];
      }
  }
  f.mbase.alloc(sizeof(int) * base.size());
  f.mfrag.alloc(sizeof(double) * frag.size());
  h2d(f.mbase.p, base.data(), sizeof(int) * base.size(), st);
  h2d(f.mfrag.p, frag.data(), sizeof(double) * frag.size(), st);
  f.mg.base = static_cast<const int*>(f.mbase.p);
  f.mg.afrag = f.mfrag.d();
  f.mg.ks = ks;
  f.mg.groups = groups;
}

static uint64_t next_band_uid() {
  static uint64_t uid = 0;
  return ++uid;
}

static void upload_factor(const FactorHost& h, FactorOwn& f, cudaStream_t s) {
  f.dev.n = h.n;
  f.dev.p = h.p;
  f.X.alloc(sizeof(double) * h.n * h.p);
  h2d(f.X.p, h.X.data(), sizeof(double) * h.n * h.p, s);
  f.dev.X = f.X.d();
  auto up = [&](bool rows, DBuf& blo, DBuf& blen, DBuf& boff, DBuf& bcoef, BandOp& op, std::vector<int>& lo,
                std::vector<int>& len) {
    std::vector<i64> off;
    std::vector<double> coef;
    int maxlen = 0;
    build_band(h, rows, lo, len, off, coef, maxlen);
    blo.alloc(sizeof(int) * lo.size());
    blen.alloc(sizeof(int) * len.size());
    boff.alloc(sizeof(i64) * off.size());
    bcoef.alloc(sizeof(double) * std::max<size_t>(coef.size(), 1));
    // pageable sources: cudaMemcpyAsync returns once the host data is staged
    h2d(blo.p, lo.data(), sizeof(int) * lo.size(), blo.s);
    h2d(blen.p, len.data(), sizeof(int) * len.size(), blen.s);
    h2d(boff.p, off.data(), sizeof(i64) * off.size(), boff.s);
    if (!coef.empty())
      h2d(bcoef.p, coef.data(), sizeof(double) * coef.size(), bcoef.s);
    op.lo = static_cast<const int*>(blo.p);
    op.len = static_cast<const int*>(blen.p);
    op.off = static_cast<const i64*>(boff.p);
    op.coef = bcoef.d();
    op.rows = rows ? h.n : h.p;
    op.cols = rows ? h.p : h.n;
    op.maxlen = maxlen;
    op.hlo = lo.data();
    op.hlen = len.data();
    op.uid = next_band_uid();
  };
  up(true, f.hlo, f.hlen, f.hoff, f.hcoef, f.dev.H, f.h_lo, f.h_len);
  up(false, f.glo, f.glen, f.goff, f.gcoef, f.dev.G, f.g_lo, f.g_len);
  build_mma(h, f.g_lo, f.g_len, f, s);
  // row-blocked copy of the H operator when every group of kRB rows reads a
  // window of at most kRW inputs (B-spline rows: 4 nonzeros, slowly moving)
  const i64 rows = h.n, groups = (rows + kRB - 1) / kRB;
  bool ok = f.dev.H.maxlen <= kRW;
  std::vector<int> wlo(static_cast<size_t>(groups), 0);
  std::vector<double> wc(static_cast<size_t>(groups * kRB * kRW), 0.0);
  for (i64 g = 0; g < groups && ok; ++g) {
    int lo = INT32_MAX, hi = 0;
    for (i64 r = g * kRB; r < std::min(rows, (g + 1) * kRB); ++r)
      if (f.h_len[r] > 0) {
        lo = std::min(lo, f.h_lo[r]);
        hi = std::max(hi, f.h_lo[r] + f.h_len[r]);
      }
    if (lo == INT32_MAX) lo = hi = 0;
    if (hi - lo > kRW || lo + kRW > h.p) {  // window must stay inside the input extent
      lo = static_cast<int>(std::max<i64>(0, std::min<i64>(lo, h.p - kRW)));
      if (hi - lo > kRW || h.p < kRW) ok = false;
    }
    wlo[static_cast<size_t>(g)] = lo;
    for (i64 r = g * kRB; r < std::min(rows, (g + 1) * kRB) && ok; ++r)
      for (int t = 0; t < f.h_len[r]; ++t)
        wc[static_cast<size_t>(((g * kRB + (r - g * kRB)) * kRW) + (f.h_lo[r] + t - lo))] = h.X[r + h.n * (f.h_lo[r] + t)];
  }
  if (ok) {
    f.rblo.alloc(sizeof(int) * groups);
    f.rbcoef.alloc(sizeof(double) * wc.size());
    h2d(f.rblo.p, wlo.data(), sizeof(int) * groups, f.rblo.s);
    h2d(f.rbcoef.p, wc.data(), sizeof(double) * wc.size(), f.rbcoef.s);
    f.dev.H.blo = static_cast<const int*>(f.rblo.p);
    f.dev.H.bcoef = f.rbcoef.d();
  }
  // wide-window row-blocked copies: G (rows = columns of X, kGB basis
  // functions per window of kGW grid rows) and H (rows of X, kHB grid rows per
  // window of kHW basis functions)
  auto blocked = [&](int RB, int RW, i64 rows, i64 in_ext, const std::vector<int>& blo_r, const std::vector<int>& blen_r,
                     bool transpose, DBuf& dlo, DBuf& dcoef, const int*& olo, const double*& ocoef) {
    const i64 groups = (rows + RB - 1) / RB;
    bool ok = dev_env("KG_NO_GB") == nullptr && in_ext >= RW;
    std::vector<int> wl(static_cast<size_t>(groups), 0);
    std::vector<double> wc(static_cast<size_t>(groups * RB * RW), 0.0);
    for (i64 g = 0; g < groups && ok; ++g) {
      int lo = INT32_MAX, hi = 0;
      for (i64 r = g * RB; r < std::min(rows, (g + 1) * RB); ++r)
        if (blen_r[r] > 0) {
          lo = std::min(lo, blo_r[r]);
          hi = std::max(hi, blo_r[r] + blen_r[r]);
        }
      if (lo == INT32_MAX) lo = hi = 0;
      if (hi - lo > RW) ok = false;
      lo = static_cast<int>(std::max<i64>(0, std::min<i64>(lo, in_ext - RW)));  // window inside the input extent
      if (hi > lo + RW) ok = false;
      wl[static_cast<size_t>(g)] = lo;
      for (i64 r = g * RB; r < std::min(rows, (g + 1) * RB) && ok; ++r)
        for (int t = 0; t < blen_r[r]; ++t) {
          const i64 c = blo_r[r] + t;  // G: X^T[r, c] = X[c, r]; H: X[r, c]
          wc[static_cast<size_t>(((g * RB + (r - g * RB)) * RW) + (c - lo))] = transpose ? h.X[c + h.n * r] : h.X[r + h.n * c];
        }
    }
    if (!ok) return;
    dlo.alloc(sizeof(int) * groups);
    dcoef.alloc(sizeof(double) * wc.size());
    h2d(dlo.p, wl.data(), sizeof(int) * groups, dlo.s);
    h2d(dcoef.p, wc.data(), sizeof(double) * wc.size(), dcoef.s);
    olo = static_cast<const int*>(dlo.p);
    ocoef = dcoef.d();
  };
  blocked(kGB, kGW, h.p, h.n, f.g_lo, f.g_len, true, f.wblo, f.wbcoef, f.dev.G.wblo, f.dev.G.wbcoef);
  blocked(kHB, kHW, h.n, h.p, f.h_lo, f.h_len, false, f.hblo, f.hbcoef, f.dev.H.hblo, f.dev.H.hbcoef);
}

// Spectral radius of X^T X for one factor: banded Gram + single-warp power
// iteration on the device; start vector exactly as spectral.cpp:17-23.
// Spectral radius of X^T X for one factor (spectral.cpp:8-42): the Gram and
// start vector are prepared per factor; every factor of a design then runs its
// power iteration in one batched launch (spectral_run).
struct SpectralJob {
  i64 p = 0;
  double immediate = -1.0;  // p == 1: |sum x^2| directly (spectral.cpp:14)
  DBuf G, glo, ghi, v0;
  int band = 0;
  const double* Gview = nullptr;  // dense Gram owned elsewhere (tensor weights); p == 1: its single entry
};

static void spectral_prepare(kg_ctx* ctx, const FactorHost& h, FactorOwn& f, SpectralJob& J) {
  const i64 p = h.p;
  J.p = p;
  // column bands of X (rows where column k is nonzero)
  std::vector<int> clo(p), chi(p);
  for (i64 k = 0; k < p; ++k) {
    i64 first = -1, last = -1;
    for (i64 i = 0; i < h.n; ++i)
      if (h.X[i + h.n * k] != 0.0) {
        if (first < 0) first = i;
        last = i;
      }
    clo[k] = first < 0 ? 0 : static_cast<int>(first);
    chi[k] = first < 0 ? 0 : static_cast<int>(last + 1);
  }
  std::vector<int> glo(p, 0), ghi(p, 0);
  int band = 0;
  for (i64 a = 0; a < p; ++a) {
    i64 first = -1, last = -1;
    for (i64 b = 0; b < p; ++b)
      if (std::max(clo[a], clo[b]) < std::min(chi[a], chi[b])) {
        if (first < 0) first = b;
        last = b;
      }
    glo[a] = first < 0 ? 0 : static_cast<int>(first);
    ghi[a] = first < 0 ? 0 : static_cast<int>(last + 1);
    band = std::max(band, ghi[a] - glo[a]);
  }
  J.band = band;
  if (p == 1) {  // spectral.cpp:14
    double s = 0.0;
    for (i64 i = 0; i < h.n; ++i) s += h.X[i] * h.X[i];
    J.immediate = std::abs(s);
    return;
  }
  std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
  std::uniform_real_distribution<double> unif(0.5, 1.5);
  std::vector<double> v0(p);
  for (i64 i = 0; i < p; ++i) v0[i] = unif(rng);
  double z = 0.0;
  for (double x : v0) z += x * x;
  if (z > 0.0) {
    const double sq = std::sqrt(z);
    for (double& x : v0) x /= sq;
  }
  J.G.alloc(sizeof(double) * p * p);
  KG_CUDA(cudaMemsetAsync(J.G.p, 0, sizeof(double) * p * p, ctx->s));
  J.glo.alloc(sizeof(int) * p);
  J.ghi.alloc(sizeof(int) * p);
  J.v0.alloc(sizeof(double) * p);
  h2d(J.glo.p, glo.data(), sizeof(int) * p, ctx->s);
  h2d(J.ghi.p, ghi.data(), sizeof(int) * p, ctx->s);
  h2d(J.v0.p, v0.data(), sizeof(double) * p, ctx->s);
  gram(ctx->L(), f.dev, J.G.d(), static_cast<int*>(J.glo.p), static_cast<int*>(J.ghi.p));
}

static std::vector<double> spectral_run(kg_ctx* ctx, std::vector<std::unique_ptr<SpectralJob>>& jobs);

// spectral_run over jobs whose Grams live in Gview (the 1 x 1 case reads its
// device entry: spectral.cpp:14 returns |G|)
static std::vector<double> spectral_run_views(kg_ctx* ctx, std::vector<std::unique_ptr<SpectralJob>>& jobs) {
  for (auto& J : jobs) {
    if (J->p == 1) {
      double g = 0.0;
      KG_CUDA(cudaMemcpyAsync(&g, J->Gview, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
      sync(ctx);
      J->immediate = std::abs(g);
    }
  }
  return spectral_run(ctx, jobs);
}

static std::vector<double> spectral_run(kg_ctx* ctx, std::vector<std::unique_ptr<SpectralJob>>& jobs) {
  std::vector<PowerJob> pj;
  std::vector<size_t> idx;
  i64 max_p = 1;
  for (size_t k = 0; k < jobs.size(); ++k) {
    SpectralJob& J = *jobs[k];
    if (J.immediate >= 0.0) continue;
    PowerJob q;
    q.p = J.p;
    q.G = J.Gview ? J.Gview : J.G.d();
    q.glo = static_cast<const int*>(J.glo.p);
    q.ghi = static_cast<const int*>(J.ghi.p);
    q.v0 = J.v0.d();
    q.band = J.band;
    pj.push_back(q);
    idx.push_back(k);
    max_p = std::max(max_p, J.p);
  }
  std::vector<double> vals(jobs.size(), 0.0);
  for (size_t k = 0; k < jobs.size(); ++k)
    if (jobs[k]->immediate >= 0.0) vals[k] = jobs[k]->immediate;
  if (pj.empty()) return vals;
  DBuf out, djobs;
  out.alloc(sizeof(double) * 3 * pj.size());
  for (size_t k = 0; k < pj.size(); ++k) pj[k].out = out.d() + 3 * k;
  djobs.alloc(sizeof(PowerJob) * pj.size());
  h2d(djobs.p, pj.data(), sizeof(PowerJob) * pj.size(), ctx->s);
  power_iterations(ctx->L(), static_cast<const PowerJob*>(djobs.p), static_cast<int>(pj.size()), max_p, 1e-14,
                   500000);
  std::vector<double> res(3 * pj.size());
  KG_CUDA(cudaMemcpyAsync(res.data(), out.p, sizeof(double) * res.size(), cudaMemcpyDeviceToHost, ctx->s));
  sync(ctx);
  static const bool trace = dev_env("KG_POWER_TRACE") != nullptr;
  for (size_t k = 0; k < pj.size(); ++k) {
    if (trace)
      std::fprintf(stderr, "kg power job %zu: p=%lld band=%d value=%.17g iterations=%.0f\n", k,
                   static_cast<long long>(pj[k].p), pj[k].band, res[3 * k], res[3 * k + 1]);
    if (res[3 * k + 2] != 0.0) throw Error(E_POWER, "power iteration did not converge after 500000 iterations");
    vals[idx[k]] = res[3 * k];
  }
  return vals;
}

// spectral_run split in two: launch on the context's side stream (after the
// jobs' inputs, which were prepared on the main stream) into page-locked
// results, then collect when the radii are first needed.
struct SpectralPending {
  std::vector<std::unique_ptr<SpectralJob>> jobs;
  std::vector<size_t> idx;
  std::vector<double> vals;
  DBuf out, djobs;
  std::vector<PowerJob> pj;
  double* host = nullptr;  // page-locked 3 doubles per power job
  cudaEvent_t done = nullptr;
  ~SpectralPending() {
    if (done) {
      cudaEventSynchronize(done);
      cudaEventDestroy(done);
    }
    if (host) cudaFreeHost(host);
  }
};

static std::unique_ptr<SpectralPending> spectral_launch(kg_ctx* ctx, std::vector<std::unique_ptr<SpectralJob>>& jobs) {
  auto S = std::make_unique<SpectralPending>();
  i64 max_p = 1;
  S->vals.assign(jobs.size(), 0.0);
  for (size_t k = 0; k < jobs.size(); ++k) {
    SpectralJob& J = *jobs[k];
    if (J.immediate >= 0.0) {
      S->vals[k] = J.immediate;
      continue;
    }
    PowerJob q;
    q.p = J.p;
    q.G = J.Gview ? J.Gview : J.G.d();
    q.glo = static_cast<const int*>(J.glo.p);
    q.ghi = static_cast<const int*>(J.ghi.p);
    q.v0 = J.v0.d();
    q.band = J.band;
    S->pj.push_back(q);
    S->idx.push_back(k);
    max_p = std::max(max_p, J.p);
  }
  S->jobs = std::move(jobs);
  if (S->pj.empty()) return S;
  S->out.alloc(sizeof(double) * 3 * S->pj.size());
  for (size_t k = 0; k < S->pj.size(); ++k) S->pj[k].out = S->out.d() + 3 * k;
  S->djobs.alloc(sizeof(PowerJob) * S->pj.size());
  h2d(S->djobs.p, S->pj.data(), sizeof(PowerJob) * S->pj.size(), ctx->s);
  KG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S->host), sizeof(double) * 3 * S->pj.size(), cudaHostAllocDefault));
  if (!ctx->side) KG_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  cudaEvent_t ready;
  KG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  KG_CUDA(cudaEventRecord(ready, ctx->s));  // job inputs and buffers are in place
  KG_CUDA(cudaStreamWaitEvent(ctx->side, ready, 0));
  KG_CUDA(cudaEventDestroy(ready));
  power_iterations({ctx->side, &ctx->launches}, static_cast<const PowerJob*>(S->djobs.p),
                   static_cast<int>(S->pj.size()), max_p, 1e-14, 500000);
  KG_CUDA(cudaMemcpyAsync(S->host, S->out.p, sizeof(double) * 3 * S->pj.size(), cudaMemcpyDeviceToHost, ctx->side));
  KG_CUDA(cudaEventCreateWithFlags(&S->done, cudaEventDisableTiming));
  KG_CUDA(cudaEventRecord(S->done, ctx->side));
  // the jobs' buffers live in S until spectral_collect has waited for `done`
  return S;
}

static std::vector<double> spectral_collect(SpectralPending& S) {
  if (S.done) KG_CUDA(cudaEventSynchronize(S.done));
  static const bool trace = dev_env("KG_POWER_TRACE") != nullptr;
  for (size_t k = 0; k < S.pj.size(); ++k) {
    if (trace)
      std::fprintf(stderr, "kg power job %zu: p=%lld band=%d value=%.17g iterations=%.0f\n", k,
                   static_cast<long long>(S.pj[k].p), S.pj[k].band, S.host[3 * k], S.host[3 * k + 1]);
    if (S.host[3 * k + 2] != 0.0) throw Error(E_POWER, "power iteration did not converge after 500000 iterations");
    S.vals[S.idx[k]] = S.host[3 * k];
  }
  return S.vals;
}

// Per-chunk X2 fragments of the slab pass (SlabArgs; d = 3, one component).
struct SlabTables {
  DBuf w0, tz, x2u, x2z, gat;
  int nch = 0, gmax = 0, PL = 0;
};

// Gather table of the scatter/gather Y step (SlabArgs::gat) from the dense
// mode-1 factor X1 (n1 x p1, column-major): the host plan kg_slab_gather_plan
// (row quad q scatters its five window partials to slots 5q .. 5q + 4 of its
// column pair's plane; basis function k sums, in ascending quad order, the
// slots of the quads that have a row with k inside its band), packed as 8
// 16-bit slots per basis function.
static void build_slab_gather(SlabTables& T, const double* X1, i64 n1, i64 p1, cudaStream_t st) {
  const int groups = static_cast<int>((p1 + 7) / 8);
  std::vector<int32_t> slots(static_cast<size_t>(groups) * 64);
  int32_t gmax = 0, PL = 0;
  if (kg_slab_gather_plan(n1, p1, X1, slots.data(), &gmax, &PL) != KG_OK) return;  // the pass keeps its DMMA form
  std::vector<int> gat(static_cast<size_t>(groups) * 8 * 4);
  for (size_t k = 0; k < static_cast<size_t>(groups) * 8; ++k)
    for (int j = 0; j < 4; ++j) gat[k * 4 + j] = slots[k * 8 + 2 * j] | (slots[k * 8 + 2 * j + 1] << 16);
  T.gat.alloc(sizeof(int) * gat.size());
  h2d(T.gat.p, gat.data(), sizeof(int) * gat.size(), st);
  T.gmax = gmax;
  T.PL = PL;
}

// Builds the slab tables from the dense mode-2 factor X2 (n x p, column-major)
// when every chunk of 8 grid rows reads an 8-wide coefficient window; returns
// null otherwise (the design then keeps the mode-1 fused route).
static std::unique_ptr<SlabTables> build_slab(const double* X, i64 n, i64 p, cudaStream_t st) {
  if (p < 8 || p > 64 || n < 1) return nullptr;
  const int nch = static_cast<int>((n + 7) / 8);
  std::vector<int> w0(static_cast<size_t>(nch)), tz(static_cast<size_t>(nch));
  std::vector<double> xu(static_cast<size_t>(nch) * 64, 0.0), xz(static_cast<size_t>(nch) * 128, 0.0);
  auto at = [&](i64 r, i64 k) { return (r >= 0 && r < n && k >= 0 && k < p) ? X[r + n * k] : 0.0; };
  for (int c = 0; c < nch; ++c) {
    i64 lo = p, hi = 0;
    for (i64 r = 8 * c; r < std::min<i64>(n, 8 * c + 8); ++r)
      for (i64 k = 0; k < p; ++k)
        if (X[r + n * k] != 0.0) {
          lo = std::min(lo, k);
          hi = std::max(hi, k + 1);
        }
    if (lo >= hi) lo = hi = 0;
    const i64 wz = std::max<i64>(0, std::min<i64>(lo, p - 8));
    if (hi > wz + 8) return nullptr;
    const i64 t0 = lo / 8, two = hi > 8 * t0 + 8 ? 1 : 0;  // aligned 8-column tiles of the Z step
    w0[static_cast<size_t>(c)] = static_cast<int>(wz);
    tz[static_cast<size_t>(c)] = static_cast<int>(t0 | (two << 16));
    for (int s2 = 0; s2 < 2; ++s2)
      for (int lane = 0; lane < 32; ++lane) {
        xu[static_cast<size_t>(c) * 64 + s2 * 32 + lane] = at(8 * c + lane / 4, wz + 4 * s2 + lane % 4);
        for (int tl = 0; tl < 2; ++tl)
          xz[static_cast<size_t>(c) * 128 + (tl * 2 + s2) * 32 + lane] =
              at(8 * c + 2 * (lane % 4) + s2, 8 * (t0 + tl) + lane / 4);
      }
  }
  auto T = std::make_unique<SlabTables>();
  T->nch = nch;
  T->w0.alloc(sizeof(int) * w0.size());
  T->tz.alloc(sizeof(int) * tz.size());
  T->x2u.alloc(sizeof(double) * xu.size());
  T->x2z.alloc(sizeof(double) * xz.size());
  h2d(T->w0.p, w0.data(), sizeof(int) * w0.size(), st);
  h2d(T->tz.p, tz.data(), sizeof(int) * tz.size(), st);
  h2d(T->x2u.p, xu.data(), sizeof(double) * xu.size(), st);
  h2d(T->x2z.p, xz.data(), sizeof(double) * xz.size(), st);
  return T;
}

}  // namespace kg

struct kg_design {
  kg_ctx* ctx = nullptr;
  kg::i64 c = 0, d = 0;
  std::vector<kg::i64> n;                  // local extents (last mode = this shard's slab)
  std::vector<kg::i64> n_full;             // global extents
  std::vector<std::vector<kg::i64>> p;     // p[r][j]
  std::vector<kg::i64> offs;
  kg::i64 N = 0, N_full = 0, P = 0;
  kg::i64 cell_base = 0;                   // global flat index of the first local cell
  std::vector<std::vector<std::unique_ptr<kg::FactorOwn>>> f;
  // Gram blocks X_{m,j}^T X_{r,j} (design.cpp:126-151 with unit weight factors)
  // as banded operators: gram[m][r][j]->dev.H maps p_{r,j} -> p_{m,j}.
  std::vector<std::vector<std::vector<std::unique_ptr<kg::FactorOwn>>>> gram;
  std::vector<std::vector<double>> spectral;
  double lipfac = 0.0;                     // sum_r prod_j rho_rj (inner.cpp:61-70)
  // The power iterations of kg_design_create run on the context's side stream
  // and are collected on first use (ensure_spectral), so the observation
  // upload that usually follows overlaps them.
  mutable std::unique_ptr<kg::SpectralPending> pending;
  bool fused = false;
  int T = 1;                               // mode-1 fibres per CTA in the fused kernels
  std::unique_ptr<kg::SlabTables> slab;    // d = 3, one component: modes 1+2 fused per slice (kg_slab.cu)
  // banded last-mode sharding (kg_halo_plan): {ok, own_lo, own_hi, t_lo, t_hi,
  // L_lo, L_hi, R_lo, R_hi} in coefficient slices of the last mode; ok = 0: all-reduce
  kg::i64 halo[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  kg::i64 scratch = 0;                     // doubles per chain scratch buffer
  kg::i64 part_cap = 0;                    // doubles in the partials buffer
};

namespace kg {
// Host -> device upload of a pageable array.  The driver stages pageable copies
// through its own small buffer at ~11 GB/s; here kStageLanes host threads each
// copy their share of the array chunk by chunk into their own page-locked ring
// slots and queue the DMA, so host copies and PCIe transfers overlap.
// Page-locked or small sources go straight to cudaMemcpyAsync.
constexpr int kStageLanes = 4, kStageSlots = 2;
constexpr size_t kStageChunk = size_t(4) << 20;
static void ensure_stage(kg_ctx* ctx) {
  if (ctx->stage) return;
  KG_CUDA(cudaHostAlloc(&ctx->stage, kStageLanes * kStageSlots * kStageChunk, cudaHostAllocDefault));
  for (int i = 0; i < kStageLanes * kStageSlots; ++i)
    KG_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
}

static void upload(kg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  cudaPointerAttributes at{};
  const bool pageable = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  if (!pageable || bytes < 2 * kStageChunk || dev_env("KG_NO_STAGE")) {
    KG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->s));
    return;
  }
  ensure_stage(ctx);
  const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
  std::vector<std::string> errs(kStageLanes);
  auto lane = [&](int l) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaSetDevice(ctx->device) != cudaSuccess) {
      errs[l] = "cudaSetDevice";
      return;
    }
    int slot = 0;
    for (size_t c = l; c < nchunks; c += kStageLanes, slot ^= 1) {
      const int id = l * kStageSlots + slot;
      char* buf = static_cast<char*>(ctx->stage) + static_cast<size_t>(id) * kStageChunk;
      const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
      if (cudaEventSynchronize(ctx->stage_ev[id]) != cudaSuccess) {  // the slot's previous DMA is done
        errs[l] = "cudaEventSynchronize";
        return;
      }
      std::memcpy(buf, static_cast<const char*>(src) + off, len);
      if (cudaMemcpyAsync(static_cast<char*>(dst) + off, buf, len, cudaMemcpyHostToDevice, ctx->s) != cudaSuccess ||
          cudaEventRecord(ctx->stage_ev[id], ctx->s) != cudaSuccess) {
        errs[l] = "cudaMemcpyAsync";
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (int l = 1; l < kStageLanes; ++l) th.emplace_back(lane, l);
  lane(0);
  for (auto& t : th) t.join();
  for (const std::string& e : errs)
    if (!e.empty()) throw Error(E_CUDA, "staged upload: " + e + " failed");
}

// Collect the design's deferred spectral radii (kg_design_create) and form
// lipschitz_upper's factor sum_r prod_j rho_rj (inner.cpp:61-70).
static void ensure_spectral(const kg_design* D) {
  if (!D || !D->pending) return;
  kg_design* M = const_cast<kg_design*>(D);  // the radii are part of the design's value; filled once
  const std::vector<double> rad = spectral_collect(*D->pending);
  M->lipfac = 0.0;
  for (i64 r = 0; r < D->c; ++r) {
    double pr = 1.0;
    for (i64 j = 0; j < D->d; ++j) {
      M->spectral[r][j] = rad[r * D->d + j];
      pr *= rad[r * D->d + j];
    }
    M->lipfac += pr;
  }
  D->pending.reset();
}
}  // namespace kg

struct kg_obs {
  kg_ctx* ctx = nullptr;
  const kg_design* design = nullptr;
  kg::DBuf y, a;
  bool unit_a = true;
  bool a_const = true;  // every prior weight equal (to a_val): weights V are then a constant
  double a_val = 1.0;
};

namespace kg {

// ------------------------------------------------------------------ chains
// Applies a sequence of banded mode contractions.  dims: current extents;
// steps: (mode j, operator, new extent).  The last step writes `out`.
struct Step {
  int mode;
  const BandOp* op;
  i64 next;
};

static void run_chain(kg_ctx* ctx, std::vector<i64> dims, const std::vector<Step>& steps, const double* in,
                      double* out, double* s0, double* s1, bool accumulate_last, bool pdl = false) {
  const double* cur = in;
  Launch L = ctx->L();
  L.pdl = pdl;
  for (size_t k = 0; k < steps.size(); ++k) {
    const Step& st = steps[k];
    const bool last = k + 1 == steps.size();
    double* dst = last ? out : (k % 2 == 0 ? s0 : s1);
    const i64 a = prod(dims, 0, st.mode), K = dims[st.mode], b = prod(dims, st.mode + 1, dims.size());
    contract(L, cur, dst, a, K, st.next, b, *st.op, last && accumulate_last);
    dims[st.mode] = st.next;
    cur = dst;
  }
}

// H chain of component r from its coefficient block: modes d-1 .. stop (stop = 0 full, 1 partial).
static std::vector<Step> h_steps(const kg_design& D, i64 r, int stop) {
  std::vector<Step> st;
  for (i64 j = D.d - 1; j >= stop; --j) st.push_back({static_cast<int>(j), &D.f[r][j]->dev.H, D.n[j]});
  return st;
}
// G chain of component r: modes start .. d-1
static std::vector<Step> g_steps(const kg_design& D, i64 r, int start) {
  std::vector<Step> st;
  for (i64 j = start; j < D.d; ++j) st.push_back({static_cast<int>(j), &D.f[r][j]->dev.G, D.p[r][j]});
  return st;
}

static std::vector<i64> coef_dims(const kg_design& D, i64 r) { return D.p[r]; }

// Max intermediate (non-final) size of every chain the solver runs.
static i64 chain_scratch(const kg_design& D) {
  i64 mx = 1;
  for (i64 r = 0; r < D.c; ++r) {
    std::vector<i64> dims = D.p[r];
    for (i64 j = D.d - 1; j >= 0; --j) {  // H: p -> n
      dims[j] = D.n[j];
      mx = std::max(mx, prod(dims, 0, dims.size()));
    }
    dims = D.n;
    for (i64 j = 0; j < D.d; ++j) {  // G: n -> p
      dims[j] = D.p[r][j];
      mx = std::max(mx, prod(dims, 0, dims.size()));
    }
  }
  return mx;
}

// ------------------------------------------------------------- fit state
struct Fit {
  kg_ctx* ctx;
  const kg_design* D;
  const kg_obs* O;
  int fam = 0, pen = 0;
  double disp = 1.0, alpha = 0.0;
  i64 n = 0, p = 0;
  // p-space
  DBuf x, xp, Sx, Sxp, best, Sbest, b, theta, Jpart, tpart;
  // n-space
  DBuf v, z, u, eta, eta_t, w, hs, P, Q, s0, s1;  // hs: generic-route eta scratch
  DBuf part, scal, errs, ctl;
  const double* zptr = nullptr;  // z or y (Gaussian shortcut)
  int n_ss = 0;
  // X^T W X route of the current inner problem: 0 = n-space pass (any weights),
  // 1 = Gram route (constant weights W = wconst I: X^T W X = wconst (x)_j X_j^T X_j,
  // the reference's xtwx_apply_tensor with constant weight factors)
  int route = 0;
  // route 0 on the fused design: objective sum v eta^2 - 2 <b, x> + sum v z^2
  // (FV_FISTA_EXP, z is not read per iteration); KG_ROUTE0_DIRECT=1 keeps sum v (eta - z)^2
  bool expand = false;
  // route 0, FV_FISTA_EXP on a d = 3 design with slab tables: the slab pass
  // (modes 1 and 2 fused per last-mode slice, kg_slab.cu) replaces the
  // mode-1 fused pass and the mode-2 chain steps
  bool slab = false;
  // banded last-mode sharding for the current fista_solve (kg_design::halo):
  // the update runs on the owned coefficient slices only and the per-gradient
  // exchange is the boundary slices with the two neighbours, not a p-sized all-reduce
  bool halo = false;
  DBuf htmp;
  // iwls = tensor: the current outer iteration's weighted Gram blocks
  // X_{m,j}^T diag(f_j) X_{r,j} (same band structure as design.gram) and the
  // Lipschitz factor (prod_j rho(G_j(f_j)) for c = 1, max(v) L-hat otherwise)
  bool tensor = false;
  double lipfac_t = 0.0;
  DBuf bt_y, bt_g, bt_c, bt_sc, bt_part;  // nu = 0: y, grad, candidate, S(candidate), partials
  std::vector<BandOp> wg;             // [(m * c + r) * d + j]
  std::vector<std::unique_ptr<DBuf>> wgcoef;
  DBuf tS, tf, text, tdense;
  std::vector<std::unique_ptr<SpectralJob>> tjobs;  // power iterations of the weighted Grams (c = 1)
  DBuf bxpart;
  double wconst = 1.0;     // the constant weight (route 1)
  bool c0_valid = false;   // F.scal[48] holds sum v z^2 for the current (v, z)
  // route 1 with one component: one fused kernel per iteration (kg_gram.cu)
  bool gstep = false;
  int persist = -1;  // -1 unknown, 0 no, 1: the whole solve runs in one cooperative kernel
  bool persist_solve = false;  // the last solve ran persistent (launch accounting)
  DBuf gpart, gcount, stheta, pX, pbar, pflags;
  // one captured FISTA graph per route
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  cudaGraph_t graph[2] = {nullptr, nullptr};
  i64 kernels_per_iter[2] = {0, 0};
  ~Fit() {
    for (int r = 0; r < 2; ++r) {
      if (exec[r]) cudaGraphExecDestroy(exec[r]);
      if (graph[r]) cudaGraphDestroy(graph[r]);
    }
  }
};

static FusedArgs fused_args(const Fit& F);
static SlabArgs slab_args(const Fit& F);


static void alloc_fit(Fit& F) {
  ensure_spectral(F.D);
  const kg_design& D = *F.D;
  F.n = D.N;
  F.p = D.P;
  const size_t pb = sizeof(double) * F.p, nb = sizeof(double) * F.n;
  for (DBuf* b : {&F.x, &F.xp, &F.Sx, &F.Sxp, &F.best, &F.Sbest, &F.b, &F.theta}) b->alloc(pb);
  for (DBuf* b : {&F.v, &F.z, &F.u, &F.eta, &F.eta_t}) b->alloc(nb);
  if (!D.fused) {
    F.w.alloc(nb);
    F.hs.alloc(nb);
  }
  if (D.fused && D.d > 1) {
    const i64 pq = D.N / D.n[0] * D.p[0][0];
    F.P.alloc(sizeof(double) * pq);
    F.Q.alloc(sizeof(double) * pq);
  } else if (D.fused) {
    F.Q.alloc(pb);
  }
  F.s0.alloc(sizeof(double) * D.scratch);
  F.s1.alloc(sizeof(double) * D.scratch);
  F.part.alloc(sizeof(double) * D.part_cap);
  F.Jpart.alloc(sizeof(double) * 2 * pgrid(F.p));
  F.bxpart.alloc(sizeof(double) * pgrid(F.p));
  F.expand = false;
  if (D.fused && dev_env("KG_ROUTE0_DIRECT") == nullptr) F.expand = fused_fast_ok(fused_args(F), FV_FISTA_EXP);
  F.slab = F.expand && D.slab && slab_ok(slab_args(F));
  if (D.halo[0] == 1) F.htmp.alloc(sizeof(double) * std::max<i64>(1, (D.halo[6] - D.halo[5]) * (D.P / D.p[0][D.d - 1])));
  F.tpart.alloc(sizeof(double) * 2 * (1 + kMaxTrials) * pgrid(F.p));
  F.scal.alloc(sizeof(double) * 64);
  F.errs.alloc(sizeof(i64) * 16);
  F.ctl.alloc(sizeof(FistaCtl));
  F.stheta.alloc(pb);
  // one-kernel Gram step: one component, d <= 4, slab fits shared memory
  const i64 pd = D.p[0][D.d - 1];
  F.gstep = D.c == 1 && D.d <= 4 && gram_step_fits(D.P / pd);
  if (F.gstep) {
    F.gpart.alloc(sizeof(double) * 12 * pd);  // 3 per CTA, four buffers (k_gauss_path)
    F.pX.alloc(2 * pb);
    F.pbar.alloc(sizeof(unsigned) * 4);
    KG_CUDA(cudaMemsetAsync(F.pbar.p, 0, sizeof(unsigned) * 4, F.ctx->s));
    F.pflags.alloc(sizeof(unsigned) * 32 * pd);  // one 128-byte line per CTA (kFlagStride)
    F.gcount.alloc(sizeof(unsigned) * 4);
    KG_CUDA(cudaMemsetAsync(F.gcount.p, 0, sizeof(unsigned) * 4, F.ctx->s));
  }
}

static void reset_errs(Fit& F) {
  KG_CUDA(cudaMemsetAsync(F.errs.p, 0x7f, sizeof(i64) * 16, F.ctx->s));  // 0x7f7f.. = "no error"
}
static const i64 kNoErr = 0x7f7f7f7f7f7f7f7fLL;

// Fused-route argument builders (c == 1).
static FusedArgs fused_args(const Fit& F) {
  const kg_design& D = *F.D;
  FusedArgs a;
  a.n1 = D.n[0];
  a.p1 = D.p[0][0];
  a.m = D.N / D.n[0];
  a.T = D.T;
  a.H = D.f[0][0]->dev.H;
  a.G = D.f[0][0]->dev.G;
  a.mg = D.f[0][0]->mg;
  a.cell_base = D.cell_base;
  return a;
}

static SlabArgs slab_args(const Fit& F) {
  const kg_design& D = *F.D;
  SlabArgs a;
  a.n1 = static_cast<int>(D.n[0]);
  a.n2 = static_cast<int>(D.n[1]);
  a.p1 = static_cast<int>(D.p[0][0]);
  a.p2 = static_cast<int>(D.p[0][1]);
  a.m3 = D.n[2];
  a.H1 = D.f[0][0]->dev.H;
  a.g1 = D.f[0][0]->mg;
  if (D.slab) {
    a.nch = D.slab->nch;
    a.w0 = static_cast<const int*>(D.slab->w0.p);
    a.tz = static_cast<const int*>(D.slab->tz.p);
    a.x2u = D.slab->x2u.d();
    a.x2z = D.slab->x2z.d();
    a.gat = static_cast<const int*>(D.slab->gat.p);
    a.gmax = D.slab->gmax;
    a.PL = D.slab->PL;
  }
  a.v = F.v.d();
  a.partial = F.part.d();
  return a;
}

static HlastArgs hlast_args(const Fit& F) {
  const kg_design& D = *F.D;
  HlastArgs h;
  h.n1 = D.n[0];
  h.p1 = D.p[0][0];
  h.m = D.N / D.n[0];
  // longer tiles than the fused kernels': a CTA's P-tile load and barrier are
  // amortised over 4x the cells (P tile <= 48 KB; fewer partials than part_cap)
  h.T = D.T;
  while (h.T * 2 <= 4 * D.T && D.p[0][0] * h.T * 2 * 8 <= 48 * 1024 && (h.m + h.T * 2 - 1) / (h.T * 2) >= 2 * 148)
    h.T *= 2;
  h.H = D.f[0][0]->dev.H;
  h.y = F.O->y.d();
  h.a = F.O->a_const ? nullptr : F.O->a.d();  // constant prior weights are not streamed
  h.a_val = F.O->a_val;
  h.fam = F.fam;
  h.disp = F.disp;
  h.partial = F.part.d();
  h.err = F.errs.l();
  h.cell_base = D.cell_base;
  return h;
}

// Fused mode-1 pass: the bulk-async pipelined kernel when a double-buffered
// tile fits shared memory, else the one-tile-per-CTA kernel.  Returns the
// number of per-CTA partials written.
static int run_fused(kg_ctx* ctx, int variant, const FusedArgs& a) {
  if (fused_tma_fits(a, variant)) {
    fused_tma(ctx->L(), variant, a);
    return fused_tma_grid(a, variant);
  }
  fused_mode1(ctx->L(), variant, a);
  return fused_grid(a);
}

// S(x) = X^T diag(v) X x into Sx, and per-CTA partials of sum v (eta - z)^2
// into F.part (returns the number of partials).
static int xwx_pass_local(Fit& F, const double* x, double* Sx) {
  const kg_design& D = *F.D;
  kg_ctx* ctx = F.ctx;
  if (F.slab) {  // H mode 3 -> slab pass (modes 1, 2 both ways) -> G mode 3
    run_chain(ctx, coef_dims(D, 0), h_steps(D, 0, 2), x, F.P.d(), F.s0.d(), F.s1.d(), false);
    SlabArgs a = slab_args(F);
    a.S = F.P.d();
    a.Q = F.Q.d();
    slab_pass(ctx->L(), a);
    std::vector<i64> dims = {D.p[0][0], D.p[0][1], D.n[2]};
    run_chain(ctx, dims, g_steps(D, 0, 2), F.Q.d(), Sx, F.s0.d(), F.s1.d(), false);
    return slab_grid(a);
  }
  if (D.fused) {
    const double* P = x;
    if (D.d > 1) {
      run_chain(ctx, coef_dims(D, 0), h_steps(D, 0, 1), x, F.P.d(), F.s0.d(), F.s1.d(), false);
      P = F.P.d();
    }
    FusedArgs a = fused_args(F);
    a.P = P;
    a.Q = D.d > 1 ? F.Q.d() : Sx;
    a.v = F.v.d();
    a.z = F.zptr;
    a.partial = F.part.d();
    const int np = run_fused(ctx, F.expand ? FV_FISTA_EXP : FV_FISTA, a);
    if (D.d > 1) {
      std::vector<i64> dims = D.n;
      dims[0] = D.p[0][0];
      run_chain(ctx, dims, g_steps(D, 0, 1), F.Q.d(), Sx, F.s0.d(), F.s1.d(), false);
    }
    return np;
  }
  for (i64 r = 0; r < D.c; ++r)
    run_chain(ctx, coef_dims(D, r), h_steps(D, r, 0), x + D.offs[r], F.hs.d(), F.s0.d(), F.s1.d(), r > 0);
  wss(ctx->L(), F.n, F.hs.d(), F.v.d(), F.zptr, F.w.d(), F.part.d());
  for (i64 r = 0; r < D.c; ++r) run_chain(ctx, D.n, g_steps(D, r, 0), F.w.d(), Sx + D.offs[r], F.s0.d(), F.s1.d(), false);
  return elem_grid(F.n);
}

// Gram route: S'(x) = ((x)_j X_j^T X_j) x (design.cpp:153-177 with unit
// weight factors; the constant weight is applied as FistaCtl::sscale), then
// per-CTA partials of wconst <x, S'x> - 2 <x, b> into F.part, so that
// sum v (Xx - z)^2 = partials + sum v z^2 needs no n-space pass.
// Gram block (m, r, j) of the current route-1 solve: the design's X^T X bands,
// or this outer iteration's tensor-weighted ones.
static const BandOp& gram_op(const Fit& F, i64 m, i64 r, i64 j) {
  const kg_design& D = *F.D;
  if (F.tensor) return F.wg[static_cast<size_t>((m * D.c + r) * D.d + j)];
  return D.gram[m][r][j]->dev.H;
}

static int gram_pass(Fit& F, const double* x, double* Sx) {
  const kg_design& D = *F.D;
  kg_ctx* ctx = F.ctx;
  for (i64 m = 0; m < D.c; ++m)
    for (i64 r = 0; r < D.c; ++r) {
      std::vector<Step> st;
      for (i64 j = D.d - 1; j >= 0; --j) st.push_back({static_cast<int>(j), &gram_op(F, m, r, j), D.p[m][j]});
      run_chain(ctx, D.p[r], st, x + D.offs[r], Sx + D.offs[m], F.s0.d(), F.s1.d(), r > 0);
    }
  gram_dots(ctx->L(), F.p, F.wconst, x, Sx, F.b.d(), F.part.d());
  return pgrid(F.p);
}

// ------------------------------------------------- halo exchange (8(f) rank 1)
// Coefficient slices of the last mode are owned by one rank each
// (kg_halo_plan); a rank's slab touches its owned slices plus the first few of
// its right neighbour's.  Per gradient: the partial of S(x) over that right
// halo goes to the right neighbour, the left neighbour's partial over this
// rank's first slices arrives and is added (own partial + left partial), and
// after the update the owned x of those first slices goes left while the
// right halo of x comes back.  ~3 slices (p1 p2 doubles each) per neighbour
// instead of all p.
static i64 halo_q(const Fit& F) { return F.D->P / F.D->p[0][F.D->d - 1]; }  // doubles per last-mode slice

static void exch_sx(Fit& F, double* Sx) {
  kg_ctx* ctx = F.ctx;
  const i64* h = F.D->halo;
  const i64 q = halo_q(F), nL = (h[6] - h[5]) * q, nR = (h[8] - h[7]) * q;
  const NcclApi* api = nccl_api();
  nccl_check(api->GroupStart(), "ncclGroupStart");
  if (nR > 0) nccl_check(api->Send(Sx + h[7] * q, nR, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->s), "ncclSend");
  if (nL > 0) nccl_check(api->Recv(F.htmp.d(), nL, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->s), "ncclRecv");
  nccl_check(api->GroupEnd(), "ncclGroupEnd");
  padd(ctx->L(), nL, F.htmp.d(), Sx + h[5] * q);
}

static void exch_x(Fit& F, double* x) {
  kg_ctx* ctx = F.ctx;
  const i64* h = F.D->halo;
  const i64 q = halo_q(F), nL = (h[6] - h[5]) * q, nR = (h[8] - h[7]) * q;
  const NcclApi* api = nccl_api();
  nccl_check(api->GroupStart(), "ncclGroupStart");
  if (nL > 0) nccl_check(api->Send(x + h[5] * q, nL, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->s), "ncclSend");
  if (nR > 0) nccl_check(api->Recv(x + h[7] * q, nR, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->s), "ncclRecv");
  nccl_check(api->GroupEnd(), "ncclGroupEnd");
}

// every rank's owned slices of x into the full vector on all ranks (exact:
// one nonzero term per element)
static void gather_owned(Fit& F, double* x) {
  const i64 q = halo_q(F);
  pmask(F.ctx->L(), F.p, F.D->halo[1] * q, F.D->halo[2] * q, x);
  ar_sum(F.ctx, x, static_cast<size_t>(F.p));
}

// the monitor's scalars of a halo step in one small all-reduce: scal[40] =
// sum v eta^2 (slab partials), scal[41..42] = |x|_1, |x|_2^2 and scal[43] =
// <b, x> over the owned slices
static void halo_scalars(Fit& F, int n_ss, int n_j, bool ex) {
  kg_ctx* ctx = F.ctx;
  sums4(ctx->L(), F.part.d(), n_ss, F.Jpart.d(), n_j, ex ? F.bxpart.d() : nullptr, n_j, F.scal.d() + 40);
  ar_sum(ctx, F.scal.d() + 40, 4);
}

// n-space pass; on a sharded context S(x) and the objective partial are
// summed over the slabs (one p-sized all-reduce + one scalar per gradient)
static int xwx_pass(Fit& F, const double* x, double* Sx) {
  const int np = xwx_pass_local(F, x, Sx);
  kg_ctx* ctx = F.ctx;
  if (!sharded(ctx)) return np;
  if (F.halo) {  // boundary slices only; the caller reduces the partials (halo_scalars)
    exch_sx(F, Sx);
    return np;
  }
  ar_sum(ctx, Sx, static_cast<size_t>(F.p));
  reduce_cols(ctx->L(), F.part.d(), np, 1, 0, F.scal.d() + 40);
  ar_sum(ctx, F.scal.d() + 40, 1);
  KG_CUDA(cudaMemcpyAsync(F.part.d(), F.scal.d() + 40, sizeof(double), cudaMemcpyDeviceToDevice, ctx->s));
  return 1;
}

static int step_pass(Fit& F, const double* x, double* Sx) {
  return F.route == 1 ? gram_pass(F, x, Sx) : xwx_pass(F, x, Sx);
}

// b = X^T (v .* z)
static void xtwz_pass(Fit& F) {
  const kg_design& D = *F.D;
  kg_ctx* ctx = F.ctx;
  if (D.fused) {
    FusedArgs a = fused_args(F);
    a.v = F.v.d();
    a.z = F.zptr;
    a.Q = D.d > 1 ? F.Q.d() : F.b.d();
    run_fused(ctx, FV_XTWZ, a);
    if (D.d > 1) {
      std::vector<i64> dims = D.n;
      dims[0] = D.p[0][0];
      run_chain(ctx, dims, g_steps(D, 0, 1), F.Q.d(), F.b.d(), F.s0.d(), F.s1.d(), false);
    }
  } else {
    vz(ctx->L(), F.n, F.v.d(), F.zptr, F.w.d());
    for (i64 r = 0; r < D.c; ++r)
      run_chain(ctx, D.n, g_steps(D, r, 0), F.w.d(), F.b.d() + D.offs[r], F.s0.d(), F.s1.d(), false);
  }
  ar_sum(ctx, F.b.d(), static_cast<size_t>(F.p));  // b = sum over slabs of X_g^T (v z)_g
}

// eta_out = H(coef) with optional reductions (HlastArgs flags) -> F.part (kHlastCols per CTA).
static int h_full(Fit& F, const double* coef, double* eta_out, HlastArgs h) {
  const kg_design& D = *F.D;
  kg_ctx* ctx = F.ctx;
  h.eta_new = eta_out;
  if (D.fused) {
    const double* P = coef;
    if (D.d > 1) {
      run_chain(ctx, coef_dims(D, 0), h_steps(D, 0, 1), coef, F.P.d(), F.s0.d(), F.s1.d(), false);
      P = F.P.d();
    }
    h.P = P;
    h.flags |= HL_WRITE;
  } else {
    for (i64 r = 0; r < D.c; ++r)
      run_chain(ctx, coef_dims(D, r), h_steps(D, r, 0), coef + D.offs[r], eta_out, F.s0.d(), F.s1.d(), r > 0);
    h.P = nullptr;
    h.flags &= ~HL_WRITE;
  }
  hlast_mode1(ctx->L(), h);
  return hlast_grid(h);
}

// ---------------------------------------------------------------- FISTA
static GramStepArgs gstep_args(Fit& F) {
  const kg_design& D = *F.D;
  GramStepArgs A;
  A.ctl = static_cast<FistaCtl*>(F.ctl.p);
  A.d = static_cast<int>(D.d);
  A.pd = D.p[0][D.d - 1];
  A.q = static_cast<int>(D.P / A.pd);
  uint32_t before = 1;
  for (i64 j = 0; j + 1 < D.d; ++j) {
    A.dims[j] = static_cast<int>(D.p[0][j]);
    A.G[j] = gram_op(F, 0, 0, j);
    A.fa[j] = FastDiv(before);
    A.fk[j] = FastDiv(static_cast<uint32_t>(D.p[0][j]));
    before *= static_cast<uint32_t>(D.p[0][j]);
  }
  A.Gd = gram_op(F, 0, 0, D.d - 1);
  A.X[0] = F.x.d();
  A.S[0] = F.Sx.d();
  A.b = F.b.d();
  A.pen = F.pen;
  A.alpha = F.alpha;
  A.part = F.gpart.d();
  A.counter = static_cast<unsigned*>(F.gcount.p);
  return A;
}

// One FISTA iteration: p-space update -> X^T W X pass on the new iterate -> control.
static void enqueue_body(Fit& F, cudaGraphConditionalHandle h, int use_handle) {
  kg_ctx* ctx = F.ctx;
  if (F.route == 1 && F.gstep) {  // update kernel + one Gram/objective/control kernel
    fista_update(ctx->L(), static_cast<FistaCtl*>(F.ctl.p), F.p, F.pen, F.alpha, F.x.d(), F.xp.d(), F.Sx.d(),
                 F.Sxp.d(), F.b.d(), F.best.d(), F.Sbest.d(), F.Jpart.d());
    GramStepArgs A = gstep_args(F);
    A.handle = h;
    A.use_handle = use_handle;
    gram_step(ctx->L(), A);
    return;
  }
  FistaCtl* c = static_cast<FistaCtl*>(F.ctl.p);
  const bool ex = F.route == 0 && F.expand;
  if (F.halo) {  // owned slices: update, x halo exchange, local pass + S(x) halo, 4-scalar all-reduce
    const i64 q = halo_q(F), o0 = F.D->halo[1] * q, on = (F.D->halo[2] - F.D->halo[1]) * q;
    fista_update(ctx->L(), c, on, F.pen, F.alpha, F.x.d() + o0, F.xp.d() + o0, F.Sx.d() + o0, F.Sxp.d() + o0,
                 F.b.d() + o0, F.best.d() + o0, F.Sbest.d() + o0, F.Jpart.d(), ex ? F.bxpart.d() : nullptr);
    exch_x(F, F.x.d());
    const int n_ss = step_pass(F, F.x.d(), F.Sx.d());
    halo_scalars(F, n_ss, ugrid(on), ex);
    fista_control(ctx->L(), c, F.scal.d() + 40, 1, F.scal.d() + 41, 1, h, use_handle,
                  ex ? F.scal.d() + 43 : nullptr, 1);
    return;
  }
  fista_update(ctx->L(), c, F.p, F.pen, F.alpha, F.x.d(), F.xp.d(), F.Sx.d(), F.Sxp.d(), F.b.d(), F.best.d(),
               F.Sbest.d(), F.Jpart.d(), ex ? F.bxpart.d() : nullptr);
  static const bool no_fork = dev_env("KG_NO_FORK") != nullptr;
  if (F.route == 0 && F.slab && !sharded(ctx) && !no_fork) {
    // Slab route: H mode 3 -> slab pass -> G mode 3.  The control kernel needs
    // only the partials of the update and of the slab pass, so it runs beside
    // the mode-3 G step (a fork / join in the captured body) instead of after it.
    const kg_design& D = *F.D;
    if (!ctx->fork) {
      KG_CUDA(cudaStreamCreateWithFlags(&ctx->fork, cudaStreamNonBlocking));
      for (cudaEvent_t& e : ctx->fork_ev) KG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // programmatic dependent launches along update -> H mode 3 -> slab pass -> G mode 3
    static const bool pdl = dev_env("KG_NO_PDL") == nullptr;
    run_chain(ctx, coef_dims(D, 0), h_steps(D, 0, 2), F.x.d(), F.P.d(), F.s0.d(), F.s1.d(), false, pdl);
    SlabArgs a = slab_args(F);
    a.S = F.P.d();
    a.Q = F.Q.d();
    Launch Lp = ctx->L();
    Lp.pdl = pdl;
    slab_pass(Lp, a);
    F.n_ss = slab_grid(a);
    KG_CUDA(cudaEventRecord(ctx->fork_ev[0], ctx->s));
    KG_CUDA(cudaStreamWaitEvent(ctx->fork, ctx->fork_ev[0], 0));
    fista_control(Launch{ctx->fork, &ctx->launches}, c, F.part.d(), F.n_ss, F.Jpart.d(), ugrid(F.p), h, use_handle,
                  ex ? F.bxpart.d() : nullptr, ugrid(F.p));
    KG_CUDA(cudaEventRecord(ctx->fork_ev[1], ctx->fork));
    std::vector<i64> dims = {D.p[0][0], D.p[0][1], D.n[2]};
    run_chain(ctx, dims, g_steps(D, 0, 2), F.Q.d(), F.Sx.d(), F.s0.d(), F.s1.d(), false, pdl);
    KG_CUDA(cudaStreamWaitEvent(ctx->s, ctx->fork_ev[1], 0));
    return;
  }
  F.n_ss = step_pass(F, F.x.d(), F.Sx.d());
  fista_control(ctx->L(), c, F.part.d(), F.n_ss, F.Jpart.d(), ugrid(F.p), h, use_handle,
                ex ? F.bxpart.d() : nullptr, ugrid(F.p));
}

// KG_HOST_LOOP=1: drive the FISTA loop from the host (one sync per
// iteration) instead of the conditional graph, so profilers can see the
// individual kernels.  Same kernels, same arithmetic.
constexpr int kHostBatch = 8;  // FISTA steps per host round trip of a sharded n-space loop

static bool host_loop_mode() {
  static const bool on = [] {
    const char* e = std::getenv("KG_HOST_LOOP");
    return e && e[0] == '1';
  }();
  return on;
}

// Captures the FISTA loop of the current route once: a gate kernel, then a
// conditional WHILE node whose body is one iteration.  Every scalar the body
// needs (lambda, step, omega, flags) is read from the device control block, and
// the Gram-route weight from F.wconst is baked in, so the graph is re-launched
// for every lambda and every outer iteration of the fit.
static void build_graph(Fit& F) {
  kg_ctx* ctx = F.ctx;
  const int r = F.route;
  cudaStream_t cap;
  KG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  KG_CUDA(cudaGraphCreate(&F.graph[r], 0));
  cudaGraphConditionalHandle h;
  KG_CUDA(cudaGraphConditionalHandleCreate(&h, F.graph[r], 0, cudaGraphCondAssignDefault));
  KG_CUDA(cudaStreamBeginCaptureToGraph(cap, F.graph[r], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  fista_gate(Launch{cap, nullptr}, static_cast<FistaCtl*>(F.ctl.p), h);
  KG_CUDA(cudaStreamEndCapture(cap, &F.graph[r]));
  size_t nn = 0;
  KG_CUDA(cudaGraphGetNodes(F.graph[r], nullptr, &nn));
  if (nn != 1) throw Error(E_CUDA, "unexpected gate capture");
  cudaGraphNode_t gate;
  KG_CUDA(cudaGraphGetNodes(F.graph[r], &gate, &nn));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  KG_CUDA(cudaGraphAddNode(&node, F.graph[r], &gate, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  KG_CUDA(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  cudaStream_t saved = ctx->s;
  i64 saved_count = ctx->launches;
  ctx->s = cap;
  ctx->launches = 0;
  try {
    enqueue_body(F, h, 1);
  } catch (...) {
    ctx->s = saved;
    ctx->launches = saved_count;
    cudaGraph_t dummy;
    cudaStreamEndCapture(cap, &dummy);
    cudaStreamDestroy(cap);
    throw;
  }
  F.kernels_per_iter[r] = ctx->launches;
  ctx->s = saved;
  ctx->launches = saved_count;
  KG_CUDA(cudaStreamEndCapture(cap, &body));
  KG_CUDA(cudaStreamDestroy(cap));
  KG_CUDA(cudaGraphInstantiate(&F.exec[r], F.graph[r], 0));
}

struct FistaOut {
  double objective = 0.0, lip = 0.0;
  i64 iterations = 0;
  bool converged = false, diverged = false, bad_weights = false;
};

struct InnerCfg {
  double nu = 1.0, tol = 1e-8;
  i64 max_iters = 2000, monitor_every = 1;
  int extrapolation = 0;
};

static int step_pass(Fit& F, const double* x, double* Sx);
static double penalty_of(int pen, double alpha, double l1, double l2);

// fista_solve with nu = 0 (inner.cpp:162-235, backtracking every iteration),
// driven from the host: delta starts at 1 and is halved until the
// majorization test holds; every quadratic is h(x) = (s <x, S x> - 2 <b, x> +
// sum v z^2) / 2n with S x from the route's X^T W X pass (the accepted
// candidate's S x is reused), so a trial costs one pass.  Results as the
// other paths: F.best / F.Sbest and the control block at PIN_CTL.
static void fista_bt0(Fit& F, double lambda, const InnerCfg& ic, const double* vmax_part, int n_vmax) {
  kg_ctx* ctx = F.ctx;
  const kg_design& D = *F.D;
  const i64 p = F.p;
  const double n = static_cast<double>(D.N_full);
  const double sscale = F.route == 1 ? F.wconst : 1.0;
  const size_t pb = sizeof(double) * static_cast<size_t>(p);
  for (DBuf* b : {&F.bt_y, &F.bt_g, &F.bt_c, &F.bt_sc}) b->alloc(pb);
  F.bt_part.alloc(sizeof(double) * 4 * pgrid(p));
  double* pin = ctx->pin();
  double* sc = F.scal.d();
  auto rd = [&](const double* dev, int k) {  // read k device scalars into pin[20 ..)
    KG_CUDA(cudaMemcpyAsync(pin + 20, dev, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  };
  if (!F.c0_valid) {  // sum v z^2
    wzz(ctx->L(), F.n, F.v.d(), F.zptr, F.part.d());
    reduce_cols(ctx->L(), F.part.d(), elem_grid(F.n), 1, 0, sc + 48);
    ar_sum(ctx, sc + 48, 1);
    F.c0_valid = true;
  }
  rd(sc + 48, 1);
  const double c0 = pin[20];
  reduce_cols(ctx->L(), vmax_part, n_vmax, 1, 1, sc + 56);  // lipschitz_upper / tensor_exact (reported)
  ar_max(ctx, sc + 56, 1);
  rd(sc + 56, 1);
  const double wmax = (F.tensor && D.c == 1) ? 1.0 : pin[20];
  FistaCtl out{};
  out.lip = wmax * (F.tensor ? F.lipfac_t : D.lipfac) / n;
  out.bad_weights = !(wmax > 0.0);
  if (out.bad_weights) {
    std::memcpy(pin + PIN_CTL, &out, sizeof(out));
    return;
  }
  auto J = [&](double l1, double l2) { return penalty_of(F.pen, F.alpha, l1, l2); };
  // x_0 = theta
  pcopy(ctx->L(), p, F.theta.d(), F.x.d(), F.xp.d(), F.best.d());
  step_pass(F, F.x.d(), F.Sx.d());
  pcopy(ctx->L(), p, F.Sx.d(), F.Sxp.d(), F.Sbest.d(), nullptr);
  bt_dots(ctx->L(), p, F.x.d(), F.Sx.d(), F.b.d(), F.bt_part.d());
  reduce_cols(ctx->L(), F.bt_part.d(), pgrid(p), 2, 0, sc + 24);
  pnorm(ctx->L(), p, F.pen, F.alpha, F.x.d(), F.Jpart.d());
  reduce_cols(ctx->L(), F.Jpart.d(), pgrid(p), 2, 0, sc + 26);
  rd(sc + 24, 4);
  double g_prev = 0.5 * (sscale * pin[20] - 2.0 * pin[21] + c0) / n + lambda * J(pin[22], pin[23]);
  double best_g = g_prev, delta = 1.0;
  i64 momentum = 1;
  const i64 me = ic.monitor_every < 1 ? 1 : ic.monitor_every;
  for (i64 it = 1; it <= ic.max_iters; ++it) {
    const double omega =
        ic.extrapolation == 0 ? static_cast<double>(momentum - 1) / static_cast<double>(momentum + 2) : 0.0;
    bt_prep(ctx->L(), p, omega, sscale, n, F.x.d(), F.xp.d(), F.Sx.d(), F.Sxp.d(), F.b.d(), F.bt_y.d(), F.bt_g.d(),
            F.bt_part.d());
    reduce_cols(ctx->L(), F.bt_part.d(), pgrid(p), 2, 0, sc + 24);
    rd(sc + 24, 2);
    const double h_y = 0.5 * (sscale * pin[20] - 2.0 * pin[21] + c0) / n;
    double h_c = 0.0, l1c = 0.0, l2c = 0.0;
    for (;;) {  // inner.cpp:170-183
      bt_trial(ctx->L(), p, delta, lambda, F.pen, F.alpha, F.bt_y.d(), F.bt_g.d(), F.bt_c.d(), F.bt_part.d());
      reduce_cols(ctx->L(), F.bt_part.d(), pgrid(p), 4, 0, sc + 24);
      step_pass(F, F.bt_c.d(), F.bt_sc.d());
      bt_dots(ctx->L(), p, F.bt_c.d(), F.bt_sc.d(), F.b.d(), F.bt_part.d());
      reduce_cols(ctx->L(), F.bt_part.d(), pgrid(p), 2, 0, sc + 28);
      rd(sc + 24, 6);
      const double gstep = pin[20], ss = pin[21];
      l1c = pin[22];
      l2c = pin[23];
      h_c = 0.5 * (sscale * pin[24] - 2.0 * pin[25] + c0) / n;
      const double bound = h_y + gstep + ss / (2.0 * delta) + 1e-12 * std::max(1.0, std::abs(h_y));
      if (h_c <= bound) break;
      delta *= 0.5;
      ++out.backtracks;
      if (delta < 1e-300) {  // DivergenceError("stepsize underflow in backtracking")
        out.diverged = 1;
        out.iterations = it;
        out.best_g = best_g;
        std::memcpy(pin + PIN_CTL, &out, sizeof(out));
        return;
      }
    }
    // x_prev = x, x = cand (S as well)
    KG_CUDA(cudaMemcpyAsync(F.xp.p, F.x.p, pb, cudaMemcpyDeviceToDevice, ctx->s));
    KG_CUDA(cudaMemcpyAsync(F.x.p, F.bt_c.p, pb, cudaMemcpyDeviceToDevice, ctx->s));
    KG_CUDA(cudaMemcpyAsync(F.Sxp.p, F.Sx.p, pb, cudaMemcpyDeviceToDevice, ctx->s));
    KG_CUDA(cudaMemcpyAsync(F.Sx.p, F.bt_sc.p, pb, cudaMemcpyDeviceToDevice, ctx->s));
    ++momentum;
    out.prox_steps += 1;
    out.iterations = it;
    if (!(it % me == 0 || it == ic.max_iters)) continue;
    const double g_cur = h_c + lambda * J(l1c, l2c);
    if (!std::isfinite(g_cur)) {  // DivergenceError("non-finite inner objective")
      out.diverged = 1;
      break;
    }
    if (g_cur <= best_g) {
      pcopy(ctx->L(), p, F.x.d(), F.best.d(), nullptr, nullptr);
      pcopy(ctx->L(), p, F.Sx.d(), F.Sbest.d(), nullptr, nullptr);
      best_g = g_cur;
    }
    if (std::abs(g_cur - g_prev) / std::max(1.0, std::abs(g_cur)) < ic.tol) {
      out.converged = 1;
      break;
    }
    g_prev = g_cur;
  }
  out.best_g = best_g;
  std::memcpy(pin + PIN_CTL, &out, sizeof(out));
}

// Enqueues fista_solve(init = theta) with weights F.v (max-partials in
// vmax_part) and working response F.zptr; F.b must hold X^T(v.*z) and, on the
// Gram route (F.route == 1), F.wconst / F.c0 the constant weight and sum v z^2.
// The result lands in F.best; the control block is copied to ctx->pin() + PIN_CTL.
static void fista_enqueue(Fit& F, double lambda, const InnerCfg& ic, const double* vmax_part, int n_vmax) {
  kg_ctx* ctx = F.ctx;
  if (F.tensor && F.D->c == 1) {  // lipschitz_tensor_exact carries no max(v): unit weight scale
    fill(ctx->L(), 1, 1.0, F.scal.d() + 60);
    vmax_part = F.scal.d() + 60;
    n_vmax = 1;
  }
  if (sharded(ctx)) {  // max(v) over all slabs (lipschitz_upper)
    reduce_cols(ctx->L(), vmax_part, n_vmax, 1, 1, F.scal.d() + 56);
    ar_max(ctx, F.scal.d() + 56, 1);
    vmax_part = F.scal.d() + 56;
    n_vmax = 1;
  }
  if (!(ic.nu >= 0.0 && ic.nu <= 1.0)) throw Error(E_INVAL, "fista_solve: nu must lie in [0,1]");
  if (ic.nu == 0.0) {  // backtracking every iteration: host-driven trials
    fista_bt0(F, lambda, ic, vmax_part, n_vmax);
    return;
  }
  F.halo = sharded(ctx) && F.D->halo[0] == 1 && F.route == 0 && F.D->c == 1;
  FistaCtl h{};
  h.lambda = lambda;
  h.tol = ic.tol;
  h.nu = ic.nu;
  h.n = static_cast<double>(F.D->N_full);
  h.lipfac = F.tensor ? F.lipfac_t : F.D->lipfac;
  h.max_iters = ic.max_iters;
  h.monitor_every = ic.monitor_every;
  h.sscale = F.route == 1 ? F.wconst : 1.0;
  h.ss_const = 0.0;  // Gram route: filled on the device below
  h.alpha = F.alpha;
  h.pen = F.pen;
  h.extrapolation = ic.extrapolation;
  h.bt_div = ic.nu > 0.0 && ic.nu < 1.0;
  FistaCtl* staged = reinterpret_cast<FistaCtl*>(ctx->pin() + PIN_STAGE);
  KG_CUDA(cudaStreamSynchronize(ctx->s));  // the pinned staging slot is reused
  *staged = h;
  KG_CUDA(cudaMemcpyAsync(F.ctl.p, staged, sizeof(FistaCtl), cudaMemcpyHostToDevice, ctx->s));
  if (F.route == 1 || F.expand) {  // sum v z^2, once per (v, z)
    if (!F.c0_valid) {
      wzz(ctx->L(), F.n, F.v.d(), F.zptr, F.part.d());
      reduce_cols(ctx->L(), F.part.d(), elem_grid(F.n), 1, 0, F.scal.d() + 48);
      ar_sum(ctx, F.scal.d() + 48, 1);
      F.c0_valid = true;
    }
    KG_CUDA(cudaMemcpyAsync(&static_cast<FistaCtl*>(F.ctl.p)->ss_const, F.scal.d() + 48, sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->s));
  }
  const bool one_kernel = F.route == 1 && F.gstep;
  if (one_kernel && F.persist < 0) F.persist = (!host_loop_mode() && fista_persist_ok(gstep_args(F))) ? 1 : 0;
  if (one_kernel && F.persist == 1 && ic.max_iters >= 1) {  // the whole solve in one cooperative launch
    PersistArgs P;
    P.g = gstep_args(F);
    P.theta = F.theta.d();
    P.X = F.pX.d();
    P.best = F.best.d();
    P.Sbest = F.Sbest.d();
    P.part = F.gpart.d();
    P.bar = static_cast<unsigned*>(F.pbar.p);
    fista_persist(ctx->L(), P);
    KG_CUDA(cudaMemcpyAsync(ctx->pin() + PIN_CTL, F.ctl.p, sizeof(FistaCtl), cudaMemcpyDeviceToHost, ctx->s));
    F.persist_solve = true;
    return;
  }
  F.persist_solve = false;
  pcopy(ctx->L(), F.p, F.theta.d(), F.x.d(), F.xp.d(), F.best.d());
  if (one_kernel) {  // S'(x_0), g_0 and the step size in one launch
    GramStepArgs A = gstep_args(F);
    A.init = 1;
    gram_step(ctx->L(), A);
    pcopy(ctx->L(), F.p, F.Sx.d(), F.Sxp.d(), F.Sbest.d(), nullptr);
  } else if (F.halo) {
    const i64 q = halo_q(F), o0 = F.D->halo[1] * q, on = (F.D->halo[2] - F.D->halo[1]) * q;
    const int n_ss = step_pass(F, F.x.d(), F.Sx.d());
    pnorm(ctx->L(), on, F.pen, F.alpha, F.x.d() + o0, F.Jpart.d());
    pcopy(ctx->L(), F.p, F.Sx.d(), F.Sxp.d(), F.Sbest.d(), nullptr);
    const bool ex = F.expand;
    if (ex) pdot(ctx->L(), on, F.b.d() + o0, F.x.d() + o0, F.bxpart.d());
    halo_scalars(F, n_ss, pgrid(on), ex);
    fista_init(ctx->L(), static_cast<FistaCtl*>(F.ctl.p), F.scal.d() + 40, 1, F.scal.d() + 41, 1, vmax_part, n_vmax,
               0, ex ? F.scal.d() + 43 : nullptr, 1);
  } else {
    const int n_ss = step_pass(F, F.x.d(), F.Sx.d());
    pnorm(ctx->L(), F.p, F.pen, F.alpha, F.x.d(), F.Jpart.d());
    pcopy(ctx->L(), F.p, F.Sx.d(), F.Sxp.d(), F.Sbest.d(), nullptr);
    const bool ex = F.route == 0 && F.expand;
    if (ex) pdot(ctx->L(), F.p, F.b.d(), F.x.d(), F.bxpart.d());
    fista_init(ctx->L(), static_cast<FistaCtl*>(F.ctl.p), F.part.d(), n_ss, F.Jpart.d(), pgrid(F.p), vmax_part,
               n_vmax, 0, ex ? F.bxpart.d() : nullptr, pgrid(F.p));
  }
  if (ic.max_iters >= 1) {
    // A sharded n-space loop is driven from the host (its all-reduces stay out
    // of graph capture) in batches of kHostBatch steps with one stream sync per
    // batch: the update and control kernels are no-ops once the device control
    // block says done, so steps enqueued past the stop leave the state as it is
    // (x is unchanged, so S(x) and its all-reduce recompute the same values),
    // and every rank enqueues the same collectives.  KG_HOST_LOOP (profiling)
    // keeps one step per batch.
    if (host_loop_mode() || (sharded(ctx) && F.route == 0)) {
      const FistaCtl* hc = reinterpret_cast<const FistaCtl*>(ctx->pin() + PIN_CTL);
      const int batch = host_loop_mode() ? 1 : kHostBatch;
      const i64 before = ctx->launches;
      KG_CUDA(cudaMemcpyAsync(ctx->pin() + PIN_CTL, F.ctl.p, sizeof(FistaCtl), cudaMemcpyDeviceToHost, ctx->s));
      sync(ctx);
      if (!hc->done && host_loop_mode()) {
        for (;;) {  // profiling: one step per host round trip
          for (int k = 0; k < batch; ++k) enqueue_body(F, cudaGraphConditionalHandle{}, 0);
          KG_CUDA(cudaMemcpyAsync(ctx->pin() + PIN_CTL, F.ctl.p, sizeof(FistaCtl), cudaMemcpyDeviceToHost, ctx->s));
          sync(ctx);
          if (hc->done) break;
        }
      } else if (!hc->done) {
        // Two batches in flight: batch j is enqueued before the host looks at
        // the control block read back after batch j - 1, so the GPU never
        // drains at a batch boundary.  Steps past the stop are no-ops for the
        // state (update and control check done; x unchanged), and every rank
        // enqueues the same collectives.
        for (cudaEvent_t& e : ctx->loop_ev)
          if (!e) KG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const FistaCtl* slot[2] = {reinterpret_cast<const FistaCtl*>(ctx->pin() + PIN_CTL),
                                   reinterpret_cast<const FistaCtl*>(ctx->pin() + PIN_CTL2)};
        auto issue = [&](int j) {
          for (int k = 0; k < batch; ++k) enqueue_body(F, cudaGraphConditionalHandle{}, 0);
          KG_CUDA(cudaMemcpyAsync(const_cast<FistaCtl*>(slot[j & 1]), F.ctl.p, sizeof(FistaCtl),
                                  cudaMemcpyDeviceToHost, ctx->s));
          KG_CUDA(cudaEventRecord(ctx->loop_ev[j & 1], ctx->s));
        };
        issue(0);
        for (int j = 1;; ++j) {
          issue(j);
          KG_CUDA(cudaEventSynchronize(ctx->loop_ev[(j - 1) & 1]));
          if (slot[(j - 1) & 1]->done) break;
        }
        sync(ctx);  // the batch still in flight only repeats the stopped state
        KG_CUDA(cudaMemcpyAsync(ctx->pin() + PIN_CTL, F.ctl.p, sizeof(FistaCtl), cudaMemcpyDeviceToHost, ctx->s));
        sync(ctx);
      }
      // fista_read() adds iterations * kernels_per_iter; undo the direct count
      const i64 its = hc->iterations;
      F.kernels_per_iter[F.route] = its > 0 ? (ctx->launches - before) / its : 0;
      ctx->launches = before;
    } else {
      if (!F.exec[F.route]) build_graph(F);
      KG_CUDA(cudaGraphLaunch(F.exec[F.route], ctx->s));
    }
  }
  fista_finalize(ctx->L(), static_cast<FistaCtl*>(F.ctl.p), F.p, F.x.d(), F.best.d(), F.Sx.d(), F.Sbest.d());
  if (F.halo) {  // owned slices back into full replicated vectors
    for (DBuf* v : {&F.x, &F.Sx, &F.best, &F.Sbest}) gather_owned(F, v->d());
    F.halo = false;
  }
  KG_CUDA(cudaMemcpyAsync(ctx->pin() + PIN_CTL, F.ctl.p, sizeof(FistaCtl), cudaMemcpyDeviceToHost, ctx->s));
}

static FistaOut fista_read(Fit& F) {
  const FistaCtl* c = reinterpret_cast<const FistaCtl*>(F.ctx->pin() + PIN_CTL);
  FistaOut o;
  o.objective = c->best_g;
  o.lip = c->lip;
  o.iterations = c->iterations;
  o.converged = c->converged;
  o.diverged = c->diverged;
  o.bad_weights = c->bad_weights;
  if (!F.persist_solve) F.ctx->launches += o.iterations * F.kernels_per_iter[F.route];
  return o;
}

// --------------------------------------------------------------- helpers
static double penalty_of(int pen, double alpha, double l1, double l2) {
  if (pen == 0) return l1;
  if (pen == 1) return l2;
  return l1 + alpha * l2;
}

static void validate_obs(Fit& F) {
  kg_ctx* ctx = F.ctx;
  reset_errs(F);
  validate_pass(ctx->L(), F.n, F.fam, F.O->y.d(), F.O->a.d(), F.errs.l(), F.D->cell_base);
  ar_min_i64(ctx, F.errs.l(), 1);  // first invalid cell over all slabs
  i64 e;
  KG_CUDA(cudaMemcpyAsync(&e, F.errs.p, sizeof(i64), cudaMemcpyDeviceToHost, ctx->s));
  sync(ctx);
  if (e == kNoErr) return;
  const i64 loc = e - F.D->cell_base;
  if (loc < 0 || loc >= F.n) throw Error(E_INVAL, "invalid observation at cell " + std::to_string(e));  // other slab
  double yi, ai;
  KG_CUDA(cudaMemcpy(&yi, F.O->y.d() + loc, sizeof(double), cudaMemcpyDeviceToHost));
  KG_CUDA(cudaMemcpy(&ai, F.O->a.d() + loc, sizeof(double), cudaMemcpyDeviceToHost));
  const std::string cell = std::to_string(e);
  if (!(ai >= 0.0) || !std::isfinite(ai))
    throw Error(E_INVAL, "observation weight must be finite and nonnegative at cell " + cell);
  if (!std::isfinite(yi)) throw Error(E_INVAL, "response must be finite at cell " + cell);
  if (F.fam == 1) throw Error(E_INVAL, "binomial response must be a proportion in [0,1] at cell " + cell);
  if (F.fam == 2) throw Error(E_INVAL, "poisson response must be nonnegative at cell " + cell);
  throw Error(E_INVAL, "gamma response must be positive at cell " + cell);
}

// lambda_max (penalty.cpp:72-85) on an allocated fit (uses F.b as scratch).
static double lambda_max_fit(Fit& F) {
  const kg_design& D = *F.D;
  kg_ctx* ctx = F.ctx;
  reset_errs(F);
  if (D.fused) {
    FusedArgs a = fused_args(F);
    a.y = F.O->y.d();
    a.a = F.O->a.d();
    a.fam = F.fam;
    a.disp = F.disp;
    a.err = F.errs.l();
    a.Q = D.d > 1 ? F.Q.d() : F.b.d();
    run_fused(ctx, FV_SCORE0, a);
    if (D.d > 1) {
      std::vector<i64> dims = D.n;
      dims[0] = D.p[0][0];
      run_chain(ctx, dims, g_steps(D, 0, 1), F.Q.d(), F.b.d(), F.s0.d(), F.s1.d(), false);
    }
  } else {
    score0(ctx->L(), F.n, F.fam, F.disp, F.O->y.d(), F.O->a.d(), F.w.d(), F.errs.l(), D.cell_base);
    for (i64 r = 0; r < D.c; ++r)
      run_chain(ctx, D.n, g_steps(D, r, 0), F.w.d(), F.b.d() + D.offs[r], F.s0.d(), F.s1.d(), false);
  }
  ar_sum(ctx, F.b.d(), static_cast<size_t>(F.p));  // G(u) summed over the slabs
  ar_min_i64(ctx, F.errs.l(), 1);
  pmaxabs(ctx->L(), F.p, F.b.d(), F.Jpart.d());
  reduce_cols(ctx->L(), F.Jpart.d(), pgrid(F.p), 1, 1, F.scal.d());
  double* pin = ctx->pin();
  KG_CUDA(cudaMemcpyAsync(pin, F.scal.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
  KG_CUDA(cudaMemcpyAsync(pin + 1, F.errs.p, sizeof(i64), cudaMemcpyDeviceToHost, ctx->s));
  sync(ctx);
  i64 e;
  std::memcpy(&e, pin + 1, sizeof(i64));
  if (e != kNoErr) throw Error(E_EVAL, "non-finite score entry at cell " + std::to_string(e), e);
  return pin[0] / static_cast<double>(D.N_full);
}

}  // namespace kg

// ------------------------------------------------------------------ result
struct kg_path_result {
  kg_ctx* ctx = nullptr;
  kg::i64 p = 0;
  std::vector<double> lambdas, objectives, initial_objectives;
  std::vector<std::vector<kg_outer_record>> traces;  // OuterTrace.iterations per model (outer.hpp:26-47)
  std::vector<kg::i64> outer_iters, inner_iters, nnz;
  std::vector<int> status;
  bool truncated = false;
  double lambda_max = 0.0;
  kg::DBuf coefs;  // n_models x p on the device
};

namespace kg {

struct ModelTrace {
  int status = 1;
  i64 outer = 0, inner = 0;
  double initial_objective = 0.0, final_objective = 0.0;
  std::vector<kg_outer_record> recs;  // one per outer iteration (OuterRecord, outer.hpp:26-33)
};

static kg_outer_record outer_rec(double objective, double alpha, double delta_k, double lip, i64 inner, bool conv,
                                 int j) {
  kg_outer_record r;
  r.objective = objective;
  r.alpha = alpha;
  r.delta_k = delta_k;
  r.lipschitz = lip;
  r.inner_iterations = inner;
  r.inner_converged = conv ? 1 : 0;
  r.armijo_j = j;
  return r;
}

// ------------------------------------------------------------ outer_solve
struct OuterCfg {
  i64 max_outer = 100, max_bt = 50;
  double alpha0 = 1.0, b = 0.5, v = 0.1, tol = 1e-8;
  int wmode = 0;
  InnerCfg inner;
};

static void check_ll_errs(Fit& F, const i64* errs) {
  if (errs[0] != kNoErr) throw Error(E_EVAL, "non-finite log-likelihood term at cell " + std::to_string(errs[0]), errs[0]);
}

// Gaussian + identity + exact weights: one inner solve per lambda
// (outer.cpp:197-231).  State carried across lambdas: theta, eta = H(theta),
// ll = loglik(eta), (l1, l2) of theta.
struct PathState {
  double ll = 0.0, l1 = 0.0, l2 = 0.0;
  double tb = 0.0, tst = 0.0;  // Gram route: <theta, b>, <theta, S' theta>
};

// Gaussian shortcut on the constant-weight route, all in p-space: with
// eta = X theta and V = w I,  loglik = <theta, b> - w/2 <theta, S' theta>
// (b = X^T V y, S' = (x)_j X_j^T X_j theta) and
// <u(eta), eta_t - eta> = <b - w S' theta, theta_t - theta>.
static ModelTrace gaussian_step_gram(Fit& F, double lambda, const OuterCfg& oc, PathState& st, int n_vmax) {
  kg_ctx* ctx = F.ctx;
  const double n = static_cast<double>(F.D->N_full);
  const double w = F.wconst;
  const double ll_cur = st.tb - 0.5 * w * st.tst;
  const double J_cur = penalty_of(F.pen, F.alpha, st.l1, st.l2);
  const double f_cur = -ll_cur / n + lambda * J_cur;
  ModelTrace tr;
  tr.initial_objective = f_cur;
  fista_enqueue(F, lambda, oc.inner, F.part.d() + F.D->part_cap - n_vmax, n_vmax);
  const int g = gauss_dots(ctx->L(), F.p, w, F.theta.d(), F.stheta.d(), F.best.d(), F.Sbest.d(), F.b.d(),
                           F.part.d());
  reduce_cols(ctx->L(), F.part.d(), g, 9, 0, F.scal.d());
  double* pin = ctx->pin();
  KG_CUDA(cudaMemcpyAsync(pin, F.scal.p, sizeof(double) * 9, cudaMemcpyDeviceToHost, ctx->s));
  sync(ctx);
  const FistaOut fo = fista_read(F);
  if (fo.bad_weights) throw Error(E_INVAL, "lipschitz_upper: weights must not be all zero");
  tr.inner = fo.iterations;
  if (fo.diverged) {
    tr.status = KG_S_INNER_DIVERGENCE;
    tr.final_objective = f_cur;
    return tr;
  }
  const double tb = pin[2], tst = pin[3], l1 = pin[5], l2 = pin[6];
  const double ll_new = tb - 0.5 * w * tst;
  const double J_t = penalty_of(F.pen, F.alpha, l1, l2);
  const double f_new = -ll_new / n + lambda * J_t;
  // Delta_k (outer.cpp:224-226): X^T u(eta) = b - w S' theta
  const double delta_k = -pin[4] / n + lambda * (J_t - J_cur);
  double f = f_cur;
  if (f_new <= f_cur) {
    pcopy(ctx->L(), F.p, F.best.d(), F.theta.d(), nullptr, nullptr);
    pcopy(ctx->L(), F.p, F.Sbest.d(), F.stheta.d(), nullptr, nullptr);
    st.tb = tb;
    st.tst = tst;
    st.l1 = l1;
    st.l2 = l2;
    f = f_new;
  }
  tr.outer = 1;
  tr.final_objective = f;
  tr.recs.push_back(outer_rec(f, 1.0, delta_k, fo.lip, fo.iterations, fo.converged, 0));
  tr.status = fo.converged ? KG_S_CONVERGED : KG_S_MAX_ITERATIONS;
  return tr;
}

static ModelTrace gaussian_step(Fit& F, double lambda, const OuterCfg& oc, PathState& st, int n_vmax) {
  if (F.route == 1) return gaussian_step_gram(F, lambda, oc, st, n_vmax);
  kg_ctx* ctx = F.ctx;
  const double n = static_cast<double>(F.D->N_full);
  const double J_cur = penalty_of(F.pen, F.alpha, st.l1, st.l2);
  const double f_cur = -st.ll / n + lambda * J_cur;
  ModelTrace tr;
  tr.initial_objective = f_cur;
  reset_errs(F);
  fista_enqueue(F, lambda, oc.inner, F.part.d() + F.D->part_cap - n_vmax, n_vmax);
  // eta_tilde = H(best); loglik(eta_tilde) and <u(eta), eta_tilde - eta> in the same pass.
  HlastArgs h = hlast_args(F);
  h.flags = HL_LL_NEW | HL_DOT | HL_U_FLY;
  h.eta_old = F.eta.d();
  const int g = h_full(F, F.best.d(), F.eta_t.d(), h);
  reduce_cols(ctx->L(), F.part.d(), g, kHlastCols, 0, F.scal.d());
  ar_sum(ctx, F.scal.d(), kHlastCols);
  pnorm(ctx->L(), F.p, F.pen, F.alpha, F.best.d(), F.Jpart.d());
  reduce_cols(ctx->L(), F.Jpart.d(), pgrid(F.p), 2, 0, F.scal.d() + 16);
  double* pin = ctx->pin();
  KG_CUDA(cudaMemcpyAsync(pin, F.scal.p, sizeof(double) * 20, cudaMemcpyDeviceToHost, ctx->s));
  ar_min_i64(ctx, F.errs.l(), 4);
  KG_CUDA(cudaMemcpyAsync(pin + PIN_ERR, F.errs.p, sizeof(i64) * 4, cudaMemcpyDeviceToHost, ctx->s));
  sync(ctx);
  const FistaOut fo = fista_read(F);
  if (fo.bad_weights) throw Error(E_INVAL, "lipschitz_upper: weights must not be all zero");
  tr.inner = fo.iterations;
  if (fo.diverged) {  // DivergenceError caught by outer_solve (outer.cpp:272-275)
    tr.status = KG_S_INNER_DIVERGENCE;
    tr.final_objective = f_cur;
    return tr;
  }
  i64 errs[4];
  std::memcpy(errs, pin + PIN_ERR, sizeof(errs));
  check_ll_errs(F, errs);
  if (errs[1] != kNoErr) throw Error(E_EVAL, "non-finite score entry at cell " + std::to_string(errs[1]), errs[1]);
  const double ll_new = pin[0] / F.disp, l1 = pin[16], l2 = pin[17];
  const double J_t = penalty_of(F.pen, F.alpha, l1, l2);
  const double f_new = -ll_new / n + lambda * J_t;
  const double delta_k = -pin[1] / n + lambda * (J_t - J_cur);  // outer.cpp:224-226
  double f = f_cur;
  if (f_new <= f_cur) {
    pcopy(ctx->L(), F.p, F.best.d(), F.theta.d(), nullptr, nullptr);
    std::swap(F.eta.p, F.eta_t.p);
    st.ll = ll_new;
    st.l1 = l1;
    st.l2 = l2;
    f = f_new;
  }
  tr.outer = 1;
  tr.final_objective = f;
  tr.recs.push_back(outer_rec(f, 1.0, delta_k, fo.lip, fo.iterations, fo.converged, 0));
  tr.status = fo.converged ? KG_S_CONVERGED : KG_S_MAX_ITERATIONS;
  return tr;
}

// General outer loop (outer.cpp:233-302) for exact / unit weights.
// iwls = tensor for one outer iteration (outer.cpp:256-263 with
// compute_weights' tensor branch, outer.cpp:53-103): F.v holds the exact GLM
// weights and F.u the score on entry.  Leaves the rank-one weights in F.v,
// z = u / v + eta in F.z, the weighted Gram blocks in F.wg and the Lipschitz
// factor in F.lipfac_t (lipschitz_tensor_exact for c = 1, inner.cpp:73-91;
// lipschitz_upper otherwise), and switches the fit to the Gram route.
static void tensor_weights(Fit& F, double* vmax_part, int n_vmax) {
  kg_ctx* ctx = F.ctx;
  const kg_design& D = *F.D;
  if (sharded(ctx)) throw Error(E_INVAL, "iwls=tensor is not supported on a sharded context");
  if (D.d > 4) throw Error(E_INVAL, "iwls=tensor supports up to 4 modes on the device");
  const int d = static_cast<int>(D.d);
  i64 next = 0;
  for (int j = 0; j < d; ++j) next += D.n[j];
  if (!F.tS.p) {  // per-fit state, built on the first outer iteration
    F.tS.alloc(sizeof(double) * next);
    F.tf.alloc(sizeof(double) * next);
    F.text.alloc(sizeof(i64) * d);
    std::vector<i64> ext(D.n.begin(), D.n.end());
    KG_CUDA(cudaMemcpyAsync(F.text.p, ext.data(), sizeof(i64) * d, cudaMemcpyHostToDevice, ctx->s));
    for (i64 m = 0; m < D.c; ++m)
      for (i64 r = 0; r < D.c; ++r)
        for (i64 j = 0; j < D.d; ++j) {
          const FactorOwn& g = *D.gram[m][r][j];
          i64 cnt = 0;
          for (size_t a = 0; a < g.h_len.size(); ++a) cnt += g.h_len[a];
          auto c = std::make_unique<DBuf>();
          c->alloc(sizeof(double) * std::max<i64>(cnt, 1));
          BandOp op = g.dev.H;
          op.coef = c->d();
          F.wg.push_back(op);
          F.wgcoef.push_back(std::move(c));
        }
    if (D.c == 1) {
      i64 pmax = 1;
      for (int j = 0; j < d; ++j) pmax = std::max(pmax, D.p[0][j]);
      F.tdense.alloc(sizeof(double) * pmax * pmax * d);
      for (int j = 0; j < d; ++j) {  // power-iteration jobs: band, seeded start (spectral.cpp:16-24)
        const FactorOwn& g = *D.gram[0][0][j];
        const i64 p = D.p[0][j];
        auto J = std::make_unique<SpectralJob>();
        J->p = p;
        std::vector<int> glo(g.h_lo.begin(), g.h_lo.end()), ghi(static_cast<size_t>(p));
        int band = 0;
        for (i64 a = 0; a < p; ++a) {
          ghi[a] = glo[a] + g.h_len[a];
          band = std::max(band, g.h_len[a]);
        }
        J->band = band;
        if (p == 1) {
          F.tjobs.push_back(std::move(J));
          continue;
        }
        std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
        std::uniform_real_distribution<double> unif(0.5, 1.5);
        std::vector<double> v0(static_cast<size_t>(p));
        for (auto& x : v0) x = unif(rng);
        double z = 0.0;
        for (double x : v0) z += x * x;
        if (z > 0.0) {
          const double sq = std::sqrt(z);
          for (double& x : v0) x /= sq;
        }
        J->glo.alloc(sizeof(int) * p);
        J->ghi.alloc(sizeof(int) * p);
        J->v0.alloc(sizeof(double) * p);
        KG_CUDA(cudaMemcpyAsync(J->glo.p, glo.data(), sizeof(int) * p, cudaMemcpyHostToDevice, ctx->s));
        KG_CUDA(cudaMemcpyAsync(J->ghi.p, ghi.data(), sizeof(int) * p, cudaMemcpyHostToDevice, ctx->s));
        KG_CUDA(cudaMemcpyAsync(J->v0.p, v0.data(), sizeof(double) * p, cudaMemcpyHostToDevice, ctx->s));
        F.tjobs.push_back(std::move(J));
      }
    }
  }
  // geometric-mean factors of the exact weights, then v, z and max(v)
  i64 off = 0;
  for (int j = 0; j < d; ++j) {
    const i64 a = prod(D.n, 0, j), b = prod(D.n, j + 1, d);
    log_slab_sums(ctx->L(), F.v.d(), a, D.n[j], b, F.tS.d() + off);
    off += D.n[j];
  }
  tensor_factors(ctx->L(), F.tS.d(), static_cast<const i64*>(F.text.p), d, F.n, F.tf.d());
  TensorExt te;
  te.d = d;
  for (int j = 0; j < d; ++j) te.ext[j] = D.n[j];
  tensor_vz(ctx->L(), F.n, te, F.tf.d(), F.u.d(), F.eta.d(), F.v.d(), F.z.d(), vmax_part);
  // weighted Gram blocks
  for (i64 m = 0; m < D.c; ++m)
    for (i64 r = 0; r < D.c; ++r) {
      i64 fo = 0;
      for (i64 j = 0; j < D.d; ++j) {
        const FactorDev& xm = D.f[m][j]->dev;
        const FactorDev& xr = D.f[r][j]->dev;
        const size_t idx = static_cast<size_t>((m * D.c + r) * D.d + j);
        wgram_band(ctx->L(), xm.X, xr.X, D.n[j], F.tf.d() + fo, xm.G.lo, xm.G.len, xr.G.lo, xr.G.len, F.wg[idx],
                   F.wgcoef[idx]->d());
        fo += D.n[j];
      }
    }
  // Lipschitz factor
  if (D.c == 1) {
    i64 pmax = 1;
    for (int j = 0; j < d; ++j) pmax = std::max(pmax, D.p[0][j]);
    for (int j = 0; j < d; ++j) {
      SpectralJob& J = *F.tjobs[static_cast<size_t>(j)];
      double* G = F.tdense.d() + pmax * pmax * j;
      if (J.p == 1) {  // spectral.cpp:14: the 1 x 1 Gram itself
        J.Gview = F.wgcoef[static_cast<size_t>(j)]->d();
      } else {
        band_dense(ctx->L(), F.wg[static_cast<size_t>(j)], F.wgcoef[static_cast<size_t>(j)]->d(), J.p, G);
        J.Gview = G;
      }
    }
    double lip = 1.0;
    std::vector<double> rad = spectral_run_views(ctx, F.tjobs);
    for (double r0 : rad) lip *= r0;
    F.lipfac_t = lip;
  } else {
    F.lipfac_t = D.lipfac;  // lipschitz_upper: max(v) enters through the vmax partials (k_fista_init)
  }
  F.tensor = true;
  F.route = 1;
  F.wconst = 1.0;
  F.c0_valid = false;
  F.zptr = F.z.d();
}

static ModelTrace outer_loop(Fit& F, double lambda, const OuterCfg& oc) {
  kg_ctx* ctx = F.ctx;
  const kg_design& D = *F.D;
  const double n = static_cast<double>(D.N_full);
  ModelTrace tr;
  // eta = H(theta), f_cur = F(theta, eta)  (outer.cpp:185-186)
  reset_errs(F);
  HlastArgs h0 = hlast_args(F);
  h0.flags = HL_LL_NEW;
  int g = h_full(F, F.theta.d(), F.eta.d(), h0);
  reduce_cols(ctx->L(), F.part.d(), g, kHlastCols, 0, F.scal.d());
  ar_sum(ctx, F.scal.d(), kHlastCols);
  pnorm(ctx->L(), F.p, F.pen, F.alpha, F.theta.d(), F.Jpart.d());
  reduce_cols(ctx->L(), F.Jpart.d(), pgrid(F.p), 2, 0, F.scal.d() + 16);
  double* pin = ctx->pin();
  KG_CUDA(cudaMemcpyAsync(pin, F.scal.p, sizeof(double) * 20, cudaMemcpyDeviceToHost, ctx->s));
  ar_min_i64(ctx, F.errs.l(), 4);
  KG_CUDA(cudaMemcpyAsync(pin + PIN_ERR, F.errs.p, sizeof(i64) * 4, cudaMemcpyDeviceToHost, ctx->s));
  sync(ctx);
  {
    i64 errs[4];
    std::memcpy(errs, pin + PIN_ERR, sizeof(errs));
    check_ll_errs(F, errs);
  }
  double J_cur = penalty_of(F.pen, F.alpha, pin[16], pin[17]);
  double f_cur = -(pin[0] / F.disp) / n + lambda * J_cur;
  tr.initial_objective = f_cur;
  tr.final_objective = f_cur;

  const int n_vmax = elem_grid(F.n);
  double* vmax_part = F.part.d() + D.part_cap - n_vmax;
  for (i64 k = 0; k < oc.max_outer; ++k) {
    reset_errs(F);
    FamilyArgs fa;
    fa.n = F.n;
    fa.fam = F.fam;
    fa.mode = oc.wmode == KG_W_UNIT ? 1 : 0;
    fa.disp = F.disp;
    fa.y = F.O->y.d();
    fa.a = F.O->a_const ? nullptr : F.O->a.d();
    fa.a_val = F.O->a_val;
    fa.eta = F.eta.d();
    fa.u = oc.wmode == KG_W_TENSOR ? F.u.d() : nullptr;  // the score is only kept for the tensor weights
    fa.v = F.v.d();
    fa.z = F.z.d();
    fa.partial = vmax_part;
    fa.err = F.errs.l() + ERR_FAM;
    fa.cell_base = D.cell_base;
    family_pass(ctx->L(), fa);
    // unit weights (outer.cpp:234-238): X^T W X is the plain Gram product
    F.route = fa.mode == 1 ? 1 : 0;
    F.wconst = 1.0;
    F.c0_valid = false;
    F.zptr = F.z.d();
    F.tensor = false;
    if (oc.wmode == KG_W_TENSOR) tensor_weights(F, vmax_part, n_vmax);  // rank-one weights, Gram route
    xtwz_pass(F);
    fista_enqueue(F, lambda, oc.inner, vmax_part, n_vmax);
    // eta_tilde = H(theta_tilde) with Delta_k's inner product and the first trials.
    // The fused pass carries only the full step t = alpha0 (accepted in the
    // common case, test_outer.cpp:107-138): every extra trial costs an exp per
    // cell.  Rejections fall through to the batched trial passes below, which
    // compute the same per-trial sums (KG_TRIALS0 sets the first batch size).
    static const int first_batch = [] {
      const char* e = dev_env("KG_TRIALS0");
      const int v = e ? std::atoi(e) : 1;
      return v < 1 ? 1 : (v > kMaxTrials ? kMaxTrials : v);
    }();
    double t_list[kMaxTrials];
    double t = oc.alpha0;
    int nt = 0;
    for (; nt < first_batch && nt <= oc.max_bt; ++nt, t *= oc.b) t_list[nt] = t;
    HlastArgs h = hlast_args(F);
    h.flags = HL_DOT | HL_TRIALS | HL_U_FLY;  // u = score(eta) recomputed from y, a, eta (not streamed)
    h.eta_old = F.eta.d();
    h.ntrial = nt;
    for (int j = 0; j < nt; ++j) h.t[j] = t_list[j];
    g = h_full(F, F.best.d(), F.eta_t.d(), h);
    reduce_cols(ctx->L(), F.part.d(), g, kHlastCols, 0, F.scal.d());
  ar_sum(ctx, F.scal.d(), kHlastCols);
    ptrials(ctx->L(), F.p, F.pen, F.alpha, F.theta.d(), F.best.d(), nt, t_list, F.tpart.d());
    reduce_cols(ctx->L(), F.tpart.d(), pgrid(F.p), 2 * (1 + kMaxTrials), 0, F.scal.d() + 16);
    KG_CUDA(cudaMemcpyAsync(pin, F.scal.p, sizeof(double) * 40, cudaMemcpyDeviceToHost, ctx->s));
    ar_min_i64(ctx, F.errs.l(), 16);
    KG_CUDA(cudaMemcpyAsync(pin + PIN_ERR, F.errs.p, sizeof(i64) * 16, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    i64 errs[16];
    std::memcpy(errs, pin + PIN_ERR, sizeof(errs));
    // reference order: score (outer.cpp:241) then working response (:252)
    if (errs[ERR_FAM] != kNoErr)
      throw Error(E_EVAL, "non-finite score entry at cell " + std::to_string(errs[ERR_FAM]), errs[ERR_FAM]);
    if (errs[ERR_FAM + 1] != kNoErr)
      throw Error(E_EVAL, "non-finite working response entry at cell " + std::to_string(errs[ERR_FAM + 1]),
                  errs[ERR_FAM + 1]);
    const FistaOut fo = fista_read(F);
    if (fo.bad_weights) throw Error(E_INVAL, "lipschitz_upper: weights must not be all zero");
    tr.inner += fo.iterations;
    if (fo.diverged) {
      tr.status = KG_S_INNER_DIVERGENCE;
      return tr;
    }
    const double dot = pin[1];
    const double J_t = penalty_of(F.pen, F.alpha, pin[16], pin[17]);
    const double delta_k = -dot / n + lambda * (J_t - J_cur);
    const double decrease = std::min(delta_k, 0.0);
    // Armijo (outer.cpp:118-143): trials in order, batches of kMaxTrials.
    bool accepted = false;
    double t_acc = 0.0, f_acc = 0.0;
    int base = 0, j_acc = -1;
    std::vector<double> lls(pin + 2, pin + 2 + nt), Js(nt);
    for (int j = 0; j < nt; ++j) Js[j] = penalty_of(F.pen, F.alpha, pin[16 + 2 + 2 * j], pin[16 + 3 + 2 * j]);
    std::vector<i64> terr(errs + 2, errs + 2 + nt);
    t = oc.alpha0;
    for (i64 j = 0; j <= oc.max_bt; ++j, t *= oc.b) {
      if (j - base >= nt) {  // next batch of trials over (eta, eta_tilde)
        base = static_cast<int>(j);
        double tt = t;
        nt = 0;
        for (; nt < kMaxTrials && base + nt <= oc.max_bt; ++nt, tt *= oc.b) t_list[nt] = tt;
        reset_errs(F);
        HlastArgs hb = hlast_args(F);
        hb.P = nullptr;
        hb.eta_new = F.eta_t.d();
        hb.eta_old = F.eta.d();
        hb.flags = HL_TRIALS;
        hb.ntrial = nt;
        for (int q = 0; q < nt; ++q) hb.t[q] = t_list[q];
        hlast_mode1(ctx->L(), hb);
        reduce_cols(ctx->L(), F.part.d(), hlast_grid(hb), kHlastCols, 0, F.scal.d());
        ar_sum(ctx, F.scal.d(), kHlastCols);
        ptrials(ctx->L(), F.p, F.pen, F.alpha, F.theta.d(), F.best.d(), nt, t_list, F.tpart.d());
        reduce_cols(ctx->L(), F.tpart.d(), pgrid(F.p), 2 * (1 + kMaxTrials), 0, F.scal.d() + 16);
        KG_CUDA(cudaMemcpyAsync(pin, F.scal.p, sizeof(double) * 40, cudaMemcpyDeviceToHost, ctx->s));
        ar_min_i64(ctx, F.errs.l(), 16);
        KG_CUDA(cudaMemcpyAsync(pin + PIN_ERR, F.errs.p, sizeof(i64) * 16, cudaMemcpyDeviceToHost, ctx->s));
        sync(ctx);
        std::memcpy(errs, pin + PIN_ERR, sizeof(errs));
        lls.assign(pin + 2, pin + 2 + nt);
        Js.resize(nt);
        for (int q = 0; q < nt; ++q) Js[q] = penalty_of(F.pen, F.alpha, pin[16 + 2 + 2 * q], pin[16 + 3 + 2 * q]);
        terr.assign(errs + 2, errs + 2 + nt);
      }
      const int q = static_cast<int>(j - base);
      if (terr[q] != kNoErr)
        throw Error(E_EVAL, "non-finite log-likelihood term at cell " + std::to_string(terr[q]), terr[q]);
      const double f_trial = -(lls[q] / F.disp) / n + lambda * Js[q];
      if (std::isfinite(f_trial) && f_trial <= f_cur + t * oc.v * decrease) {
        accepted = true;
        t_acc = t;
        f_acc = f_trial;
        J_cur = Js[q];
        j_acc = static_cast<int>(j);
        break;
      }
    }
    tr.outer += 1;
    if (!accepted) {
      tr.recs.push_back(outer_rec(f_cur, 0.0, delta_k, fo.lip, fo.iterations, fo.converged, -1));
      tr.status = KG_S_LINE_SEARCH_FAILED;
      return tr;
    }
    tr.recs.push_back(outer_rec(f_acc, t_acc, delta_k, fo.lip, fo.iterations, fo.converged, j_acc));
    ptheta_update(ctx->L(), F.p, t_acc, F.best.d(), F.theta.d());
    eta_combine(ctx->L(), F.n, t_acc, F.eta_t.d(), F.eta.d());
    tr.final_objective = f_acc;
    const double rel = std::abs(f_acc - f_cur) / std::max(1.0, std::abs(f_cur));
    f_cur = f_acc;
    if (rel < oc.tol) {
      tr.status = KG_S_CONVERGED;
      return tr;
    }
  }
  tr.status = KG_S_MAX_ITERATIONS;
  return tr;
}

static std::vector<double> lambda_sequence(double lmax, i64 nl, double ratio) {
  if (!(lmax > 0.0)) throw Error(E_INVAL, "lambda_sequence: lambda_max must be positive");
  if (nl < 1) throw Error(E_INVAL, "lambda_sequence: n_lambda must be positive");
  if (!(ratio > 0.0 && ratio < 1.0)) throw Error(E_INVAL, "lambda_sequence: lambda_min_ratio must lie in (0,1)");
  std::vector<double> out(nl);
  out[0] = lmax;
  if (nl == 1) return out;
  const double step = std::log(ratio) / static_cast<double>(nl - 1);
  for (i64 t = 1; t < nl; ++t) out[t] = lmax * std::exp(step * static_cast<double>(t));
  return out;
}

static const char* status_name(int s) {
  static const char* names[] = {"converged", "max_iterations", "line_search_failed", "inner_divergence"};
  return names[s];
}

// single_solve: outer_solve (outer.cpp:159-303) for one lambda from theta = 0:
// the model is returned with whatever status it ends in (no first-model throw).
static kg_path_result* fit_path(kg_ctx* ctx, const kg_design* D, const kg_obs* O, int fam, double disp, int pen,
                                double alpha, const kg_path_cfg& cfg, const double* lambdas_in, i64 n_lambdas_in,
                                bool single_solve = false) {
  if (fam < 0 || fam > 3) throw Error(E_INVAL, "unknown family");
  if (pen < 0 || pen > 2) throw Error(E_INVAL, "unknown penalty");
  if (!(disp > 0.0)) throw Error(E_INVAL, "dispersion must be positive");
  if (pen == KG_ELASTIC_NET && !(alpha >= 0.0)) throw Error(E_INVAL, "elastic net alpha must be nonnegative");
  if (O->design != D) throw Error(E_INVAL, "observation was created for another design");
  OuterCfg oc;
  oc.max_outer = cfg.max_outer;
  oc.max_bt = cfg.armijo_max_backtracks;
  oc.alpha0 = cfg.armijo_alpha0;
  oc.b = cfg.armijo_b;
  oc.v = cfg.armijo_v;
  oc.tol = cfg.outer_tol;
  oc.wmode = static_cast<int>(cfg.weight_mode);
  oc.inner.nu = cfg.nu;
  oc.inner.tol = cfg.inner_tol;
  oc.inner.max_iters = cfg.inner_max_iters;
  oc.inner.monitor_every = cfg.monitor_every;
  oc.inner.extrapolation = static_cast<int>(cfg.extrapolation);
  if (oc.wmode < 0 || oc.wmode > 2) throw Error(E_INVAL, "unknown weight mode");

  auto F = std::make_unique<Fit>();
  F->ctx = ctx;
  F->D = D;
  F->O = O;
  F->fam = fam;
  F->disp = disp;
  F->pen = pen;
  F->alpha = pen == KG_ELASTIC_NET ? alpha : 0.0;
  alloc_fit(*F);

  auto res = std::make_unique<kg_path_result>();
  res->ctx = ctx;
  res->p = D->P;

  // grid (path.cpp:29-45) -- lambda_max validates the data first
  std::vector<double> lambdas;
  if (!lambdas_in) {
    if (pen == KG_RIDGE)
      throw Error(E_INVAL, "fit_path: penalty has no l1 component; supply an explicit lambda sequence");
    validate_obs(*F);
    const double lmax = lambda_max_fit(*F);
    if (!(lmax > 0.0))
      throw Error(E_INVAL,
                  "fit_path: lambda_max is zero (score vanishes at theta = 0); supply an explicit lambda sequence");
    lambdas = lambda_sequence(lmax, cfg.n_lambda, cfg.lambda_min_ratio);
    res->lambda_max = lmax;
  } else {
    lambdas.assign(lambdas_in, lambdas_in + n_lambdas_in);
  }
  if (lambdas.empty()) throw Error(E_INVAL, "fit_path: empty lambda sequence");
  for (size_t t = 0; t < lambdas.size(); ++t) {
    if (!(lambdas[t] >= 0.0)) throw Error(E_INVAL, "fit_path: lambda values must be nonnegative");
    if (t > 0 && !(lambdas[t] < lambdas[t - 1]))
      throw Error(E_INVAL, "fit_path: lambda sequence must be strictly decreasing");
  }
  // outer_solve argument checks (outer.cpp:165-178)
  if (!(oc.alpha0 > 0.0) || !(oc.b > 0.0 && oc.b < 1.0) || !(oc.v > 0.0 && oc.v < 1.0))
    throw Error(E_INVAL, "outer_solve: need alpha0 > 0 and Armijo constants b, v in (0,1)");
  if (oc.max_outer < 1 || !(oc.tol > 0.0)) throw Error(E_INVAL, "outer_solve: need max_outer >= 1 and outer_tol > 0");
  if (lambdas_in) validate_obs(*F);

  const i64 nl = static_cast<i64>(lambdas.size());
  res->coefs.alloc(sizeof(double) * D->P * nl);
  DBuf nnz;
  nnz.alloc(sizeof(i64) * nl);

  // state at theta = 0: eta = 0
  KG_CUDA(cudaMemsetAsync(F->theta.p, 0, sizeof(double) * F->p, ctx->s));
  KG_CUDA(cudaMemsetAsync(F->eta.p, 0, sizeof(double) * F->n, ctx->s));
  KG_CUDA(cudaMemsetAsync(F->stheta.p, 0, sizeof(double) * F->p, ctx->s));  // S'(0) = 0
  const bool gauss_shortcut = fam == KG_GAUSSIAN && oc.wmode == KG_W_EXACT;
  PathState st;
  int n_vmax = 0;
  if (gauss_shortcut) {
    // v = a * glm_weights = a / disp, z = y: fixed along the path, so the
    // weights, X^T W z and the Lipschitz bound are computed once (the
    // reference recomputes the same values per lambda).
    n_vmax = elem_grid(F->n);
    gauss_weights(ctx->L(), F->n, disp, O->a.d(), F->v.d(), F->part.d() + D->part_cap - n_vmax);
    F->zptr = O->y.d();
    xtwz_pass(*F);
    // constant prior weights: V = a/disp is a constant, use the Gram route
    if (O->a_const) {
      F->route = 1;
      F->wconst = (std::max(1.0, 1e-10) / disp) * O->a_val;
      F->c0_valid = false;
    }
    // loglik at eta = 0
    reset_errs(*F);
    HlastArgs h = hlast_args(*F);
    h.P = nullptr;
    h.eta_new = F->eta.d();
    h.flags = HL_LL_NEW;
    hlast_mode1(ctx->L(), h);
    reduce_cols(ctx->L(), F->part.d(), hlast_grid(h), kHlastCols, 0, F->scal.d());
    ar_sum(ctx, F->scal.d(), kHlastCols);
    double* pin = ctx->pin();
    KG_CUDA(cudaMemcpyAsync(pin, F->scal.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
    ar_min_i64(ctx, F->errs.l(), 1);
    KG_CUDA(cudaMemcpyAsync(pin + PIN_ERR, F->errs.p, sizeof(i64), cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    i64 e;
    std::memcpy(&e, pin + PIN_ERR, sizeof(i64));
    check_ll_errs(*F, &e);
    st.ll = pin[0] / disp;
  }
  // Gaussian, constant weights, one component: the whole path in one cooperative launch
  if (!single_solve && gauss_shortcut && F->route == 1 && F->gstep && !host_loop_mode() && oc.inner.max_iters >= 1 &&
      oc.inner.nu != 0.0 &&
      dev_env("KG_NO_DEVICE_PATH") == nullptr && gauss_path_ok(gstep_args(*F))) {
    if (!(F->wconst > 0.0)) throw Error(E_INVAL, "lipschitz_upper: weights must not be all zero");
    if (!(oc.inner.nu >= 0.0 && oc.inner.nu <= 1.0)) throw Error(E_INVAL, "fista_solve: nu must lie in [0,1]");
    FistaCtl h{};
    h.tol = oc.inner.tol;
    h.nu = oc.inner.nu;
    h.n = static_cast<double>(D->N_full);
    h.lipfac = D->lipfac;
    h.max_iters = oc.inner.max_iters;
    h.monitor_every = oc.inner.monitor_every;
    h.sscale = F->wconst;
    h.alpha = F->alpha;
    h.pen = F->pen;
    h.extrapolation = oc.inner.extrapolation;
    h.bt_div = oc.inner.nu > 0.0 && oc.inner.nu < 1.0;
    FistaCtl* staged = reinterpret_cast<FistaCtl*>(ctx->pin() + PIN_STAGE);
    sync(ctx);
    *staged = h;
    KG_CUDA(cudaMemcpyAsync(F->ctl.p, staged, sizeof(FistaCtl), cudaMemcpyHostToDevice, ctx->s));
    wzz(ctx->L(), F->n, F->v.d(), F->zptr, F->part.d());  // sum v z^2
    reduce_cols(ctx->L(), F->part.d(), elem_grid(F->n), 1, 0, &static_cast<FistaCtl*>(F->ctl.p)->ss_const);
    ar_sum(ctx, &static_cast<FistaCtl*>(F->ctl.p)->ss_const, 1);
    DBuf dl, p2, obj, its, stat, dks;
    dl.alloc(sizeof(double) * nl);
    p2.alloc(sizeof(double) * 5 * D->p[0][D->d - 1]);
    obj.alloc(sizeof(double) * nl);
    dks.alloc(sizeof(double) * 2 * nl);
    its.alloc(sizeof(i64) * nl);
    stat.alloc(sizeof(int) * (nl + 2));
    KG_CUDA(cudaMemcpyAsync(dl.p, lambdas.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, ctx->s));
    KG_CUDA(cudaMemsetAsync(stat.p, 0, sizeof(int) * (nl + 2), ctx->s));
    PersistArgs P;
    P.g = gstep_args(*F);
    P.X = F->pX.d();
    P.part = F->gpart.d();
    P.bar = static_cast<unsigned*>(F->pbar.p);
    P.flags = static_cast<unsigned*>(F->pflags.p);
    KG_CUDA(cudaMemsetAsync(F->pflags.p, 0, F->pflags.bytes, ctx->s));
    P.lambdas = dl.d();
    P.n_lambda = static_cast<int>(nl);
    P.part2 = p2.d();
    P.coefs = res->coefs.d();
    P.obj_out = obj.d();
    P.dk_out = dks.d();
    P.iters_out = static_cast<i64*>(its.p);
    P.status_out = static_cast<int*>(stat.p) + 2;
    P.nmodels = static_cast<int*>(stat.p);
    if (const char* e = dev_env("KG_PATH_DBG")) P.dbg = std::atoi(e);
    if (!ctx->ev[0]) {
      KG_CUDA(cudaEventCreate(&ctx->ev[0]));
      KG_CUDA(cudaEventCreate(&ctx->ev[1]));
    }
    KG_CUDA(cudaEventRecord(ctx->ev[0], ctx->s));
    gauss_path(ctx->L(), P);
    KG_CUDA(cudaEventRecord(ctx->ev[1], ctx->s));
    std::vector<double> ho(nl), hdk(2 * nl);
    std::vector<i64> hi(nl);
    std::vector<int> hs(nl + 2);
    FistaCtl* hctl = reinterpret_cast<FistaCtl*>(ctx->pin() + PIN_CTL);
    KG_CUDA(cudaMemcpyAsync(ho.data(), obj.p, sizeof(double) * nl, cudaMemcpyDeviceToHost, ctx->s));
    KG_CUDA(cudaMemcpyAsync(hdk.data(), dks.p, sizeof(double) * 2 * nl, cudaMemcpyDeviceToHost, ctx->s));
    KG_CUDA(cudaMemcpyAsync(hctl, F->ctl.p, sizeof(FistaCtl), cudaMemcpyDeviceToHost, ctx->s));
    KG_CUDA(cudaMemcpyAsync(hi.data(), its.p, sizeof(i64) * nl, cudaMemcpyDeviceToHost, ctx->s));
    KG_CUDA(cudaMemcpyAsync(hs.data(), stat.p, sizeof(int) * (nl + 2), cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    const int models = hs[0], stop = hs[1];
    {  // kg_path_kernel_stats
      float ms = 0.0f;
      KG_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
      i64 steps = 0;
      const int ran = models + (stop != 0 ? 1 : 0);  // a failed model's iterations count too
      for (int t = 0; t < ran && t < nl; ++t) steps += hi[t] > 0 ? hi[t] : 0;
      const GramStepArgs& g = P.g;
      double band = 0.0;  // sum over slabs of the neighbour band length
      for (i64 sl = 0; sl < g.pd; ++sl) band += g.Gd.hlen[sl];
      const double nb = static_cast<double>(g.pd);
      const double per_step = 8.0 * (band * g.q + static_cast<double>(D->P)) + 24.0 * nb * nb;
      ctx->path_ms = ms;
      ctx->path_steps = steps;
      ctx->path_bytes = per_step * static_cast<double>(steps) + 8.0 * static_cast<double>(D->P) * (models + 2);
    }
    if (stop == 2)
      throw Error(E_RUNTIME, std::string("fit_path: first model did not converge (") + status_name(hs[2]) + ")");
    res->truncated = stop == 1;
    for (int t = 0; t < models; ++t) {
      res->lambdas.push_back(lambdas[t]);
      res->objectives.push_back(ho[t]);
      res->initial_objectives.push_back(hdk[2 * t + 1]);
      res->outer_iters.push_back(1);
      res->inner_iters.push_back(hi[t]);
      res->status.push_back(hs[2 + t]);
      res->traces.push_back({outer_rec(ho[t], 1.0, hdk[2 * t], hctl->lip, hi[t], hs[2 + t] == KG_S_CONVERGED, 0)});
    }
    return res.release();
  }
  for (i64 t = 0; t < nl; ++t) {
    ModelTrace tr = gauss_shortcut ? gaussian_step(*F, lambdas[t], oc, st, n_vmax) : outer_loop(*F, lambdas[t], oc);
    if (tr.status != KG_S_CONVERGED && !single_solve) {
      if (t == 0)
        throw Error(E_RUNTIME, std::string("fit_path: first model did not converge (") + status_name(tr.status) + ")");
      res->truncated = true;
      break;
    }
    KG_CUDA(cudaMemcpyAsync(res->coefs.d() + D->P * t, F->theta.p, sizeof(double) * D->P, cudaMemcpyDeviceToDevice,
                            ctx->s));
    res->lambdas.push_back(lambdas[t]);
    res->objectives.push_back(tr.final_objective);
    res->initial_objectives.push_back(tr.initial_objective);
    res->traces.push_back(std::move(tr.recs));
    res->outer_iters.push_back(tr.outer);
    res->inner_iters.push_back(tr.inner);
    res->status.push_back(tr.status);
  }
  sync(ctx);
  return res.release();
}

}  // namespace kg

// =================================================================== C ABI
using namespace kg;

namespace {

template <class F>
kg_status guarded(kg_ctx* ctx, F&& f) {
  struct StreamScope {  // pool allocations of this call are ordered on the context stream
    cudaStream_t saved;
    explicit StreamScope(kg_ctx* c) : saved(g_stream) { g_stream = c ? c->s : nullptr; }
    ~StreamScope() { g_stream = saved; }
  } scope(ctx);
  try {
    f();
    if (ctx) {
      ctx->err.clear();
      ctx->err_cell = -1;
    }
    return KG_OK;
  } catch (const Error& e) {
    if (ctx) {
      ctx->err = e.what();
      ctx->err_cell = e.cell;
    }
    return static_cast<kg_status>(e.code);
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    return KG_ENOMEM;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return KG_ERUNTIME;
  }
}

void set_device(kg_ctx* ctx) { KG_CUDA(cudaSetDevice(ctx->device)); }

}  // namespace

extern "C" {

void kg_path_cfg_default(kg_path_cfg* c) {
  c->n_lambda = 100;
  c->lambda_min_ratio = 1e-4;
  c->max_outer = 100;
  c->armijo_alpha0 = 1.0;
  c->armijo_b = 0.5;
  c->armijo_v = 0.1;
  c->armijo_max_backtracks = 50;
  c->weight_mode = KG_W_EXACT;
  c->outer_tol = 1e-8;
  c->nu = 1.0;
  c->inner_max_iters = 2000;
  c->inner_tol = 1e-8;
  c->extrapolation = 0;
  c->monitor_every = 1;
}

kg_status kg_ctx_create(int device, kg_ctx** out) {
  *out = nullptr;
  auto ctx = std::make_unique<kg_ctx>();
  ctx->device = device;
  kg_status st = guarded(nullptr, [&] {
    int count = 0;
    KG_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw Error(E_INVAL, "no such CUDA device");
    KG_CUDA(cudaSetDevice(device));
    KG_CUDA(cudaStreamCreateWithFlags(&ctx->s, cudaStreamNonBlocking));
    KG_CUDA(cudaMallocHost(&ctx->pinned, 4096));
    cudaMemPool_t pool;
    KG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;  // keep freed workspaces cached between fits
    KG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live_streams.insert(ctx->s);
  });
  if (st == KG_OK) *out = ctx.release();
  return st;
}

kg_status kg_ctx_create_sharded(int device, int rank, int world, const void* nccl_unique_id, kg_ctx** out) {
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return KG_EINVAL;
  kg_ctx* ctx = nullptr;
  const kg_status st = kg_ctx_create(device, &ctx);
  if (st != KG_OK) return st;
  ctx->rank = rank;
  ctx->world = world;
  if (nccl_unique_id == nullptr) {  // no communicator: this slab's local partials only
    *out = ctx;
    return KG_OK;
  }
  const kg_status s2 = guarded(ctx, [&] {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    nccl_check(nccl_api()->CommInitRank(&ctx->comm, world, id, rank), "ncclCommInitRank");
  });
  if (s2 != KG_OK) {
    kg_ctx_destroy(ctx);
    return s2;
  }
  *out = ctx;
  return KG_OK;
}

kg_status kg_nccl_unique_id(void* out128) {
  return guarded(nullptr, [&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl_api()->GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

void kg_ctx_destroy(kg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->s) cudaStreamSynchronize(ctx->s);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->fork) {
    cudaStreamSynchronize(ctx->fork);
    cudaStreamDestroy(ctx->fork);
  }
  for (cudaEvent_t e : ctx->fork_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->stage) cudaFreeHost(ctx->stage);
  for (cudaEvent_t e : ctx->stage_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->comm) nccl_api()->CommDestroy(ctx->comm);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (cudaEvent_t e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->loop_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->s) {
    {
      std::lock_guard<std::mutex> lk(g_live_mu);
      g_live_streams.erase(ctx->s);
    }
    cudaStreamDestroy(ctx->s);
  }
  delete ctx;
}

const char* kg_last_error(const kg_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }
int64_t kg_last_error_cell(const kg_ctx* ctx) { return ctx ? ctx->err_cell : -1; }
void* kg_ctx_stream(kg_ctx* ctx) { return ctx->s; }
kg_status kg_ctx_synchronize(kg_ctx* ctx) {
  return guarded(ctx, [&] { sync(ctx); });
}
void kg_ctx_shard(const kg_ctx* ctx, int* rank, int* world) {
  *rank = ctx->rank;
  *world = ctx->world;
}
kg_status kg_path_kernel_stats(const kg_ctx* ctx, double* ms, double* bytes, int64_t* steps) {
  if (!ctx || ctx->path_ms < 0.0) return KG_EINVAL;
  *ms = ctx->path_ms;
  *bytes = ctx->path_bytes;
  *steps = ctx->path_steps;
  return KG_OK;
}
int64_t kg_launch_count(const kg_ctx* ctx) { return ctx->launches; }
void kg_launch_count_reset(kg_ctx* ctx) { ctx->launches = 0; }

kg_status kg_design_create(kg_ctx* ctx, int64_t c, int64_t d, const int64_t* n, const int64_t* p,
                           const double* const* factors, kg_design** out) {
  *out = nullptr;
  auto D = std::make_unique<kg_design>();
  kg_status st = guarded(ctx, [&] {
    set_device(ctx);
    ensure_stage(ctx);
    HostArena arena{static_cast<char*>(ctx->stage), kStageLanes * kStageSlots * kStageChunk, 0};
    g_arena = &arena;
    struct ArenaGuard {  // the arena is free again only once the stream has consumed it
      kg_ctx* c;
      ~ArenaGuard() {
        g_arena = nullptr;
        cudaStreamSynchronize(c->s);
      }
    } arena_guard{ctx};
    if (c < 1) throw Error(E_INVAL, "TensorDesign: need at least one component");
    if (d < 1) throw Error(E_INVAL, "TensorDesign: need at least one marginal factor");
    D->ctx = ctx;
    D->c = c;
    D->d = d;
    D->n_full.assign(n, n + d);
    for (i64 j = 0; j < d; ++j)
      if (n[j] < 1) throw Error(E_INVAL, "ArrayDims: extents must be positive");
    D->n = D->n_full;
    D->p.assign(c, std::vector<i64>(d));
    for (i64 r = 0; r < c; ++r)
      for (i64 j = 0; j < d; ++j) {
        D->p[r][j] = p[r * d + j];
        if (D->p[r][j] < 1) throw Error(E_INVAL, "TensorDesign: factors must have at least one column");
      }
    // this shard's slab of the last mode
    const i64 nd = D->n_full[d - 1];
    const i64 lo = nd * ctx->rank / ctx->world, hi = nd * (ctx->rank + 1) / ctx->world;
    D->n[d - 1] = hi - lo;
    if (D->n[d - 1] < 1) throw Error(E_INVAL, "sharded design: fewer last-mode slices than ranks");
    D->N = prod(D->n, 0, d);
    D->N_full = prod(D->n_full, 0, d);
    D->cell_base = lo * prod(D->n_full, 0, d - 1);
    D->P = 0;
    for (i64 r = 0; r < c; ++r) {
      D->offs.push_back(D->P);
      D->P += prod(D->p[r], 0, d);
    }
    D->f.resize(c);
    D->spectral.assign(c, std::vector<double>(d, 0.0));
    D->lipfac = 0.0;
    std::vector<std::unique_ptr<SpectralJob>> sjobs;
    for (i64 r = 0; r < c; ++r) {
      for (i64 j = 0; j < d; ++j) {
        FactorHost full;
        full.n = D->n_full[j];
        full.p = D->p[r][j];
        full.X.assign(factors[r * d + j], factors[r * d + j] + full.n * full.p);
        auto fo = std::make_unique<FactorOwn>();
        // the spectral radius always uses the full factor (L-hat is global)
        upload_factor(full, *fo, ctx->s);
        sjobs.push_back(std::make_unique<SpectralJob>());
        spectral_prepare(ctx, full, *fo, *sjobs.back());
        if (j == d - 1 && (lo != 0 || hi != nd)) {  // slice the rows of X_d for this shard
          FactorHost sl;
          sl.n = hi - lo;
          sl.p = full.p;
          sl.X.resize(sl.n * sl.p);
          for (i64 k = 0; k < sl.p; ++k)
            for (i64 i = 0; i < sl.n; ++i) sl.X[i + sl.n * k] = full.X[(lo + i) + full.n * k];
          fo = std::make_unique<FactorOwn>();
          upload_factor(sl, *fo, ctx->s);
        }
        D->f[r].push_back(std::move(fo));
      }
    }
    D->pending = spectral_launch(ctx, sjobs);  // every factor in one launch, collected by ensure_spectral
    // Gram blocks X_{m,j}^T X_{r,j} of the full factors (ascending-row sums
    // over the overlap of the two column bands), uploaded as banded operators.
    D->gram.resize(c);
    for (i64 m = 0; m < c; ++m) {
      D->gram[m].resize(c);
      for (i64 r = 0; r < c; ++r)
        for (i64 j = 0; j < d; ++j) {
          const double* Xm = factors[m * d + j];
          const double* Xr = factors[r * d + j];
          const i64 nj = D->n_full[j], pm = D->p[m][j], pr_ = D->p[r][j];
          auto cband = [&](const double* X, i64 p, std::vector<i64>& lo, std::vector<i64>& hi) {
            lo.assign(p, 0);
            hi.assign(p, 0);
            for (i64 k = 0; k < p; ++k) {
              i64 f = -1, l = -1;
              for (i64 i = 0; i < nj; ++i)
                if (X[i + nj * k] != 0.0) {
                  if (f < 0) f = i;
                  l = i;
                }
              if (f >= 0) {
                lo[k] = f;
                hi[k] = l + 1;
              }
            }
          };
          std::vector<i64> mlo, mhi, rlo, rhi;
          cband(Xm, pm, mlo, mhi);
          cband(Xr, pr_, rlo, rhi);
          FactorHost g;
          g.n = pm;
          g.p = pr_;
          g.X.assign(pm * pr_, 0.0);
          for (i64 b = 0; b < pr_; ++b)
            for (i64 a = 0; a < pm; ++a) {
              double s = 0.0;
              for (i64 i = std::max(mlo[a], rlo[b]); i < std::min(mhi[a], rhi[b]); ++i) s += Xm[i + nj * a] * Xr[i + nj * b];
              g.X[a + pm * b] = s;
            }
          auto go = std::make_unique<FactorOwn>();
          upload_factor(g, *go, ctx->s);
          D->gram[m][r].push_back(std::move(go));
        }
    }
    // fused mode-1 route for one component whose mode-1 fibre tile fits shared memory
    const i64 n1 = D->n[0], p1 = D->p[0][0], m = D->N / n1;
    D->fused = c == 1 && (n1 + p1) * 8 <= 96 * 1024;
    if (D->fused) {
      i64 T = std::max<i64>(1, 2048 / n1);
      T = std::min<i64>(T, std::max<i64>(1, m / 296));  // >= 2 CTAs per SM when the array allows
      while (T > 1 && (n1 + p1) * T * 8 > 96 * 1024) --T;
      D->T = static_cast<int>(T);
    }
    if (D->fused && d == 3 && dev_env("KG_NO_SLAB") == nullptr)
      D->slab = build_slab(factors[1], D->n[1], D->p[0][1], ctx->s);
    if (D->slab) build_slab_gather(*D->slab, factors[0], n1, p1, ctx->s);
    // (KG_HALO=0 keeps the all-reduce; KG_HALO=1 also runs the owned-slice
    // path on a one-rank communicator, where it has no neighbours: a test hook)
    const char* he = std::getenv("KG_HALO");
    if (ctx->comm && (ctx->world > 1 || (he && he[0] == '1')) && c == 1 && d >= 2) {
      const NcclApi* api = nccl_api();
      if ((!he || he[0] != '0') && api->Send && api->Recv && api->GroupStart && api->GroupEnd) {
        int64_t hp[9];
        if (kg_halo_plan(D->n_full[d - 1], D->p[0][d - 1], factors[d - 1], ctx->world, ctx->rank, hp) == KG_OK)
          for (int k = 0; k < 9; ++k) D->halo[k] = hp[k];
      }
    }
    D->scratch = chain_scratch(*D);
    const i64 tiles = D->fused ? (m + D->T - 1) / D->T : 0;
    const i64 hl_tiles = (m + D->T - 1) / D->T;
    D->part_cap = std::max<i64>({tiles, static_cast<i64>(elem_grid(D->N)), hl_tiles * kHlastCols}) +
                  elem_grid(D->N) + 64;
    sync(ctx);
  });
  if (st == KG_OK) *out = D.release();
  return st;
}

void kg_design_destroy(kg_design* d) {
  if (d && d->ctx) {
    cudaSetDevice(d->ctx->device);
    d->pending.reset();  // waits for the side stream
    cudaStreamSynchronize(d->ctx->s);
  }
  delete d;
  cudaGetLastError();  // a failure here must not surface in a later, unrelated launch check
}
int64_t kg_design_n(const kg_design* d) { return d->N; }
int64_t kg_design_p(const kg_design* d) { return d->P; }
kg_status kg_design_halo(const kg_design* d, int64_t* out9) {
  if (!d || !out9) return KG_EINVAL;
  for (int k = 0; k < 9; ++k) out9[k] = d->halo[k];
  return KG_OK;
}
kg_status kg_design_spectral(kg_design* d, int64_t r, int64_t j, double* out) {
  return guarded(d->ctx, [&] {
    if (r < 0 || r >= d->c || j < 0 || j >= d->d) throw Error(E_INVAL, "factor index out of range");
    set_device(d->ctx);
    ensure_spectral(d);
    *out = d->spectral[r][j];
  });
}

kg_status kg_obs_create(kg_ctx* ctx, const kg_design* design, const double* y, const double* a, int on_device,
                        kg_obs** out) {
  *out = nullptr;
  auto O = std::make_unique<kg_obs>();
  kg_status st = guarded(ctx, [&] {
    set_device(ctx);
    O->ctx = ctx;
    O->design = design;
    const size_t nb = sizeof(double) * design->N;
    O->y.alloc(nb);
    O->a.alloc(nb);
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (on_device)
      KG_CUDA(cudaMemcpyAsync(O->y.p, y, nb, k, ctx->s));
    else
      upload(ctx, O->y.p, y, nb);
    if (a) {
      if (on_device)
        KG_CUDA(cudaMemcpyAsync(O->a.p, a, nb, k, ctx->s));
      else
        upload(ctx, O->a.p, a, nb);
      O->unit_a = false;
      // are all prior weights equal?  (then W is a constant and the Gram route applies)
      DBuf part;
      const int g = elem_grid(design->N);
      part.alloc(sizeof(double) * 2 * g);
      minmax(ctx->L(), design->N, O->a.d(), part.d());
      sync(ctx);
      std::vector<double> hp(2 * g);  // per-CTA (min, max) -> global min / max
      KG_CUDA(cudaMemcpy(hp.data(), part.p, sizeof(double) * 2 * g, cudaMemcpyDeviceToHost));
      double mn = hp[0], mx = hp[1];
      for (int i = 0; i < g; ++i) {
        mn = std::min(mn, hp[2 * i]);
        mx = std::max(mx, hp[2 * i + 1]);
      }
      if (sharded(ctx)) {  // global (min, max) over the slabs: max of (-min, max)
        double* pin = ctx->pin();
        pin[0] = -mn;
        pin[1] = mx;
        KG_CUDA(cudaMemcpyAsync(part.p, pin, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->s));
        ar_max(ctx, part.d(), 2);
        KG_CUDA(cudaMemcpyAsync(pin, part.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
        sync(ctx);
        mn = -pin[0];
        mx = pin[1];
      }
      O->a_const = mn == mx;
      O->a_val = mn;
    } else {
      fill(ctx->L(), design->N, 1.0, O->a.d());  // ObservationData(y): a = 1 (family.hpp:44-45)
    }
    sync(ctx);
  });
  if (st == KG_OK) *out = O.release();
  return st;
}

void kg_obs_destroy(kg_obs* o) { delete o; }

kg_status kg_fit_path(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, int family, double dispersion,
                      int penalty, double alpha, const kg_path_cfg* cfg, const double* lambdas, int64_t n_lambdas,
                      kg_path_result** out) {
  *out = nullptr;
  if (ctx) ctx->path_ms = -1.0;  // kg_path_kernel_stats describes this fit only
  return guarded(ctx, [&] {
    set_device(ctx);
    kg_path_cfg c;
    kg_path_cfg_default(&c);
    if (cfg) c = *cfg;
    ensure_spectral(design);
    *out = fit_path(ctx, design, obs, family, dispersion, penalty, alpha, c, lambdas, n_lambdas);
  });
}

kg_status kg_outer_solve(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, int family, double dispersion,
                         int penalty, double alpha, const kg_path_cfg* cfg, double lambda, kg_path_result** out) {
  *out = nullptr;
  return guarded(ctx, [&] {
    set_device(ctx);
    kg_path_cfg c;
    kg_path_cfg_default(&c);
    if (cfg) c = *cfg;
    if (!(lambda >= 0.0)) throw Error(E_INVAL, "outer_solve: lambda must be nonnegative");
    ensure_spectral(design);
    *out = fit_path(ctx, design, obs, family, dispersion, penalty, alpha, c, &lambda, 1, true);
  });
}

int64_t kg_result_n_models(const kg_path_result* r) { return static_cast<int64_t>(r->lambdas.size()); }
int kg_result_truncated(const kg_path_result* r) { return r->truncated ? 1 : 0; }
double kg_result_lambda_max(const kg_path_result* r) { return r->lambda_max; }
// Per-model accessors: an out-of-range t (or a NULL result) gives NaN / -1
// instead of indexing past the vectors.
static bool model_ok(const kg_path_result* r, int64_t t) {
  return r && t >= 0 && t < static_cast<int64_t>(r->lambdas.size());
}
static constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
double kg_result_lambda(const kg_path_result* r, int64_t t) { return model_ok(r, t) ? r->lambdas[t] : kNaN; }
double kg_result_objective(const kg_path_result* r, int64_t t) { return model_ok(r, t) ? r->objectives[t] : kNaN; }
double kg_result_initial_objective(const kg_path_result* r, int64_t t) {
  return model_ok(r, t) ? r->initial_objectives[t] : kNaN;
}
int64_t kg_result_outer_iters(const kg_path_result* r, int64_t t) { return model_ok(r, t) ? r->outer_iters[t] : -1; }
int64_t kg_result_inner_iters(const kg_path_result* r, int64_t t) { return model_ok(r, t) ? r->inner_iters[t] : -1; }
int kg_result_status(const kg_path_result* r, int64_t t) { return model_ok(r, t) ? r->status[t] : -1; }
int64_t kg_result_n_outer(const kg_path_result* r, int64_t t) {
  return model_ok(r, t) ? static_cast<int64_t>(r->traces[t].size()) : -1;
}
kg_status kg_result_trace(const kg_path_result* r, int64_t t, kg_outer_record* out) {
  if (!model_ok(r, t) || !out) return KG_EINVAL;
  std::copy(r->traces[t].begin(), r->traces[t].end(), out);
  return KG_OK;
}
int64_t kg_result_nonzero(const kg_path_result* r, int64_t t) {
  if (!model_ok(r, t)) return -1;
  if (cudaSetDevice(r->ctx->device) != cudaSuccess) return -1;
  std::vector<double> h(r->p);
  if (cudaMemcpy(h.data(), r->coefs.d() + r->p * t, sizeof(double) * r->p, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  int64_t k = 0;
  for (double v : h) k += v != 0.0;
  return k;
}
kg_status kg_result_nonzeros(kg_path_result* r, int64_t* out) {
  return guarded(r->ctx, [&] {
    set_device(r->ctx);
    const i64 m = static_cast<i64>(r->lambdas.size());
    if (m == 0) return;
    DBuf cnt;
    cnt.alloc(sizeof(unsigned long long) * m);
    KG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * m, r->ctx->s));
    count_nonzero(r->ctx->L(), r->coefs.d(), r->p, m, static_cast<unsigned long long*>(cnt.p));
    std::vector<unsigned long long> h(m);
    KG_CUDA(cudaMemcpyAsync(h.data(), cnt.p, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost, r->ctx->s));
    sync(r->ctx);
    for (i64 t = 0; t < m; ++t) out[t] = static_cast<int64_t>(h[t]);
  });
}
kg_status kg_result_coef(kg_path_result* r, int64_t t, double* out) {
  return guarded(r->ctx, [&] {
    set_device(r->ctx);
    if (t < 0 || t >= static_cast<int64_t>(r->lambdas.size())) throw Error(E_INVAL, "model index out of range");
    KG_CUDA(cudaMemcpy(out, r->coefs.d() + r->p * t, sizeof(double) * r->p, cudaMemcpyDeviceToHost));
  });
}
kg_status kg_result_coefs(kg_path_result* r, int64_t first, int64_t count, double* out) {
  return guarded(r->ctx, [&] {
    set_device(r->ctx);
    const int64_t m = static_cast<int64_t>(r->lambdas.size());
    if (first < 0 || count < 0 || first + count > m) throw Error(E_INVAL, "model range out of range");
    if (count)
      KG_CUDA(cudaMemcpy(out, r->coefs.d() + r->p * first, sizeof(double) * r->p * count, cudaMemcpyDeviceToHost));
  });
}
void kg_result_free(kg_path_result* r) { delete r; }

kg_status kg_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return KG_EINVAL;
  *ptr = nullptr;
  if (cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return KG_ENOMEM;
  }
  return KG_OK;
}
void kg_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"

// ============================================================ operator probes
namespace {

struct Tmp {
  std::vector<std::unique_ptr<DBuf>> bufs;
  double* get(size_t n) {
    bufs.push_back(std::make_unique<DBuf>());
    bufs.back()->alloc(sizeof(double) * std::max<size_t>(n, 1));
    return bufs.back()->d();
  }
};

void h_map_dev(kg_ctx* ctx, const kg_design* D, const double* coef, double* eta, double* s0, double* s1) {
  for (i64 r = 0; r < D->c; ++r)
    run_chain(ctx, coef_dims(*D, r), h_steps(*D, r, 0), coef + D->offs[r], eta, s0, s1, r > 0);
}

void g_map_dev(kg_ctx* ctx, const kg_design* D, const double* u, double* coef, double* s0, double* s1) {
  for (i64 r = 0; r < D->c; ++r) run_chain(ctx, D->n, g_steps(*D, r, 0), u, coef + D->offs[r], s0, s1, false);
}

}  // namespace

namespace kg {
__global__ void k_rho(const double* A, double* out, i64 n1, i64 rest, BandOp op) {
  const i64 total = rest * op.rows;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 c = idx % rest, q = idx / rest;
    const int lo = op.lo[q], len = op.len[q];
    const double* cf = op.coef + op.off[q];
    const double* col = A + n1 * c;
    double s = 0.0;
    for (int t = 0; t < len; ++t) s = fma(cf[t], col[lo + t], s);
    out[c + rest * q] = s;  // rotated: (n2..nd, r)
  }
}
}  // namespace kg

extern "C" {

kg_status kg_h_map(kg_ctx* ctx, const kg_design* D, const double* coef, double* eta) {
  return guarded(ctx, [&] {
    set_device(ctx);
    Tmp t;
    double* dc = t.get(D->P);
    double* de = t.get(D->N);
    double *s0 = t.get(D->scratch), *s1 = t.get(D->scratch);
    KG_CUDA(cudaMemcpyAsync(dc, coef, sizeof(double) * D->P, cudaMemcpyHostToDevice, ctx->s));
    h_map_dev(ctx, D, dc, de, s0, s1);
    KG_CUDA(cudaMemcpyAsync(eta, de, sizeof(double) * D->N, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  });
}

kg_status kg_g_map(kg_ctx* ctx, const kg_design* D, const double* u, double* coef) {
  return guarded(ctx, [&] {
    set_device(ctx);
    Tmp t;
    double* du = t.get(D->N);
    double* dc = t.get(D->P);
    double *s0 = t.get(D->scratch), *s1 = t.get(D->scratch);
    KG_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * D->N, cudaMemcpyHostToDevice, ctx->s));
    g_map_dev(ctx, D, du, dc, s0, s1);
    ar_sum(ctx, dc, static_cast<size_t>(D->P));  // sharded: X^T u summed over the slabs
    KG_CUDA(cudaMemcpyAsync(coef, dc, sizeof(double) * D->P, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  });
}

kg_status kg_xtwx_apply(kg_ctx* ctx, const kg_design* D, const double* v, const double* coef, double* out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    Tmp t;
    double *dv = t.get(D->N), *de = t.get(D->N), *dw = t.get(D->N);
    double *dc = t.get(D->P), *dout = t.get(D->P);
    double *s0 = t.get(D->scratch), *s1 = t.get(D->scratch);
    KG_CUDA(cudaMemcpyAsync(dv, v, sizeof(double) * D->N, cudaMemcpyHostToDevice, ctx->s));
    KG_CUDA(cudaMemcpyAsync(dc, coef, sizeof(double) * D->P, cudaMemcpyHostToDevice, ctx->s));
    h_map_dev(ctx, D, dc, de, s0, s1);
    vz(ctx->L(), D->N, dv, de, dw);
    g_map_dev(ctx, D, dw, dout, s0, s1);
    ar_sum(ctx, dout, static_cast<size_t>(D->P));
    KG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * D->P, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  });
}

kg_status kg_rho(kg_ctx* ctx, int64_t r, const double* x, int64_t ndim, const int64_t* extents, const double* a,
                 double* out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (ndim < 1) throw Error(E_INVAL, "ArrayDims: need at least one dimension");
    const i64 n1 = extents[0];
    i64 rest = 1;
    for (i64 j = 0; j < ndim; ++j) {
      if (extents[j] < 1) throw Error(E_INVAL, "ArrayDims: extents must be positive");
      if (j) rest *= extents[j];
    }
    FactorHost h;  // rho's operator is x itself (r x n1): build its row bands via a transposed "factor"
    h.n = r;
    h.p = n1;
    h.X.assign(x, x + r * n1);
    FactorOwn f;
    upload_factor(h, f, ctx->s);
    Tmp t;
    double* da = t.get(n1 * rest);
    double* dout = t.get(rest * r);
    KG_CUDA(cudaMemcpyAsync(da, a, sizeof(double) * n1 * rest, cudaMemcpyHostToDevice, ctx->s));
    const i64 total = rest * r;
    const int g = static_cast<int>(std::min<i64>((total + 255) / 256, 148 * 16));
    k_rho<<<std::max(g, 1), 256, 0, ctx->s>>>(da, dout, n1, rest, f.dev.H);
    ++ctx->launches;
    KG_CUDA(cudaGetLastError());
    KG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * total, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  });
}

kg_status kg_lambda_max(kg_ctx* ctx, const kg_design* D, const kg_obs* O, int family, double dispersion, int penalty,
                        double, double* out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (penalty == KG_RIDGE) throw Error(E_INVAL, "lambda_max: pure ridge penalty has no finite lambda_max");
    if (O->design != D) throw Error(E_INVAL, "lambda_max: data dims do not match the design");
    Fit F;
    F.ctx = ctx;
    F.D = D;
    F.O = O;
    F.fam = family;
    F.disp = dispersion;
    alloc_fit(F);
    validate_obs(F);
    *out = lambda_max_fit(F);
  });
}

kg_status kg_predict(kg_ctx* ctx, const kg_design* D, int family, const double* coef, double* eta, double* mu) {
  return guarded(ctx, [&] {
    set_device(ctx);
    Tmp t;
    double *dc = t.get(D->P), *de = t.get(D->N), *dm = t.get(D->N);
    double *s0 = t.get(D->scratch), *s1 = t.get(D->scratch);
    KG_CUDA(cudaMemcpyAsync(dc, coef, sizeof(double) * D->P, cudaMemcpyHostToDevice, ctx->s));
    h_map_dev(ctx, D, dc, de, s0, s1);
    mean_map(ctx->L(), D->N, family, de, dm);
    KG_CUDA(cudaMemcpyAsync(eta, de, sizeof(double) * D->N, cudaMemcpyDeviceToHost, ctx->s));
    KG_CUDA(cudaMemcpyAsync(mu, dm, sizeof(double) * D->N, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  });
}

kg_status kg_mse_heldout(kg_ctx* ctx, const kg_design* D, const kg_path_result* R, int family, const double* y_full,
                         const double* mask, double* mse, int64_t* argmin) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (family < KG_GAUSSIAN || family > KG_GAMMA) throw Error(E_INVAL, "unknown family");
    // path.cpp:93-110 (validated on this rank's slab; the count is summed over the slabs)
    i64 n_held = 0;
    for (i64 i = 0; i < D->N; ++i) {
      const double m = mask[i];
      if (m != 0.0 && m != 1.0) throw Error(E_INVAL, "mse_heldout: mask entries must be 0 or 1");
      if (m == 1.0) ++n_held;
    }
    Tmp t;
    double *dy = t.get(D->N), *dmask = t.get(D->N), *de = t.get(D->N), *dm = t.get(D->N);
    double *s0 = t.get(D->scratch), *s1 = t.get(D->scratch);
    const i64 models = static_cast<i64>(R->lambdas.size());
    const int g = elem_grid(D->N);
    double* part = t.get(static_cast<i64>(g));
    double* out = t.get(std::max<i64>(models, 1) + 1);
    double* pin = ctx->pin();
    if (sharded(ctx)) {
      pin[0] = static_cast<double>(n_held);
      KG_CUDA(cudaMemcpyAsync(out, pin, sizeof(double), cudaMemcpyHostToDevice, ctx->s));
      ar_sum(ctx, out, 1);
      KG_CUDA(cudaMemcpyAsync(pin, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
      sync(ctx);
      n_held = static_cast<i64>(pin[0]);
    }
    if (n_held == 0) throw Error(E_INVAL, "mse_heldout: empty held-out mask");
    if (models == 0) throw Error(E_INVAL, "mse_heldout: empty path");
    KG_CUDA(cudaMemcpyAsync(dy, y_full, sizeof(double) * D->N, cudaMemcpyHostToDevice, ctx->s));
    KG_CUDA(cudaMemcpyAsync(dmask, mask, sizeof(double) * D->N, cudaMemcpyHostToDevice, ctx->s));
    for (i64 m = 0; m < models; ++m) {  // predict (path.cpp:83-89) + masked SSE per model
      h_map_dev(ctx, D, R->coefs.d() + R->p * m, de, s0, s1);
      mean_map(ctx->L(), D->N, family, de, dm);
      masked_sse(ctx->L(), D->N, dm, dy, dmask, part);
      reduce_cols(ctx->L(), part, g, 1, 0, out + m);
    }
    ar_sum(ctx, out, static_cast<size_t>(models));
    std::vector<double> h(models);
    KG_CUDA(cudaMemcpyAsync(h.data(), out, sizeof(double) * models, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    i64 best = 0;
    for (i64 m = 0; m < models; ++m) {
      mse[m] = h[m];
      if (h[m] < h[best]) best = m;  // first minimum (path.cpp:120)
    }
    *argmin = best;
  });
}

kg_status kg_result_deviance(kg_ctx* ctx, const kg_design* D, const kg_obs* O, const kg_path_result* R, int family,
                             double* out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (family < KG_GAUSSIAN || family > KG_GAMMA) throw Error(E_INVAL, "unknown family");
    if (!R || !O || O->design != D) throw Error(E_INVAL, "deviance: observation was created for another design");
    if (R->p != D->P) throw Error(E_INVAL, "deviance: result does not match the design");
    const i64 models = static_cast<i64>(R->lambdas.size());
    if (models == 0) return;
    Tmp t;
    double* de = t.get(D->N);
    double *s0 = t.get(D->scratch), *s1 = t.get(D->scratch);
    const int g = elem_grid(D->N);
    double* part = t.get(static_cast<i64>(g));
    double* dv = t.get(models);
    for (i64 m = 0; m < models; ++m) {  // eta = H(theta_m) on the device, then the deviance terms
      h_map_dev(ctx, D, R->coefs.d() + R->p * m, de, s0, s1);
      deviance_pass(ctx->L(), D->N, family, O->y.d(), O->a.d(), de, part);
      reduce_cols(ctx->L(), part, g, 1, 0, dv + m);
    }
    ar_sum(ctx, dv, static_cast<size_t>(models));  // sharded: summed over the slabs
    KG_CUDA(cudaMemcpyAsync(out, dv, sizeof(double) * models, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
  });
}

kg_status kg_time_kernel(kg_ctx* ctx, const kg_design* D, const kg_obs* O, int which, int reps, double* avg_ms,
                         double* bytes) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (reps < 1) throw Error(E_INVAL, "reps must be positive");
    Fit F;
    F.ctx = ctx;
    F.D = D;
    F.O = O;
    alloc_fit(F);
    KG_CUDA(cudaMemsetAsync(F.x.p, 0, sizeof(double) * F.p, ctx->s));
    gauss_weights(ctx->L(), F.n, 1.0, O->a.d(), F.v.d(), F.part.d() + D->part_cap - elem_grid(F.n));
    F.zptr = O->y.d();
    cudaEvent_t e0, e1;
    KG_CUDA(cudaEventCreate(&e0));
    KG_CUDA(cudaEventCreate(&e1));
    std::function<void()> launch;
    double b = 0.0;
    if (which == 2) {  // bandwidth reference: plain read of two n-arrays
      const double* y = O->y.d();
      const double* v = F.v.d();
      launch = [&, y, v] { stream_read2(ctx->L(), F.n, y, v, F.part.d()); };
      b = 16.0 * static_cast<double>(F.n);
    } else if (which == 0 && F.slab) {
      // the slab pass the fits run (modes 1 and 2 both ways per last-mode slice)
      run_chain(ctx, coef_dims(*D, 0), h_steps(*D, 0, 2), F.x.d(), F.P.d(), F.s0.d(), F.s1.d(), false);
      SlabArgs a = slab_args(F);
      a.S = F.P.d();
      a.Q = F.Q.d();
      launch = [&, a] { slab_pass(ctx->L(), a); };
      // v read, S3 (p1 x p2 x n3) read, Q3 written
      b = 8.0 * (static_cast<double>(F.n) + 2.0 * static_cast<double>(a.p1) * a.p2 * a.m3);
    } else if (which == 6 || which == 7) {
      // slab route: the mode-3 H step (p1 p2 x p3 -> x n3) or G step (x n3 -> x p3)
      if (!F.slab) throw Error(E_INVAL, "kg_time_kernel: this design does not run the slab route");
      const i64 a_ = D->p[0][0] * D->p[0][1], K = which == 6 ? D->p[0][2] : D->n[2],
                M = which == 6 ? D->n[2] : D->p[0][2];
      double* in = F.s0.d();
      double* outp = F.s1.d();
      KG_CUDA(cudaMemsetAsync(in, 0, sizeof(double) * a_ * K, ctx->s));
      const BandOp op = which == 6 ? D->f[0][2]->dev.H : D->f[0][2]->dev.G;
      launch = [&, in, outp, a_, K, M, op] { contract(ctx->L(), in, outp, a_, K, M, 1, op, false); };
      b = 8.0 * static_cast<double>(a_ * K + a_ * M);
    } else if (which == 0 || which == 3 || which == 4) {
      if (!D->fused) throw Error(E_INVAL, "the fused pass needs a one-component design");
      const double* P = F.x.d();
      if (D->d > 1) {
        run_chain(ctx, coef_dims(*D, 0), h_steps(*D, 0, 1), F.x.d(), F.P.d(), F.s0.d(), F.s1.d(), false);
        P = F.P.d();
      }
      FusedArgs a = fused_args(F);
      a.P = P;
      a.Q = D->d > 1 ? F.Q.d() : F.Sx.d();
      a.v = F.v.d();
      a.z = F.zptr;
      a.partial = F.part.d();
      a.dbg = which == 3 ? 1 : (which == 4 ? 2 : 0);  // 3: copies only, 4: copies + phase A
      const int var = F.expand ? FV_FISTA_EXP : FV_FISTA;  // the variant the fits run
      launch = [&, a, var] { run_fused(ctx, var, a); };
      // P (p1 x m) read, v (and z unless expanded) read, Q (p1 x m) written
      b = 8.0 * ((F.expand ? 1.0 : 2.0) * static_cast<double>(F.n) + 2.0 * static_cast<double>(a.p1 * a.m));
    } else if (which == 5) {
      // G-chain step of mode 1 (after the fused mode-0 pass): (p0, n1, rest) -> (p0, p1, rest)
      if (D->d < 2) throw Error(E_INVAL, "kg_time_kernel: the G-chain step needs d >= 2");
      const i64 a_ = D->p[0][0], K = D->n[1], M = D->p[0][1], b_ = prod(D->n, 2, D->d);
      double* in = F.eta.d();
      double* outp = F.s0.d();
      KG_CUDA(cudaMemsetAsync(in, 0, sizeof(double) * a_ * K * b_, ctx->s));
      const BandOp op = D->f[0][1]->dev.G;
      launch = [&, in, outp, a_, K, M, b_, op] { contract(ctx->L(), in, outp, a_, K, M, b_, op, false); };
      b = 8.0 * static_cast<double>(a_ * K * b_ + a_ * M * b_);
    } else {
      // largest H-chain step of component 0 (modes d-1 .. 0 applied to theta)
      std::vector<i64> dims = D->p[0];
      i64 best_j = D->d - 1, best_sz = 0;
      std::vector<i64> before_best;
      for (i64 j = D->d - 1; j >= 0; --j) {
        std::vector<i64> before = dims;
        dims[j] = D->n[j];
        const i64 sz = prod(dims, 0, dims.size()) + prod(before, 0, before.size());
        if (sz > best_sz) {
          best_sz = sz;
          best_j = j;
          before_best = before;
        }
      }
      const i64 a_ = prod(before_best, 0, best_j), K = before_best[best_j],
                b_ = prod(before_best, best_j + 1, before_best.size());
      const i64 M = D->n[best_j];
      double* in = F.s0.d();
      double* outp = F.eta.d();
      KG_CUDA(cudaMemsetAsync(in, 0, sizeof(double) * a_ * K * b_, ctx->s));
      const BandOp op = D->f[0][best_j]->dev.H;
      launch = [&, in, outp, a_, K, M, b_, op] { contract(ctx->L(), in, outp, a_, K, M, b_, op, false); };
      b = 8.0 * static_cast<double>(a_ * K * b_ + a_ * M * b_);
    }
    // L2 flush between timed launches: 256 MB written (> the 126 MB L2) so
    // every launch starts from HBM, as inside a C4/C5 step.
    DBuf flush;
    flush.alloc(size_t(256) << 20);
    for (int i = 0; i < 3; ++i) launch();
    double total = 0.0;
    for (int i = 0; i < reps; ++i) {
      KG_CUDA(cudaMemsetAsync(flush.p, i & 0xff, flush.bytes, ctx->s));
      KG_CUDA(cudaEventRecord(e0, ctx->s));
      launch();
      KG_CUDA(cudaEventRecord(e1, ctx->s));
      KG_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      KG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *avg_ms = total / reps;
    *bytes = b;
  });
}

// ------------------------------------------------------- input builders
kg_status kg_bin_scatter(kg_ctx* ctx, int64_t npts, int64_t d, const double* points, const double* lo,
                         const double* hi, const int64_t* bins, int on_device, double* counts, int64_t* dropped) {
  return guarded(ctx, [&] {
    // bspline.cpp:109-121 (argument checks, same messages)
    if (d <= 0 || !lo || !hi || !bins) throw Error(E_INVAL, "bin_scatter: bounds and bins must agree on the dimension");
    if (d > kMaxBinDims) throw Error(E_INVAL, "bin_scatter: at most 8 dimensions");
    if (npts < 0 || (npts > 0 && !points) || !counts) throw Error(E_INVAL, "bin_scatter: null buffer");
    BinArgs A;
    A.d = static_cast<int>(d);
    A.npts = npts;
    static const int bin_mode = [] { const char* e = dev_env("KG_BIN_MODE"); return e ? std::atoi(e) : 0; }();
    A.mode = bin_mode;
    A.cells = 1;
    for (int64_t j = 0; j < d; ++j) {
      if (bins[j] < 1) throw Error(E_INVAL, "bin_scatter: need at least one bin");
      if (!(hi[j] > lo[j])) throw Error(E_INVAL, "bin_scatter: degenerate bounds");
      A.lo[j] = lo[j];
      A.hi[j] = hi[j];
      A.width[j] = (hi[j] - lo[j]) / static_cast<double>(bins[j]);
      A.inv[j] = 1.0 / A.width[j];
      if (bins[j] > INT32_MAX || A.cells > INT32_MAX / bins[j])
        throw Error(E_INVAL, "bin_scatter: grid too large (at most 2^31 - 1 cells)");
      A.bmax[j] = static_cast<int>(bins[j] - 1);
      A.stride[j] = static_cast<int>(A.cells);  // column-major: the first index runs fastest (bspline.cpp:145-148)
      A.cells *= bins[j];
    }
    set_device(ctx);
    int n_sm = 148;
    KG_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, ctx->device));
    Tmp t;
    double* dcounts = on_device ? counts : t.get(A.cells);
    const double* dpts = points;
    if (!on_device && npts > 0) {
      double* up = t.get(npts * d);
      KG_CUDA(cudaMemcpyAsync(up, points, sizeof(double) * npts * d, cudaMemcpyHostToDevice, ctx->s));
      dpts = up;
    }
    unsigned long long* ddrop = reinterpret_cast<unsigned long long*>(t.get(1));
    KG_CUDA(cudaMemsetAsync(dcounts, 0, sizeof(double) * A.cells, ctx->s));
    KG_CUDA(cudaMemsetAsync(ddrop, 0, sizeof(unsigned long long), ctx->s));
    A.counts = dcounts;
    A.dropped = ddrop;

    // chunks keep every CTA's u32 counters far below 2^32
    const int64_t chunk = int64_t(1) << 31;
    for (int64_t first = 0; first < npts; first += chunk) {
      BinArgs C = A;
      C.pts = dpts + first * d;
      C.npts = std::min(chunk, npts - first);
      bin_scatter(ctx->L(), C, n_sm);
    }
    int64_t* pin = reinterpret_cast<int64_t*>(ctx->pin());
    KG_CUDA(cudaMemcpyAsync(pin, ddrop, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->s));
    if (!on_device) KG_CUDA(cudaMemcpyAsync(counts, dcounts, sizeof(double) * A.cells, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    if (dropped) *dropped = pin[0];
  });
}

kg_status kg_bspline_design_dev(kg_ctx* ctx, int64_t npts, const double* points, int64_t order, int64_t nb,
                                int on_device, double* out) {
  return guarded(ctx, [&] {
    if (npts < 2) throw Error(E_INVAL, "MarginalGrid: need at least two grid points");
    if (order < 1) throw Error(E_INVAL, "bspline_design: order must be at least 1");
    if (nb < order) throw Error(E_INVAL, "bspline_design: need at least `order` basis functions");
    if (order > kMaxOrder) throw Error(E_INVAL, "bspline_design: order above 16 is host-only");
    set_device(ctx);
    Tmp t;
    const double* dpts = points;
    if (!on_device) {
      double* up = t.get(npts);
      KG_CUDA(cudaMemcpyAsync(up, points, sizeof(double) * npts, cudaMemcpyHostToDevice, ctx->s));
      dpts = up;
    }
    double* pin = ctx->pin();
    KG_CUDA(cudaMemcpyAsync(pin, dpts, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
    KG_CUDA(cudaMemcpyAsync(pin + 1, dpts + npts - 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    const double lo = pin[0], hi = pin[1];
    // clamped uniform knots, computed exactly as the host builder (bspline.cpp:30-42)
    const int64_t spans = nb - order + 1;
    const double h = (hi - lo) / static_cast<double>(spans);
    std::vector<double> knots(static_cast<size_t>(nb + order));
    for (int64_t i = 0; i < order; ++i) knots[i] = lo;
    for (int64_t i = 0; i < nb - order; ++i) knots[order + i] = lo + h * static_cast<double>(i + 1);
    for (int64_t i = 0; i < order; ++i) knots[nb + i] = hi;
    double* dk = t.get(knots.size());
    KG_CUDA(cudaMemcpyAsync(dk, knots.data(), sizeof(double) * knots.size(), cudaMemcpyHostToDevice, ctx->s));
    double* dout = on_device ? out : t.get(npts * nb);
    int* bad = reinterpret_cast<int*>(t.get(1));
    KG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->s));
    bspline_design_dev(ctx->L(), npts, dpts, static_cast<int>(order), nb, dk, dout, bad);
    int* pbad = reinterpret_cast<int*>(pin + 2);
    KG_CUDA(cudaMemcpyAsync(pbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->s));
    if (!on_device) KG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * npts * nb, cudaMemcpyDeviceToHost, ctx->s));
    sync(ctx);
    if (*pbad) throw Error(E_INVAL, "MarginalGrid: points must be strictly increasing");
  });
}

}  // extern "C"
