// Internal declarations shared by the kronglm_b200 CUDA sources.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

namespace kg {

using i64 = int64_t;

// ------------------------------------------------------------------ errors
// Codes mirror kg_status (include/kronglm_b200.h).
struct Error : std::runtime_error {
  int code;
  i64 cell;
  Error(int c, const std::string& m, i64 cl = -1) : std::runtime_error(m), code(c), cell(cl) {}
};
enum { E_INVAL = 1, E_EVAL = 2, E_RUNTIME = 3, E_DIVERGE = 4, E_POWER = 5, E_CUDA = 6, E_NCCL = 7, E_NOMEM = 8 };

#define KG_CUDA(expr)                                                                                 \
  do {                                                                                                \
    cudaError_t e__ = (expr);                                                                         \
    if (e__ != cudaSuccess)                                                                           \
      throw ::kg::Error(e__ == cudaErrorMemoryAllocation ? ::kg::E_NOMEM : ::kg::E_CUDA,              \
                        std::string(#expr) + ": " + cudaGetErrorString(e__));                         \
  } while (0)

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute:
// raise it once per (current device, kernel) to at least `bytes`.  Thread
// safe; contexts on several devices each get it set (kg_solver.cu).
void smem_attr_raw(const void* fn, int bytes);
template <class K>
inline void smem_attr(K* fn, int bytes) {
  smem_attr_raw(reinterpret_cast<const void*>(fn), bytes);
}

// Division by a loop-invariant divisor as multiply-high + shift (valid for
// numerators < 2^31); built on the host, used in kernels.
struct FastDiv {
  uint32_t d, m, s;
  __host__ __device__ explicit FastDiv(uint32_t dd = 1) : d(dd), m(0), s(0) {
    if (d > 1) {
      uint32_t l = 0;
      while ((1ull << l) < d) ++l;
      m = static_cast<uint32_t>(((1ull << (31 + l)) + d - 1) / d);
      s = l - 1;
    }
  }
#ifdef __CUDACC__
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return d == 1 ? n : (__umulhi(n, m) >> s); }
#endif
};

// Developer switches (tuning sweeps, measurement-only variants, debug traces)
// are read only when KG_DEV=1, so a production process always runs the
// default routes.  The two operational switches, KG_HOST_LOOP (drive the FISTA
// loop from the host so profilers can see its kernels) and KG_HALO (0: keep
// the p-sized all-reduce on sharded contexts), are read directly.
inline const char* dev_env(const char* name) {
  static const bool dev = [] {
    const char* e = std::getenv("KG_DEV");
    return e && e[0] == '1';
  }();
  return dev ? std::getenv(name) : nullptr;
}

// ------------------------------------------------------------ band operators
// One banded operator C (rows x cols): row m has nonzeros at columns
// [lo[m], lo[m]+len[m]) with packed coefficients coef[off[m] + t].  For the
// H direction C = X_j (n_j x p_j, row bands of X); for the G direction
// C = X_j^T (p_j x n_j, column bands of X).  Bands are derived from the
// dense factor by an exact-zero test, so skipped terms are exact zeros.
struct BandOp {
  const int* lo = nullptr;
  const int* len = nullptr;
  const i64* off = nullptr;
  const double* coef = nullptr;
  i64 rows = 0, cols = 0;
  int maxlen = 0;
  const int* hlo = nullptr;   // host copies (planning only; never dereferenced on the device)
  const int* hlen = nullptr;
  uint64_t uid = 0;           // unique per uploaded operator (plan cache key)
  // row-blocked form (H operators of B-spline factors): rows in groups of
  // kRB; group g reads the input window [blo[g], blo[g] + kRW) and row
  // 4g + r uses bcoef[(g * kRB + r) * kRW + w] (zero outside its band)
  const int* blo = nullptr;
  const double* bcoef = nullptr;
  // wide-window row-blocked form (G operators X_j^T of B-spline factors):
  // rows in groups of kGB, group g reads [wblo[g], wblo[g] + kGW) and row
  // kGB g + r uses wbcoef[(g * kGB + r) * kGW + w] (zero outside its band)
  const int* wblo = nullptr;
  const double* wbcoef = nullptr;
  // the same for H operators (rows of X_j): kHB rows per group, kHW-wide window
  const int* hblo = nullptr;
  const double* hbcoef = nullptr;
};
constexpr int kRB = 4, kRW = 8;
constexpr int kGB = 4, kGW = 32;
constexpr int kHB = 16, kHW = 8;

// Device + host copies of one factor's operators.
struct FactorDev {
  i64 n = 0, p = 0;
  double* X = nullptr;  // dense n x p column-major (Gram / power iteration)
  BandOp H, G;          // device views
  void* blob = nullptr; // owning allocation for the band arrays
  double spectral = 0.0;
};

// ------------------------------------------------------- FISTA control block
// Device-resident state of one fista_solve (inner.cpp:121-235).  Kernels of
// the iteration read their scalars from here so one captured CUDA graph
// serves every lambda and every outer iteration.
struct FistaCtl {
  // configuration
  double lambda, tol, nu, n, lipfac;
  i64 max_iters, monitor_every;
  double sscale;      // S used by the step = sscale * (stored S): 1, or the constant weight (Gram route)
  double ss_const;    // added to the reduced weighted SS (Gram route: sum v z^2)
  double alpha;       // elastic-net weight
  int pen;            // 0 lasso, 1 ridge, 2 elastic net
  int extrapolation;  // 0 fista, 1 none
  int bt_div;         // nu in (0,1)
  // state
  double delta, omega, g_prev, best_g, lip;
  i64 it, momentum, streak, prox_steps, backtracks, iterations;
  int copy_best, restart, done, converged, diverged, bad_weights;
  int pad;
};

// ----------------------------------------------------------------- kernels
// Launch wrappers (kg_kernels.cu).  All run on `s`.
struct Launch {
  cudaStream_t s;
  i64* counter;  // incremented per launch (host-side launch accounting)
  // Programmatic dependent launch: kernels that support it (k_contract_gb,
  // k_slab4: they execute griddepcontrol.wait before touching what earlier
  // kernels wrote) are launched with programmatic stream serialization, so
  // their launch and prologue overlap the tail of the kernel before them.
  // Every other kernel ignores the flag and is launched normally.
  bool pdl = false;
};

// Launch configuration of a PDL-capable kernel (see Launch::pdl).
struct PdlConfig {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1] = {};
  PdlConfig(dim3 grid, dim3 block, size_t smem, const Launch& L) {
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = L.s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = L.pdl ? 1 : 0;
  }
};

// After every kernel launch: surface launch-configuration errors immediately
// (they are otherwise silent) and count the launch.
inline void launched(const Launch& L) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(E_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
  if (L.counter) ++*L.counter;
}

void contract(const Launch& L, const double* A, double* out, i64 a, i64 K, i64 M, i64 b, const BandOp& op,
              bool accumulate);

// FV_FISTA: partials of sum v (eta - z)^2 (the reference's inner_quadratic);
// FV_FISTA_EXP: partials of sum v eta^2 only (z is not read), for the expanded
// objective sum v (eta - z)^2 = sum v eta^2 - 2 <b, x> + sum v z^2 with
// b = X^T (v .* z) (the Gram route's identity, applied on the n-space route).
enum FusedVariant { FV_FISTA = 0, FV_XTWZ = 1, FV_SCORE0 = 2, FV_FISTA_EXP = 3 };
// X1^T of a banded factor as FP64 tensor-core (DMMA m8n8k4) A fragments for
// the fused pass: output rows k in groups of kMmaK; group g reads the input
// window [base[g], base[g] + 4 ks) and afrag[(g ks + s) 32 + lane] is the A
// element lane holds at k-step s, X1[base[g] + 4 s + lane % 4, kMmaK g +
// lane / 4] (zero outside the band).  Built on the host at factor upload.
constexpr int kMmaK = 8;
struct MmaOp {
  const int* base = nullptr;
  const double* afrag = nullptr;
  int ks = 0, groups = 0;
};

struct FusedArgs {
  i64 n1 = 0, p1 = 0, m = 0;  // mode-1 extents and the number of mode-1 fibres (n / n1)
  MmaOp mg;                    // the G operator as DMMA fragments (ks == 0: unavailable)
  int T = 1;                   // fibres per CTA
  BandOp H, G;                 // mode-1 operators
  const double* P = nullptr;   // p1 x m H-partial (FISTA)
  double* Q = nullptr;         // p1 x m G-partial (out)
  const double* v = nullptr;
  const double* z = nullptr;
  const double* y = nullptr;
  const double* a = nullptr;
  int fam = 0;
  double disp = 1.0;
  double* partial = nullptr;   // one double per CTA (FISTA: sum v (eta - z)^2)
  i64* err = nullptr;          // SCORE0: first non-finite score cell
  i64 cell_base = 0;           // global flat index of local cell 0 (sharding)
  int dbg = 0;                 // measurement only: 1 = copies only, 2 = copies + phase A
};
int fused_grid(const FusedArgs& f);
// Slab pass (kg_slab.cu): modes 1 and 2 of one n-space FISTA step (FV_FISTA_EXP)
// fused per slice of the last mode of a d = 3 design: S3 = x x_3 X3 in,
// Q3 = X1^T (v .* (X1 S3 X2^T)) X2 out, one read of v.
struct SlabArgs {
  int n1 = 0, n2 = 0, p1 = 0, p2 = 0;
  i64 m3 = 0;                   // slices (local last-mode extent)
  int nch = 0;                  // chunks of 8 mode-2 grid rows
  int cg = 1, ldS = 0, ldZ = 0, ldU = 0, ldW = 0;  // set by the launcher
  BandOp H1;                    // rows of X1 (<= 4 taps)
  MmaOp g1;                     // X1^T as DMMA A fragments
  // per chunk c of X2 (8 rows 8c .. 8c + 7, 8-wide coefficient window from w0[c]):
  const int* w0 = nullptr;
  const double* x2u = nullptr;  // [c][s][lane] = X2[8c + lane/4, w0[c] + 4s + lane%4]
  // Z step: the chunk's window inside the aligned 8-column tiles t0 (and t0 + 1),
  // tz[c] = t0 | (second tile used) << 16
  const int* tz = nullptr;
  const double* x2z = nullptr;  // [c][tile][s][lane] = X2[8c + 2 (lane%4) + s, 8 (t0 + tile) + lane/4]
  // scatter/gather form of Y = X1^T w (k_slab2): basis function k sums the
  // partials of the row quads whose window holds it; gat[4k .. 4k+3] = up to 8
  // 16-bit slots (quad * 5 + tap, or the zero slot), gmax = most slots of any k
  // (0: unavailable), PL = slots per column-pair plane (= 2 mod 8, zero slot last)
  const int* gat = nullptr;
  int gmax = 0, PL = 0;
  int pf = 0;                   // v chunks prefetched into L2 ahead of the register loads (set by the launcher)
  const double* S = nullptr;    // p1 x p2 x m3
  const double* v = nullptr;    // n1 x n2 x m3
  double* Q = nullptr;          // p1 x p2 x m3 (out)
  double* partial = nullptr;    // one double per CTA: sum v eta^2
};
bool slab_ok(const SlabArgs& a);
int slab_grid(const SlabArgs& a);
void slab_pass(const Launch& L, const SlabArgs& a);

// plain streaming read of two n-arrays (bandwidth reference for kg_time_kernel)
void stream_read2(const Launch& L, i64 n, const double* x, const double* y, double* partial);
void fused_mode1(const Launch& L, int variant, const FusedArgs& f);
// bulk-async pipelined version (kg_fused.cu)
bool fused_tma_fits(const FusedArgs& f, int variant);
int fused_tma_grid(const FusedArgs& f, int variant);
void fused_tma(const Launch& L, int variant, const FusedArgs& f);
// the register-hoisted kernel applies (required for FV_FISTA_EXP)
bool fused_fast_ok(const FusedArgs& f, int variant);
void contract_tiled(const Launch& L, const double* A, double* out, i64 a, i64 K, i64 M, i64 b, const BandOp& op,
                    bool accumulate);


// H-last (+ reductions) over mode 1.  If P is null, eta_new is an input
// (already computed by a full H chain) and only the reductions run.
enum HlastFlags { HL_LL_NEW = 1, HL_DOT = 2, HL_TRIALS = 4, HL_U_FLY = 8, HL_WRITE = 16 };
constexpr int kMaxTrials = 8;
constexpr int kPathTaps = 8;  // unrolled Gram band taps of k_gauss_path (cubic B-splines: 7)
constexpr int kHlastCols = 2 + kMaxTrials;  // [ll_new, dot, trial_0..]
struct HlastArgs {
  i64 n1 = 0, p1 = 0, m = 0;
  int T = 1;
  BandOp H;
  const double* P = nullptr;
  double* eta_new = nullptr;
  const double* eta_old = nullptr;
  const double* u = nullptr;
  const double* y = nullptr;
  const double* a = nullptr;          // prior weights; nullptr: every cell has weight a_val
  double a_val = 1.0;
  int fam = 0;
  double disp = 1.0;
  int flags = 0;
  int ntrial = 0;
  double t[kMaxTrials] = {0};
  double* partial = nullptr;   // kHlastCols per CTA
  i64* err = nullptr;          // [ll_new, u_fly, trial_0..trial_7]
  i64 cell_base = 0;
};
int hlast_grid(const HlastArgs& h);
void hlast_mode1(const Launch& L, const HlastArgs& h);

// Elementwise family pass: u, v, z and max(v) partials (outer.cpp:241-267).
struct FamilyArgs {
  i64 n = 0;
  int fam = 0, mode = 0;  // mode: 0 exact, 1 unit
  double disp = 1.0;
  const double *y = nullptr, *a = nullptr, *eta = nullptr;  // a == nullptr: every cell has weight a_val
  double a_val = 1.0;
  double *u = nullptr, *v = nullptr, *z = nullptr;  // u may be nullptr (not stored)
  double* partial = nullptr;  // max(v) per CTA
  i64* err = nullptr;         // [score, working response]
  i64 cell_base = 0;
};
int elem_grid(i64 n);
void family_pass(const Launch& L, const FamilyArgs& f);
// v = a / disp (Gaussian shortcut, outer.cpp:203-205 with glm_weights = 1/disp) and max partials.
void gauss_weights(const Launch& L, i64 n, double disp, const double* a, double* v, double* partial);
// Generic-route (c > 1) elementwise pieces.
void wss(const Launch& L, i64 n, const double* eta, const double* v, const double* z, double* w, double* partial);
void vz(const Launch& L, i64 n, const double* v, const double* z, double* w);
void score0(const Launch& L, i64 n, int fam, double disp, const double* y, const double* a, double* w, i64* err,
            i64 cell_base);
// validate (family.cpp:73-109): err[0] = first bad cell, codes[] read back at that cell.
void validate_pass(const Launch& L, i64 n, int fam, const double* y, const double* a, i64* err, i64 cell_base);
void eta_combine(const Launch& L, i64 n, double t, const double* eta_t, double* eta);
void mean_map(const Launch& L, i64 n, int fam, const double* eta, double* mu);
// iwls = tensor (outer.cpp:53-103, design.cpp:126-151)
struct TensorExt {
  int d = 0;
  i64 ext[4] = {1, 1, 1, 1};
};
void log_slab_sums(const Launch& L, const double* v, i64 a, i64 K, i64 b, double* S);
void tensor_factors(const Launch& L, const double* S, const i64* ext_dev, int d, i64 n, double* f);
void tensor_vz(const Launch& L, i64 n, const TensorExt& te, const double* f, const double* u, const double* eta,
               double* v, double* z, double* vmax);
void wgram_band(const Launch& L, const double* Xm, const double* Xr, i64 n, const double* w, const int* clo_m,
                const int* clen_m, const int* clo_r, const int* clen_r, const BandOp& g, double* coef);
void band_dense(const Launch& L, const BandOp& g, const double* coef, i64 p, double* G);
// per-CTA (elem_grid(n)) partials of sum_{mask == 1} (mu - y)^2
void masked_sse(const Launch& L, i64 n, const double* mu, const double* y, const double* mask, double* part);
void fill(const Launch& L, i64 n, double v, double* x);
// per-CTA (elem_grid(n)) partials of the deviance of eta (kg_result_deviance)
void deviance_pass(const Launch& L, i64 n, int fam, const double* y, const double* a, const double* eta,
                   double* part);

// p-space
int pgrid(i64 p);
int ugrid(i64 p);  // k_fista_update's grid (its J / <b, x> partial count)
// bxpart (nullable): per-CTA partials of <b, x_new> for the expanded objective
void fista_update(const Launch& L, const FistaCtl* ctl, i64 p, int pen, double alpha, double* x, double* xp,
                  double* Sx, double* Sxp, const double* b, double* best, double* Sbest, double* Jpart,
                  double* bxpart = nullptr);
void pdot(const Launch& L, i64 p, const double* a, const double* b, double* part);
// nu = 0 (backtracking every iteration, inner.cpp:169-183), per-CTA partials
void bt_prep(const Launch& L, i64 p, double omega, double sscale, double n, const double* x, const double* xp,
             const double* Sx, const double* Sxp, const double* b, double* y, double* grad, double* part);
void bt_trial(const Launch& L, i64 p, double delta, double lambda, int pen, double alpha, const double* y,
              const double* grad, double* cand, double* part);
void bt_dots(const Launch& L, i64 p, const double* x, const double* Sx, const double* b, double* part);
void pnorm(const Launch& L, i64 p, int pen, double alpha, const double* x, double* Jpart);
// cols: 0 = J(th_t); 1 + j = J(th + t_j (th_t - th))
void ptrials(const Launch& L, i64 p, int pen, double alpha, const double* th, const double* th_t, int ntrial,
             const double* t, double* part);
void ptheta_update(const Launch& L, i64 p, double t, const double* th_t, double* th);
void pcopy(const Launch& L, i64 p, const double* src, double* d0, double* d1, double* d2);
void padd(const Launch& L, i64 n, const double* x, double* y);
// {sum ss_part, sum J_part[2r], sum J_part[2r+1], sum bx_part} into out[0..3] (one CTA, fixed order)
void sums4(const Launch& L, const double* ss_part, int n_ss, const double* J_part, int n_J, const double* bx_part,
           int n_bx, double* out);                 // y += x
void pmask(const Launch& L, i64 p, i64 lo, i64 hi, double* x);                  // x := 0 outside [lo, hi)
void pmaxabs(const Launch& L, i64 p, const double* x, double* part);
// Gram route: per-CTA partials of w <x, S x> - 2 <x, b>
void gram_dots(const Launch& L, i64 p, double w, const double* x, const double* Sx, const double* b, double* part);
// per-CTA partials of sum v z^2
void wzz(const Launch& L, i64 n, const double* v, const double* z, double* part);
// per-CTA (min, max) partials (2 per CTA)
void minmax(const Launch& L, i64 n, const double* x, double* part);
void fista_finalize(const Launch& L, const FistaCtl* ctl, i64 p, const double* x, double* best, const double* Sx,
                    double* Sbest);

// Gram product + objective partials + control in one kernel on the
// constant-weight route (kg_gram.cu); follows k_fista_update in the body.
struct GramStepArgs {
  FistaCtl* ctl = nullptr;
  int d = 0;           // number of modes (<= 4)
  int q = 1;           // slab size p_1 ... p_{d-1}
  i64 pd = 1;          // slabs (p_d)
  int dims[4] = {1, 1, 1, 1};
  BandOp Gd;           // Gram of the last mode
  BandOp G[3];         // Grams of modes 0 .. d-2
  double* X[1] = {nullptr};  // the new iterate x
  double* S[1] = {nullptr};  // S'(x) (out)
  const double* b = nullptr;
  FastDiv fa[3], fk[3];        // in-slab mode j: divide by prod_{i<j} p_i and by p_j
  int pen = 0;
  double alpha = 0.0;
  double* part = nullptr;      // 3 per CTA
  unsigned* counter = nullptr;  // zero-initialised ticket
  cudaGraphConditionalHandle handle = 0;
  int use_handle = 0;
  int init = 0;                // 1: fista_solve setup instead of a monitor step
};
bool gram_step_fits(i64 q);
void gram_step(const Launch& L, const GramStepArgs& A);

// Persistent cooperative fista_solve on the Gram route (kg_gram.cu).
struct PersistArgs {
  GramStepArgs g;             // dims, Gram operators, b, penalty, control block
  const double* theta = nullptr;  // x_0 (p)
  double* X = nullptr;        // exchange buffer of the newest iterate (p)
  double* best = nullptr;     // out: best iterate (p)
  double* Sbest = nullptr;    // out: S'(best) (p)
  double* part = nullptr;     // 3 per CTA
  unsigned* bar = nullptr;    // grid barrier {count, generation}, zero-initialised
  unsigned* flags = nullptr;  // k_gauss_path: per-CTA arrival generations (zeroed before each launch)
  // whole-path mode (k_gauss_path)
  const double* lambdas = nullptr;
  int n_lambda = 0;
  double* part2 = nullptr;    // 5 per CTA
  double* dk_out = nullptr;   // 2 n_lambda: Delta_k (outer.cpp:224-226) and the initial objective per model
  double* coefs = nullptr;    // n_lambda x p result buffer
  double* obj_out = nullptr;  // n_lambda
  i64* iters_out = nullptr;   // n_lambda
  int* status_out = nullptr;  // n_lambda
  int* nmodels = nullptr;     // [models stored, stop: 0 none, 1 truncated, 2 first model failed]
  int dbg = 0;                // debug switches (KG_PATH_DBG)
};
bool fista_persist_ok(const GramStepArgs& A);
void fista_persist(const Launch& L, const PersistArgs& P);
void count_nonzero(const Launch& L, const double* coefs, i64 p, i64 models, unsigned long long* out);
bool gauss_path_ok(const GramStepArgs& A);
void gauss_path(const Launch& L, const PersistArgs& P);

int gauss_dots(const Launch& L, i64 p, double w, const double* th, const double* Sth, const double* bt,
               const double* Sbt, const double* b, double* part);

// control / reductions (single CTA)
// bx_part (nullable): objective partials sum = ss - 2 <b, x> (+ ss_const), the expanded form
void fista_init(const Launch& L, FistaCtl* ctl, const double* ss_part, int n_ss, const double* J_part, int n_J,
                const double* vmax_part, int n_vmax, int bt_always, const double* bx_part = nullptr, int n_bx = 0);
void fista_control(const Launch& L, FistaCtl* ctl, const double* ss_part, int n_ss, const double* J_part, int n_J,
                   cudaGraphConditionalHandle h, int use_handle, const double* bx_part = nullptr, int n_bx = 0);
void fista_gate(const Launch& L, const FistaCtl* ctl, cudaGraphConditionalHandle h);
// out[c] = sum over rows of part[row * ncols + c] (fixed order); op 0 sum, 1 max
void reduce_cols(const Launch& L, const double* part, int nrows, int ncols, int op, double* out);

// Gram + power iteration for one factor (spectral.cpp:8-42)
void gram(const Launch& L, const FactorDev& f, double* G, int* glo, int* ghi);
// One power iteration per job, all jobs in one launch (one warp each).
struct PowerJob {
  i64 p = 0;
  const double* G = nullptr;  // dense p x p Gram, column-major
  const int* glo = nullptr;   // row band [glo, ghi)
  const int* ghi = nullptr;
  const double* v0 = nullptr;
  double* out = nullptr;      // [value, iterations, status]
  int band = 0;               // max row band width (banded CTA path when <= kPowerTaps)
};
constexpr int kPowerTaps = 8, kPowerBlock = 8, kPowerThreads = 512, kPowerCtaRows = 2;
void power_iterations(const Launch& L, const PowerJob* jobs_dev, int njobs, i64 max_p, double tol, i64 max_iters);

// Input builders (kg_builders.cu): bin_scatter (bspline.cpp:106-153) and the
// device bspline_design (bspline.cpp:64-104).
constexpr int kMaxBinDims = 8, kBinThreads = 512, kMaxOrder = 16;
constexpr int kBinTile = 1024, kBinStages = 3;  // points per staged tile, tiles in flight per CTA
constexpr i64 kBinSmemBytes = 220 * 1024;     // counters + stages per CTA
struct BinArgs {
  int d = 0;
  i64 npts = 0, cells = 0;
  const double* pts = nullptr;  // npts x d, point-major
  double lo[kMaxBinDims], hi[kMaxBinDims], width[kMaxBinDims], inv[kMaxBinDims];
  int bmax[kMaxBinDims], stride[kMaxBinDims];  // bins - 1 and column-major strides (cells < 2^31)
  // KG_BIN_MODE experiments: 1 direct loads (no staging), 4 force global
  // atomics, 8 force smem counters
  int mode = 0;
  double* counts = nullptr;              // cells, zeroed by the caller
  unsigned long long* dropped = nullptr;  // zeroed by the caller
};
void bin_scatter(const Launch& L, const BinArgs& A, int n_sm);
void bspline_design_dev(const Launch& L, i64 npts, const double* pts, int order, i64 nb, const double* knots,
                        double* out, int* bad);

}  // namespace kg
