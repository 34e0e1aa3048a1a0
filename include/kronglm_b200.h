/*
 * kronglm_b200 — C ABI of the B200-native GLAM fit path.
 *
 * This is the drop-in boundary for the reference's fitting path
 * (kronglm, arXiv 1510.03298).  Each entry point names the reference
 * interface it replaces (file:line under /root/reference/proj/).  Plain
 * pointers and sizes only: no C++ types, no exceptions, no torch types.
 *
 * Conventions
 *  - All arrays are FP64, column-major (Fortran order), like DenseArray
 *    (include/kronglm/array.hpp:44-47).  Coefficient vectors are the
 *    concatenation of the vec() of each component block (design.hpp:51-78).
 *  - Host buffers are caller-owned and only read/written during the call.
 *    Device memory is library-owned.  Calls on one kg_ctx are serialised on
 *    that context's CUDA stream; use one ctx per host thread.  Distinct ctxs
 *    (e.g. one per GPU, "replica" mode) may run concurrently.
 *  - Every call returns kg_status.  kg_last_error(ctx) gives the message
 *    (the reference's exception text); kg_last_error_cell(ctx) the 0-based
 *    flat cell index of an EvalError (family.hpp:53-61).
 *  - Results are bit-for-bit reproducible run to run on the same GPU and
 *    configuration (deterministic reductions, no floating-point atomics),
 *    the analogue of the reference's thread-determinism contract
 *    (tests/test_outer.cpp:363-395).
 */
#ifndef KRONGLM_B200_H
#define KRONGLM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KG_OK = 0,
  KG_EINVAL = 1,    /* std::invalid_argument (shape / config / support violations) */
  KG_EEVAL = 2,     /* kronglm::EvalError (non-finite entrywise term; see cell) */
  KG_ERUNTIME = 3,  /* std::runtime_error (e.g. first path model did not converge, path.cpp:67-70) */
  KG_EDIVERGE = 4,  /* kronglm::DivergenceError escaping fista_solve (inner.hpp:48-57) */
  KG_EPOWER = 5,    /* kronglm::PowerIterationError (spectral.hpp:10-20) */
  KG_ECUDA = 6,     /* CUDA runtime failure */
  KG_ENCCL = 7,     /* NCCL failure (sharded contexts) */
  KG_ENOMEM = 8     /* device allocation failure */
} kg_status;

/* Family / link pairs: FamilySpec::{gaussian,binomial,poisson,gamma_log} (family.hpp:26-35). */
enum { KG_GAUSSIAN = 0, KG_BINOMIAL = 1, KG_POISSON = 2, KG_GAMMA = 3 };
/* PenaltySpec::{lasso,ridge,elastic_net} (penalty.hpp:14-23). */
enum { KG_LASSO = 0, KG_RIDGE = 1, KG_ELASTIC_NET = 2 };
/* WeightMode (outer.hpp:10). */
enum { KG_W_EXACT = 0, KG_W_UNIT = 1, KG_W_TENSOR = 2 };
/* SolveStatus (outer.hpp:35). */
enum { KG_S_CONVERGED = 0, KG_S_MAX_ITERATIONS = 1, KG_S_LINE_SEARCH_FAILED = 2, KG_S_INNER_DIVERGENCE = 3 };

typedef struct kg_ctx kg_ctx;
typedef struct kg_design kg_design;
typedef struct kg_obs kg_obs;
typedef struct kg_path_result kg_path_result;

/* PathConfig + OuterConfig + InnerConfig flattened (path.hpp:9-13,
 * outer.hpp:15-24, inner.hpp:29-36).  kg_path_cfg_default() fills the
 * reference defaults. */
typedef struct {
  int64_t n_lambda;              /* 100 */
  double lambda_min_ratio;       /* 1e-4 */
  int64_t max_outer;             /* 100 */
  double armijo_alpha0;          /* 1.0 */
  double armijo_b;               /* 0.5 */
  double armijo_v;               /* 0.1 */
  int64_t armijo_max_backtracks; /* 50 */
  int64_t weight_mode;           /* KG_W_EXACT */
  double outer_tol;              /* 1e-8 */
  double nu;                     /* 1.0 */
  int64_t inner_max_iters;       /* 2000 */
  double inner_tol;              /* 1e-8 */
  int64_t extrapolation;         /* 0 = fista, 1 = none */
  int64_t monitor_every;         /* 1 */
} kg_path_cfg;

void kg_path_cfg_default(kg_path_cfg* cfg);

/* ------------------------------------------------------------- context -- */
/* One CUDA device, one stream.  Replaces nothing in the reference (which is
 * single-threaded host code); it owns streams, graphs and workspaces. */
kg_status kg_ctx_create(int device, kg_ctx** out);
/* Sharded context: the observation array is split along its
 * LAST mode into `world` contiguous slabs, rows [n_d r / world, n_d (r+1) /
 * world) for rank r; designs created on it keep only those rows of X_d and
 * observations are the rank's slab.  `nccl_unique_id` points to the 128-byte
 * ncclUniqueId made by rank 0 (kg_nccl_unique_id) and broadcast by the caller
 * (e.g. torch.distributed); the ranks then sum S(x) (a p-vector) and the
 * objective partial per gradient, b = X^T(v z) and the family scalars per
 * outer iteration, and max / min-reduce max(v) and error cells, all with
 * ncclAllReduce on the context stream.  With nccl_unique_id == NULL the
 * context computes its slab's local partials only (no cross-rank sums: the
 * caller reduces, e.g. kg_g_map partials); a fit on it is a fit of the slab.
 * Replaces nothing in the reference (single-process); libnccl.so.2 is
 * opened at run time.  KG_ENCCL if NCCL is unavailable or fails. */
kg_status kg_ctx_create_sharded(int device, int rank, int world, const void* nccl_unique_id, kg_ctx** out);
kg_status kg_nccl_unique_id(void* out128);
/* Destroy designs, observations and results made on a context before it. */
void kg_ctx_destroy(kg_ctx* ctx);
const char* kg_last_error(const kg_ctx* ctx);
int64_t kg_last_error_cell(const kg_ctx* ctx);
/* The cudaStream_t the context launches on (for CUDA-event timing). */
void* kg_ctx_stream(kg_ctx* ctx);
kg_status kg_ctx_synchronize(kg_ctx* ctx);
/* The shard this context owns: slab `rank` of `world` along the last mode. */
void kg_ctx_shard(const kg_ctx* ctx, int* rank, int* world);

/* -------------------------------------------------------------- design -- */
/* TensorDesign(std::vector<std::vector<Matrix>>) (design.hpp:17, design.cpp:19-50).
 * c components, d marginal dimensions; n[j] rows of every factor in dim j;
 * p[r*d + j] columns of factor (r, j); factors[r*d + j] -> n[j] x p[r*d+j]
 * column-major host matrix.  Uploads the factors, derives per-row and
 * per-column nonzero bands (exact-zero test) and caches the spectral radii
 * rho(X_rj^T X_rj) (spectral.cpp:8-42) for the Lipschitz bound. */
kg_status kg_design_create(kg_ctx* ctx, int64_t c, int64_t d, const int64_t* n, const int64_t* p,
                           const double* const* factors, kg_design** out);
void kg_design_destroy(kg_design* design);
int64_t kg_design_n(const kg_design* design); /* n = prod n_j (this shard's slab when sharded) */
int64_t kg_design_p(const kg_design* design); /* p = sum_r prod_j p_rj */
/* The design's halo plan on a sharded context (kg_halo_plan layout, out9[0]
 * = 0: the sharded FISTA loop all-reduces the p-vector instead). */
kg_status kg_design_halo(const kg_design* design, int64_t* out9);
/* The cached spectral radius of X_rj^T X_rj. */
kg_status kg_design_spectral(kg_design* design, int64_t r, int64_t j, double* out);

/* --------------------------------------------------------- observations -- */
/* ObservationData(y[, a]) (family.hpp:40-47).  y, a: n-arrays (a may be NULL
 * = all ones).  on_device != 0: y and a are device pointers (copied
 * device-to-device); else host pointers (uploaded).  When sharded, the
 * arrays are this rank's slab. */
kg_status kg_obs_create(kg_ctx* ctx, const kg_design* design, const double* y, const double* a, int on_device,
                        kg_obs** out);
void kg_obs_destroy(kg_obs* obs);

/* ----------------------------------------------------- operator probes -- */
/* h_map (design.cpp:89-102): coef (p) -> eta (n).  Host buffers. */
kg_status kg_h_map(kg_ctx* ctx, const kg_design* design, const double* coef, double* eta);
/* g_map (design.cpp:104-116): u (n) -> coef (p).  Host buffers. */
kg_status kg_g_map(kg_ctx* ctx, const kg_design* design, const double* u, double* coef);
/* xtwx_apply (design.cpp:118-124): G(v .* H(coef)). */
kg_status kg_xtwx_apply(kg_ctx* ctx, const kg_design* design, const double* v, const double* coef, double* out);
/* rho (array.cpp:51-72): x is r x extents[0]; a has ndim extents; out has
 * extents (extents[1..], r). */
kg_status kg_rho(kg_ctx* ctx, int64_t r, const double* x, int64_t ndim, const int64_t* extents, const double* a,
                 double* out);
/* lambda_max (penalty.cpp:72-85). */
kg_status kg_lambda_max(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, int family, double dispersion,
                        int penalty, double alpha, double* out);

/* ---------------------------------------------------------------- path -- */
/* fit_path (path.hpp:36-43, path.cpp:29-81): lambdas == NULL computes
 * lambda_max and the log grid (lambda_sequence, path.cpp:8-27); otherwise
 * the explicit strictly decreasing grid of n_lambdas values is used.  The
 * whole path is solved on the device; coefficients stay in device memory
 * until read with kg_result_coef. */
kg_status kg_fit_path(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, int family, double dispersion,
                      int penalty, double alpha, const kg_path_cfg* cfg, const double* lambdas, int64_t n_lambdas,
                      kg_path_result** out);
/* outer_solve (outer.hpp:56-60, outer.cpp:159-303) at one lambda from
 * theta = 0 (the path's first warm start, path.cpp:63): the result holds one
 * model with whatever status the solve ended in (converged, max_iterations,
 * line_search_failed, inner_divergence) -- no first-model exception -- and
 * its OuterTrace (kg_result_trace). */
kg_status kg_outer_solve(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, int family, double dispersion,
                         int penalty, double alpha, const kg_path_cfg* cfg, double lambda, kg_path_result** out);
int64_t kg_result_n_models(const kg_path_result* res);
int kg_result_truncated(const kg_path_result* res);
double kg_result_lambda_max(const kg_path_result* res);
/* Per-model accessors (FitPath fields, path.hpp:18-27): t in [0, n_models);
 * an out-of-range t returns NaN (doubles) or -1 (integers). */
double kg_result_lambda(const kg_path_result* res, int64_t t);
double kg_result_objective(const kg_path_result* res, int64_t t);
int64_t kg_result_outer_iters(const kg_path_result* res, int64_t t);
int64_t kg_result_inner_iters(const kg_path_result* res, int64_t t);
int kg_result_status(const kg_path_result* res, int64_t t);
int64_t kg_result_nonzero(const kg_path_result* res, int64_t t);

/* One OuterRecord of OuterTrace (outer.hpp:26-47): the per-outer-iteration
 * diagnostics of model t (FitPath::diagnostics, path.hpp:23). */
typedef struct {
  double objective;          /* F after the iteration (f_cur if the line search failed) */
  double alpha;              /* accepted Armijo step t (0 if the line search failed; 1 on the Gaussian shortcut) */
  double delta_k;            /* -<u(eta), eta~ - eta>/n + lambda (J(theta~) - J(theta)) (outer.cpp:118-120) */
  double lipschitz;          /* L-hat of the inner solve (inner.cpp:132-135) */
  int64_t inner_iterations;  /* fista_solve iterations */
  int32_t inner_converged;   /* 1 if the inner solve met its tolerance */
  int32_t armijo_j;          /* accepted backtracking index j (-1 if the line search failed) */
} kg_outer_record;
/* OuterTrace::initial_objective of model t (F at the warm start); NaN if t is out of range. */
double kg_result_initial_objective(const kg_path_result* res, int64_t t);
/* Number of OuterRecords of model t (-1 if t is out of range). */
int64_t kg_result_n_outer(const kg_path_result* res, int64_t t);
/* Copies the kg_result_n_outer(res, t) records of model t into out. */
kg_status kg_result_trace(const kg_path_result* res, int64_t t, kg_outer_record* out);
/* Nonzero coefficient count of every model (counted on the device): out
 * has kg_result_n_models entries. */
kg_status kg_result_nonzeros(kg_path_result* res, int64_t* out);
/* Copies the p coefficients of model t into host memory. */
kg_status kg_result_coef(kg_path_result* res, int64_t t, double* out);
/* Coefficients of models [first, first + count) in one copy: out is
 * count x p, model-major (the rows kg_result_coef returns one by one). */
kg_status kg_result_coefs(kg_path_result* res, int64_t first, int64_t count, double* out);
void kg_result_free(kg_path_result* res);

/* Page-locked host memory for result downloads (cudaHostAlloc): a
 * kg_result_coefs copy into it runs at PCIe speed instead of through the
 * driver's pageable staging.  Free with kg_host_free. */
kg_status kg_host_alloc(size_t bytes, void** ptr);
void kg_host_free(void* ptr);

/* predict (path.cpp:83-89): eta = H(coef), mu = g^{-1}(eta).  Host buffers. */
kg_status kg_predict(kg_ctx* ctx, const kg_design* design, int family, const double* coef, double* eta, double* mu);

/* ---------------------------------------------------- input builders -- */
/* bspline_design (bspline.cpp:64-104): clamped uniform cubic (order 4)
 * bases; out is npts x n_basis column-major. Host-side input builder. */
kg_status kg_bspline_design(int64_t npts, const double* points, int64_t order, int64_t n_basis, double* out);
int64_t kg_default_basis_count(int64_t n_points, int64_t ratio); /* bspline.cpp:20-26; -1 on bad args */
/* bin_scatter (bspline.cpp:106-153, decl bspline.hpp:38-45) on the device:
 * npts points of d <= 8 coordinates (point-major, npts x d) binned on the
 * regular grid bins[0] x ... x bins[d-1] over [lo_j, hi_j] (bins right-open
 * except the last, right-closed); counts (prod bins, column-major) receive
 * the counts, *dropped (may be NULL) the points outside the bounds.
 * on_device != 0: points and counts are device pointers (the counts can feed
 * kg_obs_create(on_device=1) directly); else host pointers.  lo/hi/bins are
 * host arrays.  A NaN coordinate drops the point (the reference's
 * static_cast of floor(NaN) is undefined).  Counts are exact integers. */
kg_status kg_bin_scatter(kg_ctx* ctx, int64_t npts, int64_t d, const double* points, const double* lo,
                         const double* hi, const int64_t* bins, int on_device, double* counts, int64_t* dropped);
/* bspline_design on the device: bit-identical to kg_bspline_design (same
 * knots, explicitly rounded FP64 recursion), order <= 16.  on_device: points
 * (npts) and out (npts x n_basis, column-major) are device pointers. */
kg_status kg_bspline_design_dev(kg_ctx* ctx, int64_t npts, const double* points, int64_t order, int64_t n_basis,
                                int on_device, double* out);
int64_t kg_linear_index(int64_t d, const int64_t* multi_index, const int64_t* dims); /* array.cpp:22-36; -1 bad */
/* Halo plan of banded last-mode sharding (band property
 * bspline.hpp:27-30, G chain design.cpp:104-116).  Rank r of `world` holds
 * the grid rows [n r / world, n (r + 1) / world) of the last-mode factor X
 * (n x p, column-major, host memory) and touches the coefficient slices
 * T_r = [t_lo, t_hi) its rows have nonzeros in.  Coefficient slice j is
 * OWNED by one rank: [own_lo, own_hi), own_lo = t_lo (0 for rank 0) and
 * own_hi = the next rank's t_lo (p for the last rank).  Per FISTA gradient
 * the only exchanges are the boundary slices:
 *   right halo R = [own_hi, t_hi): this rank's partial of S(x) goes to rank
 *     r + 1 (which owns it) and the updated x comes back from it;
 *   left overlap L = [own_lo, t_hi of rank r - 1): the partial of rank r - 1
 *     arrives and is added, and the updated x goes back to it.
 * out[9] = {ok, own_lo, own_hi, t_lo, t_hi, L_lo, L_hi, R_lo, R_hi}; ok = 0
 * when some rank's rows reach beyond its neighbours' owned slices (then the
 * fit falls back to the p-sized all-reduce).  Host only. */
kg_status kg_halo_plan(int64_t n, int64_t p, const double* X, int world, int rank, int64_t* out);

/* Gather plan of the slab pass (the X^T W X step of xtwx_apply,
 * design.cpp:118-124, fused per last-mode slice): the mode-1 factor X1 (n x p,
 * column-major, host memory; rows with <= 4 nonzeros inside a 5-wide window
 * per quad of grid rows).  Row quad q scatters its five window partials of
 * X1^T w to slots 5 q .. 5 q + 4 of a plane; basis function k then sums, in
 * ascending quad order, the slots of the quads that have a row with k inside
 * its nonzero band.  slots[8 k + j] (k < 8 ceil(p / 8), j < 8) = slot j of
 * basis function k, padded with the plane's always-zero slot plane - 1;
 * *gmax = most slots of any k; *plane = slots per plane (5 n / 4 rounded up to
 * = 2 mod 8, so the gather is bank-conflict free).  KG_EINVAL when n is not a
 * multiple of 4, a band leaves its quad's window, or some k needs more than 8
 * slots (the pass then keeps its DMMA form).  Host only. */
kg_status kg_slab_gather_plan(int64_t n, int64_t p, const double* X, int32_t* slots, int32_t* gmax, int32_t* plane);

/* Held-out selection (mse_heldout, path.cpp:91-126, decl path.hpp:63): for
 * every model of `res`, the sum over cells with mask == 1 of (mean(X theta_t)
 * - y_full)^2 into mse[0 .. n_models), and the first minimizing model in
 * *argmin.  y_full and mask are host arrays of this context's slab; mask
 * entries must be 0 or 1 and at least one must be 1 (KG_EINVAL otherwise).
 * Predictions are computed on the device from the resident coefficients. */
kg_status kg_mse_heldout(kg_ctx* ctx, const kg_design* design, const kg_path_result* res, int family,
                         const double* y_full, const double* mask, double* mse, int64_t* argmin);

/* Deviance of every model of `res` against `obs` into out[0 .. n_models):
 * eta_t = H(theta_t) computed on the device from the resident coefficients,
 * then Gaussian sum a (y - mu)^2, Poisson 2 sum a [y log(y/mu) - (y - mu)],
 * binomial 2 sum a [y log(y/mu) + (1-y) log((1-y)/(1-mu))], gamma 2 sum a
 * [-log(y/mu) + (y - mu)/mu] (mu with the +-30 clamp, a = 0 cells skipped,
 * 0 log 0 = 0).  Not a reference output: it is the derived quantity of the
 * parity protocol (north_star "deviance within 1e-8"), with family.cpp's
 * conventions (family.cpp:111-162).  Sharded contexts sum over the slabs. */
kg_status kg_result_deviance(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, const kg_path_result* res,
                             int family, double* out);

/* --------------------------------------------------------- measurement -- */
/* Times `reps` launches of one hot-path kernel on the context stream with
 * CUDA events, on the resident observation (inputs already in HBM).
 *   which = 0: the fused FISTA n-array pass (mode-1 H-last + weighted SS +
 *              V.* + G-first), the dominant kernel of every prox-grad step;
 *   which = 1: one banded mode contraction (the largest H-chain step).
 * avg_ms = mean device time per launch, each launch bracketed by its own
 * CUDA events after a 256 MB write that evicts L2 (so the inputs come from
 * HBM, as inside a path step); bytes = algorithmic HBM bytes per launch
 * ("roofline"). */
kg_status kg_time_kernel(kg_ctx* ctx, const kg_design* design, const kg_obs* obs, int which, int reps,
                         double* avg_ms, double* bytes);
/* Device time of the last whole-path kernel (k_gauss_path: one cooperative
 * launch runs every FISTA step of a Gaussian constant-weight lambda path),
 * measured with CUDA events around that launch on the context stream, and its
 * algorithmic bytes: per prox-grad step the neighbour bands of x read by every
 * slab, the x slabs written and the per-slab partials exchanged, plus the
 * coefficient rows stored per model ("roofline").  Returns
 * KG_EINVAL when no such launch has run on this context. */
kg_status kg_path_kernel_stats(const kg_ctx* ctx, double* ms, double* bytes, int64_t* steps);
/* Number of library kernel launches issued since the last reset (host-side
 * counter of launches, graph-replayed kernels counted per replay). */
int64_t kg_launch_count(const kg_ctx* ctx);
void kg_launch_count_reset(kg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* KRONGLM_B200_H */
