/*
 * sfw3d_cuda.h — C ABI of the B200 (sm_100a) hot path of boosted Sliding
 * Frank-Wolfe 3D deconvolution (drop-in core for the reference `sfw3d` 0.1.0).
 *
 * The reference is pure Python/numpy and has no FFI; each entry point below
 * names the reference function (file:line under pkg/src/sfw3d/) whose
 * arithmetic it replaces. The Python package `paper_2009_05473_b200` binds
 * this ABI with ctypes and keeps the reference's public function names,
 * argument meaning and exceptions (see INTEGRATION.md for the binding a
 * maintainer of the reference would add).
 *
 * Conventions
 *  - Volumes are dense (nx, ny, nz) arrays in C order (z contiguous), of
 *    storage type SFW3D_F32 or SFW3D_F64, in DEVICE memory owned by the
 *    caller (volumes.py:7-16). Host pointers are marked *_host.
 *  - An atom row is 6 doubles (w, m_x, m_y, m_z, sigma, d): the reference
 *    gradient-column / _pack order (forward.py:37, solvers.py:183-186).
 *  - Every call returns an sfw3d_status; sfw3d_last_error() returns a
 *    thread-local message for the last failure. No C++ exception crosses
 *    the ABI. SFW3D_EINVAL maps to ValueError, SFW3D_ENONFINITE to
 *    FloatingPointError (forward.py:225-228, certificate.py:207-208).
 *  - A context binds one device and one CUDA stream; all work of a call is
 *    enqueued on that stream. Calls that return values in *_host buffers
 *    synchronise the stream before returning. Contexts are independent;
 *    a context must not be used by two threads at once.
 */
#ifndef SFW3D_CUDA_H
#define SFW3D_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFW3D_ABI_VERSION 3

typedef enum {
  SFW3D_OK = 0,
  SFW3D_EINVAL = 1,      /* invalid argument (ValueError)               */
  SFW3D_ENONFINITE = 2,  /* non-finite result (FloatingPointError)       */
  SFW3D_ECUDA = 3,       /* CUDA runtime failure                         */
  SFW3D_ENOMEM = 4       /* device allocation failure                    */
} sfw3d_status;

typedef enum { SFW3D_F32 = 0, SFW3D_F64 = 1 } sfw3d_dtype;

typedef struct sfw3d_ctx sfw3d_ctx;
typedef struct sfw3d_psf sfw3d_psf;
typedef struct sfw3d_table sfw3d_table;

/* Discrete argmax record: position (i,j,k), flat candidate index
 * (sigma-major: i_sigma * n_shape + i_shape) and its eta value. */
typedef struct {
  int32_t pos[3];
  int32_t cand;
  double value;
} sfw3d_argmax;

/* ---- library / context ------------------------------------------------ */
int sfw3d_abi_version(void);
const char* sfw3d_last_error(void);
/* stream: a cudaStream_t (NULL = legacy default stream). */
int sfw3d_ctx_create(int device, void* stream, sfw3d_ctx** out);
int sfw3d_ctx_destroy(sfw3d_ctx* ctx);
int sfw3d_ctx_sync(sfw3d_ctx* ctx);
/* Number of kernels this context has launched (for launch accounting). */
int64_t sfw3d_ctx_launches(const sfw3d_ctx* ctx);

/* Per-kernel device timing for roofline accounting. When enabled, the
 * library brackets each of its kernel launches with CUDA events on the
 * context stream, grouped by kernel family ("eta_direct", "psf_pass",
 * "render", "atom_sums", "pad", "argmax", "residual", "dots", "cd",
 * "sumsq", "eta_basis"). enable = 0 disables; any call resets the counters. */
int sfw3d_ctx_profile(sfw3d_ctx* ctx, int enable);
/* Total device milliseconds and launch count of one family since the last
 * reset (synchronises the pending events). */
int sfw3d_ctx_profile_read(sfw3d_ctx* ctx, const char* family, double* total_ms,
                           int64_t* launches);
/* Measured FP32 FMA throughput of this device (a register-resident FFMA
 * loop over every SM), in TFLOP/s: the roofline denominator for the
 * correlation kernels (MEASURED_PEAKS.json has no FP32 figure). */
int sfw3d_probe_fp32(sfw3d_ctx* ctx, double* tflops);

/* Host-only helper (no device work): per-atom support radius and box
 * geometry exactly as forward.py:97-116 computes them. For each of the k
 * atom rows writes radius[k] and, per axis, start[3k] (first span value,
 * may be negative; 0 for a full axis), len[3k] and full[3k]. */
int sfw3d_atom_geometry(const int dims[3], const double* params_host, int k,
                        int32_t* radius, int32_t* start, int32_t* len, int32_t* full);

/* ---- PSF (forward.py:40-94) ------------------------------------------- */
/* kernel_host: dims[0]*dims[1]*dims[2] doubles, centred at n//2 per axis,
 * already normalised as the caller wants (Psf.__init__, forward.py:49-58).
 * The library factorises it into three 1-D tap vectors when it is
 * separable (every BASELINE PSF is), else keeps its non-zero bounding box. */
int sfw3d_psf_create(sfw3d_ctx* ctx, const int dims[3], const double* kernel_host,
                     sfw3d_psf** out);
/* separable flag and the non-zero offset box [lo, hi] per axis */
int sfw3d_psf_info(const sfw3d_psf* psf, int* separable, int32_t lo[3], int32_t hi[3]);
int sfw3d_psf_destroy(sfw3d_psf* psf);

/* K4 — out = H * in (adjoint = 0, convolve, forward.py:79-87) or
 *      out = H^T * in (adjoint = 1, correlate_adjoint, forward.py:90-94).
 * Circular; in and out are distinct device volumes of `dtype`. */
int sfw3d_psf_apply(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype,
                    const void* in_dev, void* out_dev, int adjoint);

/* ---- atoms (forward.py:119-179) --------------------------------------- */
/* K3 — out = sum_i w_i G_i over each atom's 1e-12 support box, atoms summed
 * in row order per voxel (_accumulate_atoms, forward.py:165-174). */
int sfw3d_render(sfw3d_ctx* ctx, int dtype, const int dims[3], const double* params_host,
                 int k, void* out_dev);

/* K6/K7 — raw per-atom inner products against a device volume `field`:
 * sums_host[6i + c] = < P_c(atom i), field >, with P = (G, dG/dm_x, dG/dm_y,
 * dG/dm_z, dG/dsigma, dG/dd) of the UNIT atom (weights are ignored here).
 * _gradient_rows (forward.py:209-229) and neg_eta (certificate.py:201-209)
 * finish with row = [s0 + lam, w*s1..w*s5] and [s/lam] respectively.
 * Returns SFW3D_ENONFINITE if any sum is not finite. */
int sfw3d_atom_sums(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field_dev,
                    const double* params_host, int k, double* sums_host);

/* K3-K6 fused — criterion_and_gradient (forward.py:232-257):
 *   model = H * sum_i w_i G_i ; C = 1/2 ||model - y||^2 + lam * sum_i w_i ;
 *   back = H^T * (model - y) ; grad row i = [<G_i,back> + lam, w_i <dG_i,back>].
 * grad_host may be NULL (criterion only, forward.py:182-190). back_dev, if
 * not NULL, receives the back-projection (a `dtype` volume) — also when
 * grad_host is NULL (the sharded gradient splits the atom sums over ranks). */
int sfw3d_cost_grad(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                    const double* params_host, int k, double lam, double* cost_host,
                    double* grad_host, void* back_dev);

/* K3-K6 on one rank's x-slab (multi-GPU criterion_and_gradient, SURVEY
 * §8(e); forward.py:232-257 split over z/x-slabs). `psf` is created on the
 * window dims (x1 - x0 + 1 + 2 halo, ny, nz), y_dev holds y on the window
 * planes x0 - halo .. x1 + halo of the periodic (gnx, ny, nz) volume, halo >=
 * the PSF's x half-extent. Atom x-spans are clipped to the window; the
 * residual is taken on the slab planes only. Outputs this rank's partials:
 * half_sumsq = 1/2 sum_slab (model - y)^2 and raw sums_host[6i + c] =
 * <P_c(atom i), H^T (r 1_slab)> (0 for atoms missing the window). Summed over
 * ranks: C = half_sumsq + lam sum w, row i = [s0 + lam, w s1..w s5]. */
int sfw3d_cost_grad_slab(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                         const double* params_host, int k, int gnx, int x0, int x1, int halo,
                         double* half_sumsq_host, double* sums_host);

/* The same with the partials left on the DEVICE, unsynchronised, for an
 * in-stream all-reduce (NCCL) before the one D2H: partials_dev (1 + 6k
 * doubles) = [1/2 sum_slab r^2, raw sums row-major]. Non-finite partials are
 * the caller's check after the reduction. */
int sfw3d_cost_grad_slab_dev(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                             const double* params_host, int k, int gnx, int x0, int x1, int halo,
                             double* partials_dev);

/* x-slab render (the sharded solver's blurred atoms phi_i, solvers.py:260-261):
 * the atoms of the periodic (gdims) volume clipped to the window planes
 * x0 - halo .. x1 + halo, rendered on that window (out_dev: window dims). */
int sfw3d_render_slab(sfw3d_ctx* ctx, int dtype, const int gdims[3], const double* params_host,
                      int k, int x0, int x1, int halo, void* out_dev);
/* x-slab K7 (neg_eta of the sharded refine, certificate.py:201-209): raw
 * per-atom sums over the OWNED planes [x0, x1] only; field_dev is a window of
 * x1 - x0 + 1 + 2 halo planes (plane 0 = global x0 - halo). Summed over the
 * ranks: the single-volume sfw3d_atom_sums. */
int sfw3d_atom_sums_slab(sfw3d_ctx* ctx, int dtype, const int gdims[3], const void* field_dev,
                         const double* params_host, int k, int x0, int x1, int halo,
                         double* sums_host);

/* ---- certificate (certificate.py:37-236) ------------------------------ */
/* K2 — candidate table for the (sigma, d) grid, sigma-major (sorted
 * ascending, as build_template_table sorts them, certificate.py:72-73).
 * Spatial unit atoms G_ij(m=0) on the reference's support box
 * (certificate.py:86-92) are kept on the device; the PSF is applied once to
 * the residual (factorised eta = G * (H^T * r), exact by associativity).
 * tap_tol: taps with G < tap_tol are skipped (0 keeps the reference box).
 * mode: 0 = automatic (separable Gaussian basis where its certified error
 * bound <= basis_tol, direct correlation otherwise), 1 = direct only. */
int sfw3d_table_create(sfw3d_ctx* ctx, const sfw3d_psf* psf, int n_sigma,
                       const double* sigma_host, int n_shape, const double* shape_host,
                       double tap_tol, int mode, double basis_tol, sfw3d_table** out);
/* Evaluator split for a storage dtype: candidates on the direct path and on
 * the separable basis, the taps per output voxel each path's table holds,
 * and the FP32/FP64 flops per output voxel each path EXECUTES (summed over
 * its candidates; FMA = 2, add = 1) — the FLOP counts of the roofline. */
int sfw3d_table_info(const sfw3d_table* t, int dtype, int* n_cand, int* n_direct, int* n_basis,
                     int64_t* direct_taps, int64_t* basis_taps, double* direct_flops,
                     double* basis_flops);
/* Host-only (no device work): the separable-basis fit the table uses for a
 * (sigma, d) candidate on the offset box [lo, hi]: g(s) ~ w0 [s == 0] +
 * sum_k weights[k] exp(-betas[k] s) with non-negative weights; writes up to
 * max_terms terms, the term count and the max abs error on the lattice. */
int sfw3d_basis_fit(const int32_t lo[3], const int32_t hi[3], double sigma, double d,
                    int max_terms, double* betas, double* weights, double* w0, int* n_terms,
                    double* fit_err);
/* Host-only (no device work): the SHARED separable basis a table builds for
 * the candidate grid sigma x shape (sigma-major) at storage `dtype` with
 * acceptance tolerance `tol` (the table uses basis_tol for SFW3D_F32 and
 * min(basis_tol, 1e-12) for SFW3D_F64). Every d <= 2 candidate is fitted on one
 * dictionary over the union of the candidates' support boxes:
 * g_c(s) ~ w0[c] [s == 0] + sum_t weights[c*max_terms + t] exp(-betas[t] s).
 * Writes the shared term count, up to max_terms betas, the member rows of
 * weights (zero rows elsewhere), w0, fit_err (max abs error on the common
 * box's lattice incl. the 1e-12 factor truncation; +inf for d > 2) and
 * member (1 = certificate takes the basis path) per candidate. prune and
 * loose_tol as the table options below (-1 / negative = the defaults). */
int sfw3d_basis_set_fit(const int32_t dims[3], int n_sigma, const double* sigma_host,
                        int n_shape, const double* shape_host, int dtype, double tol,
                        int prune, double loose_tol, int max_terms, int* n_terms,
                        double* betas, double* weights, double* w0, double* fit_err,
                        int32_t* member);
/* One candidate (flat sigma-major index): evaluator used for `dtype` by an
 * argmax-only evaluation (uses_basis: 0 direct, 1 shared separable basis,
 * 2 basis with exact refinement of its maxima — fp64 non-negative members
 * with an inexact fit, and the SIGNED members: candidates outside the
 * non-negative pool, e.g. d > 2, fitted with signed weights; calls that keep
 * the eta fields evaluate signed members directly), the table's SHARED basis
 * term count, the candidate's shared-basis fit error (max abs on the common
 * box lattice; for signed members the certified bound factor E, with
 * |eta~ - eta| <= E ||b||_inf / lam at every voxel; +inf when not fitted),
 * its direct tap count, the shared basis taps per voxel, and its executed
 * flops per voxel. */
int sfw3d_table_candidate(const sfw3d_table* t, int dtype, int cand, int* uses_basis,
                          int* n_terms, double* fit_err, int64_t* direct_taps,
                          int64_t* basis_taps, double* flops);
/* Table options (no reference counterpart: tuning of the B200 evaluator,
 * never of the result beyond the certified bounds). Set before the first
 * evaluation; "prune" and "loose_tol" refit the shared bases on next use.
 *   "prune"      -1 (default: prune the shared terms for >= 2^24-voxel fp32 /
 *                2^26-voxel fp64 volumes), 0 never, 1 always.
 *   "global_voxels" > 0: the voxel count the default pruning rule uses
 *                (a sharded certificate passes the GLOBAL volume's, so every
 *                rank fits the same shared terms as one GPU would).
 *   "loose_tol"  fp32 shared-term selection tolerance (< 0: default 1e-5;
 *                0: select at basis_tol itself).
 *   "refine_cap" exactly re-evaluated voxels per call before members fall
 *                back to the direct kernel (default 65536). */
int sfw3d_table_set_option(sfw3d_table* t, const char* name, double value);
/* The 1-D passes of the shared separable basis (3 per term: x, y, z filter
 * lengths), for the measurement's per-pass rooflines: a pass moves 2 volumes
 * and executes 2 * taps FLOP per voxel; filters of more than 24 taps run the
 * FP32-bound wide tiles (profile family "eta_basis_wide"), the others the
 * HBM-bound narrow tiles ("eta_basis"). *n_out = 3 * terms. */
int sfw3d_table_basis_passes(const sfw3d_table* t, int dtype, int cap, int32_t* taps_out,
                             int* n_out);
int sfw3d_table_destroy(sfw3d_table* t);
/* Diagnostics: voxels the calling thread's last sfw3d_eta_argmax re-evaluated
 * exactly (refined basis members; > 65536 means it fell back to direct). */
int sfw3d_last_refine_count(void);

/* K1 — eta_field (certificate.py:140-184): eta_c(m) = <H*G_c(.-m), r>/lam
 * for every integer m and candidate c, with the discrete argmax over the
 * window [window[2a], window[2a+1]] per axis (first C-order maximum per
 * candidate; global winner by strict '>' over sigma-major candidates).
 * per_cand_host (n_cand records) and fields_dev (n_cand volumes of dtype,
 * candidate-major) may be NULL; fields are only produced when given. */
int sfw3d_eta_argmax(sfw3d_ctx* ctx, const sfw3d_table* t, int dtype,
                     const void* residual_dev, double lam, const int32_t window[6],
                     sfw3d_argmax* best_host, sfw3d_argmax* per_cand_host,
                     void* fields_dev);

/* ---- .vol IO straight to HBM (volumes.py:96-113) ----------------------- */
/* Host-only: the dims of a .vol file after validating its magic and size. */
int sfw3d_volume_info(const char* path, int32_t dims[3]);
/* Read the float64 payload into out_dev (dims from sfw3d_volume_info) in
 * the storage dtype, streamed through pinned staging with the conversion and
 * the finite check on the device. EINVAL for a malformed file (the
 * reference's VolumeFormatError) or a non-finite payload. */
int sfw3d_volume_read(sfw3d_ctx* ctx, const char* path, int dtype, void* out_dev);
/* Write a device volume as a .vol file (float64 payload, bit-exact for fp64). */
int sfw3d_volume_write(sfw3d_ctx* ctx, const char* path, int dtype, const int dims[3],
                       const void* in_dev);

/* ---- x-slab data plane (multi-GPU certificate) ---------- */
/* Halo exchange the library requests between the passes of an x-slab
 * evaluation. `window` is a device buffer of lo + owned + hi planes of
 * plane_elems elements (dtype): planes [lo, lo + owned) are this rank's and
 * hold data; the callee must fill planes [0, lo) with the lo global planes just
 * below this rank's first plane and [lo + owned, lo + owned + hi) with the hi
 * planes just above its last (periodic; a halo wider than a neighbour's slab
 * takes planes from further ranks) before any
 * later work on the context stream reads them (enqueue on / wait from that
 * stream). Every rank calls it in the same order (collective). 0 = success. */
typedef int (*sfw3d_halo_fn)(void* user, void* window_dev, int dtype, int owned_planes,
                             int64_t plane_elems, int lo_planes, int hi_planes);
/* In-place all-reduce of n host doubles over the ranks: op 0 = sum, 1 = max. */
typedef int (*sfw3d_allreduce_fn)(void* user, double* values_host, int n, int op);

/* K1 on one rank's x-slab: the rank owns planes [x0, x0 + n_own) of the
 * periodic residual (residual_dev: those planes only, compact) of the table's
 * GLOBAL volume. b = H^T r and every shared basis term are computed on the
 * owned planes with halo exchanges of their x passes (no redundant planes);
 * refined members re-evaluate exactly on b with a template-radius halo; the
 * refinement thresholds use the all-reduced |b| statistics and member maxima.
 * window is in LOCAL coordinates (x in [0, n_own)); the records' positions
 * are local (global x = x0 + pos[0]); per_cand_host (may be NULL) receives
 * this slab's per-candidate maxima (-inf where the window misses the slab).
 * Argmax-only (no fields); every candidate must be a basis member. */
int sfw3d_eta_argmax_slab(sfw3d_ctx* ctx, const sfw3d_table* t, int dtype,
                          const void* residual_dev, int n_own, int x0, double lam,
                          const int32_t window[6], sfw3d_halo_fn halo, sfw3d_allreduce_fn allreduce,
                          void* user, sfw3d_argmax* best_host, sfw3d_argmax* per_cand_host);

/* ---- non-negative LASSO (solvers.py:111-180, 253-266) ----------------- */
/* K8 — out_host[i] = < vecs[i], v > over n elements, fp64 accumulation,
 * fixed summation order. vecs_host holds k DEVICE pointers (Gram rows and
 * the right-hand side b = Phi y, solvers.py:141-143). */
int sfw3d_dots(sfw3d_ctx* ctx, int dtype, int64_t n, const void* const* vecs_host, int k,
               const void* v_dev, double* out_host);

/* K9 — cyclic coordinate descent with the reference's update, KKT, stall
 * and sweep-cap rules (solvers.py:145-180), run in fp64 on the device.
 * gram_host is k*k row-major, w_host holds w_init on entry and the result
 * on exit. info_host[0] = sweeps, info_host[1] = 0 kkt / 1 stall / 2 cap,
 * and the final KKT residual is written to *kkt_host. */
int sfw3d_nnlasso_cd(sfw3d_ctx* ctx, int k, const double* gram_host, const double* b_host,
                     double lam, double tol, int max_iter, double* w_host,
                     int32_t* info_host, double* kkt_host);

/* K9' — the same non-negative LASSO solved by an active-set (Lawson-Hanson)
 * iteration on the device: Cholesky of the free set's Gram block in shared
 * memory, exact optimum of the QP min 1/2 w'Gw - (b - lam)'w, w >= 0, stopped
 * by the reference's KKT residual <= tol (solvers.py:161-169). Same arguments
 * as sfw3d_nnlasso_cd; info_host[0] = outer iterations, info_host[1] = 0 kkt /
 * 2 cap / 3 not applicable (k > 150 or a near-singular free block: w_host is
 * then unspecified and the caller uses sfw3d_nnlasso_cd). Used for fp32-
 * storage solves (kernel-level parity); fp64 solves keep the reference's CD
 * trajectory. */
int sfw3d_nnlasso_qp(sfw3d_ctx* ctx, int k, const double* gram_host, const double* b_host,
                     double lam, double tol, int max_iter, double* w_host,
                     int32_t* info_host, double* kkt_host);

/* K5 — out = y - sum_i w_i phi_i in list order (_residual, solvers.py:253-257);
 * out_dev may be NULL; sumsq_host (may be NULL) receives ||out||^2 in fp64. */
int sfw3d_residual(sfw3d_ctx* ctx, int dtype, int64_t n, const void* y_dev,
                   const void* const* phis_host, const double* w_host, int k,
                   void* out_dev, double* sumsq_host);

/* K5 with supports: as sfw3d_residual on a (dims) volume, with per atom i the
 * x-plane range [xrange_host[2i], xrange_host[2i+1]] (wrapped when lo > hi)
 * outside which phi_i is exactly zero (render box dilated by the PSF's x
 * extent): atoms are skipped on planes they do not reach, which leaves every
 * voxel bit-identical (r - w * 0 = r) at a fraction of the reads — the k
 * full-volume phi streams are what the weight step of a long solve costs
 * (solvers.py:253-257 at k ~ 100). */
int sfw3d_residual_ranged(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* y_dev,
                          const void* const* phis_host, const double* w_host,
                          const int32_t* xrange_host, int k, void* out_dev, double* sumsq_host);

/* ---- in-library L-BFGS-B (the reference's scipy.optimize.minimize calls) -- */
/* Objective callback: 0 = ok with *f and g[0..n) written; any other value
 * aborts the minimisation (an sfw3d_status is passed through). */
typedef int (*sfw3d_objective_fn)(void* user, const double* x, double* f, double* g);

/* L-BFGS-B with scipy's driver conventions (method="L-BFGS-B": maxcor, ftol,
 * gtol, maxiter, maxfun, maxls; nbd[i]: 0 free, 1 lower, 2 both, 3 upper).
 * x is updated in place; info = {status, iterations, evaluations}, status:
 * 0 projected gradient <= gtol, 1 relative reduction <= ftol, 2 maxiter,
 * 3 maxfun, 4 abnormal line-search termination. Host only (no context): the
 * optimiser behind sfw3d_refine_eta_max / sfw3d_local_descent, exported so
 * that it can be checked against scipy on any objective. */
int sfw3d_lbfgsb_minimize(int n, double* x, const double* lower, const double* upper,
                          const int32_t* nbd, int maxcor, double ftol, double gtol,
                          int maxiter, int maxfun, int maxls, sfw3d_objective_fn fn,
                          void* user, double* f_out, int32_t info[3]);

/* refine_eta_max (certificate.py:187-224): box-constrained L-BFGS-B ascent
 * of eta(theta) = <G_theta, back>/lam over theta = (m_x, m_y, m_z, sigma, d)
 * from `start` (projected into the box), with back = H^T r on the device
 * (correlate_adjoint, :198). Every evaluation is one sfw3d_atom_sums launch;
 * the quasi-Newton algebra runs on the calling thread (no Python callback).
 * The seed is kept when the ascent does not improve it (:221-222).
 * SFW3D_ENONFINITE as the reference's FloatingPointError (:207-208,219-220). */
int sfw3d_refine_eta_max(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* back_dev,
                         double lam, const double start[5], const double lower[5],
                         const double upper[5], int max_iter, double gtol,
                         double theta_out[5], double* eta_out, int32_t info[3]);

/* local_descent (solvers.py:197-240): joint L-BFGS-B slide of the k atom rows
 * (w, m, sigma, d) in params_host (in: start, out: result), bounds w >= 0 and
 * the (m, sigma, d) box per atom, objective sfw3d_cost_grad. The start is
 * kept (info[0] gets bit 0x100) when the result is not finite or worse
 * (:236-237). info = {status, iterations, evaluations} as above. */
int sfw3d_local_descent(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                        double* params_host, int k, double lam, const double lower[5],
                        const double upper[5], double gtol, double ftol, int max_iter,
                        double* cost_out, int32_t info[3]);

/* ---- the solver's outer loop as one call (solvers.py:286-405) ----------- */
typedef struct {
  double lam;
  int32_t max_outer_iterations;
  int32_t boosted;             /* 0 = SFW (slide after every atom), 1 = BSFW */
  double eta_threshold, eta_slack;
  double lasso_tol;
  int32_t lasso_max_iter;
  int32_t descent_max_iter;
  double descent_gtol, descent_ftol;
  double prune_rel_tol, duplicate_tol;
  double lower[5], upper[5];   /* box of (m_x, m_y, m_z, sigma, d)          */
  int32_t window[6];           /* integer position window of the grid stage */
  int32_t n_sigma, n_shape;
  const double* sigma_grid;    /* host, n_sigma                             */
  const double* shape_grid;    /* host, n_shape                             */
} sfw3d_solve_options;

/* One IterationRecord (solvers.py:77-88); absent criteria are NaN. */
typedef struct {
  int32_t index;
  double eta_max, criterion_before, criterion_after_lasso, criterion_after_descent;
  int32_t atom_count;
  double t_certificate, t_lasso, t_descent;
} sfw3d_solve_record;

enum { SFW3D_TERM_CERTIFICATE = 0, SFW3D_TERM_ITERATION_CAP = 1, SFW3D_TERM_STALLED = 2 };

/* _solve (solvers.py:286-395): the whole SFW / boosted-SFW loop on a device
 * observation y — certificate (grid argmax + L-BFGS-B ascent), phi of the
 * new atom, Gram rows (cached), non-negative LASSO, residual + criterion,
 * prune, duplicate guard, slide(s), final re-check — driven by a C++
 * controller on the calling thread. arena_dev: caller-owned device memory of
 * arena_volumes volumes of `dtype` (residual, scratch, one phi per atom:
 * max_outer_iterations + 2 always suffice; SFW3D_ENOMEM if the atoms outgrow a
 * smaller arena). rows_out: max_outer_iterations x 6 doubles
 * (w, m, sigma, d); records: max_outer_iterations entries. */
int sfw3d_solve(sfw3d_ctx* ctx, const sfw3d_psf* psf, const sfw3d_table* table, int dtype,
                const void* y_dev, const sfw3d_solve_options* opts, void* arena_dev,
                int arena_volumes, double* rows_out, int* n_atoms, double* criterion_out,
                int* termination, sfw3d_solve_record* records, int* n_records);

#ifdef __cplusplus
}
#endif
#endif /* SFW3D_CUDA_H */
