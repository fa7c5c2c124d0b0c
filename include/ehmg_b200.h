/*
 * ehmg_b200.h -- C ABI of the B200-native elastic-Helmholtz multigrid path.
 *
 * Drop-in boundary for the reference's matrix-free solver API
 * (/root/reference/proj/include/ehmg/*.hpp). Every entry point below names
 * the reference interface it replaces (file:line). Plain pointers and sizes
 * only; no torch or CUDA types cross this boundary.
 *
 * Field vectors are complex128 (interleaved re, im) in the reference
 * flatten() order (assemble.hpp:256): displacement components u_0..u_{d-1}
 * on their face boxes, then the cell-centred pressure, each block
 * axis-0-fastest. `where` says whether field pointers are host memory
 * (EHMG_HOST: copied to/from HBM inside the call) or device memory that the
 * caller keeps resident in HBM (EHMG_DEVICE).
 *
 * Ordering of EHMG_DEVICE buffers: the library runs its kernels on its own
 * non-blocking CUDA streams, so a device input must be complete before the
 * call (synchronise the stream that produced it; the Python binding does this
 * for torch's current stream). Device outputs are complete when the call
 * returns (the library synchronises its stream).
 *
 * Media are cell-sized float64 arrays, axis-0-fastest (media.hpp:13).
 * Errors: every call returns 0 on success or a negative EHMG_E* code; the
 * message (mirroring the reference's exception text) is available from
 * ehmg_last_error().
 */
#ifndef EHMG_B200_H
#define EHMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EHMG_HOST 0
#define EHMG_DEVICE 1

#define EHMG_OK 0
#define EHMG_EINVAL -1   /* std::invalid_argument in the reference */
#define EHMG_ERUNTIME -2 /* std::runtime_error (singular cell / LU failure) */
#define EHMG_ECUDA -3    /* CUDA / no device */
#define EHMG_ERANGE -4   /* std::out_of_range / std::length_error */

typedef struct ehmg_op_s* ehmg_op;
typedef struct ehmg_vanka_s* ehmg_vanka;
typedef struct ehmg_mg_s* ehmg_mg;

const char* ehmg_last_error(void);
/* Version string of the built library (sm_100a build id). */
const char* ehmg_version(void);
/* Select the CUDA device for subsequent handles (one process per GPU). */
int ehmg_set_device(int device);

/* ---- operator: operator.hpp:76 make_opdata, :437 apply_mixed_operator,
 *      :449 apply_shifted_operator (alpha folded into the mass term) ----- */
int ehmg_op_create(int ndim, const int* dims, double h, const double* lambda, const double* mu,
                   const double* rho, const double* gamma, double beta, double omega,
                   double alpha, ehmg_op* out);
int ehmg_op_destroy(ehmg_op op);
int64_t ehmg_op_n_dofs(ehmg_op op);
/* y = H x (operator.hpp:437) */
int ehmg_apply_mixed_operator(ehmg_op op, const double* x, double* y, int where);
/* r = b - H x (multigrid.hpp:210 residual) */
int ehmg_residual(ehmg_op op, const double* b, const double* x, double* r, int where);
/* CUDA stream the handle's kernels run on (cudaStream_t as an integer). */
uint64_t ehmg_op_stream(ehmg_op op);

/* ---- Vanka box smoother: vanka.hpp:27 VankaSmoother, :49 sweep -------
 * mode 0 = full, 1 = economic; order 0 = lexicographic, 1 = red-black.
 * The factorisation cache (vanka.hpp:76) is built on the device at create. */
int ehmg_vanka_create(ehmg_op op, int mode, ehmg_vanka* out);
int ehmg_vanka_destroy(ehmg_vanka v);
int ehmg_vanka_per_cell_complex_count(ehmg_vanka v); /* vanka.hpp:35 */
int ehmg_vanka_cache(ehmg_vanka v, double* out);     /* host copy of the cache */
int ehmg_vanka_sweep(ehmg_vanka v, const double* b, double* x, double w, int order, int nsweeps,
                     int where);

/* ---- transfers: transfer.hpp:188 restrict_field, :197 prolong_field,
 *      :40 coarsen_media (one cell field) -------------------------------- */
int ehmg_restrict_field(int ndim, const int* dims_fine, const double* xf, double* xc, int where);
int ehmg_prolong_field(int ndim, const int* dims_fine, const double* xc, double* xf, int where);
int ehmg_coarsen_media(int ndim, const int* dims_fine, const double* fine, double* coarse);
/* media.hpp:95 build_attenuation_profile (host arrays) */
int ehmg_attenuation_profile(int ndim, const int* dims, double gamma_phys, int layer_width,
                             double gamma_max, int absorb_top, double* out);

/* experiments.hpp:78 layered_media: seeded horizontal layers (5..10 layers,
 * per-layer vs, rho and lambda/mu ratio; same <random> engines and draw order
 * as the reference). Outputs are cell-sized host arrays; gamma = gamma_phys. */
int ehmg_layered_media(int ndim, const int* dims, double gamma_phys, uint64_t seed, double* lambda,
                       double* mu, double* rho, double* gamma);

/* BASELINE configs[1]/[3]/[4] media recipe (layered_media of experiments.hpp:78
 * extended): n_layers horizontal layers on the last axis (top = index 0) with
 * per-layer cs, cp/cs, rho drawn uniformly from ranges = {cs_lo, cs_hi,
 * ratio_lo, ratio_hi, rho_lo, rho_hi}, each multiplied by its own smooth
 * Gaussian random field (correlation length corr_cells, covariance
 * exp(-r^2/corr^2)) mapped into +-perturb; mu = rho cs^2,
 * lambda = mu ((cp/cs)^2 - 2), gamma = gamma_phys. Deterministic in `seed`
 * (splitmix64 streams; the exact recipe is in csrc/ehmg_media.cuh). Computed
 * on the device, returned as cell-sized host arrays. */
int ehmg_layered_grf_media(int ndim, const int* dims, int n_layers, const double* ranges, double perturb,
                           double corr_cells, double gamma_phys, uint64_t seed, double* lambda, double* mu,
                           double* rho, double* gamma);

/* ---- multigrid: multigrid.hpp:34 MgOptions, :75 Multigrid, :133 cycle,
 *      :136 precondition --------------------------------------------------
 * cycle: 0 two_grid, 1 v, 2 w, 3 k.
 * coarse (multigrid.hpp:22 CoarseSolverKind): 0 automatic, 1 lu, 2 kaczmarz.
 * automatic and lu solve the coarsest level exactly (CoarseSolverKind::lu,
 * multigrid.hpp:97) by an LU-derived inverse held in HBM; the reference's
 * automatic picks Kaczmarz-FGMRES in 3D (multigrid.hpp:93-95), which is not on
 * the B200 path: coarse = 2 returns EHMG_EINVAL. lu_dof_budget
 * (multigrid.hpp:42; 0 = the reference default 4000000) bounds the coarsest
 * DOF count: EHMG_ERANGE "assemble_sparse: grid exceeds DOF budget of N"
 * (assemble.hpp:209-211). The dense inverse also needs 2 N^2 complex of free
 * HBM during set-up (EHMG_ERANGE otherwise; N ~ 60000 on an idle B200).
 * kz_* (multigrid.hpp:45-49) are accepted and validated for ABI parity; they
 * only matter to the Kaczmarz solve. Zero-initialise the struct and set
 * the fields you use: zero kz_* values are read as the reference defaults. */
typedef struct {
  int n_levels;
  int cycle;
  int nu1, nu2;
  double damping;
  int vanka_mode;
  int sweep;
  int k_inner_iterations;
  double k_inner_rtol;
  /* 0: complex128 hierarchy; 1: complex64 hierarchy behind complex128
   * precondition()/cycle() calls (experiments.hpp:241 MixedPrecondition,
   * config "precision": "mixed"; V/W/two-grid cycles, red-black sweeps) */
  int precision;
  int coarse;
  int64_t lu_dof_budget;
  int kz_sweeps_per_apply;
  double kz_damping;
  double kz_rtol;
  int kz_max_iterations;
  int kz_restart;
} ehmg_mg_options;

int ehmg_multigrid_create(int ndim, const int* dims, double h, const double* lambda,
                          const double* mu, const double* rho, const double* gamma, double beta,
                          double omega, double alpha, const ehmg_mg_options* opt, ehmg_mg* out);
int ehmg_multigrid_destroy(ehmg_mg mg);
int ehmg_multigrid_n_levels(ehmg_mg mg);
/* Number of distinct Vanka factor entry sets of a level when its colour
 * updates read them through the factor dictionary (exact deduplication of
 * vanka.hpp:72's per-cell cache: homogeneous regions, sponge depth classes);
 * 0 when the level keeps the per-cell cache; -1 for a bad handle / level.
 * No reference counterpart (measurement: the bytes one update moves). */
int ehmg_multigrid_factor_sets(ehmg_mg mg, int level);
int ehmg_multigrid_cycle(ehmg_mg mg, const double* b, double* x, int where);
int ehmg_multigrid_precondition(ehmg_mg mg, const double* r, double* z, int where);
/* multigrid.hpp:136 Multigrid::precondition applied to `count` right-hand
 * sides held in host memory (r[i] -> z[i]; the multi-source runs of
 * experiments.hpp call it once per source). The host<->device copies of
 * neighbouring right-hand sides overlap the cycle of the current one (two
 * staging buffers per direction, copy streams beside the solver stream);
 * pinned host buffers are needed for the overlap. Results equal `count`
 * ehmg_multigrid_precondition calls. Pointers may repeat (an output buffer
 * reused two or more entries later is written in order). */
int ehmg_multigrid_precondition_many(ehmg_mg mg, int count, const double* const* r, double* const* z);
uint64_t ehmg_multigrid_stream(ehmg_mg mg);
/* Replay `count` preconditioner applications on device buffers and return
 * the CUDA-event time of the whole batch in milliseconds (bench helper). */
int ehmg_multigrid_time_precondition(ehmg_mg mg, const double* r_dev, double* z_dev, int count,
                                     double* ms);

/* multigrid.hpp:56 MeasureOptions / :63 MeasureResult / :143
 * measure_convergence_factor: stationary cycles from the reference's seeded
 * random start; factor = geometric-mean residual reduction per cycle. */
typedef struct {
  int warmup;
  double tol;
  int max_cycles;
  int growth_limit;
} ehmg_measure_options;

typedef struct {
  double factor;
  int cycles;
  int diverged;
  int n_history;
} ehmg_measure_result;

int ehmg_multigrid_measure_convergence(ehmg_mg mg, uint64_t seed, const ehmg_measure_options* mo,
                                       ehmg_measure_result* res, double* history, int history_cap);

/* ---- z-slab decomposed multigrid (north_star subsystem (6); no reference
 *      counterpart -- the reference is single-node CPU). Fine levels are split
 *      into z-slabs with 2 ghost planes exchanged after every field update;
 *      levels with z extent <= agg_n2 are agglomerated (replicated). In one
 *      process all slabs live on the current device and exchange by device
 *      copies; results equal ehmg_multigrid_precondition (same options).
 *      V/W cycles in complex128 or (opt->precision = 1) complex64; K-cycles
 *      need one slab per process (ehmg_dist_*) or nslabs = 1.
 * plan: la = number of distributed levels, z0[0..nslabs] = level-0 slab
 *       boundaries (pure host function, no device needed). */
typedef struct ehmg_slab_mg_s* ehmg_slab_mg;
int ehmg_slab_plan(int n2, int n_levels, int nslabs, int agg_n2, int* la, int* z0);
int ehmg_slab_multigrid_create(int ndim, const int* dims, double h, const double* lambda,
                               const double* mu, const double* rho, const double* gamma,
                               double beta, double omega, double alpha,
                               const ehmg_mg_options* opt, int nslabs, int agg_n2,
                               ehmg_slab_mg* out);
int ehmg_slab_multigrid_destroy(ehmg_slab_mg mg);
int ehmg_slab_multigrid_levels(ehmg_slab_mg mg, int* distributed, int* total);
int ehmg_slab_multigrid_precondition(ehmg_slab_mg mg, const double* r, double* z, int where);
/* bytes moved by ghost exchanges + agglomeration during the last precondition */
int64_t ehmg_slab_multigrid_exchanged_bytes(ehmg_slab_mg mg);

/* ---- one z-slab per process (one process per GPU on one node). Ranks
 *      rendezvous through a POSIX shared-memory segment named by `job`,
 *      share inbox buffers through CUDA IPC (peer copies over NVLink) and
 *      sum FGMRES reductions in rank order. Media and fields are passed as
 *      full host arrays; each rank reads its window and writes back only the
 *      planes it owns. Results equal the single-process solver's. V/W/K
 *      cycles, complex128 or complex64 hierarchy (opt->precision); the exact
 *      coarsest solve is row-partitioned over the ranks. */
typedef struct ehmg_dist_s* ehmg_dist;
int ehmg_dist_create(const char* job, int rank, int nranks, int device, int ndim, const int* dims,
                     double h, const double* lambda, const double* mu, const double* rho,
                     const double* gamma, double beta, double omega, double alpha,
                     const ehmg_mg_options* opt, int agg_n2, ehmg_dist* out);
int ehmg_dist_destroy(ehmg_dist d);
int ehmg_dist_window(ehmg_dist d, int* z0, int* z1, int* w0, int* w1);
int ehmg_dist_precondition(ehmg_dist d, const double* r, double* z);
/* bench helper: CUDA-event ms of `count` applications on the resident window */
int ehmg_dist_time_precondition(ehmg_dist d, const double* r, int count, double* ms);
int64_t ehmg_dist_exchanged_bytes(ehmg_dist d);

/* Per-launch CUDA-event profiling of the cycle kernels (bench roofline).
 * report: one "kernel level count total_ms" line per (kernel, level). */
int ehmg_profile_enable(int on);
int ehmg_profile_report(char* buf, int cap);

/* ---- Krylov: krylov.hpp:45 KrylovOptions, :55 KrylovResult, :65 fgmres,
 *      driven as in experiments.hpp:313 (A = unshifted operator, M = one
 *      multigrid cycle on the shifted hierarchy) ---------------------------
 * status: 0 converged, 1 max_iterations, 2 breakdown, 3 stalled. */
typedef struct {
  int restart;
  int max_iterations;
  double rtol;
  double stall_factor;
  int stall_cycles;
  /* B200 addition (not in krylov.hpp:45): Arnoldi orthogonalisation.
   * 0 = classical Gram-Schmidt passes (all projections of a step in one HBM
   *     pass, the update + norm in a second; with the reference's
   *     re-orthogonalisation criterion this is CGS2) -- the default;
   * 1 = modified Gram-Schmidt in the reference's order (krylov.hpp:115).
   * Distributed (z-slab) solves always use 1. */
  int orthogonalization;
} ehmg_krylov_options;

typedef struct {
  int status;
  int iterations;
  double relres;
  int n_history;
} ehmg_krylov_result;

/* The FGMRES workspace (2 restart + 3 level-0 vectors) stays on M between
 * solves (released by ehmg_multigrid_destroy); M == NULL solves unpreconditioned
 * with a per-call workspace. */
int ehmg_fgmres_solve(ehmg_op A, ehmg_mg M, const double* b, double* x, int where,
                      const ehmg_krylov_options* opt, ehmg_krylov_result* res, double* history,
                      int history_cap);
/* FGMRES over z-slab-distributed vectors (one slab per process); b and x are
 * full host arrays, x receives this rank's owned planes. */
int ehmg_dist_solve(ehmg_dist d, const double* b, double* x, const ehmg_krylov_options* opt,
                    ehmg_krylov_result* res, double* history, int history_cap);

/* ---- field BLAS-1 on device buffers (grid.hpp:129 axpy, :135 scal,
 *      :142 dot, :150 norm) ------------------------------------------------ */
int ehmg_field_dot(int64_t n, const double* x, const double* y, double* out_re_im);
int ehmg_field_norm(int64_t n, const double* x, double* out);
int ehmg_field_axpy(int64_t n, double a_re, double a_im, const double* x, double* y);

/* ---- device memory helpers for callers without their own allocator ---- */
int ehmg_device_alloc(int64_t bytes, void** out);
int ehmg_device_free(void* p);
int ehmg_memcpy(void* dst, const void* src, int64_t bytes, int kind /* 0 H2D, 1 D2H, 2 D2D */);

#ifdef __cplusplus
}
#endif
#endif
