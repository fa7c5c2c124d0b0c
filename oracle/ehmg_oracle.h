/*
 * ehmg_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference solver path
 * (/root/reference/proj/include/ehmg/{media,operator,vanka,transfer,
 * multigrid,krylov}.hpp) used ONLY as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg. The product path
 * (paper_2307_03242_b200/) never links or calls this code.
 *
 * Parity pinning: this restatement is checked against golden vectors
 * produced by the reference itself (oracle/_ref, built from the reference
 * headers by oracle/Makefile) in tests/golden/, and against the known-answer
 * values of the reference's own tests (tests/test_oracle_golden.py).
 *
 * Fields use the reference FieldVector flatten() order (assemble.hpp:256):
 * displacement components in axis order, then pressure, each block
 * axis-0-fastest, complex128 interleaved (re, im).
 */
#ifndef EHMG_ORACLE_H
#define EHMG_ORACLE_H

#include <complex.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double _Complex ocplx;

typedef struct og_op og_op;
typedef struct og_vanka og_vanka;
typedef struct og_mg og_mg;

/* -- grid ------------------------------------------------------------- */
int64_t og_n_dofs(int ndim, const int* dims);
int64_t og_n_cells(int ndim, const int* dims);

/* -- media ------------------------------------------------------------ */
/* media.hpp:95 build_attenuation_profile */
int og_attenuation_profile(int ndim, const int* dims, double gamma_phys, int layer_width,
                           double gamma_max, int absorb_top, double* out);
/* transfer.hpp:40 coarsen_media (one field) */
void og_coarsen_cell_field(int ndim, const int* dims_fine, const double* fine, double* coarse);

/* -- operator (operator.hpp:76 make_opdata, :437 apply_mixed_operator) - */
og_op* og_op_create(int ndim, const int* dims, double h, const double* lambda,
                    const double* mu, const double* rho, const double* gamma, double beta,
                    double omega, double alpha);
void og_op_destroy(og_op* op);
void og_apply(const og_op* op, const ocplx* x, ocplx* y);
/* operator.hpp:457 schur_eliminate_pressure (p entries of x ignored, y.p = 0) */
void og_schur_apply(const og_op* op, const ocplx* x, ocplx* y);
/* dense (column-major) matrix of the operator; n = n_dofs */
void og_assemble_dense(const og_op* op, ocplx* A);

/* -- Vanka (vanka.hpp:27) ---------------------------------------------- */
/* mode 0 = full, 1 = economic; order 0 = lexicographic, 1 = red-black */
og_vanka* og_vanka_create(const og_op* op, int mode);
void og_vanka_destroy(og_vanka* v);
int og_vanka_per_cell(const og_vanka* v);
const ocplx* og_vanka_cache(const og_vanka* v);
void og_vanka_sweep(og_vanka* v, const og_op* op, const ocplx* b, ocplx* x, double w, int order);

/* -- transfers (transfer.hpp:188 restrict_field, :197 prolong_field) -- */
void og_restrict(int ndim, const int* dims_fine, const ocplx* xf, ocplx* xc);
void og_prolong(int ndim, const int* dims_fine, const ocplx* xc, ocplx* xf);

/* -- Krylov (krylov.hpp:65 fgmres) ------------------------------------- */
typedef void (*og_apply_fn)(void* ctx, const ocplx* in, ocplx* out);
typedef struct {
  int restart, max_iterations;
  double rtol, stall_factor;
  int stall_cycles;
} og_krylov_opts;
typedef struct {
  int status; /* 0 converged, 1 max_iterations, 2 breakdown, 3 stalled */
  int iterations;
  double relres;
  int n_history;
  double* history; /* malloc'ed, caller frees with og_free */
} og_krylov_result;
void og_fgmres(int64_t n, og_apply_fn A, void* actx, og_apply_fn M, void* mctx, const ocplx* b,
               ocplx* x, const og_krylov_opts* opt, og_krylov_result* res);
void og_free(void* p);

/* -- multigrid (multigrid.hpp:70) --------------------------------------- */
typedef struct {
  int n_levels;
  int cycle; /* 0 two_grid, 1 v, 2 w, 3 k */
  int nu1, nu2;
  double damping;
  int vanka_mode; /* 0 full, 1 economic */
  int sweep;      /* 0 lexicographic, 1 red_black */
  int k_inner_iterations;
  double k_inner_rtol;
} og_mg_opts;
og_mg* og_mg_create(int ndim, const int* dims, double h, const double* lambda, const double* mu,
                    const double* rho, const double* gamma, double beta, double omega, double alpha,
                    const og_mg_opts* opt);
void og_mg_destroy(og_mg* mg);
int og_mg_n_levels(const og_mg* mg);
const og_op* og_mg_level_op(const og_mg* mg, int l);
void og_mg_cycle(og_mg* mg, const ocplx* b, ocplx* x);
void og_mg_precondition(og_mg* mg, const ocplx* r, ocplx* z);

/* Full solve: FGMRES on the unshifted operator preconditioned by one cycle
 * of the alpha-shifted hierarchy (experiments.hpp:258 run_solve_dim). */
void og_solve(og_mg* mg, const og_op* A0, const ocplx* b, ocplx* x, const og_krylov_opts* ko,
              og_krylov_result* res);

/* BASELINE configs[1]/[3]/[4] media recipe (csrc/ehmg_media.cuh restated) */
int og_layered_grf_media(int ndim, const int* dims, int n_layers, const double* ranges, double perturb,
                         double corr, double gamma_phys, uint64_t seed, double* lambda, double* mu,
                         double* rho, double* gamma);

#ifdef __cplusplus
}
#endif
#endif
