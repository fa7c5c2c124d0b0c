/*
 * ehmg_oracle.c -- CPU ORACLE (test infrastructure only; see ehmg_oracle.h).
 *
 * Plain-C restatement of the reference's matrix-free solver path. Every
 * function cites the reference file:line it follows; paths are relative to
 * /root/reference/proj/include/ehmg/. Scalar loops in the reference's own
 * traversal order, so rounding tracks the reference closely; the reference
 * itself (oracle/_ref) pins this file through tests/golden/.
 */
#include "ehmg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- boxes */
/* grid.hpp:21 Box: axis-0-fastest linearisation */
typedef struct {
  int n;
  int d[3];
} box_t;

static inline int64_t box_size(const box_t* b) {
  int64_t s = 1;
  for (int a = 0; a < b->n; ++a) s *= b->d[a];
  return s;
}
static inline int box_contains(const box_t* b, const int* i) {
  for (int a = 0; a < b->n; ++a)
    if (i[a] < 0 || i[a] >= b->d[a]) return 0;
  return 1;
}
static inline int64_t box_lin(const box_t* b, const int* i) {
  int64_t r = i[b->n - 1];
  for (int a = b->n - 2; a >= 0; --a) r = r * b->d[a] + i[a];
  return r;
}
static inline void box_unlin(const box_t* b, int64_t r, int* i) {
  for (int a = 0; a < b->n; ++a) {
    i[a] = (int)(r % b->d[a]);
    r /= b->d[a];
  }
}
/* Visit every index in storage order (grid.hpp:51 for_each). */
#define FOR_EACH(bx, I)                                    \
  for (int64_t _r = 0, _n = box_size(bx); _r < _n; ++_r) \
    for (int I[3] = {0, 0, 0}, _once = (box_unlin(bx, _r, I), 1); _once; _once = 0)

static box_t cell_box(int n, const int* dims) {
  box_t b = {n, {1, 1, 1}};
  for (int a = 0; a < n; ++a) b.d[a] = dims[a];
  return b;
}
static box_t face_box(int n, const int* dims, int axis) {
  box_t b = cell_box(n, dims);
  b.d[axis] += 1;
  return b;
}
static box_t edge_box(int n, const int* dims, int a, int b2) {
  box_t b = cell_box(n, dims);
  b.d[a] += 1;
  b.d[b2] += 1;
  return b;
}
/* operator.hpp:34 */
static inline int edge_pair_id(int a, int b) {
  if (a > b) {
    int t = a;
    a = b;
    b = t;
  }
  return a + b - 1;
}
static inline void shifted(const int* i, int axis, int d, int* o) {
  o[0] = i[0];
  o[1] = i[1];
  o[2] = i[2];
  o[axis] += d;
}

int64_t og_n_cells(int ndim, const int* dims) {
  box_t b = cell_box(ndim, dims);
  return box_size(&b);
}
int64_t og_n_dofs(int ndim, const int* dims) {
  int64_t s = og_n_cells(ndim, dims);
  for (int k = 0; k < ndim; ++k) {
    box_t f = face_box(ndim, dims, k);
    s += box_size(&f);
  }
  return s;
}
void og_free(void* p) { free(p); }

/* ---------------------------------------------------------------- media */
/* media.hpp:95 build_attenuation_profile */
int og_attenuation_profile(int n, const int* dims, double gamma_phys, int L, double gamma_max,
                           int absorb_top, double* out) {
  if (L < 0) return -1;
  if (L > 0)
    for (int a = 0; a < n; ++a)
      if (2 * L >= dims[a]) return -2;
  box_t cb = cell_box(n, dims);
  FOR_EACH(&cb, c) {
    double ramp = 0;
    if (L > 0)
      for (int a = 0; a < n; ++a) {
        int dist_lo = c[a], dist_hi = dims[a] - 1 - c[a];
        int skip_lo = absorb_top ? 0 : (a == n - 1);
        if (!skip_lo && dist_lo < L) {
          double d = (double)(L - dist_lo) / L;
          if (d * d > ramp) ramp = d * d;
        }
        if (dist_hi < L) {
          double d = (double)(L - dist_hi) / L;
          if (d * d > ramp) ramp = d * d;
        }
      }
    out[box_lin(&cb, c)] = L == 0 ? gamma_phys : gamma_phys + gamma_max * ramp;
  }
  return 0;
}

/* transfer.hpp:40 coarsen_media: coarse cell = mean of its 2^Dim children */
void og_coarsen_cell_field(int n, const int* df, const double* v, double* w) {
  int dc[3] = {1, 1, 1};
  for (int a = 0; a < n; ++a) dc[a] = df[a] / 2;
  box_t fb = cell_box(n, df), cb = cell_box(n, dc);
  FOR_EACH(&cb, c) {
    double s = 0;
    int nch = 1 << n;
    for (int bits = 0; bits < nch; ++bits) {
      int f[3] = {0, 0, 0};
      for (int a = 0; a < n; ++a) f[a] = 2 * c[a] + ((bits >> a) & 1);
      s += v[box_lin(&fb, f)];
    }
    w[box_lin(&cb, c)] = s / nch;
  }
}

/* ------------------------------------------------------------- operator */
struct og_op {
  int n;
  int dims[3];
  double h, beta, omega, alpha, inv_h;
  box_t cellb, faceb[3], edgeb[3];
  int64_t off[4], ndofs;
  double *mu_cell, *lamu, *inv_lamu;
  double* mu_edge[3];
  ocplx* massdiag[3];
};

/* operator.hpp:76 make_opdata (non-periodic) */
og_op* og_op_create(int n, const int* dims, double h, const double* lambda, const double* mu,
                    const double* rho, const double* gamma, double beta, double omega,
                    double alpha) {
  og_op* D = (og_op*)calloc(1, sizeof(og_op));
  D->n = n;
  for (int a = 0; a < 3; ++a) D->dims[a] = a < n ? dims[a] : 1;
  D->h = h;
  D->beta = beta;
  D->omega = omega;
  D->alpha = alpha;
  D->inv_h = 1.0 / h;
  D->cellb = cell_box(n, dims);
  int64_t o = 0;
  for (int k = 0; k < n; ++k) {
    D->faceb[k] = face_box(n, dims, k);
    D->off[k] = o;
    o += box_size(&D->faceb[k]);
  }
  D->off[n] = o;
  D->ndofs = o + box_size(&D->cellb);
  int64_t nc = box_size(&D->cellb);
  D->mu_cell = (double*)malloc(sizeof(double) * nc);
  D->lamu = (double*)malloc(sizeof(double) * nc);
  D->inv_lamu = (double*)malloc(sizeof(double) * nc);
  for (int64_t i = 0; i < nc; ++i) {
    D->mu_cell[i] = mu[i];
    double lm = lambda[i] + mu[i];
    D->lamu[i] = lm;
    D->inv_lamu[i] = 1.0 / lm;
  }
  /* mu on edges: mean of the adjacent in-range cells (operator.hpp:108) */
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b) {
      int pid = edge_pair_id(a, b);
      box_t eb = edge_box(n, dims, a, b);
      D->edgeb[pid] = eb;
      double* out = (double*)malloc(sizeof(double) * box_size(&eb));
      FOR_EACH(&eb, e) {
        double s = 0;
        int cnt = 0;
        for (int da = -1; da <= 0; ++da)
          for (int db = -1; db <= 0; ++db) {
            int c[3] = {e[0], e[1], e[2]};
            c[a] += da;
            c[b] += db;
            if (box_contains(&D->cellb, c)) {
              s += mu[box_lin(&D->cellb, c)];
              ++cnt;
            }
          }
        out[box_lin(&eb, e)] = s / cnt;
      }
      D->mu_edge[pid] = out;
    }
  /* face mass diagonal omega^2 (1 - i(gamma+alpha)) rho (operator.hpp:132) */
  double w2 = omega * omega;
  for (int k = 0; k < n; ++k) {
    box_t fb = D->faceb[k];
    ocplx* out = (ocplx*)malloc(sizeof(ocplx) * box_size(&fb));
    FOR_EACH(&fb, f) {
      double sr = 0, sg = 0;
      int cnt = 0;
      for (int d = -1; d <= 0; ++d) {
        int c[3] = {f[0], f[1], f[2]};
        c[k] += d;
        if (box_contains(&D->cellb, c)) {
          int64_t ci = box_lin(&D->cellb, c);
          sr += rho[ci];
          sg += gamma[ci];
          ++cnt;
        }
      }
      double rho_f = sr / cnt, gam_f = sg / cnt + alpha;
      out[box_lin(&fb, f)] = CMPLX(w2 * rho_f, -w2 * gam_f * rho_f);
    }
    D->massdiag[k] = out;
  }
  return D;
}

void og_op_destroy(og_op* D) {
  if (!D) return;
  free(D->mu_cell);
  free(D->lamu);
  free(D->inv_lamu);
  for (int i = 0; i < 3; ++i) {
    free(D->mu_edge[i]);
    free(D->massdiag[i]);
  }
  free(D);
}

/* Accessor: a field vector, or a unit basis vector (operator.hpp:172/212). */
typedef struct {
  const og_op* D;
  const ocplx* x;
  int unit, ucomp;
  int uat[3];
} acc_t;

static inline ocplx acc_u(const acc_t* A, int k, const int* f) {
  const box_t* fb = &A->D->faceb[k];
  if (!box_contains(fb, f)) return 0;
  if (A->unit)
    return (k == A->ucomp && f[0] == A->uat[0] && f[1] == A->uat[1] && f[2] == A->uat[2]) ? 1.0
                                                                                          : 0.0;
  return A->x[A->D->off[k] + box_lin(fb, f)];
}
static inline ocplx acc_p(const acc_t* A, const int* c) {
  const box_t* cb = &A->D->cellb;
  if (!box_contains(cb, c)) return 0;
  int n = A->D->n;
  if (A->unit)
    return (A->ucomp == n && c[0] == A->uat[0] && c[1] == A->uat[1] && c[2] == A->uat[2]) ? 1.0
                                                                                           : 0.0;
  return A->x[A->D->off[n] + box_lin(cb, c)];
}
static inline int tap_valid(const og_op* D, int k, int axis, int coord) {
  return coord >= 0 && coord < D->faceb[k].d[axis];
}

/* operator.hpp:267 dspread_cell: aligned derivative of u_k at cell c */
static ocplx dspread_cell(const og_op* D, int k, const int* c, const acc_t* A) {
  const double beta = D->beta;
#define PAIRC(b)                                        \
  ({                                                    \
    int _p[3];                                          \
    shifted(b, k, 1, _p);                               \
    acc_u(A, k, _p) - acc_u(A, k, b);                   \
  })
  ocplx v = beta * PAIRC(c);
  if (beta != 1.0) {
    double wsum = beta;
    if (D->n == 2) {
      const int t = 1 - k;
      const double w = (1.0 - beta) / 4.0;
      for (int st = -1; st <= 1; ++st) {
        if (!tap_valid(D, k, t, c[t] + st)) continue;
        const double wt = w * (double)(st == 0 ? 2 : 1);
        int b[3];
        shifted(c, t, st, b);
        v += wt * PAIRC(b);
        wsum += wt;
      }
    } else {
      const int t1 = (k + 1) % 3, t2 = (k + 2) % 3;
      const double w = (1.0 - beta) / 16.0;
      for (int s1 = -1; s1 <= 1; ++s1)
        for (int s2 = -1; s2 <= 1; ++s2) {
          if (!tap_valid(D, k, t1, c[t1] + s1) || !tap_valid(D, k, t2, c[t2] + s2)) continue;
          int b1[3], b[3];
          shifted(c, t1, s1, b1);
          shifted(b1, t2, s2, b);
          const double wt = w * (double)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
          v += wt * PAIRC(b);
          wsum += wt;
        }
    }
    v *= 1.0 / wsum;
  }
#undef PAIRC
  return v * D->inv_h;
}

/* operator.hpp:306 dspread_edge: derivative of u_k along j at edge (k,j) */
static ocplx dspread_edge(const og_op* D, int k, int j, const int* e, const acc_t* A) {
  const double beta = D->beta;
#define PAIRE(b)                                        \
  ({                                                    \
    int _m[3];                                          \
    shifted(b, j, -1, _m);                              \
    acc_u(A, k, b) - acc_u(A, k, _m);                   \
  })
  ocplx v = beta * PAIRE(e);
  if (beta != 1.0) {
    double wsum = beta;
    if (D->n == 2) {
      const int t = k;
      const double w = (1.0 - beta) / 4.0;
      for (int st = -1; st <= 1; ++st) {
        if (!tap_valid(D, k, t, e[t] + st)) continue;
        const double wt = w * (double)(st == 0 ? 2 : 1);
        int b[3];
        shifted(e, t, st, b);
        v += wt * PAIRE(b);
        wsum += wt;
      }
    } else {
      const int t1 = 3 - k - j, t2 = k;
      const double w = (1.0 - beta) / 16.0;
      for (int s1 = -1; s1 <= 1; ++s1)
        for (int s2 = -1; s2 <= 1; ++s2) {
          if (!tap_valid(D, k, t1, e[t1] + s1) || !tap_valid(D, k, t2, e[t2] + s2)) continue;
          int b1[3], b[3];
          shifted(e, t1, s1, b1);
          shifted(b1, t2, s2, b);
          const double wt = w * (double)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
          v += wt * PAIRE(b);
          wsum += wt;
        }
    }
    v *= 1.0 / wsum;
  }
#undef PAIRE
  return v * D->inv_h;
}

/* operator.hpp:344 flux_cell / :350 flux_edge */
static inline ocplx flux_cell(const og_op* D, int k, const int* c, const acc_t* A) {
  if (!box_contains(&D->cellb, c)) return 0;
  return D->mu_cell[box_lin(&D->cellb, c)] * dspread_cell(D, k, c, A);
}
static inline ocplx flux_edge(const og_op* D, int k, int j, const int* e, const acc_t* A) {
  int pid = edge_pair_id(k, j);
  return D->mu_edge[pid][box_lin(&D->edgeb[pid], e)] * dspread_edge(D, k, j, e, A);
}

/* operator.hpp:359 mass_eval: convex spreading, boundary renormalised */
static ocplx mass_eval(const og_op* D, int k, const int* f, const acc_t* A) {
  const double beta = D->beta;
  const ocplx* md = D->massdiag[k];
  const box_t* fb = &D->faceb[k];
  ocplx v = beta * (md[box_lin(fb, f)] * acc_u(A, k, f));
  if (beta == 1.0) return v;
  const double wn = (1.0 - beta) / (2 * D->n);
  double wsum = beta;
  for (int a = 0; a < D->n; ++a)
    for (int sg = -1; sg <= 1; sg += 2) {
      int fn[3];
      shifted(f, a, sg, fn);
      if (box_contains(fb, fn)) {
        v += wn * (md[box_lin(fb, fn)] * acc_u(A, k, fn));
        wsum += wn;
      }
    }
  return v * (1.0 / wsum);
}

/* operator.hpp:389 row_u_acoustic */
static ocplx row_u_acoustic(const og_op* D, int k, const int* f, const acc_t* A) {
  ocplx out = 0;
  for (int j = 0; j < D->n; ++j) {
    if (j == k) {
      int cm[3];
      shifted(f, k, -1, cm);
      ocplx wm = flux_cell(D, k, cm, A);
      ocplx wp = flux_cell(D, k, f, A);
      out += (wm - wp) * D->inv_h;
    } else {
      int ep[3];
      shifted(f, j, 1, ep);
      ocplx wm = flux_edge(D, k, j, f, A);
      ocplx wp = flux_edge(D, k, j, ep, A);
      out += (wm - wp) * D->inv_h;
    }
  }
  out -= mass_eval(D, k, f, A);
  return out;
}
/* operator.hpp:409 row_u */
static ocplx row_u(const og_op* D, int k, const int* f, const acc_t* A) {
  ocplx out = row_u_acoustic(D, k, f, A);
  int cm[3];
  shifted(f, k, -1, cm);
  out += (acc_p(A, f) - acc_p(A, cm)) * D->inv_h;
  return out;
}
/* operator.hpp:416 row_p */
static ocplx row_p(const og_op* D, const int* c, const acc_t* A) {
  ocplx out = 0;
  for (int k = 0; k < D->n; ++k) out += dspread_cell(D, k, c, A);
  out += D->inv_lamu[box_lin(&D->cellb, c)] * acc_p(A, c);
  return out;
}

/* operator.hpp:423 apply_mixed_impl / :437 apply_mixed_operator */
void og_apply(const og_op* D, const ocplx* x, ocplx* y) {
  acc_t A = {D, x, 0, 0, {0, 0, 0}};
  for (int k = 0; k < D->n; ++k) {
    const box_t* fb = &D->faceb[k];
    FOR_EACH(fb, f) { y[D->off[k] + box_lin(fb, f)] = row_u(D, k, f, &A); }
  }
  FOR_EACH(&D->cellb, c) { y[D->off[D->n] + box_lin(&D->cellb, c)] = row_p(D, c, &A); }
}

/* operator.hpp:457 schur_eliminate_pressure */
void og_schur_apply(const og_op* D, const ocplx* x, ocplx* y) {
  acc_t A = {D, x, 0, 0, {0, 0, 0}};
  for (int k = 0; k < D->n; ++k) {
    const box_t* fb = &D->faceb[k];
    FOR_EACH(fb, f) {
      ocplx v = row_u_acoustic(D, k, f, &A);
      int cm[3];
      shifted(f, k, -1, cm);
      ocplx wv[2] = {0, 0};
      const int* cs[2] = {f, cm};
      for (int s = 0; s < 2; ++s) {
        if (!box_contains(&D->cellb, cs[s])) continue;
        ocplx dv = 0;
        for (int kk = 0; kk < D->n; ++kk) dv += dspread_cell(D, kk, cs[s], &A);
        wv[s] = D->lamu[box_lin(&D->cellb, cs[s])] * dv;
      }
      v -= (wv[0] - wv[1]) * D->inv_h;
      y[D->off[k] + box_lin(fb, f)] = v;
    }
  }
  int64_t nc = box_size(&D->cellb);
  for (int64_t i = 0; i < nc; ++i) y[D->off[D->n] + i] = 0;
}

/* Position of global DOF r: component and index. */
static void dof_pos(const og_op* D, int64_t r, int* comp, int* idx) {
  int c = D->n;
  for (int k = 0; k < D->n; ++k)
    if (r < D->off[k + 1]) {
      c = k;
      break;
    }
  *comp = c;
  const box_t* b = c < D->n ? &D->faceb[c] : &D->cellb;
  idx[0] = idx[1] = idx[2] = 0;
  box_unlin(b, r - D->off[c], idx);
}

/* Dense column-major matrix via unit probes of the row kernels. All row
 * stencils reach at most one index in every axis (operator.hpp:267-421),
 * so only a +-2 window of rows around each column is probed. */
void og_assemble_dense(const og_op* D, ocplx* M) {
  const int64_t N = D->ndofs;
  memset(M, 0, sizeof(ocplx) * N * N);
  for (int64_t col = 0; col < N; ++col) {
    int cc, ci[3];
    dof_pos(D, col, &cc, ci);
    acc_t A = {D, NULL, 1, cc, {ci[0], ci[1], ci[2]}};
    for (int rc = 0; rc <= D->n; ++rc) {
      const box_t* rb = rc < D->n ? &D->faceb[rc] : &D->cellb;
      int lo2 = D->n == 3 ? -2 : 0, hi2 = D->n == 3 ? 2 : 0;
      for (int o2 = lo2; o2 <= hi2; ++o2)
        for (int o1 = -2; o1 <= 2; ++o1)
          for (int o0 = -2; o0 <= 2; ++o0) {
            int r[3] = {ci[0] + o0, ci[1] + o1, ci[2] + o2};
            if (!box_contains(rb, r)) continue;
            ocplx v = rc < D->n ? row_u(D, rc, r, &A) : row_p(D, r, &A);
            M[(D->off[rc] + box_lin(rb, r)) + col * N] = v;
          }
    }
  }
}

/* ---------------------------------------------------------------- Vanka */
struct og_vanka {
  int mode, stride, n;
  int64_t ncell;
  ocplx* cache;
};

int og_vanka_per_cell(const og_vanka* v) { return v->stride; }
const ocplx* og_vanka_cache(const og_vanka* v) { return v->cache; }

/* vanka.hpp:76 build / :85 build_cell */
og_vanka* og_vanka_create(const og_op* D, int mode) {
  og_vanka* V = (og_vanka*)calloc(1, sizeof(og_vanka));
  const int n = D->n, full = mode == 0;
  V->mode = mode;
  V->n = n;
  V->stride = n * ((full ? 4 : 2) + 4) + 1; /* vanka.hpp:35 */
  V->ncell = box_size(&D->cellb);
  V->cache = (ocplx*)calloc((size_t)(V->ncell * V->stride), sizeof(ocplx));
  FOR_EACH(&D->cellb, c) {
    ocplx* q = V->cache + box_lin(&D->cellb, c) * V->stride;
    ocplx sum_cg = 0;
    for (int k = 0; k < n; ++k) {
      int f[2][3];
      memcpy(f[0], c, sizeof(int) * 3);
      shifted(c, k, 1, f[1]);
      ocplx U[2][2] = {{0, 0}, {0, 0}}, bk[2], ck[2];
      for (int i = 0; i < 2; ++i) {
        for (int j = 0; j < 2; ++j) {
          if (!full && i != j) continue;
          acc_t A = {D, NULL, 1, k, {f[j][0], f[j][1], f[j][2]}};
          U[i][j] = row_u(D, k, f[i], &A);
        }
        acc_t Ap = {D, NULL, 1, n, {c[0], c[1], c[2]}};
        bk[i] = row_u(D, k, f[i], &Ap);
        acc_t Au = {D, NULL, 1, k, {f[i][0], f[i][1], f[i][2]}};
        ck[i] = row_p(D, c, &Au);
      }
      ocplx Ui[2][2];
      if (full) {
        ocplx det = U[0][0] * U[1][1] - U[0][1] * U[1][0];
        ocplx idet = 1.0 / det;
        Ui[0][0] = U[1][1] * idet;
        Ui[0][1] = -U[0][1] * idet;
        Ui[1][0] = -U[1][0] * idet;
        Ui[1][1] = U[0][0] * idet;
      } else {
        Ui[0][0] = 1.0 / U[0][0];
        Ui[1][1] = 1.0 / U[1][1];
        Ui[0][1] = Ui[1][0] = 0;
      }
      ocplx g0 = Ui[0][0] * bk[0] + Ui[0][1] * bk[1];
      ocplx g1 = Ui[1][0] * bk[0] + Ui[1][1] * bk[1];
      ocplx h0 = ck[0] * Ui[0][0] + ck[1] * Ui[1][0];
      ocplx h1 = ck[0] * Ui[0][1] + ck[1] * Ui[1][1];
      sum_cg += ck[0] * g0 + ck[1] * g1;
      if (full) {
        *q++ = Ui[0][0];
        *q++ = Ui[0][1];
        *q++ = Ui[1][0];
        *q++ = Ui[1][1];
      } else {
        *q++ = Ui[0][0];
        *q++ = Ui[1][1];
      }
      *q++ = g0;
      *q++ = g1;
      *q++ = h0;
      *q++ = h1;
    }
    acc_t Ap = {D, NULL, 1, n, {c[0], c[1], c[2]}};
    ocplx d = row_p(D, c, &Ap);
    *q = 1.0 / (d - sum_cg);
  }
  return V;
}

void og_vanka_destroy(og_vanka* V) {
  if (!V) return;
  free(V->cache);
  free(V);
}

/* vanka.hpp:157 corrections of one cell from the current state */
static void vanka_corr(const og_vanka* V, const og_op* D, const acc_t* A, const ocplx* b,
                       const int* c, ocplx* du, ocplx* dp) {
  const int n = D->n, full = V->mode == 0;
  const ocplx* q = V->cache + box_lin(&D->cellb, c) * V->stride;
  const int blk_w = full ? 8 : 6;
  ocplx r[3][2];
  ocplx dpa = b[D->off[n] + box_lin(&D->cellb, c)] - row_p(D, c, A);
  for (int k = 0; k < n; ++k) {
    int f[2][3];
    memcpy(f[0], c, sizeof(int) * 3);
    shifted(c, k, 1, f[1]);
    for (int i = 0; i < 2; ++i)
      r[k][i] = b[D->off[k] + box_lin(&D->faceb[k], f[i])] - row_u(D, k, f[i], A);
    const ocplx* hk = q + k * blk_w + (full ? 6 : 4);
    dpa -= hk[0] * r[k][0] + hk[1] * r[k][1];
  }
  *dp = q[V->stride - 1] * dpa;
  for (int k = 0; k < n; ++k) {
    const ocplx* blk = q + k * blk_w;
    const ocplx* gk = blk + (full ? 4 : 2);
    if (full) {
      du[2 * k + 0] = blk[0] * r[k][0] + blk[1] * r[k][1] - gk[0] * *dp;
      du[2 * k + 1] = blk[2] * r[k][0] + blk[3] * r[k][1] - gk[1] * *dp;
    } else {
      du[2 * k + 0] = blk[0] * r[k][0] - gk[0] * *dp;
      du[2 * k + 1] = blk[1] * r[k][1] - gk[1] * *dp;
    }
  }
}

static void vanka_apply_cell(const og_op* D, ocplx* x, const int* c, const ocplx* du, ocplx dp,
                             double w) {
  for (int k = 0; k < D->n; ++k) {
    int f1[3];
    shifted(c, k, 1, f1);
    x[D->off[k] + box_lin(&D->faceb[k], c)] += w * du[2 * k + 0];
    x[D->off[k] + box_lin(&D->faceb[k], f1)] += w * du[2 * k + 1];
  }
  x[D->off[D->n] + box_lin(&D->cellb, c)] += w * dp;
}

/* vanka.hpp:148 sweep_impl */
void og_vanka_sweep(og_vanka* V, const og_op* D, const ocplx* b, ocplx* x, double w, int order) {
  acc_t A = {D, x, 0, 0, {0, 0, 0}};
  const int n = D->n, nl = 2 * n + 1;
  if (order == 0) {
    ocplx du[6], dp;
    FOR_EACH(&D->cellb, c) {
      vanka_corr(V, D, &A, b, c, du, &dp);
      vanka_apply_cell(D, x, c, du, dp, w);
    }
    return;
  }
  ocplx* defer = (ocplx*)malloc(sizeof(ocplx) * V->ncell * nl);
  for (int color = 0; color < 2; ++color) {
    FOR_EACH(&D->cellb, c) {
      int par = 0;
      for (int a = 0; a < n; ++a) par += c[a];
      if ((par & 1) != color) continue;
      ocplx* slot = defer + box_lin(&D->cellb, c) * nl;
      vanka_corr(V, D, &A, b, c, slot, slot + 2 * n);
    }
    FOR_EACH(&D->cellb, c) {
      int par = 0;
      for (int a = 0; a < n; ++a) par += c[a];
      if ((par & 1) != color) continue;
      const ocplx* slot = defer + box_lin(&D->cellb, c) * nl;
      vanka_apply_cell(D, x, c, slot, slot[2 * n], w);
    }
  }
  free(defer);
}

/* ------------------------------------------------------------- transfers */
/* transfer.hpp:77 restrict_1d / :109 prolong_1d (non-periodic). A row is
 * at most 3 (index, weight) taps. */
typedef struct {
  int cnt;
  int idx[3];
  double w[3];
} tap_row;

static void renorm(tap_row* r) {
  double s = 0;
  for (int i = 0; i < r->cnt; ++i) s += r->w[i];
  for (int i = 0; i < r->cnt; ++i) r->w[i] /= s;
}

static tap_row* restrict_1d(int n_fine, int face, int* n_out) {
  if (face) {
    int nc = (n_fine - 1) / 2;
    tap_row* t = (tap_row*)calloc(nc + 1, sizeof(tap_row));
    const int offs[3] = {-1, 0, 1};
    const double ws[3] = {0.25, 0.5, 0.25};
    for (int i = 0; i <= nc; ++i) {
      for (int q = 0; q < 3; ++q) {
        int f = 2 * i + offs[q];
        if (f >= 0 && f < n_fine) {
          t[i].idx[t[i].cnt] = f;
          t[i].w[t[i].cnt++] = ws[q];
        }
      }
      renorm(&t[i]);
    }
    *n_out = nc + 1;
    return t;
  }
  int nc = n_fine / 2;
  tap_row* t = (tap_row*)calloc(nc, sizeof(tap_row));
  for (int i = 0; i < nc; ++i) {
    t[i].cnt = 2;
    t[i].idx[0] = 2 * i;
    t[i].w[0] = 0.5;
    t[i].idx[1] = 2 * i + 1;
    t[i].w[1] = 0.5;
  }
  *n_out = nc;
  return t;
}

static tap_row* prolong_1d(int n_fine, int face) {
  tap_row* t = (tap_row*)calloc(n_fine, sizeof(tap_row));
  if (face) {
    for (int f = 0; f < n_fine; ++f) {
      if (f % 2 == 0) {
        t[f].cnt = 1;
        t[f].idx[0] = f / 2;
        t[f].w[0] = 1.0;
      } else {
        t[f].cnt = 2;
        t[f].idx[0] = f / 2;
        t[f].w[0] = 0.5;
        t[f].idx[1] = f / 2 + 1;
        t[f].w[1] = 0.5;
      }
    }
  } else {
    int nc = n_fine / 2;
    for (int f = 0; f < n_fine; ++f) {
      int c = f / 2, far = (f % 2 == 0) ? c - 1 : c + 1;
      t[f].cnt = 1;
      t[f].idx[0] = c;
      t[f].w[0] = 0.75;
      if (far >= 0 && far < nc) {
        t[f].idx[1] = far;
        t[f].w[1] = 0.25;
        t[f].cnt = 2;
      }
      renorm(&t[f]);
    }
  }
  return t;
}

/* transfer.hpp:164 transfer_component: tensor product applied axis by axis */
static void transfer_component(int n, const int* df, int comp, int restricting, const ocplx* in,
                               ocplx* out) {
  int dc[3] = {1, 1, 1};
  for (int a = 0; a < n; ++a) dc[a] = df[a] / 2;
  box_t from = comp < n ? face_box(n, restricting ? df : dc, comp) : cell_box(n, restricting ? df : dc);
  box_t to = comp < n ? face_box(n, restricting ? dc : df, comp) : cell_box(n, restricting ? dc : df);
  int64_t cap = box_size(&from) > box_size(&to) ? box_size(&from) : box_size(&to);
  /* intermediate sizes never exceed max(from, to) along the sweep */
  int64_t cap2 = 1;
  for (int a = 0; a < n; ++a) cap2 *= (from.d[a] > to.d[a] ? from.d[a] : to.d[a]);
  if (cap2 > cap) cap = cap2;
  ocplx* buf = (ocplx*)malloc(sizeof(ocplx) * cap);
  ocplx* nxt = (ocplx*)malloc(sizeof(ocplx) * cap);
  memcpy(buf, in, sizeof(ocplx) * box_size(&from));
  box_t cur = from;
  for (int a = 0; a < n; ++a) {
    const int face = comp == a;
    const int n_fine = face ? df[a] + 1 : df[a];
    int nrows;
    tap_row* tab = restricting ? restrict_1d(n_fine, face, &nrows) : prolong_1d(n_fine, face);
    box_t nb = cur;
    nb.d[a] = to.d[a];
    FOR_EACH(&nb, o) {
      ocplx s = 0;
      int i[3] = {o[0], o[1], o[2]};
      const tap_row* row = &tab[o[a]];
      for (int q = 0; q < row->cnt; ++q) {
        i[a] = row->idx[q];
        s += row->w[q] * buf[box_lin(&cur, i)];
      }
      nxt[box_lin(&nb, o)] = s;
    }
    free(tab);
    ocplx* t = buf;
    buf = nxt;
    nxt = t;
    cur = nb;
  }
  memcpy(out, buf, sizeof(ocplx) * box_size(&to));
  free(buf);
  free(nxt);
}

static void comp_offsets(int n, const int* dims, int64_t* off) {
  int64_t o = 0;
  for (int k = 0; k < n; ++k) {
    off[k] = o;
    box_t f = face_box(n, dims, k);
    o += box_size(&f);
  }
  off[n] = o;
}

void og_restrict(int n, const int* df, const ocplx* xf, ocplx* xc) {
  int dc[3] = {1, 1, 1};
  for (int a = 0; a < n; ++a) dc[a] = df[a] / 2;
  int64_t of[4], oc[4];
  comp_offsets(n, df, of);
  comp_offsets(n, dc, oc);
  for (int c = 0; c <= n; ++c) transfer_component(n, df, c, 1, xf + of[c], xc + oc[c]);
}

void og_prolong(int n, const int* df, const ocplx* xc, ocplx* xf) {
  int dc[3] = {1, 1, 1};
  for (int a = 0; a < n; ++a) dc[a] = df[a] / 2;
  int64_t of[4], oc[4];
  comp_offsets(n, df, of);
  comp_offsets(n, dc, oc);
  for (int c = 0; c <= n; ++c) transfer_component(n, df, c, 0, xc + oc[c], xf + of[c]);
}

/* ---------------------------------------------------------------- FGMRES */
static double vnorm(int64_t n, const ocplx* x) {
  double s = 0;
  for (int64_t i = 0; i < n; ++i) s += creal(x[i]) * creal(x[i]) + cimag(x[i]) * cimag(x[i]);
  return sqrt(s);
}
static ocplx vdot(int64_t n, const ocplx* x, const ocplx* y) {
  ocplx s = 0;
  for (int64_t i = 0; i < n; ++i) s += conj(x[i]) * y[i];
  return s;
}
static void vaxpy(int64_t n, ocplx a, const ocplx* x, ocplx* y) {
  for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}
static void vscal(int64_t n, ocplx a, ocplx* x) {
  for (int64_t i = 0; i < n; ++i) x[i] *= a;
}

typedef struct {
  double* v;
  int n, cap;
} dvec;
static void dpush(dvec* d, double x) {
  if (d->n == d->cap) {
    d->cap = d->cap ? 2 * d->cap : 64;
    d->v = (double*)realloc(d->v, sizeof(double) * d->cap);
  }
  d->v[d->n++] = x;
}

/* krylov.hpp:65 fgmres (right-preconditioned, restarted, flexible) */
void og_fgmres(int64_t n, og_apply_fn A, void* actx, og_apply_fn M, void* mctx, const ocplx* b,
               ocplx* x, const og_krylov_opts* opt, og_krylov_result* res) {
  dvec hist = {0};
  res->status = 1;
  res->iterations = 0;
  res->relres = 1.0;
  const double bnorm = vnorm(n, b);
  if (bnorm == 0.0) {
    vscal(n, 0, x);
    res->status = 0;
    res->relres = 0.0;
    res->history = NULL;
    res->n_history = 0;
    return;
  }
  const double target = opt->rtol * bnorm;
  const int m = opt->restart;
  ocplx* r = (ocplx*)malloc(sizeof(ocplx) * n);
  ocplx* w = (ocplx*)malloc(sizeof(ocplx) * n);
  memcpy(r, b, sizeof(ocplx) * n);
  A(actx, x, w);
  vaxpy(n, -1, w, r);
  double beta = vnorm(n, r);
  dpush(&hist, beta / bnorm);
  res->relres = beta / bnorm;
  ocplx** V = (ocplx**)calloc(m + 1, sizeof(ocplx*));
  ocplx** Z = (ocplx**)calloc(m, sizeof(ocplx*));
  ocplx* H = (ocplx*)calloc((size_t)(m + 1) * m, sizeof(ocplx));
#define HH(i, j) H[(size_t)(i) * m + (j)]
  double* gc = (double*)calloc(m, sizeof(double));
  ocplx* gs = (ocplx*)calloc(m, sizeof(ocplx));
  ocplx* g = (ocplx*)calloc(m + 1, sizeof(ocplx));
  ocplx* y = (ocplx*)calloc(m, sizeof(ocplx));
  for (int i = 0; i <= m; ++i) V[i] = (ocplx*)malloc(sizeof(ocplx) * n);
  for (int i = 0; i < m; ++i) Z[i] = (ocplx*)malloc(sizeof(ocplx) * n);
  if (beta <= target) {
    res->status = 0;
    goto done;
  }
  double prev_cycle = beta;
  int stall = 0;
  while (res->iterations < opt->max_iterations) {
    for (int64_t i = 0; i < n; ++i) V[0][i] = r[i] * (1.0 / beta);
    for (int i = 0; i <= m; ++i) g[i] = 0;
    g[0] = beta;
    int broke = 0, j = 0;
    while (j < m && res->iterations < opt->max_iterations) {
      M(mctx, V[j], Z[j]);
      A(actx, Z[j], w);
      const double wpre = vnorm(n, w);
      for (int i = 0; i <= j; ++i) {
        ocplx hij = vdot(n, V[i], w);
        vaxpy(n, -hij, V[i], w);
        HH(i, j) = hij;
      }
      double wn = vnorm(n, w);
      if (wn < 0.70710678 * wpre) {
        for (int i = 0; i <= j; ++i) {
          ocplx corr = vdot(n, V[i], w);
          vaxpy(n, -corr, V[i], w);
          HH(i, j) += corr;
        }
        wn = vnorm(n, w);
      }
      HH(j + 1, j) = wn;
      ++res->iterations;
      if (!(wn > 1e-14 * (wpre > 0 ? wpre : 1.0))) {
        broke = 1;
      } else {
        for (int64_t i = 0; i < n; ++i) V[j + 1][i] = w[i] * (1.0 / wn);
      }
      for (int i = 0; i < j; ++i) {
        const ocplx a = HH(i, j), bb = HH(i + 1, j);
        HH(i, j) = gc[i] * a + gs[i] * bb;
        HH(i + 1, j) = -conj(gs[i]) * a + gc[i] * bb;
      }
      const ocplx h1 = HH(j, j), h2 = HH(j + 1, j);
      const double t = sqrt(creal(h1 * conj(h1)) + creal(h2 * conj(h2)));
      if (t == 0.0) {
        gc[j] = 1.0;
        gs[j] = 0;
      } else if (cabs(h1) == 0.0) {
        gc[j] = 0.0;
        gs[j] = 1;
      } else {
        gc[j] = cabs(h1) / t;
        gs[j] = (h1 / cabs(h1)) * conj(h2) / t;
      }
      HH(j, j) = gc[j] * h1 + gs[j] * h2;
      HH(j + 1, j) = 0;
      const ocplx gj = g[j];
      g[j] = gc[j] * gj;
      g[j + 1] = -conj(gs[j]) * gj;
      const double est = cabs(g[j + 1]);
      dpush(&hist, est / bnorm);
      ++j;
      if (broke || est <= target) break;
    }
    for (int i = j - 1; i >= 0; --i) {
      ocplx v = g[i];
      for (int l = i + 1; l < j; ++l) v -= HH(i, l) * y[l];
      if (cabs(HH(i, i)) == 0.0) {
        res->status = 2;
        goto done;
      }
      y[i] = v / HH(i, i);
    }
    for (int i = 0; i < j; ++i) vaxpy(n, y[i], Z[i], x);
    memcpy(r, b, sizeof(ocplx) * n);
    A(actx, x, w);
    vaxpy(n, -1, w, r);
    beta = vnorm(n, r);
    res->relres = beta / bnorm;
    if (beta <= target) {
      res->status = 0;
      goto done;
    }
    if (broke) {
      res->status = 2;
      goto done;
    }
    if (beta > opt->stall_factor * prev_cycle) {
      if (++stall >= opt->stall_cycles) {
        res->status = 3;
        goto done;
      }
    } else {
      stall = 0;
    }
    prev_cycle = beta;
  }
  res->status = 1;
done:
#undef HH
  for (int i = 0; i <= m; ++i) free(V[i]);
  for (int i = 0; i < m; ++i) free(Z[i]);
  free(V);
  free(Z);
  free(H);
  free(gc);
  free(gs);
  free(g);
  free(y);
  free(r);
  free(w);
  res->history = hist.v;
  res->n_history = hist.n;
}

/* ------------------------------------------------------------- multigrid */
typedef struct {
  og_op* D;
  og_vanka* sm;
  int dims[3];
  int64_t n;
  ocplx *r, *t, *bc, *ec, *corr;
} lev_t;

struct og_mg {
  og_mg_opts opt;
  int nl, ndim;
  lev_t* L;
  ocplx* lu; /* dense LU of the coarsest operator, column-major */
  int* piv;
  int64_t nco;
};

static void lu_factor(int64_t n, ocplx* a, int* piv) {
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = cabs(a[k + k * n]);
    for (int64_t i = k + 1; i < n; ++i) {
      double v = cabs(a[i + k * n]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    piv[k] = (int)p;
    if (p != k)
      for (int64_t j = 0; j < n; ++j) {
        ocplx t = a[k + j * n];
        a[k + j * n] = a[p + j * n];
        a[p + j * n] = t;
      }
    ocplx d = a[k + k * n];
    for (int64_t i = k + 1; i < n; ++i) a[i + k * n] /= d;
    for (int64_t j = k + 1; j < n; ++j) {
      ocplx akj = a[k + j * n];
      if (akj == 0) continue;
      for (int64_t i = k + 1; i < n; ++i) a[i + j * n] -= a[i + k * n] * akj;
    }
  }
}
static void lu_solve(int64_t n, const ocplx* a, const int* piv, ocplx* b) {
  for (int64_t k = 0; k < n; ++k) {
    ocplx t = b[k];
    b[k] = b[piv[k]];
    b[piv[k]] = t;
  }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j + 1; i < n; ++i) b[i] -= a[i + j * n] * b[j];
  for (int64_t j = n - 1; j >= 0; --j) {
    b[j] /= a[j + j * n];
    for (int64_t i = 0; i < j; ++i) b[i] -= a[i + j * n] * b[j];
  }
}

/* multigrid.hpp:75 constructor (coarsest solved exactly, cf. :97 LU path) */
og_mg* og_mg_create(int n, const int* dims, double h, const double* lambda, const double* mu,
                    const double* rho, const double* gamma, double beta, double omega, double alpha,
                    const og_mg_opts* opt) {
  if (opt->n_levels < 2) return NULL;
  if (opt->cycle == 0 && opt->n_levels != 2) return NULL;
  og_mg* mg = (og_mg*)calloc(1, sizeof(og_mg));
  mg->opt = *opt;
  mg->nl = opt->n_levels;
  mg->ndim = n;
  mg->L = (lev_t*)calloc(mg->nl, sizeof(lev_t));
  int d[3] = {1, 1, 1};
  for (int a = 0; a < n; ++a) d[a] = dims[a];
  int64_t nc = og_n_cells(n, d);
  double* m[4];
  const double* src[4] = {lambda, mu, rho, gamma};
  for (int f = 0; f < 4; ++f) {
    m[f] = (double*)malloc(sizeof(double) * nc);
    memcpy(m[f], src[f], sizeof(double) * nc);
  }
  double hh = h;
  for (int l = 0; l < mg->nl; ++l) {
    lev_t* L = &mg->L[l];
    memcpy(L->dims, d, sizeof d);
    L->D = og_op_create(n, d, hh, m[0], m[1], m[2], m[3], beta, omega, alpha);
    L->sm = og_vanka_create(L->D, opt->vanka_mode);
    L->n = og_n_dofs(n, d);
    L->r = (ocplx*)calloc(L->n, sizeof(ocplx));
    L->t = (ocplx*)calloc(L->n, sizeof(ocplx));
    L->bc = (ocplx*)calloc(L->n, sizeof(ocplx));
    L->ec = (ocplx*)calloc(L->n, sizeof(ocplx));
    L->corr = (ocplx*)calloc(L->n, sizeof(ocplx));
    if (l + 1 < mg->nl) {
      for (int a = 0; a < n; ++a)
        if (d[a] % 2 != 0 || d[a] / 2 < 2) {
          og_mg_destroy(mg);
          for (int f = 0; f < 4; ++f) free(m[f]);
          return NULL;
        }
      int dc[3] = {1, 1, 1};
      for (int a = 0; a < n; ++a) dc[a] = d[a] / 2;
      int64_t ncc = og_n_cells(n, dc);
      for (int f = 0; f < 4; ++f) {
        double* w = (double*)malloc(sizeof(double) * ncc);
        og_coarsen_cell_field(n, d, m[f], w);
        free(m[f]);
        m[f] = w;
      }
      memcpy(d, dc, sizeof d);
      hh = 2.0 * hh;
    }
  }
  for (int f = 0; f < 4; ++f) free(m[f]);
  lev_t* cl = &mg->L[mg->nl - 1];
  mg->nco = cl->n;
  mg->lu = (ocplx*)malloc(sizeof(ocplx) * cl->n * cl->n);
  mg->piv = (int*)malloc(sizeof(int) * cl->n);
  og_assemble_dense(cl->D, mg->lu);
  lu_factor(cl->n, mg->lu, mg->piv);
  return mg;
}

void og_mg_destroy(og_mg* mg) {
  if (!mg) return;
  for (int l = 0; l < mg->nl; ++l) {
    lev_t* L = &mg->L[l];
    og_op_destroy(L->D);
    og_vanka_destroy(L->sm);
    free(L->r);
    free(L->t);
    free(L->bc);
    free(L->ec);
    free(L->corr);
  }
  free(mg->L);
  free(mg->lu);
  free(mg->piv);
  free(mg);
}

int og_mg_n_levels(const og_mg* mg) { return mg->nl; }
const og_op* og_mg_level_op(const og_mg* mg, int l) { return mg->L[l].D; }

static void cycle_at(og_mg* mg, int l, const ocplx* b, ocplx* x);

typedef struct {
  og_mg* mg;
  int l;
} kctx_t;
static void k_apply_A(void* p, const ocplx* in, ocplx* out) {
  kctx_t* c = (kctx_t*)p;
  og_apply(c->mg->L[c->l].D, in, out);
}
static void k_apply_M(void* p, const ocplx* in, ocplx* out) {
  kctx_t* c = (kctx_t*)p;
  memset(out, 0, sizeof(ocplx) * c->mg->L[c->l].n);
  cycle_at(c->mg, c->l, in, out);
}

/* multigrid.hpp:217 cycle_at */
static void cycle_at(og_mg* mg, int l, const ocplx* b, ocplx* x) {
  if (l + 1 == mg->nl) {
    memcpy(x, b, sizeof(ocplx) * mg->nco);
    lu_solve(mg->nco, mg->lu, mg->piv, x);
    return;
  }
  lev_t* lev = &mg->L[l];
  lev_t* nxt = &mg->L[l + 1];
  for (int s = 0; s < mg->opt.nu1; ++s)
    og_vanka_sweep(lev->sm, lev->D, b, x, mg->opt.damping, mg->opt.sweep);
  og_apply(lev->D, x, lev->t);
  for (int64_t i = 0; i < lev->n; ++i) lev->r[i] = b[i] - lev->t[i];
  og_restrict(mg->ndim, lev->dims, lev->r, nxt->bc);
  memset(nxt->ec, 0, sizeof(ocplx) * nxt->n);
  const int next_coarsest = (l + 2 == mg->nl);
  switch (mg->opt.cycle) {
    case 0:
    case 1:
      cycle_at(mg, l + 1, nxt->bc, nxt->ec);
      break;
    case 2:
      cycle_at(mg, l + 1, nxt->bc, nxt->ec);
      if (!next_coarsest) cycle_at(mg, l + 1, nxt->bc, nxt->ec);
      break;
    default:
      if (next_coarsest) {
        cycle_at(mg, l + 1, nxt->bc, nxt->ec);
      } else {
        og_krylov_opts ko = {mg->opt.k_inner_iterations, mg->opt.k_inner_iterations,
                             mg->opt.k_inner_rtol, 0.99, 2};
        kctx_t c = {mg, l + 1};
        og_krylov_result kr;
        og_fgmres(nxt->n, k_apply_A, &c, k_apply_M, &c, nxt->bc, nxt->ec, &ko, &kr);
        free(kr.history);
      }
      break;
  }
  og_prolong(mg->ndim, lev->dims, nxt->ec, lev->corr);
  vaxpy(lev->n, 1, lev->corr, x);
  for (int s = 0; s < mg->opt.nu2; ++s)
    og_vanka_sweep(lev->sm, lev->D, b, x, mg->opt.damping, mg->opt.sweep);
}

void og_mg_cycle(og_mg* mg, const ocplx* b, ocplx* x) { cycle_at(mg, 0, b, x); }
void og_mg_precondition(og_mg* mg, const ocplx* r, ocplx* z) {
  memset(z, 0, sizeof(ocplx) * mg->L[0].n);
  cycle_at(mg, 0, r, z);
}

typedef struct {
  const og_op* A0;
  og_mg* mg;
} sctx_t;
static void s_apply_A(void* p, const ocplx* in, ocplx* out) {
  og_apply(((sctx_t*)p)->A0, in, out);
}
static void s_apply_M(void* p, const ocplx* in, ocplx* out) {
  og_mg_precondition(((sctx_t*)p)->mg, in, out);
}

/* experiments.hpp:320 the double-precision solve loop */
void og_solve(og_mg* mg, const og_op* A0, const ocplx* b, ocplx* x, const og_krylov_opts* ko,
              og_krylov_result* res) {
  sctx_t c = {A0, mg};
  og_fgmres(A0->ndofs, s_apply_A, &c, s_apply_M, &c, b, x, ko, res);
}

/* ------------------------------------------------ layered + GRF media
 * BASELINE configs[1]/[3]/[4] media recipe (no reference implementation:
 * the BASELINE text specifies it; the layer layout follows layered_media,
 * experiments.hpp:78-111 -- tops on the last axis, index 0 at the top,
 * mu = rho vs^2). Restated step by step from the recipe documented in
 * paper_2307_03242_b200/csrc/ehmg_media.cuh, scalar loops, same operation
 * order (no FMA contraction: the Makefile passes -ffp-contract=off). */
static uint64_t or_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int og_layered_grf_media(int ndim, const int* dims, int n_layers, const double* ranges, double perturb,
                         double corr, double gamma_phys, uint64_t seed, double* lambda, double* mu,
                         double* rho, double* gamma) {
  int d[3] = {dims[0], dims[1], ndim == 3 ? dims[2] : 1};
  const int depth = d[ndim - 1];
  if (n_layers < 1 || n_layers > 64 || depth < 2) return -1;
  /* layer draws: splitmix64 stream */
  uint64_t st = seed;
#define OR_NEXT() (st += 0x9e3779b97f4a7c15ull, or_mix64(st))
  const int nl = n_layers < depth ? n_layers : depth;
  int tops[64], nt = 1;
  tops[0] = 0;
  while (nt < nl) {
    const int dd = 1 + (int)(OR_NEXT() % (uint64_t)(depth - 1));
    int seen = 0;
    for (int i = 0; i < nt; ++i) seen |= tops[i] == dd;
    if (!seen) tops[nt++] = dd;
  }
  for (int i = 1; i < nt; ++i) /* insertion sort */
    for (int j = i; j > 0 && tops[j - 1] > tops[j]; --j) {
      int t = tops[j];
      tops[j] = tops[j - 1];
      tops[j - 1] = t;
    }
  double lcs[64], lq[64], lr[64];
  for (int l = 0; l < nl; ++l) {
    lcs[l] = ranges[0] + (ranges[1] - ranges[0]) * ((double)(OR_NEXT() >> 11) * 0x1.0p-53);
    lq[l] = ranges[2] + (ranges[3] - ranges[2]) * ((double)(OR_NEXT() >> 11) * 0x1.0p-53);
    lr[l] = ranges[4] + (ranges[5] - ranges[4]) * ((double)(OR_NEXT() >> 11) * 0x1.0p-53);
  }
#undef OR_NEXT
  /* filter taps */
  const int R = (int)ceil(2.0 * corr);
  const double s = corr / 2.0;
  double ss = 0.0;
  for (int t = -R; t <= R; ++t) ss += exp(-(double)t * t / (s * s));
  const double nrm = 1.0 / sqrt(ss);
  double* w = (double*)malloc(sizeof(double) * (size_t)(2 * R + 1));
  for (int t = -R; t <= R; ++t) w[t + R] = exp(-(double)t * t / (2.0 * s * s)) * nrm;
  const int E0 = d[0] + 2 * R, E1 = d[1] + 2 * R, E2 = ndim == 3 ? d[2] + 2 * R : 1;
  const int64_t nc = (int64_t)d[0] * d[1] * d[2];
  double* noise = (double*)malloc(sizeof(double) * (size_t)E0 * E1 * E2);
  double* t1 = (double*)malloc(sizeof(double) * (size_t)d[0] * E1 * E2);
  double* t2 = (double*)malloc(sizeof(double) * (size_t)d[0] * d[1] * E2);
  double* g[3];
  const double s3 = 1.7320508075688772;
  for (int f = 0; f < 3; ++f) {
    g[f] = (double*)malloc(sizeof(double) * (size_t)nc);
    const uint64_t key = seed ^ (0x9e3779b97f4a7c15ull * (uint64_t)(f + 1));
    for (int64_t i = 0; i < (int64_t)E0 * E1 * E2; ++i) {
      const double u = (double)(or_mix64(key + (uint64_t)i) >> 11) * 0x1.0p-53;
      noise[i] = (u * 2.0 + -1.0) * s3;
    }
    /* axis 0: (E0, E1, E2) -> (d0, E1, E2) */
    for (int64_t z = 0; z < E2; ++z)
      for (int64_t y = 0; y < E1; ++y)
        for (int x = 0; x < d[0]; ++x) {
          const double* p = noise + x + (int64_t)E0 * (y + (int64_t)E1 * z);
          double acc = 0.0;
          for (int t = 0; t <= 2 * R; ++t) acc = acc + w[t] * p[t];
          t1[x + (int64_t)d[0] * (y + (int64_t)E1 * z)] = acc;
        }
    /* axis 1: (d0, E1, E2) -> (d0, d1, E2) */
    double* o1 = ndim == 3 ? t2 : g[f];
    for (int64_t z = 0; z < E2; ++z)
      for (int y = 0; y < d[1]; ++y)
        for (int x = 0; x < d[0]; ++x) {
          const double* p = t1 + x + (int64_t)d[0] * (y + (int64_t)E1 * z);
          double acc = 0.0;
          for (int t = 0; t <= 2 * R; ++t) acc = acc + w[t] * p[(int64_t)t * d[0]];
          o1[x + (int64_t)d[0] * (y + (int64_t)d[1] * z)] = acc;
        }
    if (ndim == 3) /* axis 2: (d0, d1, E2) -> (d0, d1, d2) */
      for (int z = 0; z < d[2]; ++z)
        for (int y = 0; y < d[1]; ++y)
          for (int x = 0; x < d[0]; ++x) {
            const double* p = t2 + x + (int64_t)d[0] * (y + (int64_t)d[1] * z);
            double acc = 0.0;
            for (int t = 0; t <= 2 * R; ++t) acc = acc + w[t] * p[(int64_t)t * d[0] * d[1]];
            g[f][x + (int64_t)d[0] * (y + (int64_t)d[1] * z)] = acc;
          }
  }
  const int64_t plane = ndim == 3 ? (int64_t)d[0] * d[1] : d[0];
  for (int64_t i = 0; i < nc; ++i) {
    const int z = (int)(i / plane);
    int j = 0;
    while (j + 1 < nl && tops[j + 1] <= z) ++j;
    double fct[3];
    for (int f = 0; f < 3; ++f) {
      const double gg = g[f][i];
      fct[f] = 1.0 + perturb * (gg / sqrt(1.0 + gg * gg));
    }
    const double cs = lcs[j] * fct[0], q = lq[j] * fct[1], r = lr[j] * fct[2];
    const double m = r * cs * cs;
    mu[i] = m;
    rho[i] = r;
    lambda[i] = m * (q * q + -2.0);
    gamma[i] = gamma_phys;
  }
  for (int f = 0; f < 3; ++f) free(g[f]);
  free(noise);
  free(t1);
  free(t2);
  free(w);
  return 0;
}
