// ehmg_core.cuh -- geometry, complex arithmetic and the generic row
// evaluation of the staggered mixed elastic-Helmholtz operator.
//
// The generic rows follow the reference's row kernels term by term
// (operator.hpp:267-421) and are templated on an accessor, so the same code
// evaluates rows on a resident field (setup-free paths, small levels) and on
// unit probes (Vanka factorisation and coarsest-operator assembly, as in
// vanka.hpp:85 and assemble.hpp). The bandwidth-tuned fine-level kernels
// live in ehmg_stencil3d.cuh and are checked against these rows.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define EH_HD __host__ __device__ __forceinline__

namespace ehmg {

// ---------------------------------------------------------------- complex
typedef double2 cplx;

EH_HD cplx mk(double r, double i) { return make_double2(r, i); }
EH_HD cplx operator+(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
EH_HD cplx operator-(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
EH_HD cplx operator-(cplx a) { return mk(-a.x, -a.y); }
EH_HD cplx operator*(double s, cplx a) { return mk(s * a.x, s * a.y); }
EH_HD cplx operator*(cplx a, double s) { return mk(a.x * s, a.y * s); }
EH_HD cplx operator*(cplx a, cplx b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
EH_HD cplx& operator+=(cplx& a, cplx b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}
EH_HD cplx& operator-=(cplx& a, cplx b) {
  a.x -= b.x;
  a.y -= b.y;
  return a;
}
EH_HD cplx conj(cplx a) { return mk(a.x, -a.y); }
EH_HD double abs2(cplx a) { return a.x * a.x + a.y * a.y; }
// Smith-free division matching std::complex<double> for finite operands
// closely enough for 1e-12 parity (the divisions only appear in setup).
EH_HD cplx cdiv(cplx a, cplx b) {
  double d = b.x * b.x + b.y * b.y;
  return mk((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// complex64 fields of the single-precision hierarchy (experiments.hpp:241
// MixedPrecondition): same operations on float2.
typedef float2 cplxf;
EH_HD cplxf mkf(float r, float i) { return make_float2(r, i); }
#if defined(__CUDA_ARCH__)
// Blackwell packed FP32 pairs (FADD2 / FMUL2 / FFMA2): one instruction per
// complex64 add or real scale, two per complex product.
__device__ __forceinline__ unsigned long long f2pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ cplxf f2up(unsigned long long r) {
  cplxf o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ cplxf f2add(cplxf a, cplxf b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a.x, a.y)), "l"(f2pk(b.x, b.y)));
  return f2up(r);
}
__device__ __forceinline__ cplxf f2sub(cplxf a, cplxf b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a.x, a.y)), "l"(f2pk(b.x, b.y)));
  return f2up(r);
}
__device__ __forceinline__ cplxf f2scale(float s, cplxf a) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(s, s)), "l"(f2pk(a.x, a.y)));
  return f2up(r);
}
__device__ __forceinline__ cplxf f2mul(cplxf a, cplxf b) {
  unsigned long long t, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2pk(a.x, a.x)), "l"(f2pk(b.x, b.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2pk(-a.y, a.y)), "l"(f2pk(b.y, b.x)), "l"(t));
  return f2up(r);
}
EH_HD cplxf operator+(cplxf a, cplxf b) { return f2add(a, b); }
EH_HD cplxf operator-(cplxf a, cplxf b) { return f2sub(a, b); }
EH_HD cplxf operator*(float s, cplxf a) { return f2scale(s, a); }
EH_HD cplxf operator*(cplxf a, float s) { return f2scale(s, a); }
EH_HD cplxf operator*(cplxf a, cplxf b) { return f2mul(a, b); }
#else
EH_HD cplxf operator+(cplxf a, cplxf b) { return mkf(a.x + b.x, a.y + b.y); }
EH_HD cplxf operator-(cplxf a, cplxf b) { return mkf(a.x - b.x, a.y - b.y); }
EH_HD cplxf operator*(float s, cplxf a) { return mkf(s * a.x, s * a.y); }
EH_HD cplxf operator*(cplxf a, float s) { return mkf(a.x * s, a.y * s); }
EH_HD cplxf operator*(cplxf a, cplxf b) { return mkf(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
#endif
EH_HD cplxf operator-(cplxf a) { return mkf(-a.x, -a.y); }
EH_HD cplxf& operator+=(cplxf& a, cplxf b) {
  a = a + b;
  return a;
}
EH_HD cplxf& operator-=(cplxf& a, cplxf b) {
  a = a - b;
  return a;
}

// Field element traits: V = cplx (complex128) or cplxf (complex64).
template <class V> struct VT;
template <> struct VT<cplx> {
  typedef double R;
  EH_HD static cplx mk(double r, double i) { return make_double2(r, i); }
};
template <> struct VT<cplxf> {
  typedef float R;
  EH_HD static cplxf mk(float r, float i) { return make_float2(r, i); }
};
// widen to complex128 / narrow from complex128 (identity for cplx)
EH_HD cplx wide(cplx a) { return a; }
EH_HD cplx wide(cplxf a) { return make_double2((double)a.x, (double)a.y); }
template <class V> EH_HD V narrow(cplx a);
template <> EH_HD cplx narrow<cplx>(cplx a) { return a; }
template <> EH_HD cplxf narrow<cplxf>(cplx a) { return make_float2((float)a.x, (float)a.y); }

// --------------------------------------------------------------- geometry
// One level of the staggered grid (grid.hpp:64). 2D grids carry n[2] = 1.
// A z-slab window of a global grid stores cell planes [zoff, zoff + n[2])
// (and u2 faces [zoff, zoff + n[2]]); n/off/ndofs describe the local
// storage, gn2 the global plane count that decides boundary semantics.
struct Geo {
  int nd;
  int n[3];
  double h, inv_h;
  int64_t off[4];
  int64_t ndofs, ncells;
  int zoff, gn2;

  EH_HD int fdim(int k, int a) const { return n[a] + (a == k ? 1 : 0); }
  EH_HD bool face_ok(int k, const int* f) const {
    for (int a = 0; a < 3; ++a)
      if (f[a] < 0 || f[a] >= fdim(k, a)) return false;
    return true;
  }
  EH_HD bool cell_ok(const int* c) const {
    return c[0] >= 0 && c[0] < n[0] && c[1] >= 0 && c[1] < n[1] && c[2] >= 0 && c[2] < n[2];
  }
  EH_HD int64_t flin(int k, const int* f) const {
    return f[0] + (int64_t)fdim(k, 0) * (f[1] + (int64_t)fdim(k, 1) * f[2]);
  }
  EH_HD int64_t clin(const int* c) const {
    return c[0] + (int64_t)n[0] * (c[1] + (int64_t)n[1] * c[2]);
  }
  // Position of flat DOF r: component (nd = pressure) and index.
  EH_HD int unlin(int64_t r, int* i) const {
    int comp = nd;
    for (int k = 0; k < nd; ++k)
      if (r < off[k + 1]) {
        comp = k;
        break;
      }
    int64_t q = r - off[comp];
    int d0 = comp < nd ? fdim(comp, 0) : n[0];
    int d1 = comp < nd ? fdim(comp, 1) : n[1];
    i[0] = (int)(q % d0);
    q /= d0;
    i[1] = (int)(q % d1);
    i[2] = (int)(q / d1);
    return comp;
  }
};

inline Geo make_geo(int nd, const int* dims, double h) {
  Geo g;
  g.nd = nd;
  for (int a = 0; a < 3; ++a) g.n[a] = a < nd ? dims[a] : 1;
  g.h = h;
  g.inv_h = 1.0 / h;
  int64_t o = 0;
  for (int k = 0; k < nd; ++k) {
    g.off[k] = o;
    int64_t s = 1;
    for (int a = 0; a < 3; ++a) s *= g.fdim(k, a);
    o += s;
  }
  g.off[nd] = o;
  for (int k = nd + 1; k < 4; ++k) g.off[k] = o;
  g.ncells = (int64_t)g.n[0] * g.n[1] * g.n[2];
  g.ndofs = o + g.ncells;
  g.zoff = 0;
  g.gn2 = g.n[2];
  return g;
}

// Local geometry of the cell-plane window [z0, z1) of a global 3D grid.
inline Geo make_window(const Geo& G, int z0, int z1) {
  int d[3] = {G.n[0], G.n[1], z1 - z0};
  Geo w = make_geo(G.nd, d, G.h);
  w.zoff = z0;
  w.gn2 = G.gn2;
  return w;
}

// Operator parameters (operator.hpp:27 OperatorParams). The attenuation
// shift alpha enters only the face mass diagonal.
struct OpPar {
  double beta, omega2, alpha;
};

// Cell media packed for one 32-byte load: {mu, rho, gamma, 1/(lambda+mu)}.
typedef double4 Cell;

EH_HD void sh(const int* i, int axis, int d, int* o) {
  o[0] = i[0];
  o[1] = i[1];
  o[2] = i[2];
  o[axis] += d;
}

// ---------------------------------------------------------------- accessors
// Reads a resident field of element type V, widened to complex128 (the
// generic rows always evaluate in double).
template <class V>
struct FieldAccT {
  const V* x;
  EH_HD cplx u(const Geo& g, int k, const int* f) const {
    return g.face_ok(k, f) ? wide(x[g.off[k] + g.flin(k, f)]) : mk(0, 0);
  }
  EH_HD cplx p(const Geo& g, const int* c) const {
    return g.cell_ok(c) ? wide(x[g.off[g.nd] + g.clin(c)]) : mk(0, 0);
  }
};
typedef FieldAccT<cplx> FieldAcc;

struct UnitAcc {  // operator.hpp:212 UnitAcc
  int comp;
  int at[3];
  EH_HD cplx u(const Geo& g, int k, const int* f) const {
    return (k == comp && f[0] == at[0] && f[1] == at[1] && f[2] == at[2] && g.face_ok(k, f))
               ? mk(1, 0)
               : mk(0, 0);
  }
  EH_HD cplx p(const Geo& g, const int* c) const {
    return (comp == g.nd && c[0] == at[0] && c[1] == at[1] && c[2] == at[2] && g.cell_ok(c))
               ? mk(1, 0)
               : mk(0, 0);
  }
};

// ------------------------------------------------------ media averaging
// mu on the edge staggered in (a,b): mean of in-range cells (operator.hpp:108)
EH_HD double mu_edge(const Geo& g, const Cell* m, int a, int b, const int* e) {
  double s = 0;
  int cnt = 0;
  for (int da = -1; da <= 0; ++da)
    for (int db = -1; db <= 0; ++db) {
      int c[3] = {e[0], e[1], e[2]};
      c[a] += da;
      c[b] += db;
      if (g.cell_ok(c)) {
        s += m[g.clin(c)].x;
        ++cnt;
      }
    }
  return s / cnt;
}
// face mass diagonal omega^2 (1 - i(gamma+alpha)) rho (operator.hpp:132)
EH_HD cplx mass_diag(const Geo& g, const Cell* m, const OpPar& P, int k, const int* f) {
  double sr = 0, sg = 0;
  int cnt = 0;
  for (int d = -1; d <= 0; ++d) {
    int c[3] = {f[0], f[1], f[2]};
    c[k] += d;
    if (g.cell_ok(c)) {
      Cell q = m[g.clin(c)];
      sr += q.y;
      sg += q.z;
      ++cnt;
    }
  }
  double rho_f = sr / cnt, gam_f = sg / cnt + P.alpha;
  return mk(P.omega2 * rho_f, -P.omega2 * gam_f * rho_f);
}

// ------------------------------------------------------------ generic rows
// operator.hpp:267 dspread_cell
template <int ND, class Acc>
EH_HD cplx dspread_cell(const Geo& g, const OpPar& P, int k, const int* c, const Acc& A) {
  const double beta = P.beta;
  auto pair = [&](const int* b) {
    int q[3];
    sh(b, k, 1, q);
    return A.u(g, k, q) - A.u(g, k, b);
  };
  cplx v = beta * pair(c);
  if (beta != 1.0) {
    double wsum = beta;
    if (ND == 2) {
      const int t = 1 - k;
      const double w = (1.0 - beta) / 4.0;
      for (int st = -1; st <= 1; ++st) {
        int ct = c[t] + st;
        if (ct < 0 || ct >= g.fdim(k, t)) continue;
        const double wt = w * (double)(st == 0 ? 2 : 1);
        int b[3];
        sh(c, t, st, b);
        v += wt * pair(b);
        wsum += wt;
      }
    } else {
      const int t1 = (k + 1) % 3, t2 = (k + 2) % 3;
      const double w = (1.0 - beta) / 16.0;
      for (int s1 = -1; s1 <= 1; ++s1)
        for (int s2 = -1; s2 <= 1; ++s2) {
          int c1 = c[t1] + s1, c2 = c[t2] + s2;
          if (c1 < 0 || c1 >= g.fdim(k, t1) || c2 < 0 || c2 >= g.fdim(k, t2)) continue;
          int b1[3], b[3];
          sh(c, t1, s1, b1);
          sh(b1, t2, s2, b);
          const double wt = w * (double)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
          v += wt * pair(b);
          wsum += wt;
        }
    }
    v = v * (1.0 / wsum);
  }
  return v * g.inv_h;
}

// operator.hpp:306 dspread_edge
template <int ND, class Acc>
EH_HD cplx dspread_edge(const Geo& g, const OpPar& P, int k, int j, const int* e, const Acc& A) {
  const double beta = P.beta;
  auto pair = [&](const int* b) {
    int q[3];
    sh(b, j, -1, q);
    return A.u(g, k, b) - A.u(g, k, q);
  };
  cplx v = beta * pair(e);
  if (beta != 1.0) {
    double wsum = beta;
    if (ND == 2) {
      const int t = k;
      const double w = (1.0 - beta) / 4.0;
      for (int st = -1; st <= 1; ++st) {
        int ct = e[t] + st;
        if (ct < 0 || ct >= g.fdim(k, t)) continue;
        const double wt = w * (double)(st == 0 ? 2 : 1);
        int b[3];
        sh(e, t, st, b);
        v += wt * pair(b);
        wsum += wt;
      }
    } else {
      const int t1 = 3 - k - j, t2 = k;
      const double w = (1.0 - beta) / 16.0;
      for (int s1 = -1; s1 <= 1; ++s1)
        for (int s2 = -1; s2 <= 1; ++s2) {
          int c1 = e[t1] + s1, c2 = e[t2] + s2;
          if (c1 < 0 || c1 >= g.fdim(k, t1) || c2 < 0 || c2 >= g.fdim(k, t2)) continue;
          int b1[3], b[3];
          sh(e, t1, s1, b1);
          sh(b1, t2, s2, b);
          const double wt = w * (double)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
          v += wt * pair(b);
          wsum += wt;
        }
    }
    v = v * (1.0 / wsum);
  }
  return v * g.inv_h;
}

// operator.hpp:359 mass_eval
template <int ND, class Acc>
EH_HD cplx mass_eval(const Geo& g, const Cell* m, const OpPar& P, int k, const int* f,
                     const Acc& A) {
  const double beta = P.beta;
  cplx v = beta * (mass_diag(g, m, P, k, f) * A.u(g, k, f));
  if (beta == 1.0) return v;
  const double wn = (1.0 - beta) / (2 * ND);
  double wsum = beta;
  for (int a = 0; a < ND; ++a)
    for (int sg = -1; sg <= 1; sg += 2) {
      int fn[3];
      sh(f, a, sg, fn);
      if (g.face_ok(k, fn)) {
        v += wn * (mass_diag(g, m, P, k, fn) * A.u(g, k, fn));
        wsum += wn;
      }
    }
  return v * (1.0 / wsum);
}

// operator.hpp:389 row_u_acoustic
template <int ND, class Acc>
EH_HD cplx row_u_acoustic(const Geo& g, const Cell* m, const OpPar& P, int k, const int* f,
                          const Acc& A) {
  cplx out = mk(0, 0);
  for (int j = 0; j < ND; ++j) {
    cplx wm, wp;
    if (j == k) {
      int cm[3];
      sh(f, k, -1, cm);
      wm = g.cell_ok(cm) ? m[g.clin(cm)].x * dspread_cell<ND>(g, P, k, cm, A) : mk(0, 0);
      wp = g.cell_ok(f) ? m[g.clin(f)].x * dspread_cell<ND>(g, P, k, f, A) : mk(0, 0);
    } else {
      int ep[3];
      sh(f, j, 1, ep);
      wm = mu_edge(g, m, k, j, f) * dspread_edge<ND>(g, P, k, j, f, A);
      wp = mu_edge(g, m, k, j, ep) * dspread_edge<ND>(g, P, k, j, ep, A);
    }
    out += (wm - wp) * g.inv_h;
  }
  out -= mass_eval<ND>(g, m, P, k, f, A);
  return out;
}

// operator.hpp:409 row_u
template <int ND, class Acc>
EH_HD cplx row_u(const Geo& g, const Cell* m, const OpPar& P, int k, const int* f, const Acc& A) {
  cplx out = row_u_acoustic<ND>(g, m, P, k, f, A);
  int cm[3];
  sh(f, k, -1, cm);
  out += (A.p(g, f) - A.p(g, cm)) * g.inv_h;
  return out;
}

// operator.hpp:416 row_p
template <int ND, class Acc>
EH_HD cplx row_p(const Geo& g, const Cell* m, const OpPar& P, const int* c, const Acc& A) {
  cplx out = mk(0, 0);
  for (int k = 0; k < ND; ++k) out += dspread_cell<ND>(g, P, k, c, A);
  out += m[g.clin(c)].w * A.p(g, c);
  return out;
}

template <int ND, class Acc>
EH_HD cplx row_any(const Geo& g, const Cell* m, const OpPar& P, int comp, const int* i,
                   const Acc& A) {
  return comp < ND ? row_u<ND>(g, m, P, comp, i, A) : row_p<ND>(g, m, P, i, A);
}

}  // namespace ehmg
