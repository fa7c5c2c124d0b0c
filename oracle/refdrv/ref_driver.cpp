// ref_driver.cpp -- builds the REFERENCE's own matrix-free path into
// oracle/_ref/libehmg_ref.so (test infrastructure only).
//
// Compiled by oracle/Makefile directly against the unmodified headers under
// /root/reference/proj/include (grid, media, stencils, operator, vanka,
// transfer, krylov). Eigen is absent from this image, so shim/Eigen holds
// declaration-only forward declarations: the Eigen-typed templates (sparse
// assembly, SparseLU, Kaczmarz) are parsed but never instantiated. The
// multigrid cycle itself (multigrid.hpp:217 cycle_at) cannot be instantiated
// without Eigen's SparseLU, so it is restated here around the reference's
// own smoother/operator/transfer calls with an exact dense LU coarsest solve
// (the reference's CoarseSolverKind::lu semantics, multigrid.hpp:97).
//
// Nothing from this file ships in the product; tests/ and bench.py's
// reference arm load it to pin the oracle and time the reference CPU path.

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

// Expose VankaSmoother's factorization cache for exact cache parity checks.
#define private public
#include "ehmg/krylov.hpp"
#include "ehmg/operator.hpp"
#include "ehmg/transfer.hpp"
#include "ehmg/multigrid.hpp"  // convert_field (multigrid.hpp:311); Multigrid itself is not instantiated
#include "ehmg/vanka.hpp"
#undef private

using namespace ehmg;
using Cd = std::complex<double>;

namespace {

template <int Dim> Idx<Dim> to_idx(const int* d) {
  Idx<Dim> r{};
  for (int a = 0; a < Dim; ++a) r[a] = d[a];
  return r;
}

template <int Dim>
MediaModel<Dim> media_of(const StaggeredGrid<Dim>& g, const double* lam, const double* mu,
                         const double* rho, const double* gam) {
  MediaModel<Dim> m;
  size_t n = size_t(g.n_cells());
  m.lambda.assign(lam, lam + n);
  m.mu.assign(mu, mu + n);
  m.rho.assign(rho, rho + n);
  m.gamma.assign(gam, gam + n);
  return m;
}

template <int Dim> void load(FieldVector<double, Dim>& f, const Cd* src) {
  size_t o = 0;
  for (auto& c : f.comp)
    for (auto& z : c) z = src[o++];
}
template <int Dim> void store(const FieldVector<double, Dim>& f, Cd* dst) {
  size_t o = 0;
  for (auto& c : f.comp)
    for (auto& z : c) dst[o++] = z;
}

struct Media {
  const double *lam, *mu, *rho, *gam;
};

// ---- exact coarsest solve (dense LU on reference unit-probe rows) -------
template <class CT>
struct DenseLUT {
  using Cd = CT;
  std::int64_t n = 0;
  std::vector<Cd> a;  // column-major
  std::vector<std::int64_t> piv;
  void factor() {
    piv.resize(size_t(n));
    for (std::int64_t k = 0; k < n; ++k) {
      std::int64_t p = k;
      auto best = std::abs(a[size_t(k + k * n)]);
      for (std::int64_t i = k + 1; i < n; ++i)
        if (std::abs(a[size_t(i + k * n)]) > best) best = std::abs(a[size_t(i + k * n)]), p = i;
      piv[size_t(k)] = p;
      if (p != k)
        for (std::int64_t j = 0; j < n; ++j) std::swap(a[size_t(k + j * n)], a[size_t(p + j * n)]);
      Cd d = a[size_t(k + k * n)];
      for (std::int64_t i = k + 1; i < n; ++i) a[size_t(i + k * n)] /= d;
      for (std::int64_t j = k + 1; j < n; ++j) {
        Cd akj = a[size_t(k + j * n)];
        if (akj == Cd(0)) continue;
        for (std::int64_t i = k + 1; i < n; ++i) a[size_t(i + j * n)] -= a[size_t(i + k * n)] * akj;
      }
    }
  }
  void solve(std::vector<Cd>& b) const {
    for (std::int64_t k = 0; k < n; ++k) std::swap(b[size_t(k)], b[size_t(piv[size_t(k)])]);
    for (std::int64_t j = 0; j < n; ++j)
      for (std::int64_t i = j + 1; i < n; ++i) b[size_t(i)] -= a[size_t(i + j * n)] * b[size_t(j)];
    for (std::int64_t j = n - 1; j >= 0; --j) {
      b[size_t(j)] /= a[size_t(j + j * n)];
      for (std::int64_t i = 0; i < j; ++i) b[size_t(i)] -= a[size_t(i + j * n)] * b[size_t(j)];
    }
  }
};

using DenseLU = DenseLUT<Cd>;

// Every entry of the operator on the reference's unit-probe rows
// (UnitAcc, operator.hpp:212), fn(row, col, value) in the flatten() DOF order.
template <class Real, int Dim, class Fn> void for_each_entry(const OpData<Real, Dim>& D, Fn&& fn) {
  std::array<std::int64_t, Dim + 2> off{};
  for (int c = 0; c <= Dim; ++c)
    off[size_t(c) + 1] = off[size_t(c)] + (c < Dim ? D.faceb[size_t(c)].size() : D.cellb.size());
  for (int cc = 0; cc <= Dim; ++cc) {
    const Box<Dim>& cb = cc < Dim ? D.faceb[size_t(cc)] : D.cellb;
    for_each(cb, [&](const Idx<Dim>& ci) {
      std::int64_t col = off[size_t(cc)] + cb.lin(ci);
      UnitAcc<Real, Dim> acc{D, cc, ci};
      for (int rc = 0; rc <= Dim; ++rc) {
        const Box<Dim>& rb = rc < Dim ? D.faceb[size_t(rc)] : D.cellb;
        std::array<int, 3> lo{-2, -2, Dim == 3 ? -2 : 0}, hi{2, 2, Dim == 3 ? 2 : 0};
        for (int o2 = lo[2]; o2 <= hi[2]; ++o2)
          for (int o1 = lo[1]; o1 <= hi[1]; ++o1)
            for (int o0 = lo[0]; o0 <= hi[0]; ++o0) {
              Idx<Dim> r = ci;
              r[0] += o0;
              r[1] += o1;
              if constexpr (Dim == 3) r[2] += o2;
              if (!rb.contains(r)) continue;
              auto v = rc < Dim ? row_u(D, rc, r, acc) : row_p(D, r, acc);
              fn(off[size_t(rc)] + rb.lin(r), col, v);
            }
      }
    });
  }
}

// Banded LU with partial pivoting (the unblocked LAPACK gbtf2 scheme) on a
// DOF permutation that orders unknowns slice by slice along the longest axis,
// so the coarsest operators of the slab problems (criterion 5 of
// test_acceptance.cpp:212, 49K DOFs) factor in band storage instead of a
// dense n^2 array. Test infrastructure: same exact-solve semantics as the
// dense LU (CoarseSolverKind::lu, multigrid.hpp:97).
template <class CT>
struct BandLUT {
  std::int64_t n = 0, kl = 0, ku = 0, ld = 0;
  std::vector<CT> ab;  // A(i, j) at ab[(kl + ku + i - j) + j * ld]
  std::vector<std::int64_t> piv, perm;  // perm[new] = old DOF
  CT& at(std::int64_t i, std::int64_t j) { return ab[size_t((kl + ku + i - j) + j * ld)]; }
  const CT& at(std::int64_t i, std::int64_t j) const { return ab[size_t((kl + ku + i - j) + j * ld)]; }
  void factor() {
    piv.resize(size_t(n));
    for (std::int64_t k = 0; k < n; ++k) {
      const std::int64_t km = std::min(kl, n - 1 - k);
      std::int64_t p = k;
      auto best = std::abs(at(k, k));
      for (std::int64_t i = k + 1; i <= k + km; ++i)
        if (std::abs(at(i, k)) > best) best = std::abs(at(i, k)), p = i;
      piv[size_t(k)] = p;
      const std::int64_t ju = std::min(n - 1, k + kl + ku);
      if (p != k)
        for (std::int64_t j = k; j <= ju; ++j) std::swap(at(k, j), at(p, j));
      const CT d = at(k, k);
      for (std::int64_t i = k + 1; i <= k + km; ++i) at(i, k) /= d;
      for (std::int64_t j = k + 1; j <= ju; ++j) {
        const CT akj = at(k, j);
        if (akj == CT(0)) continue;
        for (std::int64_t i = k + 1; i <= k + km; ++i) at(i, j) -= at(i, k) * akj;
      }
    }
  }
  void solve(std::vector<CT>& v) const {
    std::vector<CT> b(static_cast<size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) b[size_t(i)] = v[size_t(perm[size_t(i)])];
    for (std::int64_t k = 0; k < n; ++k) {
      std::swap(b[size_t(k)], b[size_t(piv[size_t(k)])]);
      const std::int64_t km = std::min(kl, n - 1 - k);
      for (std::int64_t i = k + 1; i <= k + km; ++i) b[size_t(i)] -= at(i, k) * b[size_t(k)];
    }
    for (std::int64_t j = n - 1; j >= 0; --j) {
      b[size_t(j)] /= at(j, j);
      for (std::int64_t i = std::max<std::int64_t>(0, j - kl - ku); i < j; ++i) b[size_t(i)] -= at(i, j) * b[size_t(j)];
    }
    for (std::int64_t i = 0; i < n; ++i) v[size_t(perm[size_t(i)])] = b[size_t(i)];
  }
};

template <class CT> struct CoarseLUT {
  DenseLUT<CT> dense;
  BandLUT<CT> band;
  bool banded = false;
  void solve(std::vector<CT>& v) const {
    if (banded) band.solve(v);
    else dense.solve(v);
  }
};

// Real = float: the LU of the float operator in float arithmetic, as the
// reference's Multigrid<float> factors its float matrix (multigrid.hpp:97).
// Coarsest grids above kBandMin DOFs take the banded factorisation.
// (EHMG_REF_BAND_MIN overrides the threshold: the band path's own check.)
inline std::int64_t band_min() {
  const char* e = std::getenv("EHMG_REF_BAND_MIN");
  return e ? std::atoll(e) : 20000;
}
template <class Real, int Dim> CoarseLUT<std::complex<Real>> dense_lu(const OpData<Real, Dim>& D) {
  using Cd = std::complex<Real>;
  std::int64_t n = D.cellb.size();
  for (int c = 0; c < Dim; ++c) n += D.faceb[size_t(c)].size();
  CoarseLUT<Cd> out;
  if (n <= band_min()) {
    DenseLUT<Cd>& L = out.dense;
    L.n = n;
    L.a.assign(size_t(n * n), Cd(0));
    for_each_entry(D, [&](std::int64_t r, std::int64_t c, Cd v) { L.a[size_t(r + c * n)] = v; });
    L.factor();
    return out;
  }
  out.banded = true;
  BandLUT<Cd>& B = out.band;
  B.n = n;
  // slice key along the longest axis (faces of that axis sit half a cell
  // earlier), then the remaining axes from last to first, then component
  int ax = 0;
  for (int a = 1; a < Dim; ++a)
    if (D.grid.dims[a] > D.grid.dims[ax]) ax = a;
  struct Key {
    std::int64_t k[4];
    std::int64_t dof;
  };
  std::vector<Key> keys;
  keys.reserve(size_t(n));
  std::int64_t o = 0;
  for (int c = 0; c <= Dim; ++c) {
    const Box<Dim>& b = c < Dim ? D.faceb[size_t(c)] : D.cellb;
    for_each(b, [&](const Idx<Dim>& i) {
      Key key{{0, 0, 0, c}, o + b.lin(i)};
      key.k[0] = 2 * std::int64_t(i[ax]) - (c == ax ? 1 : 0);
      int q = 1;
      for (int a = Dim - 1; a >= 0; --a)
        if (a != ax) key.k[q++] = i[a];
      keys.push_back(key);
    });
    o += b.size();
  }
  std::sort(keys.begin(), keys.end(), [](const Key& x, const Key& y) {
    for (int q = 0; q < 4; ++q)
      if (x.k[q] != y.k[q]) return x.k[q] < y.k[q];
    return x.dof < y.dof;
  });
  B.perm.resize(size_t(n));
  std::vector<std::int64_t> inv(static_cast<size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) {
    B.perm[size_t(i)] = keys[size_t(i)].dof;
    inv[size_t(keys[size_t(i)].dof)] = i;
  }
  for_each_entry(D, [&](std::int64_t r, std::int64_t c, Cd v) {
    if (v == Cd(0)) return;
    const std::int64_t pr = inv[size_t(r)], pc = inv[size_t(c)];
    B.kl = std::max(B.kl, pr - pc);
    B.ku = std::max(B.ku, pc - pr);
  });
  B.ld = 2 * B.kl + B.ku + 1;
  B.ab.assign(size_t(B.ld * n), Cd(0));
  for_each_entry(D, [&](std::int64_t r, std::int64_t c, Cd v) {
    if (v == Cd(0)) return;
    B.at(inv[size_t(r)], inv[size_t(c)]) = v;
  });
  B.factor();
  return out;
}

// ---- restated cycle around the reference components --------------------
template <class Real, int Dim> struct RefMGT {
  using F = FieldVector<Real, Dim>;
  using Cd = std::complex<Real>;
  struct Lev {
    StaggeredGrid<Dim> g;
    OpData<Real, Dim> D;
    VankaSmoother<Real, Dim> sm;
    F r, t, bc, ec;
  };
  std::vector<std::unique_ptr<Lev>> L;
  CoarseLUT<Cd> lu;
  int cycle, nu1, nu2;
  int k_it = 2;          // MgOptions::k_inner_iterations default (multigrid.hpp:52)
  double k_rtol = 0.25;  // MgOptions::k_inner_rtol default
  double w;
  VankaMode mode;
  SweepOrder order;

  RefMGT(StaggeredGrid<Dim> g, MediaModel<Dim> m, OperatorParams par, int nl, int cyc, int n1,
        int n2, double w_, int vmode, int sweep)
      : cycle(cyc), nu1(n1), nu2(n2), w(w_), mode(vmode ? VankaMode::economic : VankaMode::full),
        order(sweep ? SweepOrder::red_black : SweepOrder::lexicographic) {
    for (int l = 0; l < nl; ++l) {
      auto lv = std::make_unique<Lev>(
          Lev{g, make_opdata<Real>(g, m, par), VankaSmoother<Real, Dim>(mode), F(g), F(g), F(g), F(g)});
      L.push_back(std::move(lv));
      if (l + 1 < nl) {
        m = coarsen_media(g, m);
        g = coarsen_grid(g);
      }
    }
    lu = dense_lu<Real, Dim>(L.back()->D);
  }
  void cyc(int l, const F& b, F& x) {
    const int nl = int(L.size());
    if (l + 1 == nl) {
      std::vector<Cd> v;
      for (auto& c : b.comp) v.insert(v.end(), c.begin(), c.end());
      lu.solve(v);
      size_t o = 0;
      for (auto& c : x.comp)
        for (auto& z : c) z = v[o++];
      return;
    }
    Lev& lev = *L[size_t(l)];
    Lev& nx = *L[size_t(l) + 1];
    for (int s = 0; s < nu1; ++s) lev.sm.sweep(lev.D, b, x, w, order);
    apply_mixed_operator(lev.D, x, lev.t);
    lev.r = b;
    axpy(Cd(-1), lev.t, lev.r);
    nx.bc = restrict_field(lev.g, nx.g, lev.r, false);
    nx.ec.set_zero();
    if (cycle == 3 && l + 2 != nl) {
      // K-cycle (multigrid.hpp:238-253): the coarse correction is an inner
      // FGMRES on the next level (the reference's own fgmres), preconditioned
      // by one cycle from zero
      KrylovOptions ko;
      ko.restart = k_it;
      ko.max_iterations = k_it;
      ko.rtol = k_rtol;
      auto A = [&](const F& in, F& out) { apply_mixed_operator(nx.D, in, out); };
      auto M = [&](const F& in, F& out) {
        out.set_zero();
        cyc(l + 1, in, out);
      };
      fgmres(A, M, nx.bc, nx.ec, ko);
    } else {
      cyc(l + 1, nx.bc, nx.ec);
      if (cycle == 2 && l + 2 != nl) cyc(l + 1, nx.bc, nx.ec);
    }
    F corr = prolong_field(lev.g, nx.g, nx.ec, false);
    axpy(Cd(1), corr, x);
    for (int s = 0; s < nu2; ++s) lev.sm.sweep(lev.D, b, x, w, order);
  }
};
template <int Dim> using RefMG = RefMGT<double, Dim>;

template <int Dim>
int apply_t(const int* dims, double h, Media M, double beta, double omega, double alpha,
            const Cd* x, Cd* y, int schur) {
  StaggeredGrid<Dim> g(to_idx<Dim>(dims), h);
  auto D = make_opdata<double, Dim>(g, media_of<Dim>(g, M.lam, M.mu, M.rho, M.gam),
                                    {beta, omega, alpha, false});
  FieldVector<double, Dim> X(g), Y(g);
  load(X, x);
  if (schur) schur_eliminate_pressure(D, X, Y);
  else apply_mixed_operator(D, X, Y);
  store(Y, y);
  return 0;
}

template <int Dim>
int vanka_t(const int* dims, double h, Media M, double beta, double omega, double alpha, int mode,
            int order, double w, int nsweeps, const Cd* b, Cd* x, Cd* cache_out) {
  StaggeredGrid<Dim> g(to_idx<Dim>(dims), h);
  auto D = make_opdata<double, Dim>(g, media_of<Dim>(g, M.lam, M.mu, M.rho, M.gam),
                                    {beta, omega, alpha, false});
  VankaSmoother<double, Dim> sm(mode ? VankaMode::economic : VankaMode::full);
  FieldVector<double, Dim> B(g), X(g);
  load(B, b);
  load(X, x);
  for (int s = 0; s < nsweeps; ++s)
    sm.sweep(D, B, X, w, order ? SweepOrder::red_black : SweepOrder::lexicographic);
  sm.ensure_cache(D);
  store(X, x);
  if (cache_out) std::copy(sm.cache_.begin(), sm.cache_.end(), cache_out);
  return 0;
}

template <int Dim> int transfer_t(const int* dims_f, int restricting, const Cd* in, Cd* out) {
  StaggeredGrid<Dim> gf(to_idx<Dim>(dims_f), 1.0);
  StaggeredGrid<Dim> gc = coarsen_grid(gf);
  FieldVector<double, Dim> xi(restricting ? gf : gc);
  load(xi, in);
  FieldVector<double, Dim> xo =
      restricting ? restrict_field(gf, gc, xi, false) : prolong_field(gf, gc, xi, false);
  store(xo, out);
  return 0;
}

template <int Dim> int coarsen_t(const int* dims_f, const double* in, double* out) {
  StaggeredGrid<Dim> gf(to_idx<Dim>(dims_f), 1.0);
  MediaModel<Dim> m = MediaModel<Dim>::homogeneous(gf, 1, 1, 1, 0);
  m.lambda.assign(in, in + gf.n_cells());
  auto mc = coarsen_media(gf, m);
  std::copy(mc.lambda.begin(), mc.lambda.end(), out);
  return 0;
}

template <int Dim>
int mg_t(const int* dims, double h, Media M, double beta, double omega, double alpha, int nl,
         int cyc, int nu1, int nu2, double w, int vmode, int sweep, int ncycles, const Cd* b, Cd* x,
         double* seconds) {
  StaggeredGrid<Dim> g(to_idx<Dim>(dims), h);
  RefMG<Dim> mg(g, media_of<Dim>(g, M.lam, M.mu, M.rho, M.gam), {beta, omega, alpha, false}, nl,
                cyc, nu1, nu2, w, vmode, sweep);
  for (auto& lv : mg.L) lv->sm.ensure_cache(lv->D);
  FieldVector<double, Dim> B(g), X(g);
  load(B, b);
  load(X, x);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < ncycles; ++i) mg.cyc(0, B, X);
  if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  store(X, x);
  return 0;
}

template <int Dim>
int solve_t(const int* dims, double h, Media M, double beta, double omega, double alpha, int nl,
            int cyc, int nu1, int nu2, double w, int vmode, int sweep, int restart, int max_it,
            double rtol, const Cd* b, Cd* x, int* iters, int* status, double* relres,
            double* hist, int hist_cap, int* n_hist, int mixed = 0) {
  StaggeredGrid<Dim> g(to_idx<Dim>(dims), h);
  auto media = media_of<Dim>(g, M.lam, M.mu, M.rho, M.gam);
  std::unique_ptr<RefMG<Dim>> mgd;
  std::unique_ptr<RefMGT<float, Dim>> mgf;
  if (mixed)
    mgf = std::make_unique<RefMGT<float, Dim>>(g, media, OperatorParams{beta, omega, alpha, false}, nl, cyc, nu1,
                                               nu2, w, vmode, sweep);
  else
    mgd = std::make_unique<RefMG<Dim>>(g, media, OperatorParams{beta, omega, alpha, false}, nl, cyc, nu1, nu2,
                                       w, vmode, sweep);
  FieldVector<float, Dim> rf(g), zf(g);
  auto D0 = make_opdata<double, Dim>(g, media, {beta, omega, 0.0, false});
  using F = FieldVector<double, Dim>;
  F B(g), X(g);
  load(B, b);
  load(X, x);
  KrylovOptions ko;
  ko.restart = restart;
  ko.max_iterations = max_it;
  ko.rtol = rtol;
  auto A = [&](const F& in, F& out) { apply_mixed_operator(D0, in, out); };
  // experiments.hpp:241 MixedPrecondition for mixed
  auto Mp = [&](const F& r, F& z) {
    if (mixed) {
      convert_field(r, rf);
      zf.set_zero();
      mgf->cyc(0, rf, zf);
      convert_field(zf, z);
    } else {
      z.set_zero();
      mgd->cyc(0, r, z);
    }
  };
  KrylovResult res = fgmres(A, Mp, B, X, ko);
  store(X, x);
  *iters = res.iterations;
  *status = int(res.status);
  *relres = res.relres;
  int nh = std::min<int>(hist_cap, int(res.history.size()));
  for (int i = 0; i < nh; ++i) hist[i] = res.history[size_t(i)];
  *n_hist = int(res.history.size());
  return 0;
}

// multigrid.hpp:143 measure_convergence_factor restated around the
// restated cycle (RefMGT::cyc) and the reference's apply/norm/scal.
template <class Real, int Dim>
int measure_t(const int* dims, double h, Media M, double beta, double omega, double alpha, int nl, int cyc,
              int nu1, int nu2, double w, int vmode, int sweep, std::uint64_t seed, int warmup, double tol,
              int max_cycles, int growth_limit, double* factor, int* cycles, int* diverged, double* hist,
              int hist_cap, int* n_hist) {
  StaggeredGrid<Dim> g(to_idx<Dim>(dims), h);
  auto media = media_of<Dim>(g, M.lam, M.mu, M.rho, M.gam);
  RefMGT<Real, Dim> mg(g, media, OperatorParams{beta, omega, alpha, false}, nl, cyc, nu1, nu2, w, vmode, sweep);
  using C = std::complex<Real>;
  auto& D = mg.L[0]->D;
  auto x = make_field(D), zero = make_field(D), t = make_field(D);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (auto& comp : x.comp)
    for (auto& v : comp) v = C(Real(dist(rng)), Real(dist(rng)));
  for (int i = 0; i < warmup; ++i) mg.cyc(0, zero, x);
  auto rnorm = [&]() {
    apply_mixed_operator(D, x, t);
    return norm(t);
  };
  double r0 = rnorm();
  *factor = 0.0;
  *cycles = 0;
  *diverged = 0;
  *n_hist = 0;
  if (r0 == 0.0) return 0;
  scal(C(Real(1.0 / r0)), x);
  std::vector<double> hs;
  double prev = 1.0;
  int growths = 0;
  while (*cycles < max_cycles) {
    mg.cyc(0, zero, x);
    ++*cycles;
    double rn = rnorm();
    hs.push_back(rn);
    if (rn > prev) {
      if (++growths >= growth_limit) {
        *diverged = 1;
        break;
      }
    } else {
      growths = 0;
    }
    prev = rn;
    if (rn < tol) break;
    if (!std::isfinite(rn) || rn > 1e12) {
      *diverged = 1;
      break;
    }
  }
  *factor = std::pow(hs.empty() ? 1.0 : hs.back(), 1.0 / std::max(1, *cycles));
  *n_hist = int(hs.size());
  for (int i = 0; i < std::min(hist_cap, int(hs.size())); ++i) hist[i] = hs[size_t(i)];
  return 0;
}

template <class F> int guard(F&& f) {
  try {
    return f();
  } catch (const std::exception&) {
    return -1;
  }
}

}  // namespace

extern "C" {

int ref_apply(int ndim, const int* dims, double h, const double* lam, const double* mu,
              const double* rho, const double* gam, double beta, double omega, double alpha,
              const Cd* x, Cd* y) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    return ndim == 2 ? apply_t<2>(dims, h, M, beta, omega, alpha, x, y, 0)
                     : apply_t<3>(dims, h, M, beta, omega, alpha, x, y, 0);
  });
}

int ref_schur_apply(int ndim, const int* dims, double h, const double* lam, const double* mu,
                    const double* rho, const double* gam, double beta, double omega, double alpha,
                    const Cd* x, Cd* y) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    return ndim == 2 ? apply_t<2>(dims, h, M, beta, omega, alpha, x, y, 1)
                     : apply_t<3>(dims, h, M, beta, omega, alpha, x, y, 1);
  });
}

int ref_vanka(int ndim, const int* dims, double h, const double* lam, const double* mu,
              const double* rho, const double* gam, double beta, double omega, double alpha,
              int mode, int order, double w, int nsweeps, const Cd* b, Cd* x, Cd* cache_out) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    return ndim == 2 ? vanka_t<2>(dims, h, M, beta, omega, alpha, mode, order, w, nsweeps, b, x, cache_out)
                     : vanka_t<3>(dims, h, M, beta, omega, alpha, mode, order, w, nsweeps, b, x, cache_out);
  });
}

int ref_transfer(int ndim, const int* dims_f, int restricting, const Cd* in, Cd* out) {
  return guard([&] {
    return ndim == 2 ? transfer_t<2>(dims_f, restricting, in, out)
                     : transfer_t<3>(dims_f, restricting, in, out);
  });
}

int ref_coarsen(int ndim, const int* dims_f, const double* in, double* out) {
  return guard([&] { return ndim == 2 ? coarsen_t<2>(dims_f, in, out) : coarsen_t<3>(dims_f, in, out); });
}

int ref_attenuation(int ndim, const int* dims, double gamma_phys, int L, double gamma_max,
                    int absorb_top, double* out) {
  return guard([&] {
    SpongeConfig s;
    s.layer_width = L;
    s.gamma_max = gamma_max;
    s.absorb_top = absorb_top != 0;
    std::vector<double> v;
    if (ndim == 2) v = build_attenuation_profile(StaggeredGrid<2>(to_idx<2>(dims), 1.0), gamma_phys, s);
    else v = build_attenuation_profile(StaggeredGrid<3>(to_idx<3>(dims), 1.0), gamma_phys, s);
    std::copy(v.begin(), v.end(), out);
    return 0;
  });
}

int ref_mg_cycles(int ndim, const int* dims, double h, const double* lam, const double* mu,
                  const double* rho, const double* gam, double beta, double omega, double alpha,
                  int nl, int cyc, int nu1, int nu2, double w, int vmode, int sweep, int ncycles,
                  const Cd* b, Cd* x, double* seconds) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    return ndim == 2 ? mg_t<2>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, ncycles, b, x, seconds)
                     : mg_t<3>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, ncycles, b, x, seconds);
  });
}

int ref_solve(int ndim, const int* dims, double h, const double* lam, const double* mu,
              const double* rho, const double* gam, double beta, double omega, double alpha, int nl,
              int cyc, int nu1, int nu2, double w, int vmode, int sweep, int restart, int max_it,
              double rtol, const Cd* b, Cd* x, int* iters, int* status, double* relres,
              double* hist, int hist_cap, int* n_hist) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    return ndim == 2 ? solve_t<2>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, restart, max_it, rtol, b, x, iters, status, relres, hist, hist_cap, n_hist)
                     : solve_t<3>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, restart, max_it, rtol, b, x, iters, status, relres, hist, hist_cap, n_hist);
  });
}

int ref_measure(int ndim, const int* dims, double h, const double* lam, const double* mu, const double* rho,
                const double* gam, double beta, double omega, double alpha, int nl, int cyc, int nu1, int nu2,
                double w, int vmode, int sweep, std::uint64_t seed, int warmup, double tol, int max_cycles,
                int growth_limit, int mixed, double* factor, int* cycles, int* diverged, double* hist,
                int hist_cap, int* n_hist) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    if (ndim == 2)
      return mixed ? measure_t<float, 2>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, seed, warmup, tol, max_cycles, growth_limit, factor, cycles, diverged, hist, hist_cap, n_hist)
                   : measure_t<double, 2>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, seed, warmup, tol, max_cycles, growth_limit, factor, cycles, diverged, hist, hist_cap, n_hist);
    return mixed ? measure_t<float, 3>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, seed, warmup, tol, max_cycles, growth_limit, factor, cycles, diverged, hist, hist_cap, n_hist)
                 : measure_t<double, 3>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, seed, warmup, tol, max_cycles, growth_limit, factor, cycles, diverged, hist, hist_cap, n_hist);
  });
}

// FGMRES in double around a complex64 hierarchy (precision "mixed")
int ref_solve_mixed(int ndim, const int* dims, double h, const double* lam, const double* mu,
                    const double* rho, const double* gam, double beta, double omega, double alpha, int nl,
                    int cyc, int nu1, int nu2, double w, int vmode, int sweep, int restart, int max_it,
                    double rtol, const Cd* b, Cd* x, int* iters, int* status, double* relres,
                    double* hist, int hist_cap, int* n_hist) {
  Media M{lam, mu, rho, gam};
  return guard([&] {
    return ndim == 2 ? solve_t<2>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, restart, max_it, rtol, b, x, iters, status, relres, hist, hist_cap, n_hist, 1)
                     : solve_t<3>(dims, h, M, beta, omega, alpha, nl, cyc, nu1, nu2, w, vmode, sweep, restart, max_it, rtol, b, x, iters, status, relres, hist, hist_cap, n_hist, 1);
  });
}

}  // extern "C"
