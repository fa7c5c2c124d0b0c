// ehmg_b200_adapter.hpp -- C++ adapter a reference maintainer adds next to
// the reference headers (proj/include/ehmg) to route its solve path to the
// B200 library through the C ABI in ehmg_b200.h.
//
// Reference types in, reference types out:
//   b200::Multigrid<Dim>  mirrors ehmg::Multigrid<double, Dim>
//                         (multigrid.hpp:70: ctor :75, cycle :133,
//                         precondition :136, n_levels, coarse_kind)
//   b200::Operator<Dim>   mirrors make_opdata + apply_mixed_operator
//                         (operator.hpp:76, :437)
//   b200::solve           mirrors fgmres(A, M, b, x, ko) as driven by
//                         experiments.hpp:313 (A = unshifted operator,
//                         M = one cycle of the shifted hierarchy)
// Errors keep the reference's exception types: EHMG_EINVAL ->
// std::invalid_argument, EHMG_ERANGE -> std::length_error (assemble.hpp:210),
// anything else -> std::runtime_error.
//
// Compiled against the reference headers by tests/test_adapter.py.
#pragma once

#include <algorithm>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ehmg/krylov.hpp"
#include "ehmg/multigrid.hpp"
#include "ehmg_b200.h"

namespace ehmg::b200 {

inline void check(int rc) {
  if (rc == EHMG_OK) return;
  const std::string msg = ehmg_last_error();
  if (rc == EHMG_EINVAL) throw std::invalid_argument(msg);
  if (rc == EHMG_ERANGE) throw std::length_error(msg);
  throw std::runtime_error(msg);
}

// FieldVector <-> one flat complex128 buffer in flatten() order (assemble.hpp:256)
template <int Dim> std::vector<std::complex<double>> flatten(const FieldVector<double, Dim>& f) {
  std::vector<std::complex<double>> out;
  for (const auto& c : f.comp) out.insert(out.end(), c.begin(), c.end());
  return out;
}
template <int Dim> void unflatten(const std::vector<std::complex<double>>& v, FieldVector<double, Dim>& f) {
  size_t o = 0;
  for (auto& c : f.comp)
    for (auto& z : c) z = v[o++];
}

inline ehmg_mg_options to_c(const MgOptions& mo) {
  ehmg_mg_options o{};
  o.n_levels = mo.n_levels;
  o.cycle = int(mo.cycle);            // two_grid, v, w, k
  o.nu1 = mo.nu1;
  o.nu2 = mo.nu2;
  o.damping = mo.damping;
  o.vanka_mode = int(mo.vanka_mode);  // full, economic
  o.sweep = int(mo.sweep);            // lexicographic, red_black
  o.k_inner_iterations = mo.k_inner_iterations;
  o.k_inner_rtol = mo.k_inner_rtol;
  o.precision = 0;
  o.coarse = int(mo.coarse);          // automatic, lu, kaczmarz
  o.lu_dof_budget = mo.lu_dof_budget;
  o.kz_sweeps_per_apply = mo.kz_sweeps_per_apply;
  o.kz_damping = mo.kz_damping;
  o.kz_rtol = mo.kz_rtol;
  o.kz_max_iterations = mo.kz_max_iterations;
  o.kz_restart = mo.kz_restart;
  return o;
}

template <int Dim> class Operator {
 public:
  Operator(const StaggeredGrid<Dim>& g, const MediaModel<Dim>& m, const OperatorParams& par) {
    if (par.periodic) throw std::invalid_argument("b200: periodic operators are LFA-probe only");
    m.validate(g);
    check(ehmg_op_create(Dim, g.dims.data(), g.h, m.lambda.data(), m.mu.data(), m.rho.data(),
                         m.gamma.data(), par.beta, par.omega, par.alpha, &h_));
  }
  ~Operator() { ehmg_op_destroy(h_); }
  Operator(const Operator&) = delete;
  Operator& operator=(const Operator&) = delete;
  void apply(const FieldVector<double, Dim>& x, FieldVector<double, Dim>& y) const {
    auto xf = flatten(x), yf = xf;
    check(ehmg_apply_mixed_operator(h_, reinterpret_cast<const double*>(xf.data()),
                                    reinterpret_cast<double*>(yf.data()), EHMG_HOST));
    unflatten(yf, y);
  }
  ehmg_op handle() const { return h_; }

 private:
  ehmg_op h_ = nullptr;
};

template <int Dim> class Multigrid {
 public:
  Multigrid(const StaggeredGrid<Dim>& g, const MediaModel<Dim>& m, const OperatorParams& par,
            const MgOptions& mo)
      : opt_(mo) {
    if (par.periodic) throw std::invalid_argument("b200: periodic hierarchies are LFA-probe only");
    m.validate(g);
    const ehmg_mg_options o = to_c(mo);
    check(ehmg_multigrid_create(Dim, g.dims.data(), g.h, m.lambda.data(), m.mu.data(), m.rho.data(),
                                m.gamma.data(), par.beta, par.omega, par.alpha, &o, &h_));
  }
  ~Multigrid() { ehmg_multigrid_destroy(h_); }
  Multigrid(const Multigrid&) = delete;
  Multigrid& operator=(const Multigrid&) = delete;

  int n_levels() const { return ehmg_multigrid_n_levels(h_); }
  const MgOptions& options() const { return opt_; }
  CoarseSolverKind coarse_kind() const { return CoarseSolverKind::lu; }
  bool coarse_exact() const { return true; }

  void cycle(const FieldVector<double, Dim>& b, FieldVector<double, Dim>& x) {
    auto bf = flatten(b), xf = flatten(x);
    check(ehmg_multigrid_cycle(h_, reinterpret_cast<const double*>(bf.data()),
                               reinterpret_cast<double*>(xf.data()), EHMG_HOST));
    unflatten(xf, x);
  }
  void precondition(const FieldVector<double, Dim>& r, FieldVector<double, Dim>& z) {
    auto rf = flatten(r), zf = rf;
    check(ehmg_multigrid_precondition(h_, reinterpret_cast<const double*>(rf.data()),
                                      reinterpret_cast<double*>(zf.data()), EHMG_HOST));
    unflatten(zf, z);
  }
  ehmg_mg handle() const { return h_; }

 private:
  MgOptions opt_;
  ehmg_mg h_ = nullptr;
};

// fgmres(A, M, b, x, ko) of experiments.hpp:313 on the B200 path. `shifted`
// carries the preconditioner's alpha; A is the same operator with alpha = 0.
// orthogonalization: 0 = classical Gram-Schmidt passes (B200 default),
// 1 = the reference's MGS order (krylov.hpp:115).
template <int Dim>
KrylovResult solve(const StaggeredGrid<Dim>& g, const MediaModel<Dim>& m, const OperatorParams& shifted,
                   const MgOptions& mo, const FieldVector<double, Dim>& b, FieldVector<double, Dim>& x,
                   const KrylovOptions& ko, int orthogonalization = 0) {
  OperatorParams phys = shifted;
  phys.alpha = 0.0;
  Operator<Dim> A(g, m, phys);
  Multigrid<Dim> M(g, m, shifted, mo);
  auto bf = flatten(b), xf = flatten(x);
  ehmg_krylov_options k{ko.restart, ko.max_iterations, ko.rtol, ko.stall_factor, ko.stall_cycles,
                        orthogonalization};
  ehmg_krylov_result r{};
  std::vector<double> hist(size_t(ko.max_iterations) + size_t(ko.max_iterations / std::max(1, ko.restart)) + 8);
  check(ehmg_fgmres_solve(A.handle(), M.handle(), reinterpret_cast<const double*>(bf.data()),
                          reinterpret_cast<double*>(xf.data()), EHMG_HOST, &k, &r, hist.data(),
                          int(hist.size())));
  unflatten(xf, x);
  KrylovResult out;
  out.status = KrylovStatus(r.status);  // converged, max_iterations, breakdown, stalled
  out.iterations = r.iterations;
  out.relres = r.relres;
  out.history.assign(hist.begin(), hist.begin() + std::min<size_t>(size_t(r.n_history), hist.size()));
  return out;
}

}  // namespace ehmg::b200
