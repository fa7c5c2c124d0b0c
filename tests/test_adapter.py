"""CPU: the C++ adapter of INTEGRATION.md (include/ehmg_b200_adapter.hpp)
compiles against the reference's own headers (/root/reference/proj/include,
with the declaration-only Eigen shim of oracle/refdrv) and links against the
B200 library; its calls map the C ABI's errors onto the reference's
exception types. Without a GPU the solve fails loudly (no CPU fallback)."""
import os
import subprocess

import pytest

from paper_2307_03242_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"

PROGRAM = r"""
#include <cstdio>
#include <cstring>
#include "ehmg_b200_adapter.hpp"
using namespace ehmg;
int main(int argc, char** argv) {
  StaggeredGrid<2> g;
  g.dims = {16, 16};
  g.h = 1.0 / 16;
  MediaModel<2> m;
  const size_t n = 16 * 16;
  m.lambda.assign(n, 2.0); m.mu.assign(n, 1.0); m.rho.assign(n, 1.0); m.gamma.assign(n, 0.01);
  OperatorParams par; par.beta = 2.0 / 3.0; par.omega = 2 * 3.141592653589793 * 16 / 10; par.alpha = 0.5;
  MgOptions mo; mo.n_levels = 2; mo.nu1 = mo.nu2 = 2; mo.damping = 0.55;
  mo.vanka_mode = VankaMode::full; mo.sweep = SweepOrder::red_black;
  const char* what = argc > 1 ? argv[1] : "solve";
  try {
    if (!std::strcmp(what, "kaczmarz")) {
      mo.coarse = CoarseSolverKind::kaczmarz;
      b200::Multigrid<2> M(g, m, par, mo);
    } else if (!std::strcmp(what, "budget")) {
      mo.coarse = CoarseSolverKind::lu;
      mo.lu_dof_budget = 100;
      b200::Multigrid<2> M(g, m, par, mo);
    } else {
      FieldVector<double, 2> b, x;
      b.comp[0].assign(17 * 16, 0.0); b.comp[1].assign(16 * 17, 0.0); b.comp[2].assign(n, 0.0);
      b.comp[0][17 * 8 + 8] = 1.0;
      x = b;
      for (auto& c : x.comp) for (auto& z : c) z = 0.0;
      KrylovOptions ko; ko.restart = 10; ko.max_iterations = 200;
      KrylovResult r = b200::solve(g, m, par, mo, b, x, ko);
      std::printf("status %s iterations %d relres %.3e\n", to_string(r.status), r.iterations, r.relres);
    }
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what()); return 2;
  } catch (const std::length_error& e) {
    std::printf("length_error: %s\n", e.what()); return 3;
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what()); return 4;
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def adapter_exe(tmp_path_factory):
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers absent (only in the build container)")
    B.build()
    d = tmp_path_factory.mktemp("adapter")
    src = d / "adapter_main.cpp"
    src.write_text(PROGRAM)
    exe = d / "adapter_main"
    cmd = ["g++", "-std=c++20", "-O1", "-w", f"-I{REF_INC}",
           f"-I{os.path.join(ROOT, 'oracle', 'refdrv', 'shim')}", f"-I{os.path.join(ROOT, 'include')}",
           str(src), "-o", str(exe), f"-L{os.path.dirname(B.LIB)}", "-lehmg_b200",
           f"-Wl,-rpath,{os.path.dirname(B.LIB)}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return str(exe)


def _run(exe, what):
    p = subprocess.run([exe, what], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout


def test_adapter_rejects_kaczmarz_as_invalid_argument(adapter_exe):
    rc, out = _run(adapter_exe, "kaczmarz")
    assert rc == 2 and "kaczmarz" in out, out


def test_adapter_honours_lu_dof_budget_as_length_error(adapter_exe):
    rc, out = _run(adapter_exe, "budget")
    # coarsest 8x8 grid = 208 DOFs > 100 (assemble.hpp:209-211 text)
    assert rc == 3 and "assemble_sparse: grid exceeds DOF budget of 100" in out, out


def test_adapter_solve_without_gpu_fails_loudly(adapter_exe):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc, out = _run(adapter_exe, "solve")
    assert rc == 4 and "no CUDA device" in out, out
