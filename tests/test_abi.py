"""CPU: the C-ABI library loads, exports every symbol include/ehmg_b200.h
declares, and fails loudly (no CPU fallback) without a CUDA device."""
import os
import re
import subprocess

import numpy as np
import pytest

import __graft_entry__
from paper_2307_03242_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ehmg_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(ehmg_[a-z0-9_]+)\(", src,
                                 re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    B.build()
    assert os.path.exists(B.LIB)
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(ehmg_\w+)", out))
    decl = declared_symbols()
    assert len(decl) >= 30
    missing = [s for s in decl if s not in exported]
    assert not missing, missing


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2307_03242_b200 as E
    g = E.StaggeredGrid((8, 8), 0.125)
    m = E.MediaModel.homogeneous(g, 2, 1, 1, 0.01)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        E.make_opdata(g, m, E.OperatorParams(2 / 3, 10.0, 0.1))
    with pytest.raises(RuntimeError):
        E.Multigrid(g, m, E.OperatorParams(2 / 3, 10.0, 0.1), E.MgOptions())


def test_host_validation_mirrors_reference_messages():
    import paper_2307_03242_b200 as E
    with pytest.raises(ValueError, match="need >= 2 cells"):
        E.StaggeredGrid((1, 4), 0.1)
    with pytest.raises(ValueError, match="h must be positive"):
        E.StaggeredGrid((4, 4), 0.0)
    g = E.StaggeredGrid((4, 4), 0.25)
    m = E.MediaModel.homogeneous(g, 1, 1, -1)
    with pytest.raises(ValueError, match="rho must be positive"):
        m.validate(g)
    with pytest.raises(ValueError, match="dims must be even"):
        E.coarsen_grid(E.StaggeredGrid((9, 8), 0.1))
    assert E.coarsen_grid(E.StaggeredGrid((8, 6), 0.125)).dims == (4, 3)
    assert E.middle_of_top_row(E.StaggeredGrid((8, 6, 4), 0.25)) == (4, 3, 0)
    f = E.make_point_source(E.StaggeredGrid((8, 4), 0.25), 2, (3, 1))
    assert np.abs(f).max() == pytest.approx(16.0)
    with pytest.raises(IndexError):
        E.make_point_source(E.StaggeredGrid((8, 4), 0.25), 0, (9, 0))


def test_graft_entry_has_build_and_smoke():
    assert callable(__graft_entry__.build) and callable(__graft_entry__.smoke)


def test_krylov_options_struct_matches_header():
    """The ctypes mirror of ehmg_krylov_options carries every header field
    (incl. the B200 orthogonalization switch) and rejects unknown variants."""
    import ctypes
    import paper_2307_03242_b200 as E
    from paper_2307_03242_b200 import ehmg as H
    src = open(HEADER).read()
    body = src[:src.index("} ehmg_krylov_options;")]
    body = body[body.rindex("typedef struct {"):]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"^\s*(?:int|double)\s+([a-z_]+);", body, re.M)
    assert [f for f, _ in H._KOpts._fields_] == fields
    assert ctypes.sizeof(H._KOpts) == 32  # int int double double int int
    assert E.KrylovOptions().orthogonalization == "classical"
    assert H._ORTH == {"classical": 0, "modified": 1}
    with pytest.raises(ValueError, match="unknown orthogonalization"):
        E.KrylovOptions(orthogonalization="householder")
