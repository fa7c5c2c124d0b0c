"""A/B timing of the 3D operator apply across library builds.

    python tools/ab_stencil.py LIB.so [LIB2.so ...] [--n 256] [--reps 20]

Each library is loaded through ctypes, an operator is built at n^3 with the
bench media, and `reps` applies on resident device buffers are timed with CUDA
events on the operator's stream (development tool; not part of the product).
"""
import argparse
import ctypes as C
import math
import sys

import numpy as np
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--homogeneous", action="store_true", help="constant media (uniform-media tile path)")
    ap.add_argument("--one", action="store_true", help="(internal) time one library in this process")
    ap.add_argument("--cmp", action="store_true", help="(internal) compare with the first library's output")
    a = ap.parse_args()
    if not a.one:
        # one process per library: two builds of the same library cannot share a process
        import subprocess
        for i, path in enumerate(a.libs):
            subprocess.run([sys.executable, __file__, path, "--n", str(a.n), "--reps", str(a.reps), "--one"]
                           + (["--cmp"] if i else []) + (["--homogeneous"] if a.homogeneous else []), check=False)
        return
    n = a.n
    nc = n ** 3
    rng = np.random.default_rng(5)
    lam = 2.0 * rng.uniform(0.8, 1.2, nc)
    mu = rng.uniform(0.8, 1.2, nc)
    rho = rng.uniform(0.8, 1.2, nc)
    gam = 0.01 * rng.uniform(0.5, 1.5, nc)
    if a.homogeneous:
        lam, mu, rho, gam = np.full(nc, 2.0), np.ones(nc), np.ones(nc), np.full(nc, 0.01)
    y_ref = None
    dims = (C.c_int * 3)(n, n, n)
    dp = lambda v: v.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for path in a.libs:
        L = C.CDLL(path)
        L.ehmg_op_n_dofs.restype = C.c_int64
        L.ehmg_op_stream.restype = C.c_uint64
        op = C.c_void_p()
        rc = L.ehmg_op_create(3, dims, C.c_double(1.0 / n), dp(lam), dp(mu), dp(rho), dp(gam),
                              C.c_double(2 / 3), C.c_double(2 * math.pi * n / 10), C.c_double(0.5),
                              C.byref(op))
        assert rc == 0, rc
        N = L.ehmg_op_n_dofs(op)
        torch.manual_seed(0)
        x = torch.randn(N, dtype=torch.complex128, device="cuda")
        y = torch.empty_like(x)
        bvec = torch.randn(N, dtype=torch.complex128, device="cuda")
        r = torch.empty_like(x)
        st = torch.cuda.ExternalStream(L.ehmg_op_stream(op))
        L.ehmg_last_error.restype = C.c_char_p
        for _ in range(3):
            rc = L.ehmg_apply_mixed_operator(op, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1)
            if rc:
                print(path, "apply failed:", L.ehmg_last_error().decode())
                break
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            L.ehmg_apply_mixed_operator(op, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        for _ in range(2):
            L.ehmg_residual(op, C.c_void_p(bvec.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(r.data_ptr()), 1)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(a.reps):
            L.ehmg_residual(op, C.c_void_p(bvec.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(r.data_ptr()), 1)
        e1.record(st)
        torch.cuda.synchronize()
        msr = e0.elapsed_time(e1) / a.reps
        ref = f"/tmp/ab_stencil_ref_{n}.pt"
        if not a.cmp:
            torch.save({"y": y.cpu(), "r": r.cpu()}, ref)
            err = errr = 0.0
        else:
            d = torch.load(ref)
            y_ref, r_ref = d["y"].cuda(), d["r"].cuda()
            err = float((y - y_ref).abs().max() / y_ref.abs().max())
            errr = float((r - r_ref).abs().max() / r_ref.abs().max())
        print(f"{path}: apply {ms:.4f} ms ({N / ms / 1e6:.2f} GDOF/s)  residual {msr:.4f} ms  "
              f"rel diff vs first lib: apply {err:.2e} residual {errr:.2e}")
        L.ehmg_op_destroy(op)
        sys.stdout.flush()


if __name__ == "__main__":
    main()
