"""Validate the reference arm's DOF-ratio extrapolation: time one reference
V(2,2) cycle (oracle/_ref = the reference headers) at 32^3 (3 levels), 64^3
(4 levels) and 128^3 (5 levels) on one host core, and 64^3 with every host
core running a replica, then extrapolate each to 256^3 (5 levels) exactly as
bench.py does. Output: profiles/round2/ref_extrapolation.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

out = {"host_cores": os.cpu_count(), "rows": []}
for n, lv, threads in [(32, 3, 1), (64, 4, 1), (128, 5, 1), (32, 3, os.cpu_count()), (64, 4, os.cpu_count())]:
    t0 = time.perf_counter()
    rate, kind, per, wall, lv = bench.run_cpu_sample(1, threads, n, lv)
    row = {"cells": n, "levels": lv, "threads": threads, "kind": kind, "s_per_cycle": round(per, 3),
           "extrapolated_256_vcycles_per_s": rate, "wall_s": round(time.perf_counter() - t0, 1)}
    out["rows"].append(row)
    print(json.dumps(row), flush=True)
base = {(r["cells"], r["threads"]): r["extrapolated_256_vcycles_per_s"] for r in out["rows"]}
one = base[(128, 1)]
out["single_core_error_vs_128"] = {f"{n}^3": round(base[(n, 1)] / one - 1, 4) for n in (32, 64)}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "ref_extrapolation.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out["single_core_error_vs_128"]))
