"""Summarise an ncu report (.ncu-rep) or an ncu launch-list CSV into text
for profiles/ (run here, without a GPU)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Issued Ipc Active", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
        "Issued Instructions", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
       "gpu__time_duration.sum"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def report(path):
    out = [f"# ncu summary: {path}"]
    det = run([path, "--page", "details", "--csv"])
    rows = list(csv.reader(io.StringIO(det)))
    if rows:
        h = rows[0]
        iN, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        iK = h.index("Kernel Name")
        out.append(f"kernel: {rows[1][iK]}")
        seen = set()
        for r in rows[1:]:
            if r[iN] in KEYS and r[iN] not in seen:
                seen.add(r[iN])
                out.append(f"  {r[iN]:45s} {r[iV]:>16s} {r[iU]}")
    raw = list(csv.reader(io.StringIO(run([path, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        d = dict(zip(raw[0], raw[2]))
        u = dict(zip(raw[0], raw[1]))
        for k in RAW:
            if k in d:
                out.append(f"  {k:45s} {d[k]:>16s} {u.get(k, '')}")
    sass = list(csv.reader(io.StringIO(run([path, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(sass) > 2:
        h = sass[1]
        iS, iE = h.index("Source"), h.index("Instructions Executed")
        iW = h.index("Warp Stall Sampling (All Samples)")
        op, st = collections.Counter(), collections.Counter()
        for r in sass[2:]:
            s = r[iS].strip().split()
            if not s:
                continue
            o = (s[1] if s[0].startswith("@") else s[0]).split(".")[0]
            op[o] += int(r[iE] or 0)
            st[o] += int(r[iW] or 0)
        tot, stt = sum(op.values()), max(1, sum(st.values()))
        out.append(f"  instruction mix (warp-level, total {tot}):")
        for o, c in op.most_common(12):
            out.append(f"    {o:10s} {c:12d} {100 * c / tot:5.1f}%   stall-samples {100 * st[o] / stt:5.1f}%")
    return "\n".join(out)


SETUP = ("cutlass", "trsm", "getr", "ipiv", "k_identity", "vanka_build", "vanka_to_soa", "coarse_matrix",
         "laswp", "laset", "coarsen_media", "swap")


def launches(path, steady=False):
    """steady: only the launches after the last setup kernel (LU inverse,
    Vanka factorisation): the cycles the bench times."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    iK, iV, iG = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    agg = collections.defaultdict(lambda: [0, 0.0])
    body = rows[hi + 1:]
    if steady:
        last = max([i for i, r in enumerate(body) if any(k in r[iK] for k in SETUP)], default=-1)
        body = body[last + 1:]
    for r in body:
        agg[(r[iK].split("(")[0], r[iG])][0] += 1
        agg[(r[iK].split("(")[0], r[iG])][1] += float(r[iV].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = [f"# ncu launch list summary: {path} (gpu__time_duration.sum, cold-cache, serialised"
           + (", launches after the last setup kernel)" if steady else ")"),
           f"{'kernel':40s} {'grid':16s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}"]
    for (k, g), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:40]:40s} {g:16s} {c:8d} {t / 1e6:10.3f} {100 * t / tot:6.1f}% {t / c / 1e3:9.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    p = sys.argv[1]
    print(launches(p, "--steady" in sys.argv) if p.endswith(".csv") else report(p))
