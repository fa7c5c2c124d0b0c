"""Static SASS instruction mix per kernel of an object / library (cuobjdump -sass).
    python tools/sass_mix.py FILE [kernel-substring]
Loops are found from backward branches; the mix of each loop body is printed."""
import collections, re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
want = sys.argv[2] if len(sys.argv) > 2 else ""
kern = None; ins = {}
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m: kern = m.group(1); ins[kern] = []; continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and kern: ins[kern].append((int(m.group(1), 16), m.group(2).strip()))
for k, L in ins.items():
    if want not in k: continue
    print("==", k[:110], len(L), "instructions")
    addr = {a: i for i, (a, _) in enumerate(L)}
    loops = []
    for i, (a, s) in enumerate(L):
        m = re.search(r"BRA(?:\.U)?(?:\.\w+)*\s+(?:!?U?P\d,\s*)?`?\(?0x([0-9a-f]+)", s)
        if m:
            tgt = int(m.group(1), 16)
            if tgt in addr and addr[tgt] < i and i - addr[tgt] > 200: loops.append((addr[tgt], i))
    for (lo, hi) in loops:
        c = collections.Counter()
        for a, s in L[lo:hi + 1]:
            p = s.split()
            o = p[1] if p[0].startswith("@") else p[0]
            c[o.split(".")[0]] += 1
        tot = sum(c.values())
        fp = c["DADD"] + c["DFMA"] + c["DMUL"]; lsu = c["SHFL"] + c["LDS"] + c["STS"] + c["STG"] + c["LDG"]
        print(f" loop [{lo},{hi}] {tot} instrs: FP64 {fp} LSU {lsu} other {tot-fp-lsu}")
        print("   ", " ".join(f"{o}:{v}" for o, v in c.most_common(28)))
