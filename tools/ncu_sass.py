"""Per-SASS-instruction executed counts and stall samples of an ncu report (source page), grouped into
runs of equal execution count (basic blocks): python tools/ncu_sass.py rep [min_share_pct]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source")
tot_i = sum(float(r[ie] or 0) for r in data); tot_s = sum(float(r[ss] or 0) for r in data)
blocks = []; cur = None
for r in data:
    n = float(r[ie] or 0)
    if cur is None or n != cur["n"]:
        cur = {"n": n, "rows": []}; blocks.append(cur)
    cur["rows"].append(r)
print(f"total instr {tot_i:.3e}  samples {tot_s:.0f}")
for b in blocks:
    bi = b["n"] * len(b["rows"]); bs = sum(float(r[ss] or 0) for r in b["rows"])
    if 100 * bi / tot_i >= thr or 100 * bs / tot_s >= thr:
        print(f"--- block x{b['n']:.3e} len {len(b['rows'])}  instr {100*bi/tot_i:5.1f}%  stall {100*bs/tot_s:5.1f}%  first {b['rows'][0][0][-5:]}")
        if len(sys.argv) > 3:
            for r in b["rows"]: print("     ", r[src].strip()[:90], r[ss])
