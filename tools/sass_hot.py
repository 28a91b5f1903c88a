"""Group an ncu source-page CSV (--page source --csv --print-source sass) into runs of equal
execution count and print where the stall samples and shared wavefronts go.

    python tools/sass_hot.py src.csv [min_samples]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]


def f(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError, IndexError):
        return 0.0


runs = []
for r in rows[2:]:
    if len(r) < len(h):
        break
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    ex = f(r, "Instructions Executed")
    s = f(r, "Warp Stall Sampling (All Samples)")
    wf = f(r, "L1 Wavefronts Shared")
    stl = {k[6:]: f(r, k) for k in st}
    if runs and runs[-1]["ex"] == ex:
        R = runs[-1]
        R["n"] += 1; R["s"] += s; R["wf"] += wf
        R["ops"][op] = R["ops"].get(op, 0) + 1
        for k, v in stl.items():
            R["st"][k] = R["st"].get(k, 0) + v
    else:
        runs.append(dict(a=r[ix["Address"]][-5:], ex=ex, n=1, s=s, wf=wf, ops={op: 1}, st=stl))
tot = sum(r["s"] for r in runs)
print(f"total samples {tot:.0f}")
for r in runs:
    if r["s"] >= thr:
        top = sorted(r["ops"].items(), key=lambda t: -t[1])[:4]
        ss = sorted(r["st"].items(), key=lambda t: -t[1])[:4]
        print(f"{r['a']} ex={r['ex']:8.0f} n={r['n']:4d} samp={r['s']:5.0f} ({100 * r['s'] / tot:4.1f}%) "
              f"wf={r['wf']:9.0f} {top} {[(k, int(v)) for k, v in ss]}")
