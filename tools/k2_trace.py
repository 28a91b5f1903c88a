"""Phase breakdown of the symmetric projector from a -DPK_FS_TRACE=1 build (timing experiments).

    K2V_BUILD=1 tools/k2v.sh "tr:-DPK_FS_TRACE=1"      # here: builds libpactgpu_vtr.so
    PK_LIB=paper_2404_10928_b200/libpactgpu_vtr.so python tools/k2_trace.py [--config cfg3]

Per CTA (clock64 stamps, fp_sym_f32_kernel): entry, after griddepcontrol.wait, then per
segment: start (scale known, windows initialised), first / last warp out of the scatter loop,
after the end-of-scatter barrier, after each staging round; end.  Prints the mean over CTAs of
each phase in microseconds (SM clock from nvidia-smi / --mhz).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200 import _native as N  # noqa: E402
from paper_2404_10928_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--frames", type=int, default=1)
ap.add_argument("--mhz", type=float, default=1965.0)
ap.add_argument("--ctas", type=int, default=148)
a = ap.parse_args()
cfg = CONFIGS[a.config]
grid, ring, ac, ph = pk.make_scene(cfg.n, cfg.sensors, cfg.samples, seed=0)
op = pk.operator_for(grid, ring, ac, pk.CudaPool(0, "float32"), frames=a.frames)
y = op.matvec(np.tile(ph.values, a.frames))
p1 = N.SolverParams(alpha=8.8e-8, beta=8.8e-10, step=333.0, tv_epsilon=1e-3, tolerance=0.0,
                    iterations=3, nonneg=0)
params = (N.SolverParams * a.frames)(*([p1] * a.frames))
lib = N.load()
lib.pk_debug_fs_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
ms = (ctypes.c_float * 3)()
n = ctypes.c_int32()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    N.check(lib.pk_profile_iterations(op.handle, params, y.data_ptr(), ms, ctypes.byref(n), s))
torch.cuda.synchronize()
print("per-launch us (CUDA events): K1 %.1f  K2 %.1f  K3 %.1f" % tuple(1e3 * v / 3 for v in ms))
tr = np.zeros((1024, 64), dtype=np.int64)
N.check(lib.pk_debug_fs_trace(tr.ctypes.data, tr.nbytes))
us = 1.0 / a.mhz
rows = []
tot_extra = {}
for c in range(a.ctas):
    t = tr[c]
    if t[1] == 0:
        continue
    c0, nseg = t[1], int(t[2])
    d = {"wait": (t[3] - c0) * us, "end": (t[63] - c0) * us, "gt0": t[0]}
    segs = []
    prev = t[3]
    for k in range(min(nseg, 7)):
        b = 4 + 8 * k
        st, wmin, wmax, bar = t[b], t[b + 1], t[b + 2], t[b + 3]
        rounds = [x for x in t[b + 4:b + 6] if x > 0 and x >= bar]
        if t[b + 6] > 0 and t[b + 6] >= bar and rounds:
            tot_extra["transpose0"] = tot_extra.get("transpose0", 0.0) + (t[b + 6] - bar) * us
            tot_extra["issue0"] = tot_extra.get("issue0", 0.0) + (rounds[0] - t[b + 6]) * us
            tot_extra["nt"] = tot_extra.get("nt", 0) + 1
        if len(rounds) == 2:
            tot_extra["round0"] = tot_extra.get("round0", 0.0) + (rounds[0] - bar) * us
            tot_extra["round1"] = tot_extra.get("round1", 0.0) + (rounds[1] - rounds[0]) * us
            tot_extra["nr"] = tot_extra.get("nr", 0) + 1
        segs.append({
            "pre": (st - prev) * us,            # scale / init before the scatter
            "scatter_first": (wmin - st) * us,  # first warp out
            "scatter_tail": (wmax - wmin) * us, # last warp out - first warp out
            "barrier": (bar - wmax) * us,
            "staging": ((rounds[-1] if rounds else bar) - bar) * us,
        })
        prev = rounds[-1] if rounds else bar
    d["post"] = (t[63] - prev) * us
    d["segs"] = segs
    rows.append(d)
gt = np.array([r["gt0"] for r in rows])
print(f"CTAs {len(rows)}, entry spread (globaltimer) {(gt.max() - gt.min()) / 1e3:.2f} us")
ends = np.array([r["end"] for r in rows])
print(f"CTA duration: mean {ends.mean():.2f}  min {ends.min():.2f}  max {ends.max():.2f} us")
print(f"griddep wait: mean {np.mean([r['wait'] for r in rows]):.2f} us")
nsg = np.array([len(r["segs"]) for r in rows])
print(f"segments per CTA: mean {nsg.mean():.2f}")
tot = {}
for r in rows:
    for k, sgm in enumerate(r["segs"]):
        for key, v in sgm.items():
            tot[key] = tot.get(key, 0.0) + v
    tot["post"] = tot.get("post", 0.0) + r["post"]
for key, v in tot.items():
    print(f"  {key:14s} per CTA {v / len(rows):7.2f} us")
if tot_extra.get("nt"):
    print("round 0 (per segment): transposition + fence + barrier %.2f  bulk issue %.2f us" % (
        tot_extra["transpose0"] / tot_extra["nt"], tot_extra["issue0"] / tot_extra["nt"]))
if tot_extra.get("nr"):
    print("staging rounds (per segment): round0 %.2f  round1 %.2f us" % (tot_extra["round0"] / tot_extra["nr"], tot_extra["round1"] / tot_extra["nr"]))
order = np.argsort(ends)
def line(i):
    r = rows[i]
    sc = sum(s["scatter_first"] + s["scatter_tail"] for s in r["segs"])
    st = sum(s["staging"] for s in r["segs"])
    pre = sum(s["pre"] for s in r["segs"])
    return (f"  cta {i:3d} end {r['end']:6.2f} segs {len(r['segs'])} wait {r['wait']:5.2f} pre {pre:5.2f} "
            f"scatter {sc:6.2f} staging {st:5.2f} | " + " ".join(f"{s['scatter_first'] + s['scatter_tail']:.1f}" for s in r["segs"]))
print("fastest:")
for i in order[:6]:
    print(line(i))
print("slowest:")
for i in order[-10:]:
    print(line(i))
