"""Phase breakdown of the symmetric back-projector from a -DPK_BP_TRACE=1 build.

    K2V_BUILD=1 tools/k2v.sh "bt:-DPK_BP_TRACE=1"
    PK_LIB=paper_2404_10928_b200/libpactgpu_vbt.so python tools/k1_trace.py [--config cfg3]

Per CTA (consumer thread 0): entry, after griddepcontrol.wait, first chunk staged, end of the
chunk loop, end of the last flush (clock64), chunks and partial slots.
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
a = ap.parse_args()
cfg = CONFIGS[a.config]
grid, ring, ac, ph = pk.make_scene(cfg.n, cfg.sensors, cfg.samples, seed=0)
op = pk.operator_for(grid, ring, ac, pk.CudaPool(0, "float32"), frames=a.frames)
y = op.matvec(np.tile(ph.values, a.frames))
p1 = N.SolverParams(alpha=8.8e-8, beta=8.8e-10, step=333.0, tv_epsilon=1e-3, tolerance=0.0,
                    iterations=3, nonneg=0)
params = (N.SolverParams * a.frames)(*([p1] * a.frames))
lib = N.load()
lib.pk_debug_bp_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
ms = (ctypes.c_float * 3)()
n = ctypes.c_int32()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    N.check(lib.pk_profile_iterations(op.handle, params, y.data_ptr(), ms, ctypes.byref(n), s))
torch.cuda.synchronize()
print("per-launch us (CUDA events): K1 %.1f  K2 %.1f  K3 %.1f" % tuple(1e3 * v / 3 for v in ms))
tr = np.zeros((1536, 16), dtype=np.int64)
N.check(lib.pk_debug_bp_trace(tr.ctypes.data, tr.nbytes))
us = 1.0 / a.mhz
rows = [t for t in tr if t[1] != 0 and t[3] > 0]
gt = np.array([t[0] for t in rows])
print(f"CTAs {len(rows)}, entry spread {(gt.max() - gt.min()) / 1e3:.2f} us")
ph = {
    "griddep wait": [(t[2] - t[1]) * us for t in rows],
    "pipeline fill": [(t[4] - t[2]) * us for t in rows],
    "chunk loop": [(t[5] - t[4]) * us for t in rows],
    "last flush": [(t[6] - t[5]) * us for t in rows],
    "total": [(t[6] - t[1]) * us for t in rows],
    "end (global, from first entry)": [(t[0] - gt.min()) / 1e3 + (t[6] - t[1]) * us for t in rows],
}
for k, v in ph.items():
    v = np.array(v)
    print(f"  {k:32s} mean {v.mean():6.2f}  min {v.min():6.2f}  max {v.max():6.2f} us")
ch = np.array([t[3] for t in rows]); sl = np.array([t[7] for t in rows])
print(f"chunks per CTA: mean {ch.mean():.1f} min {ch.min()} max {ch.max()}; slots per CTA: mean {sl.mean():.2f} max {sl.max()}")
loop = np.array(ph["chunk loop"])
order = np.argsort(loop)
for i in list(order[:4]) + list(order[-6:]):
    t = rows[i]
    print(f"  cta loop {loop[i]:6.2f} us chunks {t[3]} slots {t[7]}  us/chunk {loop[i] / t[3]:.3f}")
# per-chunk clocks of consumer warp 0 vs chunk (tile, base sensors)
lib.pk_debug_bp_chunks.argtypes = [ctypes.c_void_p, ctypes.c_int64]
cc = np.zeros((1536, 64), dtype=np.int32)
N.check(lib.pk_debug_bp_chunks(cc.ctypes.data, cc.nbytes))
cap = 1 << 20
chunks = np.zeros(cap, np.int32); c0 = np.zeros(cap, np.int32); tiles = np.zeros(cap, np.int32)
lib.pk_debug_bp_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
nch = lib.pk_debug_bp_plan(op.handle, chunks.ctypes.data, c0.ctypes.data, tiles.ctypes.data, cap)
qt = (cfg.n // 2 + 31) // 32
ntiles = qt * (qt + 1) // 2
recs = []
for cta in range(len(rows)):
    a0, a1 = c0[cta], c0[cta + 1]
    for c in range(a0, min(a1, a0 + 64)):
        if c == a0:
            continue  # (the first chunk includes the pipeline fill)
        t = chunks[c] >> 16; k = chunks[c] & 0xffff
        tp = tiles[t % ntiles]
        tx, ty = tp >> 16, tp & 0xffff
        recs.append((cc[cta, c - a0], tx, ty, k))
recs = np.array(recs)
diag = recs[:, 1] == recs[:, 2]
for name, sel in (("diagonal", diag), ("off-diagonal", ~diag)):
    v = recs[sel, 0] * us
    print(f"{name:12s} chunks {sel.sum():6d}: us per chunk mean {v.mean():.3f} p10 {np.percentile(v, 10):.3f} "
          f"p90 {np.percentile(v, 90):.3f} max {v.max():.3f}")
off = recs[~diag]
# dependence on the base sensors (chunk k covers sensors 2k, 2k+1): angle bins
M = cfg.sensors
ang = (off[:, 3] * 2 / M * 360.0)
for lo_ in range(0, 360, 45):
    sel = (ang >= lo_) & (ang < lo_ + 45)
    if sel.any():
        print(f"  sensor angle {lo_:3d}-{lo_ + 45:3d}: us per chunk {off[sel, 0].mean() * us:.3f}")

# per tile (off-diagonal and diagonal) mean cost, and per sensor angle (16 bins) per tile class
print("per tile: (tx, ty) us per chunk")
for (tx, ty) in sorted(set((int(r[1]), int(r[2])) for r in recs)):
    sel = (recs[:, 1] == tx) & (recs[:, 2] == ty)
    print(f"  ({tx},{ty}) {recs[sel, 0].mean() * us:.3f} (n {sel.sum()})")
for name, sel0 in (("off-diagonal", ~diag), ("diagonal", diag)):
    r = recs[sel0]
    ang = (r[:, 3] * 2 / M * 360.0)
    line = " ".join(f"{r[(ang >= a0) & (ang < a0 + 22.5), 0].mean() * us:.2f}" if ((ang >= a0) & (ang < a0 + 22.5)).any() else "-"
                    for a0 in np.arange(0, 360, 22.5))
    print(f"{name} by sensor angle (22.5 deg bins): {line}")
