"""Pinned solver parameters (alpha, beta, step) of the BASELINE configurations, computed by
the fp64 CPU oracle exactly as the reference's resolve_config does (recon.py:199-283:
alpha = 1e-3 max|2 K^T y|, beta = alpha / 100, step = 1 / (2 sigma_max^2 + 8 beta / eps) from
50 seeded power iterations) on y = K phantom of make_scene(seed 0).

Both bench arms (ours and --impl reference) use these committed values, so the two JSON
lines describe the same workload.  Output: paste into workloads.PINNED.

    python tools/pin_configs.py cfg1 cfg2 cfg3 cfg5
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from paper_2404_10928_b200.workloads import CONFIGS  # noqa: E402

out = {}
for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5"]:
    cfg = CONFIGS[name]
    t0 = time.perf_counter()
    s = O.make_scene(cfg.n, cfg.sensors, cfg.samples, 0)
    op = O.Operator.of(s)
    y = op.forward(s.phantom)
    alpha, beta = O.resolve_regularization(op, y)
    step = O.resolve_step(op, beta, 1e-3)
    out[name] = (alpha, beta, step)
    print(f"{name}: alpha={alpha!r} beta={beta!r} step={step!r} ({time.perf_counter() - t0:.1f} s)",
          flush=True)
print(json.dumps(out))
