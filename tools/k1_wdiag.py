"""Print the back-projector's tuned diagonal cut weight and slot count of a config's plan.

    python tools/k1_wdiag.py [--config cfg3] [--frames 4]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--frames", type=int, default=1)
ap.add_argument("--concurrency", type=int, default=1)
a = ap.parse_args()
cfg = CONFIGS[a.config]
grid, ring, ac, ph = pk.make_scene(cfg.n, cfg.sensors, cfg.samples, seed=0)
t0 = time.time()
op = pk.operator_for(grid, ring, ac, pk.CudaPool(0, "float32"), frames=a.frames, concurrency=a.concurrency)
print(f"{a.config} x{a.frames} conc {a.concurrency}: plan {time.time() - t0:.2f} s, bp_split (slots) {op.info.bp_split}")
