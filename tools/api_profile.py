"""Wall time of the public API calls (the reference harness's view), in the harness's order:
python tools/api_profile.py [n M Q]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.harness import _scene  # noqa: E402

n, M, Q = (int(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (128, 128, 1024)))
grid, ring, ac, ph, K, y, cfg = _scene(n, M, Q, 0, pk.ReconConfig(iterations=10), 0)
f32, f64 = pk.CudaPool(0, "float32"), pk.CudaPool(0, "float64")


def t(fn, k=5):
    out = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        out.append((time.perf_counter() - t0) * 1e3)
    return " ".join(f"{v:.2f}" for v in out)


print("bp f32 ms", t(lambda: pk.back_project(K, y, pool=f32)))
print("ir f64 ms", t(lambda: pk.iterative_reconstruct(K, y, cfg, pool=f64)))
print("ir f32 ms", t(lambda: pk.iterative_reconstruct(K, y, cfg, pool=f32)))
print("bp f32 ms", t(lambda: pk.back_project(K, y, pool=f32)))
print("ir f32 ms", t(lambda: pk.iterative_reconstruct(K, y, cfg, pool=f32)))

if len(sys.argv) > 4:  # the harness in the same process, then the direct calls again
    rep = pk.bench_recon(n, M, Q, pk.ReconConfig(iterations=10), reps=5)
    print("harness iterative_parallel (fp32) ms", rep.entry("iterative_parallel").wall_seconds * 1e3)
    print("ir f32 ms", t(lambda: pk.iterative_reconstruct(K, y, cfg, pool=f32)))
    g2, r2, a2, p2, K2, y2, c2 = _scene(n, M, Q, 0, pk.ReconConfig(iterations=10), 0)
    print("ir f32 (new scene objects) ms", t(lambda: pk.iterative_reconstruct(K2, y2, c2, pool=f32)))
    print("ir f32 (old K, new cfg) ms", t(lambda: pk.iterative_reconstruct(K, y, c2, pool=f32)))
    print("cfg", cfg)
    print("c2 ", c2)
