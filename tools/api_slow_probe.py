"""Which reference cycles does one bench_recon leave behind (they pinned device memory and
slowed the next public calls until a gc pass)?  python tools/api_slow_probe.py"""
import collections
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.harness import _scene  # noqa: E402

n, M, Q = 512, 512, 2048
grid, ring, ac, ph, K, y, cfg = _scene(n, M, Q, 0, pk.ReconConfig(iterations=10), 0)
f32 = pk.CudaPool(0, "float32")


def t(k=5):
    out = []
    for _ in range(k):
        t0 = time.perf_counter()
        pk.iterative_reconstruct(K, y, cfg, pool=f32)
        out.append((time.perf_counter() - t0) * 1e3)
    return " ".join(f"{v:.2f}" for v in out)


print("before", t())
gc.collect()
gc.set_debug(gc.DEBUG_SAVEALL)
pk.bench_recon(n, M, Q, pk.ReconConfig(iterations=10), reps=5)
print("after harness", t())
gc.collect()
print(collections.Counter(type(o).__name__ for o in gc.garbage).most_common(25))
import torch  # noqa: E402
big = [o for o in gc.garbage if isinstance(o, torch.Tensor)]
print("tensors in garbage:", [(tuple(x.shape), str(x.device), x.dtype) for x in big][:10])
for o in gc.garbage:
    if type(o).__name__ in ("frame", "function", "cell"):
        print(type(o).__name__, getattr(o, "f_code", getattr(o, "__code__", None)))
gc.set_debug(0)
gc.garbage.clear()
print("after gc", t())
