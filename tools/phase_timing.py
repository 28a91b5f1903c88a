"""Phase breakdown of the symmetric projector (experiment build with -DPK_PHASE_TIMING):
    PK_LIB=paper_2404_10928_b200/libpactgpu_timing.so python tools/phase_timing.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200 import _native as N  # noqa: E402

grid, ring, ac, ph = pk.make_scene(512, 512, 2048, seed=0)
op = pk.operator_for(grid, ring, ac, pk.CudaPool(0, "float32"))
lib = N.load()
buf = (ctypes.c_ulonglong * 8)()
x = torch.tensor(np.random.default_rng(0).random(grid.size), device="cuda", dtype=torch.float32)
op.matvec(x)
lib.pk_phase_cycles_read(buf)
op.matvec(x)
torch.cuda.synchronize()
lib.pk_phase_cycles_read(buf)
names = ["zero", "barrier", "scatter", "flush"]
tot = sum(buf[i] for i in range(4))
for i in range(4):
    print(f"{names[i]:8s} {buf[i] / tot * 100:5.1f} %  ({buf[i] / 1e6:.1f} Mcycles over all warps)")
