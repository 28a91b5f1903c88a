"""Alias conftest: the reference's own test suite re-run against the drop-in.

tools/refsuite/run.sh copies the reference package and its tests into the git-ignored
scratch directory .reftest/ (never committed) together with this file, and runs pytest there
on the GPU box.  Every public name that the reference package `pactkit` and this drop-in
both export is rebound, in `pactkit` and in the submodule that defines it, to the drop-in's
object before the test modules import them; names the drop-in does not provide (the numba
kernels module, the CLI, bench_matmul, file readers of images) stay the reference's.  The
reference tests pass `pool=None` or a `WorkerPool`, which the drop-in maps to its fp64
device mode (device.resolve_pool), so the suite exercises the CUDA path at the reference's
own fp64 tolerances.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, HERE)   # the copied reference package (pactkit/)
sys.path.insert(0, REPO)   # the drop-in

import pytest  # noqa: E402

import pactkit  # noqa: E402
from pactkit import bench, forward, geometry, kernels, recon  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402

MODULES = ("bench", "forward", "geometry", "kernels", "recon", "cli")
REBOUND = []
for name in sorted(n for n in dir(pactkit) if not n.startswith("_") and n not in MODULES):
    if not hasattr(pk, name):
        continue
    new = getattr(pk, name)
    for mod in (pactkit, bench, forward, geometry, recon):
        if hasattr(mod, name):
            setattr(mod, name, new)
    REBOUND.append(name)


def pytest_report_header(config):
    return [f"refsuite: {len(REBOUND)} pactkit names bound to the drop-in: {', '.join(REBOUND)}"]


@pytest.fixture(scope="session", autouse=True)
def compiled_kernels():
    kernels.warm_up()  # (the reference's own numba kernels, used by the tests that stay on them)
