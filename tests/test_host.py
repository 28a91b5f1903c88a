"""Host-side logic of the drop-in package (no GPU): geometry mirror bit-exactness, config
validation, operator construction and the C-ABI library's symbol table."""

import ctypes
import hashlib
import json
import os
import re
import warnings

import numpy as np
import pytest

import paper_2404_10928_b200 as pk
from paper_2404_10928_b200 import _native
from conftest import GOLDEN, ROOT


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_scene_geometry_bit_exact_with_reference():
    for rec in json.load(open(os.path.join(GOLDEN, "geometry.json"))):
        if rec.get("custom"):
            g = pk.make_grid(24, 20, 2e-4, (1e-3, -2e-3))
            ring = pk.make_ring(12, 9e-3, (3.3e-3, -0.1e-3), g)
            assert sha(g.pixel_coords()) == rec["pixel_coords"]
            assert sha(ring.positions) == rec["positions"]
            assert sha(pk.make_vessel_phantom(g, 5, 3).values) == rec["phantom"]
            continue
        g, ring, ac, ph = pk.make_scene(rec["n"], rec["M"], rec["Q"], seed=rec["seed"])
        assert ac.dt.hex() == rec["dt"]
        assert ring.radius.hex() == rec["radius"]
        assert [v.hex() for v in g.origin] == rec["origin"]
        assert sha(g.pixel_coords()) == rec["pixel_coords"]
        assert sha(ring.positions) == rec["positions"]
        assert sha(ph.values) == rec["phantom"]


def test_recon_config_validation():
    with pytest.raises(ValueError):
        pk.ReconConfig(alpha=-1.0)
    with pytest.raises(ValueError):
        pk.ReconConfig(iterations=0)
    with pytest.raises(ValueError):
        pk.ReconConfig(step=0.0)
    with pytest.raises(ValueError):
        pk.ReconConfig(step="fast")
    with pytest.raises(ValueError):
        pk.ReconConfig(tv_epsilon=0.0)


def test_build_time_matrix_is_lazy_and_validates():
    g, ring, ac, _ = pk.make_scene(512, 512, 2048)
    K = pk.build_time_matrix(g, ring, ac)  # 2.2 TB dense -- must not be formed
    assert K.rows == 512 * 2048 and K.cols == 512 * 512
    assert K.provenance["truncated_pairs"] == 0
    assert K.layout() == (512, 2048)
    bad = pk.TransducerRing(8, 1e-3)
    with pytest.raises(pk.GeometryError):
        pk.build_time_matrix(pk.centered_grid(64, 64, 1e-4), bad, pk.AcousticConfig())


def test_truncation_warning_count_matches_reference():
    t = json.load(open(os.path.join(GOLDEN, "kat.json")))["truncation"]
    g = pk.centered_grid(16, 16, 1e-4)
    ring = pk.make_ring(4, 5e-3, (0, 0), g)
    with pytest.warns(pk.TruncationWarning):
        K = pk.build_time_matrix(g, ring, pk.AcousticConfig(c=1500.0, dt=1e-7, q_s=8, q_n=8))
    assert K.provenance["truncated_pairs"] == t["truncated_pairs"]


def test_sensor_data_and_field_validation():
    with pytest.raises(ValueError):
        pk.SensorData("time", 2, 3, np.zeros(5))
    with pytest.raises(ValueError):
        pk.SensorData("time", 1, 2, np.array([0.0, np.nan]))
    g = pk.make_grid(2, 2, 1.0)
    with pytest.raises(ValueError):
        pk.ImageField(g, np.zeros(3))
    with pytest.raises(ValueError):
        pk.CudaPool(dtype="float16")


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "pactgpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(pk_\w+)\s*\(", txt, re.M)))


def test_abi_library_exports_every_header_symbol():
    """The C-ABI library loads without a GPU and exports what include/pactgpu.h declares."""
    _native.build()
    lib = _native.load()
    syms = _header_symbols()
    assert len(syms) >= 12
    bound = {name for name, _, _ in _native.SYMBOLS}
    for s in syms:
        assert hasattr(lib, s), s
        assert s in bound, f"{s} not bound in _native.SYMBOLS"
    assert lib.pk_version() >= 10000


def test_abi_rejects_bad_arguments_without_gpu():
    lib = _native.load()
    h = ctypes.c_void_p()
    assert lib.pk_plan_create(None, ctypes.byref(h)) == _native.PK_ERR_INVALID
    xx = np.zeros(1)
    dp = ctypes.POINTER(ctypes.c_double)
    desc = _native.GeometryDesc(nx=0, ny=1, pixel_x=xx.ctypes.data_as(dp), pixel_y=xx.ctypes.data_as(dp),
                                sensors=1, sensor_xy=xx.ctypes.data_as(dp), sensor_begin=0,
                                sensor_end=1, samples=4, c=1.0, dt=1.0, dtype=0, device=0)
    assert lib.pk_plan_create(ctypes.byref(desc), ctypes.byref(h)) == _native.PK_ERR_INVALID
    assert b"grid" in lib.pk_last_error()


def test_no_cpu_fallback_when_no_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g, ring, ac, ph = pk.make_scene(16, 8, 40)
    K = pk.build_time_matrix(g, ring, ac)
    with pytest.raises(_native.NativeUnavailable):
        pk.forward_project(K, ph)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2404_10928_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace("oracle/", ""), f


def test_stop_point_rules():
    """Speculative sharded solve: the stopping rules of recon.py:346-363 applied afterwards."""
    import math

    from paper_2404_10928_b200.sharded import stop_point

    dec = [(10.0 - i, 0.0, 0.0, 0.0) for i in range(6)]
    k, why, hist = stop_point(dec, 20.0, 1.0, 1.0, 0.0)
    assert (k, why, len(hist)) == (6, "max_iterations", 6)
    bad = dec[:3] + [(math.nan, 0.0, 0.0, 0.0)] + dec[3:]
    assert stop_point(bad, 20.0, 1.0, 1.0, 0.0)[:2] == (3, "divergence")
    nonfin = dec[:2] + [(1.0, 0.0, 0.0, 1.0)]
    assert stop_point(nonfin, 20.0, 1.0, 1.0, 0.0)[:2] == (2, "divergence")
    grow = [(1.0 + i, 0.0, 0.0, 0.0) for i in range(8)]
    assert stop_point(grow, 0.5, 1.0, 1.0, 0.0)[:2] == (5, "divergence")
    flat = [(1.0, 0.0, 0.0, 0.0)] * 4
    assert stop_point(flat, 2.0, 1.0, 1.0, 1e-6)[:2] == (2, "tolerance")
    # l1 / tv weights enter the objective
    k, why, hist = stop_point([(1.0, 2.0, 3.0, 0.0)], 100.0, 0.5, 0.25, 0.0)
    assert hist[0] == (1.0 + 1.0 + 0.75, 1.0, 1.0, 0.75)


def test_pactmat_pactsig_round_trip_and_reference_layout(tmp_path):
    """PACTMAT / PACTSIG (forward.py:276-330): header line + little-endian float64 payload,
    complex interleaved; files written byte-for-byte as the reference lays them out are read
    back exactly, and our writer produces the same bytes."""
    import paper_2404_10928_b200 as pk

    rng = np.random.default_rng(0)
    A = rng.standard_normal((6, 5))
    ref_bytes = b"PACTMAT time 6 5\n" + A.astype("<f8").tobytes()
    (tmp_path / "a.mat").write_bytes(ref_bytes)
    K = pk.read_matrix(tmp_path / "a.mat")
    assert K.domain == "time" and np.array_equal(K.entries, A)
    pk.write_matrix(K, tmp_path / "b.mat")
    assert (tmp_path / "b.mat").read_bytes() == ref_bytes
    C = rng.standard_normal((4, 3)) + 1j * rng.standard_normal((4, 3))
    (tmp_path / "c.mat").write_bytes(b"PACTMAT frequency 4 3\n" + C.view(np.float64).astype("<f8").tobytes())
    Kc = pk.read_matrix(tmp_path / "c.mat")
    assert Kc.domain == "frequency" and np.array_equal(Kc.entries, C)
    y = pk.SensorData("frequency", 2, 3, rng.standard_normal(6) + 1j * rng.standard_normal(6))
    pk.write_signal(y, tmp_path / "y.sig")
    raw = (tmp_path / "y.sig").read_bytes()
    assert raw.startswith(b"PACTSIG frequency 2 3\n")
    y2 = pk.read_signal(tmp_path / "y.sig")
    assert y2.domain == "frequency" and np.array_equal(y2.values, y.values)
    (tmp_path / "bad").write_bytes(b"PACTSIG time 2 3\n" + b"\0" * 8)
    with pytest.raises(ValueError):
        pk.read_signal(tmp_path / "bad")
    with pytest.raises(ValueError):
        pk.read_matrix(tmp_path / "y.sig")


def test_measurement_matrix_reference_constructor():
    """MeasurementMatrix(domain, entries, provenance) as forward.py:70-91 declares it: keyword
    `entries=` and dataclasses.replace(K, entries=...) work."""
    import dataclasses

    A = np.arange(12.0).reshape(4, 3)
    K = pk.MeasurementMatrix(domain="time", entries=A)
    assert K.rows == 4 and K.cols == 3 and np.array_equal(K.entries, A)
    assert not K.entries.flags.writeable
    K2 = dataclasses.replace(K, entries=2 * A)
    assert np.array_equal(K2.entries, 2 * A) and K2.domain == "time"
    K3 = pk.MeasurementMatrix("frequency", A + 1j)
    assert K3.entries.dtype == np.complex128
    with pytest.raises(ValueError):
        pk.MeasurementMatrix("time", np.zeros(3))
    with pytest.raises(ValueError):
        pk.MeasurementMatrix("time")  # neither entries nor provenance
    g, ring, ac, _ = pk.make_scene(16, 8, 40)
    lazy = pk.MeasurementMatrix("time", None, {"grid": g, "ring": ring, "acoustic": ac})
    assert lazy.geometry_backed and lazy.rows == 320


def test_pool_policy_is_explicit():
    """pool=None and a reference WorkerPool keep the reference's fp64 numerics; fp32 needs
    an explicit CudaPool."""
    from paper_2404_10928_b200.device import resolve_pool

    class WorkerPool:  # what pactkit.kernels.WorkerPool looks like (kernels.py:55-73)
        worker_count = 8

    assert resolve_pool(None) == pk.CudaPool(0, "float64")
    assert resolve_pool(WorkerPool()) == pk.CudaPool(0, "float64")
    f32 = pk.CudaPool(0, "float32")
    assert resolve_pool(f32) is f32
    with pytest.raises(TypeError):
        resolve_pool("float32")
    pk.set_default_pool(f32)
    try:
        assert resolve_pool(None) is f32
    finally:
        pk.set_default_pool(None)
    assert pk.default_pool().dtype == "float64"


def test_reconstruct_frames_routes_non_time_operators_per_frame(monkeypatch):
    """A frequency-domain (or explicit) K never reaches the time-domain batched plans
    (complex y would be truncated and solved with the wrong operator)."""
    from paper_2404_10928_b200 import solver

    g, ring, ac, _ = pk.make_scene(16, 8, 40)
    Kf = pk.build_freq_matrix(g, ring, ac)
    y = pk.SensorData("frequency", 8, 40, np.ones(320, dtype=complex))
    seen = []
    monkeypatch.setattr(solver, "iterative_reconstruct",
                        lambda K, y, config, pool=None: seen.append(K.domain) or "solved")
    out = solver.reconstruct_frames(Kf, [y, y], pk.ReconConfig(iterations=2),
                                    pool=pk.CudaPool(0, "float32"), batch=1)
    assert out == ["solved", "solved"] and seen == ["frequency", "frequency"]
    Ke = pk.MeasurementMatrix("time", np.eye(4))
    assert solver.geometry_path(Ke) is None and solver.geometry_path(Kf) == "frequency"
    assert solver.geometry_path(pk.build_time_matrix(g, ring, ac)) == "time"
