"""The CPU oracle against the reference's own outputs (tests/golden, made by running
pactkit itself -- tests/golden/make_golden.py).  Pins the oracle before it is trusted."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

SMALL = [(16, 8, 40, 0), (32, 16, 64, 3), (64, 32, 128, 1), (32, 64, 64, 0)]
STOP = ["max_iterations", "tolerance", "divergence"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _load(n, M, Q, seed):
    return np.load(os.path.join(GOLDEN, f"scene_{n}_{M}_{Q}_{seed}.npz"))


def test_geometry_matches_reference(oracle):
    for rec in json.load(open(os.path.join(GOLDEN, "geometry.json"))):
        if rec.get("custom"):
            continue
        if rec["n"] > 512:
            continue  # 1024^2 phantom is covered by test_host (same generator)
        s = oracle.make_scene(rec["n"], rec["M"], rec["Q"], rec["seed"])
        pix = np.empty((s.ny, s.nx, 2))
        pix[:, :, 0] = s.xx[None, :]
        pix[:, :, 1] = s.yy[:, None]
        assert sha(pix.reshape(-1, 2)) == rec["pixel_coords"]
        assert sha(s.pos) == rec["positions"]
        assert sha(s.phantom) == rec["phantom"]
        assert s.dt.hex() == rec["dt"]


@pytest.mark.parametrize("scene", SMALL)
def test_products_bit_exact(oracle, scene):
    g = _load(*scene)
    s = oracle.make_scene(*scene)
    op = oracle.Operator.of(s)
    assert np.array_equal(op.forward(s.phantom), g["y"])
    assert np.array_equal(op.adjoint(g["r"]), g["KTr"])


@pytest.mark.parametrize("scene", SMALL)
def test_reconstruction_bit_exact(oracle, scene):
    g = _load(*scene)
    s = oracle.make_scene(*scene)
    op = oracle.Operator.of(s)
    alpha, beta, step = g["pinned"]
    variants = {
        "default": dict(iterations=10),
        "nonneg": dict(iterations=10, nonneg=True),
        "tolerance": dict(iterations=40, tolerance=0.2),
        "divergence": dict(iterations=50, step_override=1e9),
        "data_only": dict(iterations=10, zero_reg=True),
    }
    for name, kw in variants.items():
        a, b, st = alpha, beta, step
        if kw.pop("zero_reg", False):
            a, b = 0.0, 0.0
        st = kw.pop("step_override", st)
        out = oracle.reconstruct(op, g["y"], a, b, st, **kw)
        meta = g[f"{name}_meta"]
        assert out["iterations_run"] == int(meta[0]), name
        assert out["stopped_by"] == STOP[int(meta[1])], name
        assert np.array_equal(out["image"], g[f"{name}_image"]), name
        h = np.stack([out["objective_history"], out["data_term_history"], out["l1_history"],
                      out["tv_history"]])
        assert np.array_equal(h, g[f"{name}_hist"]), name


@pytest.mark.parametrize("scene", SMALL[:3])
def test_calibration_matches_reference(oracle, scene):
    g = _load(*scene)
    s = oracle.make_scene(*scene)
    op = oracle.Operator.of(s)
    a, b = oracle.resolve_regularization(op, g["y"])
    assert a == g["pinned"][0] and b == g["pinned"][1]  # serial adjoint: bit-exact
    st = oracle.resolve_step(op, b, 1e-3)
    assert st == pytest.approx(g["pinned"][2], rel=1e-12)  # reference uses BLAS GEMV


def test_known_answer_delays(oracle):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    for case in kat["delays"]:
        dt = float.fromhex(case["dt"])
        op = oracle.Operator([0.0], [0.0], [[float.fromhex(case["radius"]), 0.0]], case["c"], dt, case["q"])
        K = op.dense()
        col = K[:, 0]
        nz = np.flatnonzero(col)
        assert nz.tolist() == case["rows"]
        assert [float(v).hex() for v in col[nz]] == case["vals"]


def test_truncation_case(oracle):
    t = json.load(open(os.path.join(GOLDEN, "kat.json")))["truncation"]
    xx, yy = oracle.pixel_vectors(16, 16, 1e-4, oracle.centred_origin(16, 16, 1e-4))
    pos = oracle.ring_positions(4, 5e-3)
    op = oracle.Operator(xx, yy, pos, 1500.0, 1e-7, 8)
    assert op.truncated_pairs() == t["truncated_pairs"]
    x = np.random.default_rng(3).standard_normal(256)
    r = np.random.default_rng(4).standard_normal(op.rows)
    np.testing.assert_allclose(op.forward(x), t["Kx"], rtol=1e-13, atol=1e-20)
    np.testing.assert_allclose(op.adjoint(r), t["KTr"], rtol=1e-13, atol=1e-20)


def test_config1_reference_run(oracle):
    """BASELINE config 1 (128^2, 128 x 1024, 10 iterations): y bit-exact, image bit-exact."""
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    s = oracle.make_scene(128, 128, 1024, 0)
    op = oracle.Operator.of(s)
    y = op.forward(s.phantom)
    assert sha(y) == str(g["y_sha"])
    alpha, beta, step = g["pinned"]
    out = oracle.reconstruct(op, y, alpha, beta, step, 10)
    assert out["iterations_run"] == 10
    assert oracle.rel_l2(out["image"], g["image"]) <= 1e-12
    np.testing.assert_allclose(out["objective_history"], g["hist"][0], rtol=1e-12)


def test_thread_count_independent(oracle):
    s = oracle.make_scene(32, 16, 64, 3)
    a = oracle.Operator.of(s, threads=1)
    b = oracle.Operator.of(s, threads=5)
    assert np.array_equal(a.forward(s.phantom), b.forward(s.phantom))
    r = np.random.default_rng(0).standard_normal(a.rows)
    assert np.array_equal(a.adjoint(r), b.adjoint(r))


def test_frequency_operator_matches_reference(oracle):
    """The frequency-domain oracle (forward.py:218-234) against the reference's own products
    and 10-iteration reconstruction (tests/golden/freq_16_8_40_0.npz)."""
    g = np.load(os.path.join(GOLDEN, "freq_16_8_40_0.npz"))
    s = oracle.make_scene(16, 8, 40, 0)
    op = oracle.FreqDense(s, int(g["q_n"]))
    y = op.forward(s.phantom)
    assert np.max(np.abs(y - g["y"])) <= 1e-14 * np.max(np.abs(g["y"]))
    khr = op.adjoint(g["r"])
    assert np.max(np.abs(khr - g["KHr"])) <= 1e-13 * np.max(np.abs(g["KHr"]))
    alpha, beta, step = g["pinned"]
    a2, b2 = oracle.resolve_regularization(op, g["y"])
    assert abs(a2 - alpha) <= 1e-12 * alpha and abs(b2 - beta) <= 1e-12 * beta
    out = oracle.reconstruct(op, g["y"], alpha, beta, step, 10)
    assert out["iterations_run"] == int(g["meta"][0])
    assert oracle.rel_l2(out["image"], g["image"]) <= 1e-12
    np.testing.assert_allclose(out["objective_history"], g["hist"][0], rtol=1e-12)


@pytest.mark.parametrize("sc", [(64, 32, 128, 1), (128, 128, 1024, 0)])
def test_c_index_equals_numpy_hypot(oracle, sc):
    """The C oracle's index rule (glibc hypot, / c dt, floor) is numpy's bit for bit -- it is
    the reference index of the large-config census (tests/test_gpu_census.py)."""
    n, M, Q, seed = sc
    s = oracle.make_scene(n, M, Q, seed)
    s0, fr = oracle.Operator.of(s).index()
    ref_s0, ref_fr = oracle.numpy_index(s.xx, s.yy, s.pos, s.c, s.dt)
    assert np.array_equal(s0, ref_s0) and np.array_equal(fr, ref_fr)
