"""Explicit-matrix mode on the device: a MeasurementMatrix given by its
entries (read_matrix / PACTMAT, forward.py:70-121, 297-330) runs the hand-written pk_dense_*
kernels -- streaming GEMV / GEMV^H (the reference's kernels.py:195-225) and the device-resident
solver loop (recon.py:286-377).  Checked against numpy products of the same entries, the
reference's own reconstructions (tests/golden), and BASELINE config 1's dense K (17.2 GB,
formed on the device bit-identical to build_time_matrix) against the reference's output."""

import os

import numpy as np
import pytest

import paper_2404_10928_b200 as pk
from conftest import GOLDEN
from paper_2404_10928_b200 import measurement as meas

pytestmark = pytest.mark.gpu

F32 = pk.CudaPool(0, "float32")
F64 = pk.CudaPool(0, "float64")
SMALL = [(16, 8, 40, 0), (32, 16, 64, 3), (64, 32, 128, 1), (32, 64, 64, 0)]
STOP = ["max_iterations", "tolerance", "divergence"]
PROD_TOL = {"float32": 2e-6, "float64": 1e-13}
IMG_TOL = {"float32": 1e-4, "float64": 1e-10}


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("pool", [F32, F64], ids=["f32", "f64"])
def test_dense_products_vs_numpy(pool):
    tol = PROD_TOL[pool.dtype]
    rng = np.random.default_rng(2)
    g, ring, ac, ph = pk.make_scene(32, 16, 64, seed=3)
    A = pk.build_time_matrix(g, ring, ac).entries  # the reference's dense K (fp64 index rule)
    op = meas.DenseOperator(A, pool)
    x = rng.standard_normal(A.shape[1])
    xc = x + 1j * rng.standard_normal(A.shape[1])
    y = rng.standard_normal(A.shape[0])
    yc = y + 1j * rng.standard_normal(A.shape[0])
    assert rel(op.matvec(x).cpu().numpy(), A @ x) <= tol
    assert rel(op.matvec(xc).cpu().numpy(), A @ xc) <= tol
    assert rel(op.adjoint(y, 2.0).cpu().numpy(), 2.0 * (A.T @ y)) <= tol
    assert rel(op.adjoint(yc).cpu().numpy(), A.T @ yc) <= tol
    # complex entries: the frequency-domain K (build_freq_matrix, forward.py:218-234)
    grid, ring, ac, ph = pk.make_scene(16, 8, 40, seed=0)
    Af = pk.build_freq_matrix(grid, ring, ac).entries
    opf = meas.DenseOperator(Af, pool)
    assert opf.cplx and opf.info.complex_entries == 1
    x = rng.standard_normal(Af.shape[1])
    yc = rng.standard_normal(Af.shape[0]) + 1j * rng.standard_normal(Af.shape[0])
    assert rel(opf.matvec(x).cpu().numpy(), Af @ x) <= tol
    assert rel(opf.matvec(x + 1j * x[::-1]).cpu().numpy(), Af @ (x + 1j * x[::-1])) <= tol
    assert rel(opf.adjoint(yc, 3.0).cpu().numpy(), 3.0 * (Af.conj().T @ yc)) <= tol
    with pytest.raises(ValueError):
        op.matvec(np.zeros(A.shape[1] + 1))


def test_dense_rejects_unaligned_rows():
    """Rows must fill whole 16-byte loads (2 fp64 / 4 fp32 columns)."""
    from paper_2404_10928_b200._native import PkError

    with pytest.raises(PkError):
        meas.DenseOperator(np.ones((4, 7)), F64)


@pytest.mark.parametrize("pool", [F32, F64], ids=["f32", "f64"])
@pytest.mark.parametrize("twopass", [False, True], ids=["auto", "twopass"])
def test_dense_reconstruction_vs_reference_golden(pool, twopass, monkeypatch):
    """Explicit K solves against the reference's own reconstructions: 4 scenes x 5 variants
    (default, nonneg, tolerance stop, divergence stop, data only)."""
    if twopass:
        monkeypatch.setenv("PK_DENSE_TWOPASS", "1")
    meas._dense_cache.clear()
    for sc in SMALL:
        n, M, Q, seed = sc
        g, ring, ac, ph = pk.make_scene(n, M, Q, seed=seed)
        gold = np.load(os.path.join(GOLDEN, f"scene_{n}_{M}_{Q}_{seed}.npz"))
        A = pk.build_time_matrix(g, ring, ac).entries
        K = pk.MeasurementMatrix("time", A, {"grid": g})
        op = meas.device_operator(K, pool)
        assert isinstance(op, meas.DenseOperator)
        assert op.info.fused == int(pool.dtype == "float32" and not twopass)
        alpha, beta, step = gold["pinned"]
        y = pk.SensorData("time", M, Q, gold["y"])
        variants = {
            "default": pk.ReconConfig(alpha, beta, 10, step),
            "nonneg": pk.ReconConfig(alpha, beta, 10, step, nonneg=True),
            "tolerance": pk.ReconConfig(alpha, beta, 40, step, tolerance=0.2),
            "divergence": pk.ReconConfig(alpha, beta, 50, 1e9),
            "data_only": pk.ReconConfig(0.0, 0.0, 10, step),
        }
        for name, cfg in variants.items():
            res = pk.iterative_reconstruct(K, y, cfg, pool=pool)
            meta = gold[f"{name}_meta"]
            assert res.iterations_run == int(meta[0]), (sc, name)
            assert res.stopped_by == STOP[int(meta[1])], (sc, name)
            if name != "divergence":
                assert rel(res.image.values, gold[f"{name}_image"]) <= IMG_TOL[pool.dtype], (sc, name)
                h = np.stack([res.objective_history, res.data_term_history, res.l1_history,
                              res.tv_history])
                np.testing.assert_allclose(h, gold[f"{name}_hist"], rtol=IMG_TOL[pool.dtype], atol=1e-300)
    meas._dense_cache.clear()


@pytest.mark.parametrize("pool", [F32, F64], ids=["f32", "f64"])
def test_dense_frequency_reconstruction_vs_reference(pool):
    """Explicit complex K (the frequency-domain matrix) against the reference's own run."""
    gl = np.load(os.path.join(GOLDEN, "freq_16_8_40_0.npz"))
    grid, ring, ac, ph = pk.make_scene(16, 8, 40, seed=0)
    ac = pk.AcousticConfig(c=ac.c, dt=ac.dt, q_s=ac.q_s, q_n=int(gl["q_n"]))
    A = pk.build_freq_matrix(grid, ring, ac).entries
    K = pk.MeasurementMatrix("frequency", A, {"grid": grid})
    alpha, beta, step = (float(v) for v in gl["pinned"])
    ys = pk.SensorData("frequency", ring.count, ac.q_n, gl["y"])
    res = pk.iterative_reconstruct(K, ys, pk.ReconConfig(alpha, beta, 10, step), pool=pool)
    assert res.iterations_run == int(gl["meta"][0])
    assert rel(res.image.values, gl["image"]) <= IMG_TOL[pool.dtype]
    np.testing.assert_allclose(res.objective_history, gl["hist"][0], rtol=IMG_TOL[pool.dtype])


@pytest.mark.slow
@pytest.mark.parametrize("pool", [F64, F32], ids=["f64", "f32"])
def test_config1_dense_vs_reference(pool):
    """BASELINE config 1 with the reference's dense K (131072 x 16384, formed on the device,
    fp64 bit-identical to build_time_matrix): products against the geometry kernels and the
    10-iteration reconstruction against the reference's own output (tests/golden/cfg1.npz)."""
    import torch

    gold = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
    Kg = pk.build_time_matrix(g, ring, ac)
    Kd = pk.dense_time_matrix(g, ring, ac, pool)
    try:
        y_geo = pk.forward_project(Kg, ph, pool=F64)
        y_den = pk.forward_project(Kd, ph)
        assert rel(y_den.values, y_geo.values) <= PROD_TOL[pool.dtype] * 10
        r = np.random.default_rng(1).standard_normal(Kd.rows)
        a_den = Kd.dense_operator.adjoint(r).double().cpu().numpy()
        a_geo = pk.operator_for(g, ring, ac, F64).adjoint(r).cpu().numpy()
        assert rel(a_den, a_geo) <= PROD_TOL[pool.dtype] * 10
        alpha, beta, step = gold["pinned"]
        res = pk.iterative_reconstruct(Kd, y_geo, pk.ReconConfig(alpha, beta, 10, step), pool=pool)
        assert res.iterations_run == 10
        err = rel(res.image.values, gold["image"])
        print(f"config 1 dense {pool.dtype}: image rel L2 vs reference {err:.3e}")
        assert err <= IMG_TOL[pool.dtype]
        np.testing.assert_allclose(res.objective_history, gold["hist"][0], rtol=1e-5)
    finally:
        Kd.dense_operator.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("frames", [1, 5, 32, 64, 100])
def test_tensor_core_products_vs_numpy(frames):
    """Frame-batched products on the tensor cores (pk_dense_matmat / rmatmat: tcgen05 tf32 with
    the 3xTF32 split, TMEM accumulation drained every 128 products into fp32): every frame of
    K X and K^T Y against the fp64 numpy products of the same fp32 entries, at fp32 accuracy,
    including frame counts that are not a multiple of the tile (zero-padded frames not stored)
    and split-K reductions."""
    rng = np.random.default_rng(frames)
    g, ring, ac, ph = pk.make_scene(64, 32, 256, seed=1)
    A = pk.build_time_matrix(g, ring, ac).entries  # 8192 x 4096
    op = meas.DenseOperator(A, F32)
    try:
        A32 = A.astype(np.float32).astype(np.float64)
        X = rng.random((frames, A.shape[1]))
        Y = rng.standard_normal((frames, A.shape[0]))
        Xf, Yf = X.astype(np.float32).astype(np.float64), Y.astype(np.float32).astype(np.float64)
        got = op.matmat(X).double().cpu().numpy()
        ref = Xf @ A32.T
        assert got.shape == (frames, A.shape[0])
        for f in range(frames):
            assert rel(got[f], ref[f]) <= 1e-5
        gt = op.rmatmat(Y).double().cpu().numpy()
        reft = Yf @ A32
        for f in range(frames):
            assert rel(gt[f], reft[f]) <= 1e-5
        # one frame through the tensor cores agrees with the streaming GEMV
        assert rel(got[0], op.matvec(X[0]).double().cpu().numpy()) <= 1e-5
    finally:
        op.close()


@pytest.mark.slow
def test_tensor_core_products_config1():
    """BASELINE config 1's dense K (131072 x 16384, formed on the device) with 64 frames
    through the tensor cores: each frame equals the geometry kernels' fp64 product to fp32
    accuracy (the forward splits no K; the adjoint runs split-K over 131072 rows)."""
    import torch

    g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
    Kd = pk.dense_time_matrix(g, ring, ac, F32)
    op64 = pk.operator_for(g, ring, ac, F64)
    try:
        rng = np.random.default_rng(7)
        X = np.stack([pk.make_vessel_phantom(g, s).values for s in range(60)] + [rng.random(g.size) for _ in range(4)])
        got = Kd.dense_operator.matmat(X).double().cpu().numpy()
        for f in (0, 17, 59, 63):
            assert rel(got[f], op64.matvec(X[f]).cpu().numpy()) <= 1e-5
        R = rng.standard_normal((8, Kd.rows))
        gt = Kd.dense_operator.rmatmat(R).double().cpu().numpy()
        for f in (0, 7):
            assert rel(gt[f], op64.adjoint(R[f]).cpu().numpy()) <= 1e-5
    finally:
        Kd.dense_operator.close()
        torch.cuda.empty_cache()
