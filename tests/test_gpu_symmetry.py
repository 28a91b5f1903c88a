"""The symmetric kernels (D4 back-projector, rotation projector) against the generic ones
and the fp64 oracle.  Every BASELINE scene (centred square grid, M % 4 == 0) selects them
automatically; PK_SYM / PK_FSYM = 0 forces the generic kernels."""

import numpy as np
import pytest

import paper_2404_10928_b200 as pk

pytestmark = pytest.mark.gpu
F32 = pk.CudaPool(0, "float32")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _plan(monkeypatch, g, ring, ac, sym, fsym):
    monkeypatch.setenv("PK_SYM", sym)
    monkeypatch.setenv("PK_FSYM", fsym)
    pk.clear_plan_cache()
    return pk.operator_for(g, ring, ac, F32)


@pytest.mark.parametrize("cfg", [(64, 32, 128), (96, 64, 512), (128, 128, 1024), (256, 256, 2048)])
def test_symmetric_products_match_oracle(monkeypatch, oracle, cfg):
    n, M, Q = cfg
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=2)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 2))
    op = _plan(monkeypatch, g, ring, ac, "1", "1")
    # both symmetric kernels forced on; the projector's quadrant strips are 64 or 32 columns
    # wide (whichever stores fewer window words per projection)
    assert op.info.symmetric == 3
    assert op.info.fp_tile in (32, 64)
    rng = np.random.default_rng(9)
    x = ph.values + 0.05 * rng.random(g.size)          # dense, non-negative
    assert rel(op.matvec(x).double().cpu().numpy(), o.forward(x)) <= 5e-5
    y = o.forward(ph.values)                              # a smooth measured trace
    assert rel(op.adjoint(y).double().cpu().numpy(), o.adjoint(y)) <= 2e-5
    pk.clear_plan_cache()


@pytest.mark.parametrize("sym,fsym", [("1", "1"), ("1", "0"), ("0", "0")])
def test_symmetric_and_generic_reconstructions_agree(monkeypatch, oracle, sym, fsym):
    n, M, Q = 128, 128, 1024
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=0)
    K = pk.build_time_matrix(g, ring, ac)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 0))
    y = o.forward(ph.values)
    alpha, beta = oracle.resolve_regularization(o, y)
    step = oracle.resolve_step(o, beta, 1e-3)
    ref = oracle.reconstruct(o, y, alpha, beta, step, 10)
    op = _plan(monkeypatch, g, ring, ac, sym, fsym)
    assert op.info.symmetric & 1 == int(sym)
    res = pk.iterative_reconstruct(K, pk.SensorData("time", M, Q, y),
                                   pk.ReconConfig(alpha, beta, 10, step), pool=F32)
    assert res.iterations_run == 10
    assert rel(res.image.values, ref["image"]) <= 1e-4
    np.testing.assert_allclose(res.objective_history, ref["objective_history"], rtol=1e-5)
    pk.clear_plan_cache()


def test_symmetric_projector_deterministic(monkeypatch):
    g, ring, ac, ph = pk.make_scene(64, 32, 128, seed=1)
    K = pk.build_time_matrix(g, ring, ac)
    _plan(monkeypatch, g, ring, ac, "1", "1")
    y1 = pk.forward_project(K, ph, pool=F32)
    y2 = pk.forward_project(K, ph, pool=F32)
    assert np.array_equal(y1.values, y2.values)
    grad = pk.data_gradient(K, ph, y1, pool=F32)
    assert np.max(np.abs(grad.values)) <= 1e-18
    # the symmetric back-projector adds its partial slots in a fixed order: bitwise repeatable
    rng = np.random.default_rng(3)
    r = pk.SensorData("time", 32, 128, rng.standard_normal(32 * 128))
    b1 = pk.back_project(K, r, pool=F32)
    b2 = pk.back_project(K, r, pool=F32)
    assert np.array_equal(b1.values, b2.values)
    pk.clear_plan_cache()


@pytest.mark.parametrize("scale", [1e-30, 1.0, 1e25])
def test_symmetric_adjoint_fixed_point_range(monkeypatch, oracle, scale):
    """The symmetric back-projector (fp32 partial slots summed in a fixed order) keeps fp32
    relative accuracy for tiny and huge traces."""
    n, M, Q = 96, 64, 512
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=4)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 4))
    op = _plan(monkeypatch, g, ring, ac, "1", "0")
    assert op.info.symmetric & 1
    rng = np.random.default_rng(5)
    y = scale * rng.standard_normal(M * Q)
    assert rel(op.adjoint(y).double().cpu().numpy(), o.adjoint(y)) <= 2e-4
    pk.clear_plan_cache()


@pytest.mark.parametrize("variant", ["nonneg", "tolerance", "divergence"])
def test_symmetric_kernels_solver_variants(monkeypatch, oracle, variant):
    """Symmetric back-projector + projector (forced on) through the stopping rules and the
    non-negativity clamp, on a ring whose sensor count is not a multiple of 32 (a partial
    sensor group) and a grid whose quadrant is not a multiple of the tiles."""
    n, M, Q = 96, 36, 512
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=5)
    K = pk.build_time_matrix(g, ring, ac)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 5))
    y = o.forward(ph.values)
    alpha, beta = oracle.resolve_regularization(o, y)
    step = oracle.resolve_step(o, beta, 1e-3)
    kw = {"nonneg": dict(iterations=10, nonneg=True),
          "tolerance": dict(iterations=40, tolerance=0.2),
          "divergence": dict(iterations=50)}[variant]
    st = 1e9 if variant == "divergence" else step
    ref = oracle.reconstruct(o, y, alpha, beta, st, **kw)
    op = _plan(monkeypatch, g, ring, ac, "1", "1")
    assert op.info.symmetric == 3
    res = pk.iterative_reconstruct(K, pk.SensorData("time", M, Q, y),
                                   pk.ReconConfig(alpha, beta, step=st, **kw), pool=F32)
    assert res.iterations_run == ref["iterations_run"]
    assert res.stopped_by == ref["stopped_by"]
    if variant != "divergence":
        assert rel(res.image.values, ref["image"]) <= 1e-4
    pk.clear_plan_cache()


def test_symmetric_kernels_truncated_window(monkeypatch, oracle):
    """Delays beyond the acquisition window (TruncationWarning scenes): the clamped paths
    of both symmetric kernels against the oracle's dropped weights."""
    import warnings

    n, M = 64, 32
    s = oracle.make_scene(n, M, 128, 0)
    Q = 100  # shorter than the farthest delay (~122 samples at 128)
    g, ring, ac, ph = pk.make_scene(n, M, 128, seed=0)
    ac = pk.AcousticConfig(c=ac.c, dt=ac.dt, q_s=Q, q_n=Q)
    o = oracle.Operator(s.xx, s.yy, s.pos, s.c, s.dt, Q)
    assert o.truncated_pairs() > 0
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        op = _plan(monkeypatch, g, ring, ac, "1", "1")
    assert op.info.symmetric & 1
    rng = np.random.default_rng(8)
    x = ph.values + 0.05 * rng.random(g.size)
    assert rel(op.matvec(x).double().cpu().numpy(), o.forward(x)) <= 5e-5
    r = rng.standard_normal(M * Q)
    assert rel(op.adjoint(r).double().cpu().numpy(), o.adjoint(r)) <= 2e-4
    pk.clear_plan_cache()


def test_throughput_grid_matches_latency_grid(oracle):
    """pk_geometry_desc.concurrency > 1 halves the back-projector's persistent grid: the
    reconstruction agrees with the latency-mode plan to fp32 rounding and with the oracle."""
    import torch

    n, M, Q, N = 512, 512, 2048, 3  # occupancy-limited grid: the throughput mode halves it
    s = oracle.make_scene(n, M, Q, 0)
    o = oracle.Operator.of(s)
    y = o.forward(s.phantom)
    alpha, beta = oracle.resolve_regularization(o, y)
    step = 333.156  # survey-pinned config 3 step
    ref = oracle.reconstruct(o, y, alpha, beta, step, N)
    grid, ring, ac, _ = pk.make_scene(n, M, Q, 0)
    params = pk.solver.solver_params(pk.ReconConfig(alpha, beta, N, step), alpha, beta, step)
    xs = []
    for conc in (1, 2):
        op = pk.operator_for(grid, ring, ac, pk.CudaPool(0, "float32"), concurrency=conc)
        assert op.info.bp_split >= 1
        x, hist, status = op.reconstruct(y, params)
        torch.cuda.synchronize()
        assert int(status[0, 0]) == N
        xs.append(x[0].double().cpu().numpy())
    assert np.linalg.norm(xs[0] - xs[1]) <= 1e-5 * np.linalg.norm(xs[0])
    for xv in xs:
        assert np.linalg.norm(xv - ref["image"]) <= 1e-4 * np.linalg.norm(ref["image"])


@pytest.mark.parametrize("spin", ["20000", "0"])
def test_fused_update_matches_epilogue_kernel(monkeypatch, oracle, spin):
    """PK_SYM_FUSE=1 runs the update in the back-projector's tail (per-tile arrival counters,
    bounded wait, claimed units); the image, history and status are bitwise those of the
    separate epilogue kernel, with waiting CTAs (spin) or the final arrivers alone (0)."""
    n, M, Q = 256, 256, 2048
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=4)
    K = pk.build_time_matrix(g, ring, ac)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 4))
    y = o.forward(ph.values)
    alpha, beta = oracle.resolve_regularization(o, y)
    cfg = pk.ReconConfig(alpha, beta, 6, 2651.3)
    out = {}
    for fuse in ("0", "1"):
        monkeypatch.setenv("PK_SYM_FUSE", fuse)
        monkeypatch.setenv("PK_SYM_SPIN_NS", spin)
        pk.clear_plan_cache()
        res = [pk.iterative_reconstruct(K, pk.SensorData("time", M, Q, y), cfg, pool=F32) for _ in range(2)]
        assert np.array_equal(res[0].image.values, res[1].image.values)  # graph replay
        out[fuse] = res[1]
    pk.clear_plan_cache()
    assert np.array_equal(out["0"].image.values, out["1"].image.values)
    assert np.array_equal(out["0"].objective_history, out["1"].objective_history)
    assert out["1"].iterations_run == 6


@pytest.mark.parametrize("batch", [2, 4])
def test_batched_symmetric_frames_match_oracle(oracle, batch):
    """Batched plans keep both symmetric kernels (frame-major chunks and segments, one residual
    CTA per (trace, frame)): every frame of a 256^2 batch (BASELINE config 2/4 geometry) within
    1e-4 of its fp64 oracle solve, and equal to the single-frame plan to fp32 rounding."""
    n, M, Q, N = 256, 256, 2048, 4
    grid, ring, ac, _ = pk.make_scene(n, M, Q, 0)
    K = pk.build_time_matrix(grid, ring, ac)
    op = pk.operator_for(grid, ring, ac, F32, frames=batch)
    assert op.info.symmetric == 3 and op.info.frames == batch
    ys, refs = [], []
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 0))
    alpha, beta, step = 2.0817e-8, 2.0817e-10, 2651.30  # survey-pinned config 2
    for f in range(batch):
        s = oracle.make_scene(n, M, Q, 0)
        ph = pk.make_vessel_phantom(grid, 10 + f).values * (1.0 + f)
        y = o.forward(ph)
        ys.append(pk.SensorData("time", M, Q, y))
        refs.append(oracle.reconstruct(o, y, alpha, beta, step, N)["image"])
    cfg = pk.ReconConfig(alpha, beta, N, step)
    many = pk.reconstruct_frames(K, ys, cfg, pool=F32, batch=batch, pinned=(alpha, beta, step))
    singles = [pk.iterative_reconstruct(K, y, cfg, pool=F32) for y in ys]
    for r, s1, ref in zip(many, singles, refs):
        assert r.iterations_run == N
        assert rel(r.image.values, ref) <= 1e-4
        assert rel(r.image.values, s1.image.values) <= 1e-5
    # standalone batched products: each frame's projection and adjoint match the oracle
    rng = np.random.default_rng(5)
    xs = rng.random((batch, n * n))
    yb = op.matvec(xs.ravel()).double().cpu().numpy().reshape(batch, -1)
    rb = rng.standard_normal((batch, M * Q))
    gb = op.adjoint(rb.ravel()).double().cpu().numpy().reshape(batch, -1)
    for f in range(batch):
        assert rel(yb[f], o.forward(xs[f])) <= 5e-5
        assert rel(gb[f], o.adjoint(rb[f])) <= 2e-4
    pk.clear_plan_cache()


@pytest.mark.parametrize("lw,t", [("184", "32"), ("256", "32"), ("256", "64"), ("320", "64")])
def test_projector_window_variants_match_oracle(monkeypatch, oracle, lw, t):
    """Every staging-round schedule of the projector's bulk reductions (4 images at once,
    2 + 2 with the second round aliasing the transposed rows, 1 + 1 + waits) and both strip
    widths give the same projection (fp32 rounding of the oracle) and reconstruction."""
    n, M, Q = 256, 256, 2048
    monkeypatch.setenv("PK_FSYM_LW", lw)
    monkeypatch.setenv("PK_FSYM_T", t)
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=6)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 6))
    op = _plan(monkeypatch, g, ring, ac, "1", "1")
    assert op.info.symmetric == 3 and op.info.fp_window == int(lw) and op.info.fp_tile == int(t)
    rng = np.random.default_rng(11)
    x = ph.values + 0.05 * rng.random(g.size)
    assert rel(op.matvec(x).double().cpu().numpy(), o.forward(x)) <= 5e-5
    pk.clear_plan_cache()


def test_tuned_chunk_ranges_agree(monkeypatch, oracle):
    """The back-projector's diagonal cut weight is timed once per geometry and process: a
    second plan of the same geometry reuses the choice (bitwise equal solves), and pinned
    weights (PK_SYM_WDIAG) at both ends of the candidate range give the same image to fp32
    rounding and the oracle's to 1e-4."""
    n, M, Q, N = 128, 128, 1024, 6
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=3)
    K = pk.build_time_matrix(g, ring, ac)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, 3))
    y = o.forward(ph.values)
    alpha, beta = oracle.resolve_regularization(o, y)
    step = oracle.resolve_step(o, beta, 1e-3)
    ref = oracle.reconstruct(o, y, alpha, beta, step, N)["image"]
    cfg = pk.ReconConfig(alpha, beta, N, step)
    sd = pk.SensorData("time", M, Q, y)
    pk.clear_plan_cache()
    a = pk.iterative_reconstruct(K, sd, cfg, pool=F32)
    split_a = pk.operator_for(g, ring, ac, F32).info.bp_split
    pk.clear_plan_cache()
    b = pk.iterative_reconstruct(K, sd, cfg, pool=F32)
    assert pk.operator_for(g, ring, ac, F32).info.bp_split == split_a
    assert np.array_equal(a.image.values, b.image.values)
    imgs = []
    for w in ("18", "26"):
        monkeypatch.setenv("PK_SYM_WDIAG", w)
        pk.clear_plan_cache()
        imgs.append(pk.iterative_reconstruct(K, sd, cfg, pool=F32).image.values)
    pk.clear_plan_cache()
    assert rel(imgs[0], imgs[1]) <= 1e-5
    for im in imgs + [a.image.values]:
        assert rel(im, ref) <= 1e-4


@pytest.mark.parametrize("frames", [1, 2, 4])
def test_multi_strip_epilogue_matches_one_strip_kernel(monkeypatch, frames):
    """The solver epilogue with one CTA per (tile, image, block of 2 or 4 strips)
    (bp_sym_epik_kernel; 2 strips by default) is bitwise
    the one-strip kernel (PK_SYM_EPIK=1): same slot order per pixel, the skipped zero padding
    is exact.  Image, history and status, one frame and 2- and 4-frame batches."""
    n, M, Q, N = 256, 256, 2048, 6
    grid, ring, ac, ph = pk.make_scene(n, M, Q, 5)
    alpha, beta, step = 2.0817e-8, 2.0817e-10, 2651.30  # survey-pinned config 2
    params = pk.solver.solver_params(pk.ReconConfig(alpha, beta, N, step), alpha, beta, step)
    out = {}
    for ks in ("1", "2", "4"):
        monkeypatch.setenv("PK_SYM_EPIK", ks)
        pk.clear_plan_cache()
        op = pk.operator_for(grid, ring, ac, F32, frames=frames)
        assert op.info.symmetric == 3
        y = op.matvec(np.tile(ph.values, frames))
        runs = [[t.cpu().numpy() for t in op.reconstruct(y, params)] for _ in range(2)]
        for a_, b_ in zip(runs[0], runs[1]):
            assert np.array_equal(a_, b_)  # graph replay
        out[ks] = runs[1]
    pk.clear_plan_cache()
    assert (out["1"][2][:, 0] == N).all()
    for ks in ("2", "4"):
        for a_, b_ in zip(out["1"], out[ks]):
            assert np.array_equal(a_, b_)
