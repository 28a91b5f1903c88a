"""Generate the golden fixtures of tests/golden/ by running the REFERENCE itself.

Run in the build container only (needs /root/reference; the GPU box does not have it):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py [--cfg1]

Fixtures (all small):
  geometry.json     sha256 of pixel_coords / ring.positions / phantom bytes and dt for a
                    list of make_scene() calls (pins the host geometry mirror bit-exact)
  kat.json          known-answer delays of the reference's own tests (test_forward.py:51-92)
  scene_<n>_<M>_<Q>_<seed>.npz
                    y = forward_project(K, phantom), K^T of a seeded trace, pinned config
                    (resolve_config), 10-iteration reconstructions (default / nonneg /
                    tolerance / divergence variants) with histories
  cfg1.npz          BASELINE config 1 (128^2, 128 x 1024, 10 it): sha256(y), pinned config,
                    image and histories of the reference's iterative_reconstruct (--cfg1;
                    needs ~17 GB RAM for the dense matrix)
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

import pactkit as pk

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


GEOM_SCENES = [(16, 8, 40, 0), (32, 16, 64, 3), (64, 32, 128, 1), (128, 128, 1024, 0),
               (256, 256, 2048, 0), (512, 512, 2048, 0), (1024, 1024, 4096, 0),
               (256, 256, 2048, 1), (256, 256, 2048, 7), (64, 64, 64, 11)]
SMALL = [(16, 8, 40, 0), (32, 16, 64, 3), (64, 32, 128, 1), (32, 64, 64, 0)]


def geometry():
    out = []
    for n, M, Q, seed in GEOM_SCENES:
        g, ring, ac, ph = pk.make_scene(n, M, Q, seed=seed)
        out.append({"n": n, "M": M, "Q": Q, "seed": seed, "dt": ac.dt.hex(),
                    "radius": ring.radius.hex(), "origin": [v.hex() for v in g.origin],
                    "pixel_coords": sha(g.pixel_coords()), "positions": sha(ring.positions),
                    "phantom": sha(ph.values), "phantom_nnz": int(np.count_nonzero(ph.values))})
    # non-centred grid / off-centre ring
    g = pk.make_grid(24, 20, 2e-4, (1e-3, -2e-3))
    ring = pk.make_ring(12, 9e-3, (3.3e-3, -0.1e-3), g)
    out.append({"custom": True, "pixel_coords": sha(g.pixel_coords()), "positions": sha(ring.positions),
                "phantom": sha(pk.make_vessel_phantom(g, 5, 3).values)})
    json.dump(out, open(os.path.join(HERE, "geometry.json"), "w"), indent=1)


def kat():
    cases = []
    ac = pk.AcousticConfig(c=2048.0, dt=2.0**-13, q_s=32, q_n=32)
    grid = pk.make_grid(1, 1, 1e-6, (0, 0))
    for delay in (10.0, 10.5):
        ring = pk.make_ring(1, delay * ac.dt * ac.c, (0, 0), grid)
        K = pk.build_time_matrix(grid, ring, ac)
        col = K.entries[:, 0]
        nz = np.flatnonzero(col)
        cases.append({"c": ac.c, "dt": ac.dt.hex(), "q": ac.q_s, "radius": ring.radius.hex(),
                      "rows": nz.tolist(), "vals": [float(col[i]).hex() for i in nz]})
    ac = pk.AcousticConfig(c=1500.0, dt=1e-7, q_s=64, q_n=64)
    rng = np.random.default_rng(0)
    for _ in range(10):
        radius = float(rng.uniform(2.0, 60.0) * ac.dt * ac.c)
        ring = pk.make_ring(1, radius, (0, 0), grid)
        K = pk.build_time_matrix(grid, ring, ac)
        col = K.entries[:, 0]
        nz = np.flatnonzero(col)
        cases.append({"c": ac.c, "dt": ac.dt.hex(), "q": ac.q_s, "radius": ring.radius.hex(),
                      "rows": nz.tolist(), "vals": [float(col[i]).hex() for i in nz]})
    # truncation: window far too short (test_forward.py:123-132)
    g = pk.centered_grid(16, 16, 1e-4)
    ring = pk.make_ring(4, 5e-3, (0, 0), g)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        K = pk.build_time_matrix(g, ring, pk.AcousticConfig(c=1500.0, dt=1e-7, q_s=8, q_n=8))
    x = np.random.default_rng(3).standard_normal(g.size)
    r = np.random.default_rng(4).standard_normal(K.rows)
    trunc = {"truncated_pairs": K.provenance["truncated_pairs"], "Kx": (K.entries @ x).tolist(),
             "KTr": (K.entries.T @ r).tolist()}
    json.dump({"delays": cases, "truncation": trunc}, open(os.path.join(HERE, "kat.json"), "w"), indent=1)


def small():
    for n, M, Q, seed in SMALL:
        g, ring, ac, ph = pk.make_scene(n, M, Q, seed=seed)
        K = pk.build_time_matrix(g, ring, ac)
        y = pk.forward_project(K, ph)
        r = np.random.default_rng(17).standard_normal(K.rows)
        kt = pk.kernels.matvec_adjoint_serial(K.entries, r)
        cfg = pk.resolve_config(pk.ReconConfig(iterations=10), K, y)
        res = {}
        variants = {
            "default": cfg,
            "nonneg": pk.ReconConfig(cfg.alpha, cfg.beta, 10, cfg.step, nonneg=True),
            "tolerance": pk.ReconConfig(cfg.alpha, cfg.beta, 40, cfg.step, tolerance=0.2),
            "divergence": pk.ReconConfig(cfg.alpha, cfg.beta, 50, 1e9),
            "data_only": pk.ReconConfig(0.0, 0.0, 10, cfg.step),
        }
        for name, c in variants.items():
            out = pk.iterative_reconstruct(K, y, c)
            res[name] = out
        arrays = {"y": y.values, "r": r, "KTr": kt,
                  "pinned": np.array([cfg.alpha, cfg.beta, cfg.step])}
        for name, out in res.items():
            arrays[f"{name}_image"] = out.image.values
            arrays[f"{name}_hist"] = np.stack([out.objective_history, out.data_term_history,
                                               out.l1_history, out.tv_history])
            arrays[f"{name}_meta"] = np.array([out.iterations_run,
                                               ["max_iterations", "tolerance", "divergence"].index(out.stopped_by),
                                               out.step_used])
        np.savez_compressed(os.path.join(HERE, f"scene_{n}_{M}_{Q}_{seed}.npz"), **arrays)
        print("wrote scene", n, M, Q, seed, {k: (v.iterations_run, v.stopped_by) for k, v in res.items()})


def freq():
    """Frequency-domain operator (build_freq_matrix, forward.py:218-234): products and a
    10-iteration reconstruction of the reference on a small scene."""
    g, ring, ac, ph = pk.make_scene(16, 8, 40, seed=0)
    ac = pk.AcousticConfig(c=ac.c, dt=ac.dt, q_s=ac.q_s, q_n=12)
    K = pk.build_freq_matrix(g, ring, ac)
    y = pk.forward_project(K, ph)
    rng = np.random.default_rng(21)
    r = rng.standard_normal(K.rows) + 1j * rng.standard_normal(K.rows)
    khr = pk.kernels.matvec_adjoint_serial(K.entries, r)
    cfg = pk.resolve_config(pk.ReconConfig(iterations=10), K, y)
    out = pk.iterative_reconstruct(K, y, cfg)
    np.savez_compressed(os.path.join(HERE, "freq_16_8_40_0.npz"),
                        q_n=np.array(12), y=y.values, r=r, KHr=khr,
                        pinned=np.array([cfg.alpha, cfg.beta, cfg.step]), image=out.image.values,
                        hist=np.stack([out.objective_history, out.data_term_history,
                                       out.l1_history, out.tv_history]),
                        meta=np.array([out.iterations_run,
                                       ["max_iterations", "tolerance", "divergence"].index(out.stopped_by)]))
    print("wrote freq fixture", out.iterations_run, out.stopped_by, cfg)


def cfg1():
    t = time.time()
    g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
    K = pk.build_time_matrix(g, ring, ac)
    y = pk.forward_project(K, ph, pool=pk.WorkerPool())
    cfg = pk.resolve_config(pk.ReconConfig(iterations=10), K, y)
    out = pk.iterative_reconstruct(K, y, cfg, pool=pk.WorkerPool())
    np.savez_compressed(
        os.path.join(HERE, "cfg1.npz"),
        y_sha=np.array(sha(y.values)), y_norm=np.array(np.linalg.norm(y.values)),
        pinned=np.array([cfg.alpha, cfg.beta, cfg.step]),
        image=out.image.values,
        hist=np.stack([out.objective_history, out.data_term_history, out.l1_history, out.tv_history]),
        meta=np.array([out.iterations_run, 0]),
    )
    print("cfg1 done in", time.time() - t, "s; pinned", cfg.alpha, cfg.beta, cfg.step)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg1", action="store_true")
    ap.add_argument("--only-freq", action="store_true")
    a = ap.parse_args()
    if a.only_freq:
        freq()
        sys.exit(0)
    geometry()
    kat()
    small()
    freq()
    if a.cfg1:
        cfg1()
