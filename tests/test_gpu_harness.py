"""The reference's benchmark harness (pactkit/bench.py:206-340) with the device path:
bench_recon / profile_breakdown report shapes, verification and breakdown invariants, and
the report type on the CPU (no compute)."""
import json

import numpy as np
import pytest

import paper_2404_10928_b200 as pk
from paper_2404_10928_b200.harness import BenchEntry, BenchReport


def test_report_type_cpu():
    r = BenchReport("s")
    r.entries += [BenchEntry("a", 1.0, 2, "x"), BenchEntry("b", 0.5, 2, "y", True)]
    r.speedups.append({"baseline": "a", "candidate": "b", "speedup": 2.0,
                       "below_measurement_floor": False})
    r.breakdown = {"gradient_products": {"seconds": 0.9, "percent": 90.0}}
    assert r.entry("b").verification is True and r.speedup("a", "b") == 2.0
    assert r.verification_ok()
    d = json.loads(r.to_json())
    assert d["verification"] and [e["label"] for e in d["entries"]] == ["a", "b"]
    assert "speedup a -> b: 2.00x" in r.to_text()
    r.entries.append(BenchEntry("c", 1.0, 1, "z", False))
    assert not r.verification_ok()
    with pytest.raises(KeyError):
        r.entry("missing")
    with pytest.raises(KeyError):
        r.speedup("b", "a")


@pytest.mark.gpu
def test_bench_recon_device():
    rep = pk.bench_recon(64, 32, 128, pk.ReconConfig(iterations=10), reps=2)
    assert [e.label for e in rep.entries] == ["back_projection", "iterative_serial",
                                              "iterative_parallel"]
    assert rep.verification_ok(), rep.metrics
    assert rep.metrics["rel_l2_f32_vs_f64"] <= 1e-4
    assert all(len(e.checksum) == 64 and e.wall_seconds > 0 for e in rep.entries)
    assert rep.speedup("iterative_serial", "iterative_parallel") > 0
    assert 0.0 <= rep.metrics["rmse_ir"] < rep.metrics["rmse_bp"]  # IR beats BP (bench.py:243)


@pytest.mark.gpu
def test_profile_breakdown_device():
    rep = pk.profile_breakdown(64, 32, 128, pk.ReconConfig(iterations=6))
    assert set(rep.breakdown) == {"gradient_products", "tv_gradient", "prox", "objective", "other"}
    total = sum(v["percent"] for v in rep.breakdown.values())
    assert abs(total - 100.0) < 1e-6
    assert rep.breakdown["gradient_products"]["seconds"] > 0
    assert rep.metrics["iterations_run"] == 6 and rep.metrics["kernel_launches"] > 0
    assert rep.entry("iterative_run").wall_seconds > 0


@pytest.mark.gpu
def test_bench_recon_verified_against_oracle(oracle):
    """The harness's verification with the CPU oracle in the reference's serial-kernel role
    (bench.py:230-235): fp64 device image <= 1e-10, fp32 <= 1e-4 of the oracle's."""

    def ref(K, y, cfg):
        o = oracle.Operator(*K.grid.axis_vectors(), K.ring.positions, K.acoustic.c,
                            K.acoustic.dt, K.acoustic.q_s)
        return oracle.reconstruct(o, y.values, cfg.alpha, cfg.beta, cfg.step, cfg.iterations)["image"]

    rep = pk.bench_recon(64, 32, 128, pk.ReconConfig(iterations=10), reps=1, reference=ref)
    assert [e.label for e in rep.entries] == ["iterative_reference", "back_projection",
                                              "iterative_serial", "iterative_parallel"]
    assert rep.verification_ok(), rep.metrics
    assert rep.entry("iterative_serial").verification is True
    assert rep.metrics["rel_l2_f64_vs_reference"] <= 1e-10
    assert rep.metrics["rel_l2_f32_vs_reference"] <= 1e-4


@pytest.mark.gpu
def test_stage_seconds_split():
    """iterative_reconstruct(stage_seconds=...) books the graph solve under the reference's
    four stage keys (recon.py:303-347) by the plan's per-kernel device times."""
    import time

    g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
    K = pk.build_time_matrix(g, ring, ac)
    F32 = pk.CudaPool(0, "float32")
    y = pk.forward_project(K, ph, pool=F32)
    cfg = pk.resolve_config(pk.ReconConfig(iterations=10), K, y, pool=F32)
    pk.iterative_reconstruct(K, y, cfg, pool=F32)  # graph captured
    stages = {}
    t0 = time.perf_counter()
    pk.iterative_reconstruct(K, y, cfg, pool=F32, stage_seconds=stages)
    wall = time.perf_counter() - t0
    assert set(stages) == {"gradient_products", "tv_gradient", "prox", "objective"}
    assert stages["gradient_products"] > stages["tv_gradient"] > 0.0
    assert stages["objective"] > 0.0 and stages["prox"] == 0.0  # beta > 0: the update is TV + prox
    assert sum(stages.values()) <= wall
    # accumulates like the reference's dict
    pk.iterative_reconstruct(K, y, cfg, pool=F32, stage_seconds=stages)
    assert stages["gradient_products"] > 0.0
