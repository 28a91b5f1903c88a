"""Index generation (north_star "geometry and index generation
bit-exact") on every pair of the BASELINE configurations, config 5 included (1.07e9 pairs,
sensor blocks):

* fp64 validation kernels (pk_index_dump): s0 and frac bit-identical to the reference's
  rule floor(np.hypot(p - s) / (c dt)) (forward.py:153-182);
* fp32 production kernels (pk_delay_census_f32: the delay exactly as the generic, the
  D4-symmetric back-projector and the rotation-symmetric projector evaluate it): a census of
  the pairs whose s0 differs, with the bound of DESIGN.md section 2 -- every difference is
  one sample, only for pairs whose exact delay lies within delta of an integer, and the fp32
  delay itself is within delta = 4e-7 Q samples of the exact one on every pair.  Because the
  interpolation weights ((1-f) w at s0-1, f w at s0) are continuous across an integer delay,
  a flipped s0 moves at most delta*w of weight, the same as the fraction error of any pair.

The reference index (np.hypot / floor) comes from the fp64 C oracle's or_index, which
tests/test_oracle.py pins to numpy bit for bit.
"""

import numpy as np
import pytest

import paper_2404_10928_b200 as pk

pytestmark = pytest.mark.gpu

F32 = pk.CudaPool(0, "float32")
F64 = pk.CudaPool(0, "float64")
CFGS = [(128, 128, 1024), (256, 256, 2048), (512, 512, 2048), (1024, 1024, 4096)]
DELTA_PER_SAMPLE = 4e-7  # |u_fp32 - u| <= 4e-7 Q (~4 ulp of the largest delay)


@pytest.mark.parametrize("cfg", CFGS, ids=["cfg1", "cfg2", "cfg3", "cfg5"])
def test_index_rule_every_pair(oracle, cfg):
    import torch

    n, M, Q = cfg
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=0)
    op64 = pk.operator_for(g, ring, ac, F64)
    op32 = pk.operator_for(g, ring, ac, F32)
    sym = op32.info.symmetric
    rules = [0] + ([1] if sym & 1 else []) + ([2] if sym & 2 else [])
    # every BASELINE scene runs the D4 back-projector; the rotation-symmetric projector needs
    # its window to fit (config 1's short c*dt keeps the generic projector, rule 0)
    assert sym & 1 and (sym & 2 or n == 128), sym
    xx, yy = g.axis_vectors()
    delta = DELTA_PER_SAMPLE * Q
    stats = {r: [0, 0.0] for r in rules}  # mismatching pairs, max |du|
    block = max(1, (1 << 24) // g.size)
    for m0 in range(0, M, block):
        m1 = min(M, m0 + block)
        o = oracle.Operator(xx, yy, ring.positions, ac.c, ac.dt, Q, m0, m1)
        ref_s0, ref_fr = o.index()
        s0, fr = op64.index_dump(m0, m1)
        assert np.array_equal(s0.cpu().numpy(), ref_s0), f"fp64 s0 differs in sensors [{m0}, {m1})"
        assert np.array_equal(fr.cpu().numpy(), ref_fr), f"fp64 frac differs in sensors [{m0}, {m1})"
        rs0 = torch.from_numpy(ref_s0).cuda()
        ru = rs0.double() + torch.from_numpy(ref_fr).cuda()
        for r in rules:
            c0, cf = op32.delay_census(r, m0, m1)
            c0 = c0.long()
            du = (c0.double() + cf.double() - ru).abs()
            ds = (c0 - rs0).abs()
            assert int(ds.max()) <= 1, f"rule {r}: s0 off by more than one sample"
            stats[r][0] += int((ds != 0).sum())
            stats[r][1] = max(stats[r][1], float(du.max()))
    pairs = M * g.size
    for r in rules:
        miss, dmax = stats[r]
        print(f"{cfg} rule {r}: {miss} of {pairs} pairs ({miss / pairs:.2e}) differ in s0 by one "
              f"sample; max |u_fp32 - u| = {dmax:.3e} samples (bound {delta:.3e})")
        assert dmax <= delta
        # a flip needs the exact delay within dmax of an integer: a 2*dmax-wide band
        assert miss <= 4.0 * dmax * pairs + 16
