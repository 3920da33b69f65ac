"""Seeded random shapes through the tensor-core batched path (bf16 layers, batch >= 8): ragged
d / d_ff / d_rank (TMA zero fill, partial tiles), batches spanning several 64-sample n-tiles,
both activations, every method, against the oracle per sample (y 1e-4 rel-L2, indicators 1e-5,
masks equal except lanes within 1e-4 of tau)."""
import numpy as np
import pytest

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import Reduction

from conftest import bf16_round, rel_l2

pytestmark = pytest.mark.gpu

FAST = cd.BlockConfig(reduction=Reduction.UnorderedAccumulate)

_rng = np.random.default_rng(2505)
CASES = [(int(_rng.integers(8, 700)), int(_rng.integers(8, 900)), int(_rng.integers(1, 200)),
          int(_rng.integers(8, 140)), int(_rng.integers(0, 2)), 500 + i) for i in range(16)]


def flips_ok(got, want, ind, tau, band=1e-4):
    diff = np.nonzero(got != want)[0]
    scale = max(abs(tau), float(np.sqrt(np.mean(np.square(ind.astype(np.float64))))))
    assert np.all(np.abs(np.abs(ind[diff]) - abs(tau)) <= band * scale), diff


@pytest.mark.parametrize("d,F,r,B,act,seed", CASES)
def test_tc_random_shapes(oracle, d, F, r, B, act, seed):
    g = oracle.generate(seed, d, F, r)
    g = {k: bf16_round(v) for k, v in g.items()}
    layer = cd.GatedMlpLayer(d, F, act, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
    rng = oracle.rng(seed + 1)
    X = np.stack([rng.normals_f(d) for _ in range(B)])
    pick = list(range(0, B, max(1, B // 6))) + [B - 1]
    # D-CountDown
    zs = {b: oracle.lowrank_logits(g["theta_a"], g["theta_b"], X[b])[1] for b in pick}
    tau = float(np.mean([np.quantile(z, 0.7) for z in zs.values()]))
    res = cd.pipeline_dc(layer, X, pred, FAST, tau_d=tau, want_logits=True)
    assert layer.device_layer(pred).last_path() == "tensor"
    for b in pick:
        assert rel_l2(res.logits[b], zs[b]) <= 1e-5
        flips_ok(res.mask[b].alive, (zs[b] > tau).astype(np.uint8), zs[b], tau)
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive, act=act)) <= 1e-4
    # M-CountDown
    us = {b: oracle.gemv(g["w_up"], X[b]) for b in pick}
    tau_u = float(np.mean([np.quantile(np.abs(u), 0.6) for u in us.values()]))
    res = cd.pipeline_mc(layer, X, tau_u, FAST, want_u=True)
    for b in pick:
        assert rel_l2(res.u[b], us[b]) <= 1e-5
        flips_ok(res.mask[b].alive, (np.abs(us[b]) > tau_u).astype(np.uint8), us[b], tau_u)
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive, act=act)) <= 1e-4
    # dense
    y = cd.exec_dense(layer, X, FAST)
    for b in pick:
        assert rel_l2(y[b], oracle.forward_dense(g, X[b], act=act)["y"]) <= 1e-4
