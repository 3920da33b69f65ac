"""Tensor-parallel shards on the device: every rank's d_ff slice of one
layer is built on the single available GPU (TPLayer -> cd_layer_create_shard + the predictor's
theta_b rows of the slice), each shard runs its own kernels (the fused batch-1 kernels, the
tensor-core batched path), and the partial outputs are summed as the NCCL all-reduce would.

Contract (north_star): masks are shard-local and equal the slices of the single-device mask
(thresholds are lane-local; near-threshold lanes counted), and the summed y equals the oracle's
forward_sparse on the concatenated mask within 1e-4 relative L2 (sharded sums re-associate).
"""
import numpy as np
import pytest
import torch

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import _capi
from paper_2505_17701_b200.tp import TPLayer, shard_range

from conftest import bf16_round, rel_l2

pytestmark = pytest.mark.gpu


def run_shards(tps, method, X, tau, F):
    """Each rank's partial y (batch x d) and its mask slice; returns (sum of partials, mask)."""
    B, d = X.shape
    x_dev = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
    y_sum = torch.zeros((B, d), device="cuda")
    mask = np.zeros((B, F), np.uint8)
    for t in tps:
        b0, b1 = t.rows
        y = torch.empty((B, d), device="cuda")
        m = torch.empty((B, b1 - b0), dtype=torch.uint8, device="cuda")
        t.dev.forward_device(method, x_dev, y, tau, cd.Reduction.UnorderedAccumulate, B, mask_out=m)
        torch.cuda.synchronize()
        y_sum += y  # the all-reduce
        mask[:, b0:b1] = m.cpu().numpy()
    return y_sum.cpu().numpy(), mask


def flips_ok(got, want, ind, tau, band=1e-4):
    diff = np.nonzero(got != want)[0]
    scale = max(abs(tau), float(np.sqrt(np.mean(np.square(ind.astype(np.float64))))))
    assert np.all(np.abs(np.abs(ind[diff]) - abs(tau)) <= band * scale), diff


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 16])
def test_tp_shards_sum_to_oracle(oracle, world, B):
    d, F, r = 1024, 4096, 128
    g = oracle.generate(300 + world, d, F, r)
    g = {k: bf16_round(v) for k, v in g.items()}
    layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"])
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]))
    tps = [TPLayer(layer, pred, world, rank, device=0, device_dtype="bf16") for rank in range(world)]
    assert [t.rows for t in tps] == [shard_range(F, world, k) for k in range(world)]
    rng = oracle.rng(17 + B)
    X = np.stack([rng.normals_f(d) for _ in range(B)])
    zs = [oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)[1] for x in X]
    tau = float(np.mean([np.quantile(z, 0.9) for z in zs]))
    y, mask = run_shards(tps, _capi.METHOD_DC, X, tau, F)
    if B >= 8:
        assert tps[0].dev.last_path() == "tensor"
    for b in range(B):
        flips_ok(mask[b], (zs[b] > tau).astype(np.uint8), zs[b], tau)
        assert rel_l2(y[b], oracle.forward_sparse(g, X[b], mask[b])) <= 1e-4
    us = [oracle.gemv(g["w_up"], x) for x in X]
    tau_u = float(np.mean([np.quantile(np.abs(u), 0.8) for u in us]))
    y, mask = run_shards(tps, _capi.METHOD_MC, X, tau_u, F)
    for b in range(B):
        flips_ok(mask[b], (np.abs(us[b]) > tau_u).astype(np.uint8), us[b], tau_u)
        assert rel_l2(y[b], oracle.forward_sparse(g, X[b], mask[b])) <= 1e-4
    y, _ = run_shards(tps, _capi.METHOD_DENSE, X, 0.0, F)
    for b in range(B):
        assert rel_l2(y[b], oracle.forward_dense(g, X[b])["y"]) <= 1e-4


@pytest.mark.slow
def test_tp8_llama_shape_dc90(oracle):
    """BASELINE configs[3]'s per-GPU work: the Llama-3.1-8B FFN split 8 ways (1792 neurons per
    rank), D-CountDown at 90%, batch 1."""
    d, F, r = 4096, 14336, 512
    g = oracle.generate(42, d, F, r)
    g = {k: bf16_round(v) for k, v in g.items()}
    layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"])
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]))
    tps = [TPLayer(layer, pred, 8, rank, device=0, device_dtype="bf16") for rank in range(8)]
    x = cd.synth_normals(9, d)
    _, z = oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)
    tau = float(np.quantile(z, 0.9))
    y, mask = run_shards(tps, _capi.METHOD_DC, x[None, :], tau, F)
    flips_ok(mask[0], (z > tau).astype(np.uint8), z, tau)
    assert rel_l2(y[0], oracle.forward_sparse(g, x, mask[0])) <= 1e-4
