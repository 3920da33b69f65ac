"""Batched decode (B >= 8) and dense prefill on the tcgen05 tensor cores (SURVEY.md section 8f
row 1, BASELINE.json config 5) against the CPU oracle.

Caller-supplied masks (exec_*, mask_override) stay on the CUDA-core kernels at every batch size
(dead lanes are never read); the tensor-core path serves the thresholding calls.
The reference semantics are per sample (blocked_exec.cpp:252-298 / :350-379; main.cpp:239-282):
each sample's y must equal the oracle's forward_sparse on that sample's own mask.  Decode runs
activations as bf16 (hi, lo) pairs, so the contract is the fast path's: y within 1e-4 relative
L2 of the oracle on the bf16 weights, indicators within 1e-5, index sets equal except lanes
within 1e-4 relative of the threshold.  Prefill (dense, > 256 tokens) uses plain bf16
activations: 1e-2 (the north_star bf16 bound).
"""
import numpy as np
import pytest

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import Reduction

from conftest import bf16_round, rel_l2

pytestmark = pytest.mark.gpu

FAST = cd.BlockConfig(reduction=Reduction.UnorderedAccumulate)


def make(oracle, seed, d, F, r, act=0):
    g = oracle.generate(seed, d, F, r)
    for k in ("w_up", "w_gate", "w_down", "theta_a", "theta_b"):
        g[k] = bf16_round(g[k])
    layer = cd.GatedMlpLayer(d, F, act, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
    return g, layer, pred


def batch(oracle, seed, B, d):
    rng = oracle.rng(seed)
    return np.stack([rng.normals_f(d) for _ in range(B)])


def flips_ok(got, want, ind, tau, band=1e-4):
    diff = np.nonzero(got != want)[0]
    scale = max(abs(tau), float(np.sqrt(np.mean(np.square(ind.astype(np.float64))))))
    assert np.all(np.abs(np.abs(ind[diff]) - abs(tau)) <= band * scale), diff
    return len(diff)


TC_SHAPES = [  # (seed, d, F, r): ragged d / F / r (TMA zero fill), multi-tile, > 1 k-block
    (201, 64, 128, 16),
    (202, 200, 300, 40),
    (203, 130, 500, 24),
    (204, 512, 1024, 128),
]


@pytest.mark.parametrize("B", [8, 13, 64, 70])
@pytest.mark.parametrize("shape", TC_SHAPES)
def test_tc_dc_pipeline(oracle, shape, B):
    seed, d, F, r = shape
    g, layer, pred = make(oracle, seed, d, F, r)
    X = batch(oracle, seed + B, B, d)
    zs = [oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)[1] for x in X]
    tau = float(np.mean([np.quantile(z, 0.8) for z in zs]))
    res = cd.pipeline_dc(layer, X, pred, FAST, tau_d=tau, want_logits=True)
    assert layer.device_layer(pred).last_path() == "tensor"
    for b in range(B):
        assert rel_l2(res.logits[b], zs[b]) <= 1e-5
        flips_ok(res.mask[b].alive, (zs[b] > tau).astype(np.uint8), zs[b], tau)
        assert res.mask[b].alive_count == int(res.mask[b].alive.sum())
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive)) <= 1e-4


@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("B", [3, 5, 8, 33, 64])  # M-CountDown takes the tensor cores from batch 3
@pytest.mark.parametrize("shape", TC_SHAPES[1:])
def test_tc_mc_pipeline(oracle, shape, B, act):
    seed, d, F, r = shape
    g, layer, _ = make(oracle, seed, d, F, r, act)
    X = batch(oracle, seed + 7 * B, B, d)
    us = [oracle.gemv(g["w_up"], x) for x in X]
    tau = float(np.mean([np.quantile(np.abs(u), 0.7) for u in us]))
    res = cd.pipeline_mc(layer, X, tau, FAST, want_u=True)
    assert layer.device_layer().last_path() == "tensor"
    for b in range(B):
        assert rel_l2(res.u[b], us[b]) <= 1e-5
        flips_ok(res.mask[b].alive, (np.abs(us[b]) > tau).astype(np.uint8), us[b], tau)
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive, act=act)) <= 1e-4


@pytest.mark.parametrize("B", [3, 8, 40])
def test_tc_cats_pipeline(oracle, B):
    seed, d, F, r = 202, 200, 300, 40
    g, layer, _ = make(oracle, seed, d, F, r, 1)
    X = batch(oracle, 99, B, d)
    hs = [np.array([oracle.act(1, v) for v in oracle.gemv(g["w_gate"], x)], np.float32) for x in X]
    tau = float(np.mean([np.quantile(np.abs(h), 0.6) for h in hs]))
    res = cd.pipeline_cats(layer, X, tau, FAST, want_act=True)
    assert layer.device_layer().last_path() == "tensor"
    for b in range(B):
        assert rel_l2(res.act[b], hs[b]) <= 1e-5
        flips_ok(res.mask[b].alive, (np.abs(hs[b]) > tau).astype(np.uint8), hs[b], tau)
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive, act=1)) <= 1e-4


@pytest.mark.parametrize("B", [8, 64, 65])
def test_batched_caller_masks_never_read_dead_lanes(oracle, B):
    """exec_dc / exec_mc / pipeline_dc(mask_override) at batch >= 8 on a bf16 layer: the rows
    and u entries of lanes dead in EVERY sample are NaN-poisoned (test_blocked_exec.cpp:101-116
    at batch scale) and must not reach y.  Caller-supplied masks therefore stay on the CUDA-core
    kernels (the row-union GEMM would read them); per-sample masks include all-dead and
    all-live rows."""
    seed, d, F, r = 203, 130, 500, 24
    g, layer_ok, pred = make(oracle, seed, d, F, r)
    X = batch(oracle, 5, B, d)
    rng = np.random.default_rng(B)
    masks = (rng.random((B, F)) < 0.3).astype(np.uint8)
    masks[:, :50] = 0        # dead in every sample: poisoned below
    masks[0] = 0
    masks[1, 50:] = 1
    want = [oracle.forward_sparse(g, X[b], masks[b]) for b in range(B)]
    bad = {k: v.copy() for k, v in g.items()}
    for k in ("w_up", "w_gate", "w_down"):
        bad[k][:50] = np.nan
    layer = cd.GatedMlpLayer(d, F, 0, bad["w_up"], bad["w_gate"], bad["w_down"], device_dtype="bf16")
    y = cd.exec_dc(layer, X, masks, FAST)
    assert layer.device_layer().last_path() == "fast"
    assert np.all(np.isfinite(y)) and np.all(y[0] == 0)
    U = np.stack([oracle.gemv(g["w_up"], X[b]) for b in range(B)])
    U[:, :50] = np.nan
    y_mc = cd.exec_mc(layer, X, U, masks, FAST)
    assert np.all(np.isfinite(y_mc))
    for b in range(B):
        assert rel_l2(y[b], want[b]) <= 1e-4
        assert rel_l2(y_mc[b], want[b]) <= 1e-4
    res = cd.pipeline_dc(layer_ok, X, pred, FAST, mask_override=masks)
    assert layer_ok.device_layer(pred).last_path() == "fast"
    for b in range(B):
        assert np.array_equal(res.mask[b].alive, masks[b])
        assert rel_l2(res.y[b], want[b]) <= 1e-4


@pytest.mark.parametrize("B", [8, 64, 300])
def test_tc_dense_and_prefill(oracle, B):
    """Dense batch: split (hi/lo) decode up to 256 tokens, plain-bf16 prefill beyond."""
    seed, d, F, r = 204, 512, 1024, 128
    g, layer, _ = make(oracle, seed, d, F, r)
    X = batch(oracle, 11, B, d)
    y = cd.exec_dense(layer, X, FAST)
    assert layer.device_layer().last_path() == "tensor"
    tol = 1e-4 if B <= 256 else 1e-2
    for b in range(0, B, max(1, B // 16)):
        assert rel_l2(y[b], oracle.forward_dense(g, X[b])["y"]) <= tol


def test_tc_matches_cuda_core_path(oracle):
    """Same batch through the tensor cores and (tensor engine off) the CUDA-core fused chain."""
    seed, d, F, r = 202, 200, 300, 40
    g, _, _ = make(oracle, seed, d, F, r)
    X = batch(oracle, 3, 16, d)
    outs = {}
    for tc in ("1", "0"):
        layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
        pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
        layer.device_layer(pred).set_engines(tensor=(tc == "1"))
        outs[tc] = cd.pipeline_dc(layer, X, pred, FAST, tau_d=0.05, want_logits=True)
        assert layer.device_layer(pred).last_path() == ("tensor" if tc == "1" else "fast")
    for b in range(16):
        assert rel_l2(outs["1"].logits[b], outs["0"].logits[b]) <= 1e-5
        both = outs["1"].mask[b].alive & outs["0"].mask[b].alive
        flips_ok(outs["1"].mask[b].alive, outs["0"].mask[b].alive, outs["0"].logits[b], 0.05)
        if np.array_equal(outs["1"].mask[b].alive, outs["0"].mask[b].alive):
            assert rel_l2(outs["1"].y[b], outs["0"].y[b]) <= 1e-4
        assert both.sum() > 0


@pytest.mark.slow
def test_tc_qwen_b64_decode_and_prefill(oracle):
    """BASELINE.json config 5: Qwen2.5-14B FFN shape (5120 x 13824, SiLU), batch-64 decode at
    ~80% sparsity (DC and MC) and a dense prefill chunk, against the oracle on sampled rows."""
    d, F, r = 5120, 13824, 512
    g, layer, pred = make(oracle, 42, d, F, r)
    X = batch(oracle, 77, 64, d)
    zs = [oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)[1] for x in X[:4]]
    tau = float(np.mean([np.quantile(z, 0.8) for z in zs]))
    res = cd.pipeline_dc(layer, X, pred, FAST, tau_d=tau, want_logits=True)
    assert layer.device_layer(pred).last_path() == "tensor"
    for b in range(4):
        assert rel_l2(res.logits[b], zs[b]) <= 1e-5
        flips_ok(res.mask[b].alive, (zs[b] > tau).astype(np.uint8), zs[b], tau)
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive)) <= 1e-4
    sp = 1 - np.mean([m.alive_count for m in res.mask]) / F
    assert 0.7 <= sp <= 0.9
    union = np.any(np.stack([m.alive for m in res.mask]), axis=0).mean()
    assert union > 0.99  # the row union at B=64 is ~all rows
    P = batch(oracle, 78, 512, d)
    y = cd.exec_dense(layer, P, FAST)
    for b in (0, 257, 511):
        assert rel_l2(y[b], oracle.forward_dense(g, P[b])["y"]) <= 1e-2


@pytest.mark.slow
def test_tc_prefill_2048_tokens_sampled(oracle):
    """BASELINE.json config 5 prefill chunk at full size: Qwen2.5-14B FFN, 2048 tokens through the
    repo's own tcgen05 gate/up and down kernels (whole 256 x 256 tiles on every CTA plus the
    stream-K remainder), 64 sampled tokens across every token tile vs the oracle's forward_dense
    (bf16 activations: the north_star 1e-2 bound)."""
    d, F, r = 5120, 13824, 512
    g, layer, _ = make(oracle, 42, d, F, r)
    P = batch(oracle, 79, 2048, d)
    y = cd.exec_dense(layer, P, FAST)
    assert layer.device_layer().last_path() == "tensor"
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([rng.integers(0, 2048, 56), [0, 255, 256, 1023, 1791, 1792, 2046, 2047]]))
    assert len(rows) >= 60
    for b in rows:
        assert rel_l2(y[b], oracle.forward_dense(g, P[b])["y"]) <= 1e-2, b


@pytest.mark.parametrize("shape,B", [((200, 300, 8), 600), ((130, 500, 8), 257), ((512, 1024, 8), 1100)])
def test_tc_prefill_ragged(oracle, shape, B):
    """Prefill on ragged shapes: d not a multiple of 4 (scalar epilogue) or of the 256-column tile,
    F not a multiple of 64 (TMA zero fill along K), partial token tiles."""
    d, F, r = shape
    g, layer, _ = make(oracle, 300 + d, d, F, r)
    X = batch(oracle, 12, B, d)
    y = cd.exec_dense(layer, X, FAST)
    assert layer.device_layer().last_path() == "tensor"
    for b in list(range(0, B, max(1, B // 24))) + [B - 1]:
        assert rel_l2(y[b], oracle.forward_dense(g, X[b])["y"]) <= 1e-2, b
