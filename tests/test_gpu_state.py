"""Handle state across calls: the saved host-call graph, replaced predictors, regrown
workspaces, engine selection and the finite-weights routing of the row-union GEMM.

Each case would silently give wrong results if the library replayed a graph that holds stale
device pointers, leaked the replaced predictor, or sent a layer with a non-finite weight to the
tensor cores (where a dead lane's rows ARE read, unlike the reference's pipelines).
"""
import numpy as np
import pytest

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import DataError, Reduction

from conftest import bf16_round, rel_l2

pytestmark = pytest.mark.gpu

FAST = cd.BlockConfig(reduction=Reduction.UnorderedAccumulate)


def _case(oracle, seed, d, F, r, dtype="bf16"):
    g = oracle.generate(seed, d, F, r)
    if dtype == "bf16":
        g = {k: bf16_round(v) for k, v in g.items()}
    return g


def test_alternating_predictors_on_one_layer(oracle):
    """Two predictors attached in turn to one layer, each used for >= 2 consecutive host calls
    (the second call captures a graph): every call matches the oracle with the predictor in
    use, and device memory does not grow with the number of switches."""
    d, F, r = 512, 2048, 64
    g = _case(oracle, 301, d, F, r)
    g2 = _case(oracle, 302, d, F, r)
    layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
    preds = [cd.Predictor(cd.LowRankPredictor(d, r, F, gg["theta_a"], gg["theta_b"]), "bf16") for gg in (g, g2)]
    rng = oracle.rng(9)
    sizes = []
    for rnd in range(6):
        k = rnd % 2
        gg = g if k == 0 else g2
        for _ in range(3):
            x = rng.normals_f(d)
            _, z = oracle.lowrank_logits(gg["theta_a"], gg["theta_b"], x)
            tau = float(np.quantile(z, 0.8))
            got = cd.pipeline_dc(layer, x, preds[k], FAST, tau_d=tau, want_logits=True)
            assert rel_l2(got.logits, z) <= 1e-5, f"round {rnd}: logits of the other predictor"
            assert rel_l2(got.y, oracle.forward_sparse(g, x, got.mask.alive)) <= 1e-4
        sizes.append(layer.device_layer().device_bytes())
    assert sizes[-1] == sizes[1], f"device bytes grow with predictor switches: {sizes}"


def test_tensor_core_graph_survives_workspace_regrow(oracle):
    """A batch-16 host call is replayed from a saved graph; a larger device-pointer call then
    regrows the tensor-core workspace (the old buffer is freed).  The next batch-16 host calls
    must not replay the graph that holds the freed pointer."""
    import torch
    d, F, r = 384, 1536, 48
    g = _case(oracle, 303, d, F, r)
    layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
    rng = oracle.rng(10)

    def check_b16():
        X = np.stack([rng.normals_f(d) for _ in range(16)])
        res = cd.pipeline_dc(layer, X, pred, FAST, tau_d=0.05)
        assert layer.device_layer(pred).last_path() == "tensor"
        for b in range(16):
            assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive)) <= 1e-4

    for _ in range(3):
        check_b16()
    dev = layer.device_layer(pred)
    big = 512
    xb = torch.from_numpy(np.stack([rng.normals_f(d) for _ in range(big)])).cuda()
    yb = torch.empty(big, d, device="cuda")
    dev.forward_device(cd._capi.METHOD_DENSE, xb, yb, batch=big)
    torch.cuda.synchronize()
    for _ in range(3):
        check_b16()


def test_engine_selection_keeps_results(oracle):
    """cd_layer_set_engines: fused / chain, host graph on / off -- same contract."""
    d, F, r = 512, 2048, 64
    g = _case(oracle, 304, d, F, r)
    x = g["x"]
    _, z = oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)
    tau = float(np.quantile(z, 0.9))
    for fused in (True, False):
        for hg in (True, False):
            layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
            pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
            layer.device_layer(pred).set_engines(fused=fused, host_graph=hg)
            for _ in range(3):
                got = cd.pipeline_dc(layer, x, pred, FAST, tau_d=tau)
                assert rel_l2(got.y, oracle.forward_sparse(g, x, got.mask.alive)) <= 1e-4
            # kernels of the step: the persistent kernel, or latent + indicator + sparse
            # (plus the staging copies of the host call)
            assert layer.device_layer(pred).last_launches() >= (1 if fused else 3)
    with pytest.raises(DataError):
        cd._capi.check(cd._capi.lib().cd_layer_set_engines(layer.device_layer(pred).raw, 64))


def test_nonfinite_weight_keeps_batched_calls_off_the_row_union(oracle):
    """A NaN in the gate and down rows of a neuron that is dead for every sample: the
    reference never reads those rows (finite y).  The library routes such a layer's batched
    thresholding calls to the CUDA-core kernels instead of the row-union GEMM."""
    d, F, r, B = 256, 1024, 32, 16
    g = _case(oracle, 305, d, F, r)
    rng = oracle.rng(12)
    X = np.stack([rng.normals_f(d) for _ in range(B)])
    Z = np.stack([oracle.lowrank_logits(g["theta_a"], g["theta_b"], X[b])[1] for b in range(B)])
    tau = float(np.quantile(Z, 0.8))
    dead = int(np.argmin(Z.max(axis=0)))
    assert Z[:, dead].max() < tau
    gp = dict(g)
    gp["w_gate"] = g["w_gate"].copy()
    gp["w_down"] = g["w_down"].copy()
    gp["w_gate"][dead, :] = np.nan
    gp["w_down"][dead, :] = np.nan
    layer = cd.GatedMlpLayer(d, F, 0, gp["w_up"], gp["w_gate"], gp["w_down"], device_dtype="bf16")
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
    res = cd.pipeline_dc(layer, X, pred, FAST, tau_d=tau)
    assert layer.device_layer(pred).last_path() == "fast"
    assert np.isfinite(res.y).all()
    for b in range(B):
        assert res.mask[b].alive[dead] == 0
        assert rel_l2(res.y[b], oracle.forward_sparse(g, X[b], res.mask[b].alive)) <= 1e-4
    # the same layer without the poison takes the tensor cores
    clean = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
    cd.pipeline_dc(clean, X, pred, FAST, tau_d=tau)
    assert clean.device_layer(pred).last_path() == "tensor"


def test_cdwn1_header_fields_read_exactly(reference, tmp_path):
    """cd_layer_load_cdwn1: a uint64 seed above 2^53 is kept exactly; a string where a number
    belongs is the reference's 'bad header field' DataError."""
    import oracle as O
    good = tmp_path / "good.cdwn"
    reference.write_model(good, 5, 8, 16, 4, 0, 0.5)
    raw = open(good, "rb").read()
    hlen = int(np.frombuffer(raw[5:9], np.uint32)[0])
    header = raw[9:9 + hlen].decode()

    def with_header(h, name):
        p = tmp_path / name
        hb = h.encode()
        open(p, "wb").write(raw[:5] + np.uint32(len(hb)).tobytes() + hb + raw[9 + hlen:])
        return p

    big = (1 << 63) + 12345
    p = with_header(header.replace('"seed":5', f'"seed":{big}'), "seed.cdwn")
    assert reference.read_model(p) is not None
    dev = cd.DeviceLayer.load(str(p), "f32")
    assert dev.seed == big
    p = with_header(header.replace('"d_model":8', '"d_model":"8"'), "str.cdwn")
    with pytest.raises(O.ReferenceError_, match="bad header field"):
        reference.read_model(p)
    with pytest.raises(DataError, match="bad header field"):
        cd.DeviceLayer.load(str(p), "f32")
