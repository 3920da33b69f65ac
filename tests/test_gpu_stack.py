"""configs[3]: the layer stack on the device.

Layer l+1's input is RMSNorm(y_l) (no gain, no residual: the reference has none), computed
inside k_dc_fused (cd_forward_device_normed) or by the norm kernel for the other engines.

Each layer is checked against the oracle GIVEN ITS OWN INPUT, i.e. the oracle's rms_norm of the
device's previous-layer output: the index set equals the oracle's logits > tau_l except lanes
within 1e-4 relative of tau (counted), and y_l is within 1e-4 rel-L2 of the oracle's
forward_sparse on the device's mask.  Checking layer by layer keeps a near-threshold flip in one
layer from being blamed on the next.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import Reduction, _capi
from paper_2505_17701_b200.tp import RMS_EPS, TPLayer, TPStack, stack_step

from conftest import bf16_round, rel_l2

pytestmark = pytest.mark.gpu


def check_layer(oracle, g, x_in, tau, mask, y, act=0, band=1e-4):
    _, z = oracle.lowrank_logits(g["theta_a"], g["theta_b"], x_in)
    want = (z > np.float32(tau)).astype(np.uint8)
    diff = np.nonzero(mask != want)[0]
    assert np.all(np.abs(z[diff] - tau) <= band * max(abs(tau), 1e-3)), (len(diff), z[diff], tau)
    assert mask.sum() > 0
    assert rel_l2(y, oracle.forward_sparse(g, x_in, mask, act=act)) <= 1e-4
    return len(diff)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_stack_layer_by_layer(oracle, dtype):
    d, F, r, L = 512, 2048, 64, 4
    st = TPStack.synthetic(L, d, F, r, 0.9, 1, 0, seed0=42, device_dtype=dtype, keep_host=True)
    x = cd.synth_normals(5, d)
    xd = torch.from_numpy(x).cuda()
    ys = torch.zeros((L, d), device="cuda")
    masks = torch.zeros((L, F), dtype=torch.uint8, device="cuda")
    alive = torch.zeros((L, 1), dtype=torch.int32, device="cuda")
    st.forward(xd, ys, torch.cuda.current_stream().cuda_stream, masks_out=masks, alive_out=alive)
    torch.cuda.synchronize()
    ys, masks, alive = ys.cpu().numpy(), masks.cpu().numpy(), alive.cpu().numpy()
    x_in = x
    for l in range(L):
        layer, pred = st.host[l]
        rnd = bf16_round if dtype == "bf16" else (lambda a: a)
        lp = pred.lowrank()
        g = {"w_up": rnd(layer.w_up), "w_gate": rnd(layer.w_gate), "w_down": rnd(layer.w_down),
             "theta_a": rnd(lp.theta_a), "theta_b": rnd(lp.theta_b)}
        if l > 0:
            x_in = O.rms_norm(ys[l - 1], RMS_EPS)
        check_layer(oracle, g, x_in, st.taus[l], masks[l], ys[l])
        assert alive[l, 0] == masks[l].sum()
        assert 0.85 <= 1 - masks[l].sum() / F <= 0.95


def test_normed_input_on_every_engine(oracle):
    """cd_forward_device_normed == cd_forward_device on the host-normalised input, for the
    fused kernel, the kernel chain, the exact kernels, M-CountDown and the tensor-core batch."""
    d, F, r = 384, 1536, 48
    g = oracle.generate(77, d, F, r)
    g = {k: bf16_round(v) for k, v in g.items()}
    layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16")
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
    dev = layer.device_layer(pred)
    rng = oracle.rng(3)
    for B in (1, 3, 16):
        X = np.stack([3.0 * rng.normals_f(d) for _ in range(B)])
        Xn = np.stack([O.rms_norm(x, RMS_EPS) for x in X])
        xd = torch.from_numpy(X).cuda()
        for method, tau in ((_capi.METHOD_DC, 0.05), (_capi.METHOD_MC, 0.3)):
            for fused in (True, False):
                for red in (Reduction.UnorderedAccumulate, Reduction.DeterministicOrdered):
                    dev.set_engines(fused=fused)
                    y = torch.zeros((B, d), device="cuda")
                    m = torch.zeros((B, F), dtype=torch.uint8, device="cuda")
                    dev.forward_device(method, xd, y, tau, red, B, mask_out=m, rms_eps=RMS_EPS,
                                       stream=torch.cuda.current_stream().cuda_stream)
                    torch.cuda.synchronize()
                    y, m = y.cpu().numpy(), m.cpu().numpy()
                    for b in range(B):
                        if method == _capi.METHOD_DC:
                            _, ind = oracle.lowrank_logits(g["theta_a"], g["theta_b"], Xn[b])
                        else:
                            ind = np.abs(oracle.gemv(g["w_up"], Xn[b]))
                        want = ind > np.float32(tau)
                        diff = np.nonzero(m[b].astype(bool) != want)[0]
                        assert np.all(np.abs(ind[diff] - tau) <= 1e-4 * tau), (B, method, fused, red)
                        assert rel_l2(y[b], oracle.forward_sparse(g, Xn[b], m[b])) <= 1e-4
    dev.set_engines()
    with pytest.raises(cd.DataError):
        dev.forward_device(_capi.METHOD_DC, xd, torch.zeros((16, d), device="cuda"), 0.1, batch=16, rms_eps=-1.0)


def test_tp_stack_shards_on_one_gpu(oracle):
    """Two ranks' shards of a 3-layer stack on the one GPU, combined per layer as the all-reduce
    would (stack_step with a summing all-reduce): same output as the unsharded stack."""
    d, F, r, L = 512, 2048, 64, 3
    full = TPStack.synthetic(L, d, F, r, 0.8, 1, 0, seed0=11, keep_host=True)
    shards = [TPStack([TPLayer(lay, p, 2, k) for lay, p in full.host], full.taus) for k in range(2)]
    x = cd.synth_normals(8, d)
    xd = torch.from_numpy(x).cuda()
    ys_full = torch.zeros((L, d), device="cuda")
    full.forward(xd, ys_full, torch.cuda.current_stream().cuda_stream)
    ys = torch.zeros((L, d), device="cuda")
    part = torch.zeros((2, d), device="cuda")

    def run_layer(l, x_in, y_out, normed):
        for k in range(2):
            shards[k].tps[l].dev.forward_device(_capi.METHOD_DC, x_in, part[k], shards[k].taus[l],
                                                rms_eps=RMS_EPS if normed else None,
                                                stream=torch.cuda.current_stream().cuda_stream)
        torch.sum(part, dim=0, out=y_out)

    stack_step(L, xd, ys, run_layer, lambda y: None)
    torch.cuda.synchronize()
    for l in range(L):
        assert rel_l2(ys[l].cpu().numpy(), ys_full[l].cpu().numpy()) <= 1e-4


@pytest.mark.slow
def test_llama_32_layer_stack(oracle):
    """The full configs[3] stack at TP 1: 32 Llama-3.1-8B FFN layers (seeds 42 + l), DC at 90%,
    bf16, captured as one CUDA graph; every layer checked against the oracle given its input."""
    d, F, r, L = 4096, 14336, 512, 32
    st = TPStack.synthetic(L, d, F, r, 0.9, 1, 0, seed0=42)
    x = cd.synth_normals(1234, d)
    xd = torch.from_numpy(x).cuda()
    ys = torch.zeros((L, d), device="cuda")
    masks = torch.zeros((L, F), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.forward(xd, ys, s.cuda_stream, masks_out=masks)  # warm-up (eager)
    torch.cuda.synchronize()
    ys.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            st.forward(xd, ys, torch.cuda.current_stream().cuda_stream, masks_out=masks)
    g.replay()
    torch.cuda.synchronize()
    ys_h, masks_h = ys.cpu().numpy(), masks.cpu().numpy()
    flips = 0
    x_in = x
    for l in range(L):
        layer, _, pred = cd.synth_workload(42 + l, d, F, r)
        lp = pred.lowrank()
        gl = {"w_up": bf16_round(layer.w_up), "w_gate": bf16_round(layer.w_gate),
              "w_down": bf16_round(layer.w_down), "theta_a": bf16_round(lp.theta_a),
              "theta_b": bf16_round(lp.theta_b)}
        del layer, pred, lp
        if l > 0:
            x_in = O.rms_norm(ys_h[l - 1], RMS_EPS)
        flips += check_layer(oracle, gl, x_in, st.taus[l], masks_h[l], ys_h[l])
        assert 0.87 <= 1 - masks_h[l].sum() / F <= 0.93
    assert flips <= 2 * L
