"""The exact thing bench.py times, output-checked (VERDICT r1 weak #1c): a CUDA graph of
PDL-chained k_dc_fused launches over 8 rotating device layers of the Llama-3.1-8B FFN
(BASELINE configs[1]), every step's y checked against the oracle.

Each launch's own-work cap comes from the previous launch's active count and its queue counters
from the launch two before, so the chained graph exercises state the single-call tests do not.
Fast-path contract per step (blocked_exec UnorderedAccumulate, test_blocked_exec.cpp:87-99):
y within 1e-4 relative L2 of the oracle's forward_sparse on the mask the kernel chose, and that
mask equal to the exact logits > tau except lanes within 1e-4 relative of tau."""
import numpy as np
import pytest

import paper_2505_17701_b200 as cd

from conftest import bf16_round, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("pdl_chain", [True, False])
def test_bench_graph_rotating_handles_vs_oracle(oracle, pdl_chain):
    torch = pytest.importorskip("torch")
    d, F, r, NL, NX, STEPS = 4096, 14336, 512, 8, 16, 48
    g = oracle.generate(42, d, F, r)
    g = {k: (bf16_round(v) if k != "x" else v) for k, v in g.items()}
    pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]), "bf16")
    devs = [cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"], device_dtype="bf16").device_layer(pred)
            for _ in range(NL)]
    for dv in devs:
        dv.set_engines(pdl_chain=pdl_chain)  # the bench's mode (True) and the library default
    X = np.stack([cd.synth_normals(9000 + i, d) for i in range(NX)])
    Z = np.stack([oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)[1] for x in X])
    tau = float(np.mean([np.quantile(z, 0.9) for z in Z]))
    xs = torch.from_numpy(X).cuda()
    ys = torch.zeros((STEPS, d), device="cuda")
    ms = torch.zeros((STEPS, F), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()

    def step(i, cs):
        devs[i % NL].forward_device(cd._capi.METHOD_DC, xs[i % NX], ys[i], tau, mask_out=ms[i], stream=cs)

    with torch.cuda.stream(s):
        for i in range(2 * NL):  # warm: host-side graphs, launch tags, previous active counts
            step(i, s.cuda_stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for i in range(STEPS):
                step(i, torch.cuda.current_stream().cuda_stream)
    for rep in range(3):
        ys.zero_()
        ms.zero_()
        with torch.cuda.stream(s):
            graph.replay()
        torch.cuda.synchronize()
        Y, M = ys.cpu().numpy(), ms.cpu().numpy()
        flips = 0
        for i in range(STEPS):
            z = Z[i % NX]
            diff = np.nonzero(M[i] != (z > np.float32(tau)))[0]
            flips += len(diff)
            assert np.all(np.abs(z[diff] - tau) <= 1e-4 * max(abs(tau), 1e-30) + 1e-6), (rep, i, diff)
            assert rel_l2(Y[i], oracle.forward_sparse(g, X[i % NX], M[i])) <= 1e-4, (rep, i)
        assert flips <= 4 * STEPS
