"""Quick GPU probe: small-shape parity smoke + Llama-shape timings (development tool)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import Reduction  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.float64(a) - b) / max(np.linalg.norm(np.float64(b)), 1e-30))


def small_checks():
    o = oracle.Oracle()
    for (seed, d, F, r) in [(101, 20, 48, 6), (104, 64, 256, 16), (106, 512, 2048, 64)]:
        g = o.generate(seed, d, F, r)
        layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"])
        pred = cd.Predictor(cd.LowRankPredictor(d, r, F, g["theta_a"], g["theta_b"]))
        x = g["x"]
        want = o.pipeline_dc(g, x)
        for red in (Reduction.DeterministicOrdered, Reduction.UnorderedAccumulate):
            t0 = time.time()
            got = cd.pipeline_dc(layer, x, pred, cd.BlockConfig(reduction=red))
            ym = o.forward_sparse(g, x, got.mask.alive)
            print(f"DC d={d} F={F} red={int(red)} alive {got.mask.alive_count}/{want['alive']} "
                  f"maskeq={np.array_equal(got.mask.alive, want['mask'])} bits={np.array_equal(got.y, want['y'])} "
                  f"rel={rel(got.y, ym):.2e} {1e3*(time.time()-t0):.1f}ms", flush=True)
        u = o.gemv(g["w_up"], x)
        tau = float(np.sort(np.abs(u))[::-1][F // 4])
        want = o.pipeline_mc(g, x, tau)
        for red in (Reduction.DeterministicOrdered, Reduction.UnorderedAccumulate):
            got = cd.pipeline_mc(layer, x, tau, cd.BlockConfig(reduction=red))
            ym = o.forward_sparse(g, x, got.mask.alive)
            print(f"MC d={d} F={F} red={int(red)} alive {got.mask.alive_count}/{want['alive']} "
                  f"maskeq={np.array_equal(got.mask.alive, want['mask'])} bits={np.array_equal(got.y, want['y'])} "
                  f"rel={rel(got.y, ym):.2e}", flush=True)
        yd = cd.exec_dense(layer, x, cd.BlockConfig(reduction=Reduction.UnorderedAccumulate))
        print(f"dense rel={rel(yd, o.forward_dense(g, x)['y']):.2e}", flush=True)


def timings():
    d, F, r = 4096, 14336, 512
    t0 = time.time()
    layer, x0, pred = cd.synth_workload(42, d, F, r, device_dtype="bf16")
    print(f"synth {time.time()-t0:.1f}s", flush=True)
    NL = 6
    devs = []
    for i in range(NL):
        L = cd.GatedMlpLayer(d, F, 0, layer.w_up, layer.w_gate, layer.w_down, device_dtype="bf16")
        devs.append(L.device_layer(pred))
    print(f"upload {time.time()-t0:.1f}s", flush=True)
    NX = 16
    X = np.stack([cd.synth_normals(1000 + i, d) for i in range(NX)])
    z = devs[0].predict_logits(X)
    xs = torch.from_numpy(X).cuda()
    ys = torch.empty((NX, d), device="cuda")
    s = torch.cuda.Stream()
    for k in (0.5, 0.7, 0.8, 0.9, None):
        if k is None:
            method, tau, name = 0, 0.0, "dense"
        else:
            tau = float(np.mean([np.quantile(z[i], k) for i in range(NX)]))
            method, name = 2, f"dc@{k}"
        steps = NL * 4
        with torch.cuda.stream(s):
            for i in range(3):
                devs[i % NL].forward_device(method, xs[i % NX], ys[i % NX], tau, stream=s.cuda_stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            cs = torch.cuda.current_stream().cuda_stream
            for i in range(steps):
                devs[i % NL].forward_device(method, xs[i % NX], ys[i % NX], tau, stream=cs)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        R = 20
        e0.record()
        for _ in range(R):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (R * steps)
        alive = (z > tau).sum(axis=1).mean() if k is not None else F
        byts = cd.costmodel.device_bytes("dense" if k is None else "dc", d, F, r, int(alive), 2)["total_bytes"]
        print(f"{name}: {us:.2f} us/token  alive~{alive:.0f}  {byts/us/1e3:.0f} GB/s "
              f"({byts/us/1e3/6545.6*100:.1f}% of 6545.6)", flush=True)


if __name__ == "__main__":
    small_checks()
    timings()
