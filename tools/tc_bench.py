"""tc_bench.py -- time the tensor-core batched path (BASELINE.json config 5: Qwen2.5-14B FFN
shape, batch-64 decode at ~80% sparsity + dense prefill) with CUDA graphs and events.

  python tools/tc_bench.py [--steps 20] [--prefill 2048] [--cases dc,mc,dense,prefill]
Prints one JSON object per case.  Development tool; bench.py carries the contract numbers.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prefill", type=int, default=2048)
    ap.add_argument("--cases", default="dc,mc,dense,prefill")
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2505_17701_b200 as cd
    from paper_2505_17701_b200 import _capi

    D, F, R = 5120, 13824, 512
    layer, _, pred = cd.synth_workload(42, D, F, R, device_dtype="bf16")
    dev = layer.device_layer(pred)
    B = a.batch
    xs = np.stack([cd.synth_normals(5000 + i, D) for i in range(B)])
    z = np.atleast_2d(cd.predict_logits(pred, xs[:8]))
    tau_dc = float(np.mean([np.quantile(r, 0.8) for r in z]))
    u = np.abs(cd.pipeline_mc(layer, xs[:8], float("inf"), cd.BlockConfig(reduction=cd.Reduction.DeterministicOrdered),
                              want_u=True).u)
    tau_mc = float(np.mean([np.quantile(r, 0.8) for r in u]))
    x_dev = torch.from_numpy(xs).cuda()
    P = a.prefill
    xp = torch.randn(P, D, device="cuda")
    stream = torch.cuda.Stream()
    wbytes = 3 * F * D * 2
    for case in a.cases.split(","):
        if case == "prefill":
            method, nb, x, tau = _capi.METHOD_DENSE, P, xp, 0.0
        else:
            method = {"dc": _capi.METHOD_DC, "mc": _capi.METHOD_MC, "dense": _capi.METHOD_DENSE}[case]
            nb, x, tau = B, x_dev, {"dc": tau_dc, "mc": tau_mc, "dense": 0.0}[case]
        y = torch.empty(nb, D, device="cuda")
        alive = torch.zeros(nb, dtype=torch.int32, device="cuda")

        def step(cs):
            dev.forward_device(method, x, y, tau=tau, batch=nb, alive_out=alive, stream=cs)

        with torch.cuda.stream(stream):
            for _ in range(3):
                step(stream.cuda_stream)
        torch.cuda.synchronize()
        path = dev.last_path()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if a.no_graph:
            e0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(a.steps):
                    step(stream.cuda_stream)
            e1.record(stream)
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(a.steps):
                        step(torch.cuda.current_stream().cuda_stream)
            g.replay()
            torch.cuda.synchronize()
            e0.record(stream)
            with torch.cuda.stream(stream):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.steps
        flops = 2 * 3 * F * D * nb
        sp = 1 - alive.float().mean().item() / F
        print(json.dumps({"case": case, "batch": nb, "path": path, "us_per_step": round(us, 2),
                          "tokens_per_s": round(nb / us * 1e6, 1), "weight_gbs": round(wbytes / us / 1e3, 1),
                          "tflops": round(flops / us / 1e6, 1), "sparsity": round(sp, 4)}), flush=True)


if __name__ == "__main__":
    main()
