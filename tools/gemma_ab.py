"""Gemma-2-9B FFN decode step time at a batch (4 rotating replicas, graph of 64 steps, >= 60 ms
of replays).  usage: CD_LIB_DIR=... python tools/gemma_ab.py [dc|mc] [batch]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_17701_b200 as cd  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "dc"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
D, F, R, NL = 3584, 14336, 512, 4
layer, _, pred = cd.synth_workload(142, D, F, R, activation=cd.Activation.GeluTanh, device_dtype="bf16")
devs = [layer.device_layer(pred)] + [cd.GatedMlpLayer(D, F, 1, layer.w_up, layer.w_gate, layer.w_down,
                                                      device_dtype="bf16").device_layer(pred) for _ in range(NL - 1)]
for dv in devs:
    dv.set_engines(pdl_chain=True)
X = np.stack([cd.synth_normals(60 + i, D) for i in range(16)])
if method == "dc":
    z = devs[0].predict_logits(X)
    tau = float(np.mean([np.quantile(z[i], 0.9) for i in range(16)]))
    mid = cd._capi.METHOD_DC
else:
    u = np.abs(cd.pipeline_mc(layer, X, float("inf"), want_u=True).u)
    tau = float(np.mean([np.quantile(u[i], 0.9) for i in range(16)]))
    mid = cd._capi.METHOD_MC
xs = torch.from_numpy(X).cuda()
ys = torch.zeros((NL, 16, D), device="cuda")
s = torch.cuda.Stream()
nx = 16 // B


def fwd(i):
    li, xi = i % NL, (i // NL) % nx
    devs[li].forward_device(mid, xs[xi * B:(xi + 1) * B], ys[li, :B], tau, batch=B, stream=s.cuda_stream)


with torch.cuda.stream(s):
    for i in range(2 * NL):
        fwd(i)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(64):
            fwd(i)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    torch.cuda.synchronize()
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(40):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{method} B={B} path={devs[0].last_path()} us/step={1e3 * e0.elapsed_time(e1) / (40 * 64):.2f}", flush=True)
