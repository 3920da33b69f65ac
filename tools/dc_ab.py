"""A/B timing of the headline step (Llama FFN, D-CountDown k, batch 1, 8 rotating replicas,
graph of 400 PDL-chained steps replayed >= 60 ms) for the library in CD_LIB_DIR.

usage: CD_LIB_DIR=_lib_x python tools/dc_ab.py [k] [reps]
prints one line per rep: "pf=<0|1> us=<us/token>"
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_17701_b200 as cd  # noqa: E402

k = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
method = os.environ.get("AB_METHOD", "dc")
d, F, r, NL, NX, STEPS = 4096, 14336, 512, 8, 16, 400
layer, _, pred = cd.synth_workload(42, d, F, r, device_dtype="bf16")
devs = [layer.device_layer(pred)] + [cd.GatedMlpLayer(d, F, 0, layer.w_up, layer.w_gate, layer.w_down,
                                                      device_dtype="bf16").device_layer(pred) for _ in range(NL - 1)]
for dv in devs:
    dv.set_engines(pdl_chain=os.environ.get("AB_COOP") != "1")
X = np.stack([cd.synth_normals(1000 + i, d) for i in range(NX)])
mid = {"dc": cd._capi.METHOD_DC, "mc": cd._capi.METHOD_MC, "dense": cd._capi.METHOD_DENSE}[method]
if method == "dc":
    z = devs[0].predict_logits(X)
    tau = float(np.mean([np.quantile(z[i], k) for i in range(NX)]))
elif method == "mc":
    u = np.abs(cd.pipeline_mc(layer, X, float("inf"), want_u=True).u)
    tau = float(np.mean([np.quantile(u[i], k) for i in range(NX)]))
else:
    tau = 0.0
xs = torch.from_numpy(X).cuda()
ys = torch.zeros((NL, NX, d), device="cuda")
s = torch.cuda.Stream()


def fwd(i):
    devs[i % NL].forward_device(mid, xs[i % NX], ys[i % NL, i % NX], tau, stream=s.cuda_stream)


def timed(g, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(n):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(reps):
    for pf in (0, 1):
        for i, dv in enumerate(devs):
            dv.set_prefetch(devs[(i + 1) % NL] if pf else None)
        with torch.cuda.stream(s):
            for i in range(2 * NL):
                fwd(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for i in range(STEPS):
                    fwd(i)
        one = timed(g, 1)
        n = max(2, int(np.ceil(60.0 / one)))
        ms = timed(g, n)
        print(f"{method} k={k} pf={pf} us={1e3 * ms / (n * STEPS):.3f}", flush=True)
        del g
