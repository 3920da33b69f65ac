"""Run N decode steps of one method at the Llama shape without graphs (for ncu capture).

usage: python tools/prof_step.py [dc|mc|dense] [k] [steps] [dtype]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_17701_b200 as cd  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "dc"
k = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dtype = sys.argv[4] if len(sys.argv) > 4 else "bf16"
d, F, r = 4096, 14336, 512
layer, x0, pred = cd.synth_workload(42, d, F, r if method == "dc" else 0, device_dtype=dtype)
dev = layer.device_layer(pred)
NX = 8
X = np.stack([cd.synth_normals(1000 + i, d) for i in range(NX)])
if method == "dc":
    z = dev.predict_logits(X)
    tau = float(np.mean([np.quantile(z[i], k) for i in range(NX)]))
    mid = 2
elif method == "mc":
    u = np.abs(cd.pipeline_mc(layer, X, float("inf"), want_u=True).u)
    tau = float(np.mean([np.quantile(u[i], k) for i in range(NX)]))
    mid = 1
else:
    tau, mid = 0.0, 0
xs = torch.from_numpy(X).cuda()
ys = torch.empty((NX, d), device="cuda")
s = torch.cuda.Stream()
for i in range(steps):
    dev.forward_device(mid, xs[i % NX], ys[i % NX], tau, stream=s.cuda_stream)
torch.cuda.synchronize()
print(f"{method} k={k} tau={tau:.4f} steps={steps} launches/step={dev.last_launches()}")
