"""N steps of one method at a batch size (Gemma-2-9B shape by default), no graphs, for ncu.
usage: python tools/prof_batch.py [dc|mc] [batch] [steps] [d] [F] [act]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_17701_b200 as cd  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "mc"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
d = int(sys.argv[4]) if len(sys.argv) > 4 else 3584
F = int(sys.argv[5]) if len(sys.argv) > 5 else 14336
act = int(sys.argv[6]) if len(sys.argv) > 6 else 1
layer, _, pred = cd.synth_workload(42, d, F, 512, activation=cd.Activation(act), device_dtype="bf16")
dev = layer.device_layer(pred)
X = np.stack([cd.synth_normals(1000 + i, d) for i in range(16)])
if method == "dc":
    z = dev.predict_logits(X)
    tau = float(np.mean([np.quantile(z[i], 0.9) for i in range(16)]))
    mid = cd._capi.METHOD_DC
else:
    u = np.abs(cd.pipeline_mc(layer, X, float("inf"), want_u=True).u)
    tau = float(np.mean([np.quantile(u[i], 0.9) for i in range(16)]))
    mid = cd._capi.METHOD_MC
xs = torch.from_numpy(X).cuda()
ys = torch.empty((16, d), device="cuda")
s = torch.cuda.Stream()
for i in range(steps):
    j = (i * B) % 16
    dev.forward_device(mid, xs[j:j + B], ys[j:j + B], tau, batch=B, stream=s.cuda_stream)
torch.cuda.synchronize()
print(f"{method} B={B} launches/step={dev.last_launches()} path={dev.last_path()}")
