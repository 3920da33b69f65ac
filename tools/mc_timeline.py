"""Phase stamps of k_mc_fused (CD_MC_TL development hook): Llama shape, MC 90%, batch 1, steps
chained in a CUDA graph (PDL); stamps of the last step, µs from the earliest CTA start.
0 start, 1 first W_up stage landed, 2 stage 1 done, 3 first record landed, 4 stage 3 done, 5 end."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("CD_LIB_DIR", "_lib_tl")  # the phase-stamp hooks exist only in the timeline build
sys.path.insert(0, ROOT)
tl = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
os.environ["CD_MC_TL"] = str(tl.data_ptr())
import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import _capi  # noqa: E402

D, F = 4096, 14336
layer, _, _ = cd.synth_workload(42, D, F, 0, device_dtype="bf16")
dev = layer.device_layer()
xs = np.stack([cd.synth_normals(100 + i, D) for i in range(4)])
u = np.abs(cd.pipeline_mc(layer, xs, float("inf"), cd.BlockConfig(reduction=cd.Reduction.DeterministicOrdered),
                          want_u=True).u)
tau = float(np.mean([np.quantile(r, 0.9) for r in u]))
x = torch.from_numpy(xs[0]).cuda()
y = torch.empty(D, device="cuda")
s = torch.cuda.Stream()
for _ in range(5):
    dev.forward_device(_capi.METHOD_MC, x, y, tau=tau, stream=s.cuda_stream)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            dev.forward_device(_capi.METHOD_MC, x, y, tau=tau, stream=torch.cuda.current_stream().cuda_stream)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
with torch.cuda.stream(s):
    g.replay()
e1.record(s)
torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) * 1e3 / 20:.2f} us/step")
t = tl.view(1024, 8).cpu().numpy()[:148].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
for k, name in enumerate(["start", "stage1_first", "stage1_done", "rec_first", "stage3_done", "end"]):
    col = rel[:, k]
    print(f"  {name:13s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
