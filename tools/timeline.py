"""Per-CTA phase timeline of one decode step (needs the _lib_tl build: CD_LIB_DIR=_lib_tl)."""
import ctypes as C
import os
import sys

import numpy as np

os.environ.setdefault("CD_LIB_DIR", "_lib_tl")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import _capi  # noqa: E402

K, CT, P = 8, 160, 8
NAMES = {0: "latent", 1: "ind_dc", 2: "sparse_dc", 3: "sparse_mc", 4: "st3_recs", 5: "dc_fused", 6: "fused_st2", 7: "fused_prod"}


def read():
    buf = np.zeros(K * CT * P, np.uint64)
    L = _capi.lib()
    L.cd_debug_timeline.argtypes = [C.c_void_p, C.c_int64]
    _capi.check(L.cd_debug_timeline(buf.ctypes.data_as(C.c_void_p), buf.size))
    return buf.reshape(K, CT, P).astype(np.int64)


def show(tl, label):
    cyc = tl[7, :148, 7].copy()
    s2 = tl[7, :148, 6].copy()
    tl[7, :, 7] = 0
    tl[7, :, 6] = 0
    c1 = tl[7, :148, 0:5].copy()
    tl[7, :, 0:5] = 0
    if (c1 > 0).any():
        m = np.median(c1[c1[:, 0] > 0], axis=0)
        print("    stage-1 cycles (thread 0): compute %d, transpose %d, bar %d, final+store %d, bar %d" % tuple(m))
    nrec = tl[4, :148, 7].copy()
    tl[4, :, 7] = 0
    if (nrec > 0).any():
        print(f"    stage-3 records per CTA: min {nrec.min()} median {np.median(nrec):.0f} max {nrec.max()}")
    if (s2 > 0).any():
        print(f"    stage-2 loop cycles (thread 0): median {np.median(s2[s2 > 0]):.0f}, max {s2.max():.0f}")
    if (cyc > 0).any():
        dur = (tl[5, :148, 7] - tl[5, :148, 0]) / 1e3
        ok = (cyc > 0) & (dur > 0)
        print(f"    fused kernel SM clock: median {np.median(cyc[ok] / dur[ok]) / 1e3:.0f} MHz "
              f"(cycles / globaltimer us over each CTA's lifetime)")
    nz = tl[tl > 0]
    t0 = nz.min()
    print(f"--- {label} (us relative to first stamp)")
    for k in range(K):
        if not (tl[k] > 0).any():
            continue
        parts = []
        for p in range(P):
            col = tl[k, :148, p]
            col = col[col > 0]
            if len(col):
                parts.append(f"p{p}:{(col.min()-t0)/1e3:6.2f}/{(np.median(col)-t0)/1e3:6.2f}/{(col.max()-t0)/1e3:6.2f}")
        print(f"  {NAMES.get(k, k):10s} " + "  ".join(parts))


method = sys.argv[1] if len(sys.argv) > 1 else "dc"
k = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
d, F, r = 4096, 14336, 512
layer, x0, pred = cd.synth_workload(42, d, F, r if method == "dc" else 0, device_dtype="bf16")
dev = layer.device_layer(pred)
X = np.stack([cd.synth_normals(1000 + i, d) for i in range(4)])
if method == "dc":
    z = dev.predict_logits(X)
    tau, mid = float(np.quantile(z[0], k)), 2
elif method == "mc":
    u = np.abs(cd.pipeline_mc(layer, X, float("inf"), want_u=True).u)
    tau, mid = float(np.quantile(u[0], k)), 1
else:
    tau, mid = 0.0, 0
xs = torch.from_numpy(X).cuda()
ys = torch.empty((4, d), device="cuda")
s = torch.cuda.Stream()
for i in range(5):
    dev.forward_device(mid, xs[i % 4], ys[i % 4], tau, stream=s.cuda_stream)
torch.cuda.synchronize()
read()
dev.forward_device(mid, xs[0], ys[0], tau, stream=s.cuda_stream)
show(read(), f"{method} k={k} single step, stream launch")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(4):
        dev.forward_device(mid, xs[i], ys[i], tau, stream=torch.cuda.current_stream().cuda_stream)
g.replay(); torch.cuda.synchronize(); read()
g.replay(); torch.cuda.synchronize()
show(read(), f"{method} k={k} graph of 4 steps (stamps of the last step)")
