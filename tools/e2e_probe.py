"""Where does a synchronous host-buffer call's time go?  Llama shape, DC 90%, batch 1.
(a) cd_pipeline_dc host call; (b) forward_device + synchronize; (c) one step in a graph + sync;
(d) K steps in one graph (per step)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import _capi  # noqa: E402
from paper_2505_17701_b200._capi import check, lib, ptr  # noqa: E402

D, F, R = 4096, 14336, 512
layer, _, pred = cd.synth_workload(42, D, F, R, device_dtype="bf16")
dev = layer.device_layer(pred)
x = cd.synth_normals(5, D)
z = cd.predict_logits(pred, x)
tau = float(np.quantile(z, 0.9))
N = 300
yh = np.empty(D, np.float32)
ah = np.empty(1, np.int64)
L = lib()


def timeit(name, fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    torch.cuda.synchronize()
    print(f"{name:48s} {1e6 * (time.perf_counter() - t0) / N:8.2f} us/call", flush=True)


timeit("(a) cd_pipeline_dc host call", lambda: check(L.cd_pipeline_dc(dev.raw, 1, ptr(x), tau, None, 1, ptr(yh), None,
                                                                     ptr(ah), None)))
print("host call launches:", dev.last_launches(), "path:", dev.last_path(), flush=True)
dev.set_engines(pdl_chain=True)
timeit("(a2) cd_pipeline_dc host call, PDL chain", lambda: check(L.cd_pipeline_dc(dev.raw, 1, ptr(x), tau, None, 1,
                                                                              ptr(yh), None, ptr(ah), None)))
dev.set_engines()
xd = torch.from_numpy(x).cuda()
yd = torch.empty(D, device="cuda")
s = torch.cuda.Stream()


def dev_call():
    dev.forward_device(_capi.METHOD_DC, xd, yd, tau=tau, stream=s.cuda_stream)
    s.synchronize()


timeit("(b) forward_device + stream sync", dev_call)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        dev.forward_device(_capi.METHOD_DC, xd, yd, tau=tau, stream=torch.cuda.current_stream().cuda_stream)


def g_call():
    g.replay()
    torch.cuda.synchronize()


timeit("(c) 1-step graph replay + sync", g_call)
xh = torch.from_numpy(x).pin_memory()
yh_t = torch.empty(D).pin_memory()


def g_copy_call():
    with torch.cuda.stream(s):
        xd.copy_(xh, non_blocking=True)
        g.replay()
        yh_t.copy_(yd, non_blocking=True)
    s.synchronize()


timeit("(d) H2D + graph + D2H + sync (torch)", g_copy_call)
timeit("(e) empty stream sync", lambda: s.synchronize())
