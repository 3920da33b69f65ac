"""Per-CTA phase table of the LAST step of a 400-step graph over 8 rotating Llama replicas
(headline config), CD_TIMELINE build.  usage: python tools/timeline_cta.py [k] [pf]"""
import ctypes as C
import os
import sys

os.environ.setdefault("CD_LIB_DIR", "_lib_tl")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import _capi  # noqa: E402

K, CT, P = 8, 160, 8


def read():
    buf = np.zeros(K * CT * P, np.uint64)
    L = _capi.lib()
    L.cd_debug_timeline.argtypes = [C.c_void_p, C.c_int64]
    _capi.check(L.cd_debug_timeline(buf.ctypes.data_as(C.c_void_p), buf.size))
    return buf.reshape(K, CT, P).astype(np.int64)


k = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
pf = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d, F, r, NL, NX, STEPS = 4096, 14336, 512, 8, 16, 400
layer, _, pred = cd.synth_workload(42, d, F, r, device_dtype="bf16")
devs = [layer.device_layer(pred)] + [cd.GatedMlpLayer(d, F, 0, layer.w_up, layer.w_gate, layer.w_down,
                                                      device_dtype="bf16").device_layer(pred) for _ in range(NL - 1)]
for dv in devs:
    dv.set_engines(pdl_chain=os.environ.get("AB_COOP") != "1")
X = np.stack([cd.synth_normals(1000 + i, d) for i in range(NX)])
z = devs[0].predict_logits(X)
tau = float(np.mean([np.quantile(z[i], k) for i in range(NX)]))
xs = torch.from_numpy(X).cuda()
ys = torch.zeros((NL, NX, d), device="cuda")
s = torch.cuda.Stream()
for i, dv in enumerate(devs):
    dv.set_prefetch(devs[(i + 1) % NL] if pf else None)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(STEPS):
            devs[i % NL].forward_device(cd._capi.METHOD_DC, xs[i % NX], ys[i % NL, i % NX], tau,
                                        stream=torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
read()
g.replay()
torch.cuda.synchronize()
tl = read()[:, :148]
cyc = tl[2].copy()
xw = np.concatenate([tl[3], tl[7]], axis=1)[:, :13].astype(np.int64)  # per-warp x arrival (clock64)
tl[3] = 0
tl[7] = 0
rel = np.where((xw > 0) & (cyc[:, 0:1] > 0), xw - cyc[:, 0:1], np.iinfo(np.int64).min)
print("  per-warp x arrival after thread 0's wait mark (cycles, median over CTAs; n):",
      " ".join(f"{np.median(rel[rel[:, w] > -10**12, w]):.0f}({(rel[:, w] > -10**12).sum()})"
               if (rel[:, w] > -10**12).any() else "-" for w in range(13)))
tl[2] = 0
ok = (cyc[:, 0] > 0) & (cyc[:, 7] > 0)
if ok.any():
    names = ["wait->x", "x->bar(tag)", "bar->theta_a", "theta_a->s1cmp", "s1cmp->bar", "bar->pub", "pub->gathered"]
    d = np.diff(cyc[ok], axis=1)
    print("  thread-0 clock64 segments (cycles, median / p90 over CTAs with latent columns):")
    print("   " + "  ".join(f"{n} {np.median(d[:, i]):.0f}/{np.percentile(d[:, i], 90):.0f}" for i, n in enumerate(names)))
cnt = tl[1, :, 7].copy()
tl[1, :, 7] = 0
nrec = tl[4, :, 7].copy()
tl[4, :, 7] = 0
t0 = tl[5, :, 1].min()  # first CTA past griddepcontrol.wait
us = lambda a: (a - t0) / 1e3
cols = [("start", tl[5, :, 0]), ("wait", tl[5, :, 1]), ("theta_a", tl[1, :, 4]), ("theta_b", tl[1, :, 5]), ("x", tl[0, :, 0]), ("s1cmp", tl[0, :, 1]),
        ("s1bar", tl[0, :, 2]), ("s1pub", tl[0, :, 3]), ("s1done", tl[5, :, 2]), ("gath", tl[5, :, 3]),
        ("regs", tl[6, :, 0]), ("s2done", tl[6, :, 1]), ("prodgo", tl[6, :, 5]), ("own8", tl[1, :, 0]),
        ("rec0", tl[4, :, 0]), ("rec3", tl[4, :, 1]), ("ownall", tl[1, :, 1]), ("steal0", tl[1, :, 2]),
        ("stealN", tl[1, :, 3]), ("lastrec", tl[4, :, 3]), ("sentinel", tl[6, :, 4]), ("s3done", tl[5, :, 6]),
        ("end", tl[5, :, 7])]
print(f"k={k} pf={pf}: us after the first CTA passed griddepcontrol.wait; min / p50 / p90 / max over CTAs")
for name, c in cols:
    v = c[c > 0]
    if len(v):
        q = us(np.percentile(v, [0, 50, 90, 100]))
        print(f"  {name:9s} " + " ".join(f"{x:7.2f}" for x in q) + f"   (n={len(v)})")
own, kept, stolen = cnt & 0xFFFF, (cnt >> 16) & 0xFFFF, cnt >> 32
print(f"  n_own min/med/max {own.min()}/{np.median(own):.0f}/{own.max()}  kept med {np.median(kept):.0f}  "
      f"stolen min/med/max {stolen.min()}/{np.median(stolen):.0f}/{stolen.max()}  records min/med/max "
      f"{nrec.min()}/{np.median(nrec):.0f}/{nrec.max()}  total own {own.sum()}")
order = np.argsort(-tl[5, :, 7])
print("  slowest CTAs: cta own kept stolen recs | s2done ownall stealN lastrec s3done end")
for c in order[:10]:
    print(f"   {c:4d} {own[c]:3d} {kept[c]:3d} {stolen[c]:3d} {nrec[c]:3d} | " +
          " ".join(f"{us(tl[a, c, b]):6.2f}" if tl[a, c, b] > 0 else "     -" for a, b in
                   ((6, 1), (1, 1), (1, 3), (4, 3), (5, 6), (5, 7))))
