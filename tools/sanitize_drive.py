"""Small calls through every engine, for compute-sanitizer (tools/sanitize.sh): fused batch-1
D-/M-CountDown (bf16 and f32, cooperative and PDL-chained), the batch-2..4 fused kernel, the
multi-kernel chains, the exact kernels, the tensor-core decode (two n-tiles) and prefill
(2-CTA clusters), the host-call CUDA graph, device top-m."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import Reduction  # noqa: E402

FAST = cd.BlockConfig(reduction=Reduction.UnorderedAccumulate)
ORD = cd.BlockConfig(reduction=Reduction.DeterministicOrdered)
d, F, r = 256, 1024, 64
keep = []
for dtype in ("bf16", "f32"):
    layer, x, pred = cd.synth_workload(5, d, F, r, device_dtype=dtype)
    keep += [layer, pred]
    X = np.stack([cd.synth_normals(100 + i, d) for i in range(4)])
    dev = layer.device_layer(pred)
    for pdl in (False, True):
        dev.set_engines(pdl_chain=pdl)
        for xb in (x, X[:2], X):
            cd.pipeline_dc(layer, xb, pred, FAST, tau_d=0.05)
            cd.pipeline_mc(layer, xb, 0.5, FAST)
    dev.set_engines(fused=False)
    cd.pipeline_dc(layer, X, pred, FAST, tau_d=0.05)
    cd.pipeline_mc(layer, X, 0.5, FAST)
    dev.set_engines()
    cd.pipeline_dc(layer, x, pred, ORD, tau_d=0.05)
    cd.pipeline_mc(layer, x, 0.5, ORD)
    cd.exec_dense(layer, x, FAST)
    for _ in range(3):  # host-call graph capture + replay
        cd.pipeline_dc(layer, x, pred, FAST, tau_d=0.05)
lb, _, pb = cd.synth_workload(6, 512, 1024, 128, device_dtype="bf16")
X = np.stack([cd.synth_normals(200 + i, 512) for i in range(70)])
cd.pipeline_dc(lb, X, pb, FAST, tau_d=0.05)
cd.pipeline_mc(lb, X, 0.5, FAST)
cd.exec_dense(lb, np.stack([cd.synth_normals(300 + i, 512) for i in range(300)]), FAST)
z = lb.device_layer(pb).predict_logits(X[:8])
cd.top_m_threshold(z[0], 100)
# release every handle before exit, so memcheck's leak check sees the library's own frees
for obj in keep + [lb, pb]:
    h = getattr(obj, "_dev", None) or getattr(obj, "_handle", None)
    if h is not None:
        h.close()
print("sanitize drive ok")
