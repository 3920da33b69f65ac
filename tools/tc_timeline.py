"""Phase stamps of the tensor-core gate/up kernel (CD_TC_TL development hook), one MC batch-64
step at the Qwen shape.  Prints per-CTA µs since the earliest CTA start for:
0 start, 1 first TMA, 2 last MMA commit, 3/4/5 epilogue segment 0/1/2+ begin, 6 epilogue end, 7 exit."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("CD_LIB_DIR", "_lib_tl")  # the phase-stamp hooks exist only in the timeline build
sys.path.insert(0, ROOT)
tl = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
os.environ["CD_TC_TL"] = str(tl.data_ptr())
import paper_2505_17701_b200 as cd  # noqa: E402
from paper_2505_17701_b200 import _capi  # noqa: E402

D, F, R = 5120, 13824, 512
layer, _, pred = cd.synth_workload(42, D, F, R, device_dtype="bf16")
dev = layer.device_layer(pred)
x = torch.randn(64, D, device="cuda")
y = torch.empty(64, D, device="cuda")
for method in (_capi.METHOD_MC, _capi.METHOD_DC):
    for _ in range(3):
        tl.zero_()
        dev.forward_device(method, x, y, tau=0.5, batch=64)
        torch.cuda.synchronize()
    t = tl.view(1024, 8).cpu().numpy().astype(np.int64)
    n = int((t[:, 0] > 0).sum())
    t = t[:n]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print("method", method, "CTAs", n)
    names = (["start", "mmaA_end", "prod_swait", "prod_sgo", "epiA_end", "epiB_end", "fin_flags", "fin_start"]
             if os.environ.get("CD_TC_FUSED", "1") != "0" else
             ["start", "tma0", "mma_end", "epi0", "epi1", "epi2", "epi_end", "exit"])
    for k, name in enumerate(names):
        col = rel[:, k]
        if np.all(np.isnan(col)):
            continue
        print(f"  {name:8s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f}")

    # the CTAs whose phase-A epilogue ends last (they gate "s complete")
    order = np.argsort(-np.nan_to_num(rel[:, 4]))
    F_ = F
    nkbA = (D + 63) // 64 + ((R + 63) // 64 if method == _capi.METHOD_DC else 0)
    tiles = (F_ + 127) // 128
    U = tiles * nkbA
    print("  latest epiA_end: cta | range units [lo, hi) tiles | mmaA_end fin_start epiA_end")
    for c in order[:6]:
        lo, hi = c * U // n, (c + 1) * U // n
        print(f"   {c:4d} | [{lo}, {hi}) tiles {lo // nkbA}..{(hi - 1) // nkbA} | "
              f"{rel[c, 1]:6.2f} {rel[c, 7]:6.2f} {rel[c, 4]:6.2f}")
