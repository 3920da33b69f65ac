"""Generate tests/golden/golden.npz from the UNMODIFIED reference library (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref first):
    make -C oracle ref && python tests/golden/make_golden.py

Each case is identified by (seed, d, F, r, act); the inputs are NOT stored -- they are the
reference bench()'s seeded RNG stream (blocked_exec.cpp:396-415), which the oracle must
regenerate bit-for-bit (a 64-bit FNV-1a of every generated array is stored to pin that).
Stored outputs, all produced by the reference library itself:
  forward_dense u/h/s/y (gated_mlp.cpp:46-59), predict_logits (predictor.cpp:128-138),
  pipeline_mc at tau = top-(F/4) |u| (blocked_exec.cpp:316-328; mask, alive, y, traffic),
  pipeline_dc with the predictor's own z > 0 mask (blocked_exec.cpp:350-379),
  forward_sparse on the ideal top-(F/3) |s| mask (sparsity.cpp:44-71), and
  forward_practical MC at that tau (sparsity.cpp:90-121).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

CASES = [  # (seed, d, F, r, act)
    (101, 20, 48, 6, 0),
    (102, 24, 96, 8, 1),
    (103, 17, 53, 5, 0),
    (104, 64, 256, 16, 1),
    (42, 128, 448, 32, 0),
]


def fnv1a64(a: np.ndarray) -> int:
    """64-bit FNV-1a over the array bytes (the reference checksums y the same way,
    model_io.cpp:82-92, there as 32-bit)."""
    h = 0xcbf29ce484222325
    for b in np.ascontiguousarray(a).tobytes():
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def main():
    ref = O.Reference()
    out = {}
    for (seed, d, F, r, act) in CASES:
        k = f"s{seed}_d{d}_F{F}_r{r}_a{act}"
        g = ref.generate(seed, d, F, r, act)
        for name in ("w_up", "w_gate", "w_down", "x", "theta_a", "theta_b"):
            out[f"{k}/hash_{name}"] = np.array([fnv1a64(g[name])], np.uint64)
        x = g["x"]
        tr = ref.forward_dense(g, x, act)
        for n in ("u", "h", "s", "y"):
            out[f"{k}/dense_{n}"] = tr[n]
        out[f"{k}/logits"] = ref.predict_logits(g["theta_a"], g["theta_b"], x)
        tau_u, _ = ref.top_m_threshold(tr["u"], F // 4)
        mc = ref.pipeline_mc(g, x, tau_u, act=act)
        out[f"{k}/mc_tau"] = np.array([tau_u], np.float32)
        out[f"{k}/mc_mask"] = mc["mask"]
        out[f"{k}/mc_y"] = mc["y"]
        out[f"{k}/mc_traffic"] = np.array(mc["traffic"], np.int64)
        dc = ref.pipeline_dc(g, x, act=act)
        out[f"{k}/dc_mask"] = dc["mask"]
        out[f"{k}/dc_y"] = dc["y"]
        out[f"{k}/dc_traffic"] = np.array(dc["traffic"], np.int64)
        _, ideal = ref.top_m_threshold(tr["s"], F // 3)
        out[f"{k}/ideal_mask"] = ideal
        out[f"{k}/sparse_y"] = ref.forward_sparse(g, x, ideal, act)
        pr = ref.forward_practical("mc", g, x, tau_hat=tau_u, act=act)
        out[f"{k}/practical_mc_mask"] = pr["mask"]
        out[f"{k}/practical_mc_y"] = pr["y"]
    # scalar known answers
    out["alive_counts"] = np.array([ref.alive_count_for(k, 14336) for k in (0.7, 0.8, 0.9)], np.int64)
    xs = np.linspace(-20, 20, 401).astype(np.float32)
    out["act_x"] = xs
    out["act_silu"] = ref.activation(0, xs)
    out["act_gelu"] = ref.activation(1, xs)
    out["rng_normals_seed7"] = ref.rng_normals(7, 64)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
