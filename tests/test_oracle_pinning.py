"""Pin the CPU oracle (oracle/countdown_oracle.c) before trusting it (CPU only).

1. Against the committed golden fixtures (tests/golden/golden.npz, produced by the unmodified
   reference library via tests/golden/make_golden.py): bit-for-bit.
2. Against the reference library itself (oracle/_ref, when built here): bit-for-bit on
   fresh random cases, including near-tie and NaN-poisoned inputs.
3. The reference's own unit tests (test_numerics / gated_mlp / sparsity / blocked_exec /
   costmodel / predictor / calibration) compiled against the reference library.
4. The reference's frozen integers (test_sparsity.cpp:59-70, test_costmodel.cpp:21-53).
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def fnv1a64(a):
    h = 0xcbf29ce484222325
    for b in np.ascontiguousarray(a).tobytes():
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def cases(golden):
    keys = sorted({k.split("/")[0] for k in golden.files if "/" in k})
    out = []
    for k in keys:
        s, d, F, r, a = k.split("_")
        out.append((k, int(s[1:]), int(d[1:]), int(F[1:]), int(r[1:]), int(a[1:])))
    return out


def test_golden_generation_bitwise(oracle, golden):
    """numerics.cpp:11-24 (splitmix64 + Box-Muller with spare), gated_mlp.cpp:61-75,
    predictor.cpp:52-69: identical streams."""
    for k, seed, d, F, r, act in cases(golden):
        g = oracle.generate(seed, d, F, r)
        for name in ("w_up", "w_gate", "w_down", "x", "theta_a", "theta_b"):
            assert fnv1a64(g[name]) == int(golden[f"{k}/hash_{name}"][0]), (k, name)


def test_golden_dense_and_logits_bitwise(oracle, golden):
    for k, seed, d, F, r, act in cases(golden):
        g = oracle.generate(seed, d, F, r)
        tr = oracle.forward_dense(g, g["x"], act)
        for n in ("u", "h", "s", "y"):
            assert np.array_equal(bits(tr[n]), bits(golden[f"{k}/dense_{n}"])), (k, n)
        _, z = oracle.lowrank_logits(g["theta_a"], g["theta_b"], g["x"])
        assert np.array_equal(bits(z), bits(golden[f"{k}/logits"])), k


def test_golden_pipelines_bitwise(oracle, golden):
    for k, seed, d, F, r, act in cases(golden):
        g = oracle.generate(seed, d, F, r)
        x = g["x"]
        tau = float(golden[f"{k}/mc_tau"][0])
        u = oracle.gemv(g["w_up"], x)
        t2, _ = oracle.top_m_threshold(u, F // 4)
        assert np.float32(t2) == np.float32(tau)
        mc = oracle.pipeline_mc(g, x, tau, act=act)
        assert np.array_equal(mc["mask"], golden[f"{k}/mc_mask"]), k
        assert np.array_equal(bits(mc["y"]), bits(golden[f"{k}/mc_y"])), k
        assert oracle.traffic_split("mc", d, F, 0, mc["alive"]) == tuple(golden[f"{k}/mc_traffic"])
        dc = oracle.pipeline_dc(g, x, tau_d=0.0, act=act)
        assert np.array_equal(dc["mask"], golden[f"{k}/dc_mask"]), k
        assert np.array_equal(bits(dc["y"]), bits(golden[f"{k}/dc_y"])), k
        assert oracle.traffic_split("dc", d, F, r, dc["alive"]) == tuple(golden[f"{k}/dc_traffic"])
        ideal = golden[f"{k}/ideal_mask"]
        tr = oracle.forward_dense(g, x, act)
        _, m2 = oracle.top_m_threshold(tr["s"], F // 3)
        assert np.array_equal(m2, ideal)
        assert np.array_equal(bits(oracle.forward_sparse(g, x, ideal, act)), bits(golden[f"{k}/sparse_y"]))
        # forward_practical MC == pipeline_mc semantics (sparsity.cpp:103-111)
        assert np.array_equal(mc["mask"], golden[f"{k}/practical_mc_mask"])
        assert np.array_equal(bits(mc["y"]), bits(golden[f"{k}/practical_mc_y"]))


def test_golden_scalars(oracle, golden):
    assert [oracle.alive_count_for(k, 14336) for k in (0.7, 0.8, 0.9)] == list(golden["alive_counts"])
    xs = golden["act_x"]
    silu = np.array([oracle.act(0, float(v)) for v in xs], np.float32)
    gelu = np.array([oracle.act(1, float(v)) for v in xs], np.float32)
    assert np.array_equal(bits(silu), bits(golden["act_silu"]))
    assert np.array_equal(bits(gelu), bits(golden["act_gelu"]))
    r = oracle.rng(7)
    assert np.array_equal(np.array([r.normal() for _ in range(64)]), golden["rng_normals_seed7"])


def test_frozen_integers(oracle):
    """test_sparsity.cpp:59-70 and test_costmodel.cpp:21-53."""
    assert [oracle.alive_count_for(k, 14336) for k in (0.7, 0.8, 0.9)] == [4300, 2867, 1433]
    d, F, r = 4096, 14336, 512
    assert sum(oracle.traffic_split("dense", d, F)) == 176287744
    assert oracle.traffic_split("dense", d, F) == (176160768, 65536, 61440)
    want_mc = {0.7: 94077132, 0.8: 82336563, 0.9: 70587801}
    want_dc = {0.7: 62374912, 0.8: 44766208, 0.9: 27145216}
    for k in (0.7, 0.8, 0.9):
        s = oracle.alive_count_for(k, F)
        assert sum(oracle.traffic_split("mc", d, F, 0, s)) == want_mc[k]
        assert sum(oracle.traffic_split("dc", d, F, r, s)) == want_dc[k]
    assert oracle.L.cdo_flops_dense(d, F, 5) == 352407552
    assert oracle.L.cdo_flops_mc(d, F, 1433, 5) == 140956054
    assert oracle.L.cdo_flops_dc(d, F, r, 1433, 5) == 54114710
    assert oracle.L.cdo_traffic_dc_oracle(d, F, 1433) == 17707008


def test_hand_examples(oracle):
    """test_numerics.cpp:105-120, test_predictor.cpp:60-70, test_gated_mlp.cpp:28-37."""
    w = np.array([[1, 1], [2, 0]], np.float32)
    assert oracle.gemv(w, np.array([3, 4], np.float32)).tolist() == [7.0, 6.0]
    _, z = oracle.lowrank_logits(np.array([[2.0]], np.float32), np.array([[3.0, -1.0]], np.float32),
                                 np.array([1.0], np.float32))
    assert z.tolist() == [6.0, -2.0]
    one = np.ones((1, 1), np.float32)
    L = dict(w_up=10 * one, w_gate=3 * one, w_down=one)
    y = oracle.forward_dense(L, np.array([1.0], np.float32))["y"]
    assert y[0] == np.float32(10.0) * np.float32(oracle.act(0, 3.0))


# ----------------------------------------------------------------------------- vs live reference
@pytest.mark.parametrize("seed,d,F,r,act", [(7, 33, 120, 9, 0), (8, 64, 200, 12, 1), (9, 5, 7, 2, 0)])
def test_oracle_matches_reference_library(oracle, reference, seed, d, F, r, act):
    g = oracle.generate(seed, d, F, r)
    gr = reference.generate(seed, d, F, r, act)
    for n in g:
        assert np.array_equal(bits(g[n]), bits(gr[n])), n
    x = g["x"]
    a = oracle.forward_dense(g, x, act)
    b = reference.forward_dense(g, x, act)
    for n in ("u", "h", "s", "y"):
        assert np.array_equal(bits(a[n]), bits(b[n])), n
    _, z = oracle.lowrank_logits(g["theta_a"], g["theta_b"], x)
    assert np.array_equal(bits(z), bits(reference.predict_logits(g["theta_a"], g["theta_b"], x)))
    for m in (0, 1, F // 3, F - 1, F):
        ta, ma = oracle.top_m_threshold(a["s"], m)
        tb, mb = reference.top_m_threshold(a["s"], m)
        assert (np.isinf(ta) and np.isinf(tb) and np.sign(ta) == np.sign(tb)) or ta == tb
        assert np.array_equal(ma, mb)
    # ties: top-m resolves ties to the lower index (numerics.cpp:105-142)
    v = np.array([1, -2, 2, 2, 0, -2, 1], np.float32)
    for m in range(8):
        assert np.array_equal(oracle.top_m_threshold(v, m)[1], reference.top_m_threshold(v, m)[1])
    tau = float(np.median(np.abs(a["u"])))
    pm, rm = oracle.pipeline_mc(g, x, tau, act=act), reference.pipeline_mc(g, x, tau, act=act)
    assert np.array_equal(pm["mask"], rm["mask"]) and np.array_equal(bits(pm["y"]), bits(rm["y"]))
    pd, rd = oracle.pipeline_dc(g, x, act=act), reference.pipeline_dc(g, x, act=act)
    assert np.array_equal(pd["mask"], rd["mask"]) and np.array_equal(bits(pd["y"]), bits(rd["y"]))
    # blocked executors == semantic forward, any block shape, Ordered (test_blocked_exec.cpp:72-85)
    _, ideal = oracle.top_m_threshold(a["s"], max(1, F // 3))
    want = oracle.forward_sparse(g, x, ideal, act)
    for blk in ((1, 1), (3, 4), (8, 1), (16, 256)):
        y, _ = reference.exec_dc(g, x, ideal, blk, 0, act)
        assert np.array_equal(bits(y), bits(want))
    # calibration (calibration.cpp:11-37)
    xs = np.stack([oracle.rng(1000 + i).normals_f(d) for i in range(5)])
    assert oracle.calibrate_mc(g["w_up"], xs, 0.7) == reference.calibrate_mc(g["w_up"], xs, 0.7)


def test_reference_unit_tests_pass():
    """The reference's own doctest suites against the reference library (oracle/_ref)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests_cpu")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_unit_tests_cpu not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_reference_model_handle_matches_per_call_pipeline(reference):
    """bench.py --impl reference times pipeline_dc on a reference layer / predictor built once;
    it must be bit-identical to the per-call path (with and without a mask override)."""
    g = reference.generate(42, 256, 1024, 32)
    h = reference.model(g)
    try:
        for mo in (None, (np.arange(1024) % 3 == 0).astype(np.uint8)):
            a = reference.model_pipeline_dc(h, g["x"], 256, mo)
            b = reference.pipeline_dc(g, g["x"], mo)
            assert np.array_equal(a["y"].view(np.uint32), b["y"].view(np.uint32)) and a["alive"] == b["alive"]
    finally:
        reference.model_free(h)
