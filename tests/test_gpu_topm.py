"""Device top-m (kernels_topm.cu) against the reference's top_m_threshold (numerics.cpp:105-142)
and calibrate (calibration.cpp:11-37), both run from the unmodified reference library.

Contract: bit-identical tau and identical masks -- larger magnitude first, ties to the lower
index, tau = the (m+1)-th magnitude, +inf / -inf at m = 0 / n; calibrate's tau_hat equal as a
double.  Edge cases the reference tests: m = 0, m = n, n = 1, heavy ties, negative zeros.
"""
import numpy as np
import pytest

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import DataError

pytestmark = pytest.mark.gpu


def f32_bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("n", [1, 2, 17, 1000, 4097, 13824, 14336])
def test_top_m_matches_reference(reference, n):
    rng = np.random.default_rng(n)
    v = rng.standard_normal(n).astype(np.float32)
    for m in sorted({0, 1, n // 3, n // 2, max(0, n - 1), n}):
        tau, mask = cd.top_m_threshold(v, m)
        rt, rm = reference.top_m_threshold(v, m)
        assert f32_bits(tau) == f32_bits(rt), (n, m, tau, rt)
        assert np.array_equal(mask, rm), (n, m)
        assert int(mask.sum()) == m


def test_top_m_ties_go_to_the_lower_index(reference):
    rng = np.random.default_rng(7)
    for n in (64, 1000, 14336):
        # few distinct magnitudes, both signs, +0 / -0: every threshold sits inside a tie
        v = (rng.integers(-4, 5, n).astype(np.float32) * np.float32(0.25))
        v[rng.integers(0, n, n // 10)] = -0.0
        for m in (1, n // 7, n // 2, n - 3):
            tau, mask = cd.top_m_threshold(v, m)
            rt, rm = reference.top_m_threshold(v, m)
            assert f32_bits(tau) == f32_bits(rt) and np.array_equal(mask, rm), (n, m)


def test_top_m_batched_and_signed(reference):
    rng = np.random.default_rng(3)
    V = rng.standard_normal((5, 3000)).astype(np.float32)
    taus, masks = cd.top_m_threshold(V, 301)
    for b in range(5):
        rt, rm = reference.top_m_threshold(V[b], 301)
        assert f32_bits(taus[b]) == f32_bits(rt) and np.array_equal(masks[b], rm)
    # signed order: the (m+1)-th largest VALUE, ties to the lower index (lexsort)
    taus, masks = cd.top_m_threshold(V, 301, signed=True)
    for b in range(5):
        order = np.lexsort((np.arange(3000), -V[b]))
        assert f32_bits(taus[b]) == f32_bits(V[b][order[301]])
        want = np.zeros(3000, np.uint8)
        want[order[:301]] = 1
        assert np.array_equal(masks[b], want)


def test_top_m_errors_follow_the_reference():
    with pytest.raises(DataError, match="empty vector"):
        cd.top_m_threshold(np.zeros(0, np.float32), 0)
    with pytest.raises(DataError, match=r"m = 5 outside \[0, 4\]"):
        cd.top_m_threshold(np.ones(4, np.float32), 5)


@pytest.mark.slow
def test_calibrate_bitwise_at_llama_shape(reference):
    """calibrate(MC) at the Llama-3.1-8B shape: tau_hat bitwise the reference's (exact u folds +
    exact top-m + the ascending double mean); CATS checked against the reference's trace h."""
    d, F = 4096, 14336
    g = reference.generate(42, d, F, 0)
    layer = cd.GatedMlpLayer(d, F, 0, g["w_up"], g["w_gate"], g["w_down"])
    xs = np.stack([reference.rng_normals(600 + i, d).astype(np.float32) for i in range(6)])
    for k in (0.7, 0.9):
        got, per = cd.calibrate(layer, xs, k, cd.SparsityMethod.MCountdown, per_sample=True)
        assert got == reference.calibrate_mc(g["w_up"], xs, k)
    m = cd.alive_count_for(0.8, F)
    got, per = cd.calibrate(layer, xs, 0.8, cd.SparsityMethod.Cats, per_sample=True)
    acc = 0.0
    for b, x in enumerate(xs):
        h = reference.forward_dense(g, x)["h"]
        t, _ = reference.top_m_threshold(h, m)
        assert f32_bits(per[b]) == f32_bits(t)
        acc += float(np.float32(t))
    assert got == acc / len(xs)
