"""CDWN1 model files (model_io.cpp:94-224), SURVEY.md section 8f row 2.

Host side (CPU): paper_2505_17701_b200.read_model / write_model against the UNMODIFIED
reference (oracle/_ref built with model_io.cpp): byte-identical files, bit-identical weights,
and the same DataError for every malformed input the reference rejects.  Device side (GPU):
the C-ABI loader cd_layer_load_cdwn1 uploads the same layer the host arrays give.
"""
import os

import numpy as np
import pytest

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import DataError


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("seed,d,F,r,act", [(101, 20, 48, 6, 0), (7, 33, 70, 0, 1)])
def test_reference_file_reads_bitwise_and_rewrites_identically(reference, tmp_path, seed, d, F, r, act):
    path = tmp_path / "m.cdwn"
    reference.write_model(path, seed, d, F, r, act, 0.7)
    want = reference.read_model(path)
    mf = cd.read_model(str(path))
    assert (mf.layer.d_model, mf.layer.d_inter, int(mf.layer.activation), mf.seed) == (d, F, act, seed)
    for a, b in ((mf.layer.w_up, want["w_up"]), (mf.layer.w_gate, want["w_gate"]), (mf.layer.w_down, want["w_down"])):
        assert np.array_equal(bits(a), bits(b))
    if r:
        lp = mf.predictor.lowrank()
        assert np.array_equal(bits(lp.theta_a), bits(want["theta_a"]))
        assert np.array_equal(bits(lp.theta_b), bits(want["theta_b"]))
        assert mf.predictor_k == 0.7
    else:
        assert mf.predictor is None
    out = tmp_path / "again.cdwn"
    cd.write_model(str(out), mf)
    assert open(out, "rb").read() == open(path, "rb").read()
    assert cd.checksum_hex(mf.layer.w_up[:3]) == cd.checksum_hex(want["w_up"][:3])


def _corrupt(src, dst, fn):
    b = bytearray(open(src, "rb").read())
    open(dst, "wb").write(bytes(fn(b)))


@pytest.mark.parametrize("what", ["magic", "truncated", "payload", "nonfinite", "activation"])
def test_malformed_files_rejected_like_reference(reference, tmp_path, what):
    import oracle as O
    good = tmp_path / "good.cdwn"
    reference.write_model(good, 5, 8, 16, 4, 0, 0.5)
    bad = tmp_path / "bad.cdwn"
    hlen = int(np.frombuffer(open(good, "rb").read()[5:9], np.uint32)[0])

    def mutate(b):
        if what == "magic":
            b[0:5] = b"XDWN1"
        elif what == "truncated":
            del b[7:]
        elif what == "payload":
            del b[-4:]
        elif what == "nonfinite":
            b[9 + hlen + 8:9 + hlen + 12] = np.float32(np.nan).tobytes()
        elif what == "activation":
            h = bytes(b[9:9 + hlen]).replace(b'"silu"', b'"relu"')
            b[9:9 + hlen] = h
        return b

    _corrupt(good, bad, mutate)
    with pytest.raises(O.ReferenceError_) as ref_err:
        reference.read_model(bad)
    assert ref_err.value.code == 2  # DataError
    with pytest.raises(DataError) as ours:
        cd.read_model(str(bad))
    ref_msg = str(ref_err.value).split("] ", 1)[1]
    assert str(ours.value).split(":")[0] == ref_msg.split(":")[0]


@pytest.mark.gpu
def test_device_loader_matches_host_arrays(reference, oracle, tmp_path):
    path = tmp_path / "m.cdwn"
    reference.write_model(path, 106, 512, 2048, 64, 0, 0.9)
    dev = cd.DeviceLayer.load(str(path), "f32")
    assert (dev.d_model, dev.d_inter, dev.d_rank, dev.seed, dev.predictor_kind) == (512, 2048, 64, 106, "lowrank")
    g = oracle.generate(106, 512, 2048, 64)
    x = g["x"][None, :]
    _, z = oracle.lowrank_logits(g["theta_a"], g["theta_b"], g["x"])
    tau = float(np.quantile(z, 0.8))
    y, mask, alive, _ = dev.pipeline_dc(x, tau, cd.Reduction.DeterministicOrdered)
    want = oracle.pipeline_dc(g, g["x"], tau_d=tau)
    assert np.array_equal(mask[0], want["mask"]) and np.array_equal(bits(y[0]), bits(want["y"]))
    bad = tmp_path / "bad.cdwn"
    open(bad, "wb").write(b"XDWN1" + open(path, "rb").read()[5:])
    with pytest.raises(DataError, match="bad magic"):
        cd.DeviceLayer.load(str(bad))


@pytest.mark.gpu
def test_device_loader_bf16_batched_tensor_cores(reference, oracle, tmp_path):
    """A CDWN1 file loaded straight to bf16 device weights serves a batch of 16 on the
    tensor-core path; each sample matches the oracle on the bf16-rounded weights (1e-4)."""
    from conftest import bf16_round, rel_l2
    path = tmp_path / "m.cdwn"
    reference.write_model(path, 107, 384, 1536, 48, 1, 0.9)
    dev = cd.DeviceLayer.load(str(path), "bf16")
    g = oracle.generate(107, 384, 1536, 48)
    g = {k: bf16_round(v) for k, v in g.items()}
    rng = oracle.rng(5)
    X = np.stack([rng.normals_f(384) for _ in range(16)])
    y, mask, alive, z = dev.pipeline_dc(X, 0.05, cd.Reduction.UnorderedAccumulate, None, True)
    assert dev.last_path() == "tensor"
    for b in range(16):
        _, zb = oracle.lowrank_logits(g["theta_a"], g["theta_b"], X[b])
        assert rel_l2(z[b], zb) <= 1e-5
        assert rel_l2(y[b], oracle.forward_sparse(g, X[b], mask[b], act=1)) <= 1e-4
        assert alive[b] == int(mask[b].sum())
