"""CPU-side checks of the drop-in boundary (no GPU needed, no compute calls).

* libcountdown_b200.so loads and exports every function include/countdown_b200.h declares,
  and the ctypes binding covers exactly that set;
* the library is sm_100a code (cuobjdump) and reports loud failures without a device;
* the host mirror of the reference API validates arguments with the reference's error
  taxonomy (DataError) before any device work (gated_mlp.cpp:8-26, blocked_exec.cpp:24-36);
* the host-side synthetic workload is bit-identical to the oracle's (numerics.cpp:11-24).
"""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

import paper_2505_17701_b200 as cd
from paper_2505_17701_b200 import _capi


def test_header_symbols_exported_and_bound():
    syms = _capi.header_symbols()
    assert len(syms) >= 20
    L = _capi.lib()
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/countdown_b200.h but not exported"
    assert set(syms) == set(_capi._SIGNATURES), set(syms) ^ set(_capi._SIGNATURES)
    # nothing else is exported with default visibility
    nm = shutil.which("nm")
    if nm:
        out = subprocess.run([nm, "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
        exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln and ln.split()[-1].startswith("cd_")}
        assert exported == set(syms), exported ^ set(syms)


def test_library_is_sm100a_only():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    archs = {tok for ln in out.splitlines() for tok in ln.replace(".", " ").split() if tok.startswith("sm_")}
    assert archs == {"sm_100a"}, archs


def test_fails_loudly_without_gpu():
    """No CPU fallback: with no device every compute entry point reports an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _capi.lib()
    out = C.c_void_p()
    w = np.zeros((4, 8), np.float32)
    rc = L.cd_layer_create(0, 8, 4, 0, 0, _capi.ptr(w), _capi.ptr(w), _capi.ptr(w), C.byref(out))
    assert rc == _capi.CD_ERR_CUDA
    assert L.cd_last_error().decode()
    layer = cd.GatedMlpLayer(8, 4, cd.Activation.Silu, w, w, w)
    with pytest.raises(cd.CudaError):
        cd.exec_dense(layer, np.zeros(8, np.float32))


def test_data_errors_before_device_work():
    w = np.zeros((4, 8), np.float32)
    bad = cd.GatedMlpLayer(8, 4, cd.Activation.Silu, w, w, np.zeros((4, 7), np.float32))
    with pytest.raises(cd.DataError):
        bad.validate()
    layer = cd.GatedMlpLayer(8, 4, cd.Activation.Silu, w, w, w)
    with pytest.raises(cd.DataError):
        cd.exec_dc(layer, np.zeros(8, np.float32), np.ones(5, np.uint8))   # mask lanes
    with pytest.raises(cd.DataError):
        cd.exec_dc(layer, np.zeros(7, np.float32), np.ones(4, np.uint8))   # x length
    with pytest.raises(cd.DataError):
        cd.forward_practical(layer, np.zeros(8, np.float32),
                             cd.SparsityConfig(cd.SparsityMethod.MCountdown, cd.SparsityMode.Practical, 0.5),
                             cd.PracticalContext())
    with pytest.raises(cd.DataError):
        cd.alive_count_for(1.0, 10)
    with pytest.raises(cd.DataError):
        cd.realized_sparsity(cd.ActivationMask())
    L = _capi.lib()
    # null handles / arguments are data errors at the ABI, before any CUDA call
    assert L.cd_exec_dense(None, 1, None, 1, None) == _capi.CD_ERR_DATA
    assert L.cd_layer_destroy(None) == _capi.CD_OK
    assert L.cd_bench_stages(None, 0, 2, 1, None, 0.0, 0, 1, None, None) == _capi.CD_ERR_DATA


def test_synth_matches_oracle(oracle):
    """cd_synth_layer (host C++) reproduces the reference bench() workload bit-for-bit."""
    layer, x, pred = cd.synth_workload(1234, 24, 80, 6)
    g = oracle.generate(1234, 24, 80, 6)
    for a, b in ((layer.w_up, g["w_up"]), (layer.w_gate, g["w_gate"]), (layer.w_down, g["w_down"]),
                 (x, g["x"]), (pred.lowrank().theta_a, g["theta_a"]), (pred.lowrank().theta_b, g["theta_b"])):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(cd.synth_normals(77, 33), oracle.rng(77).normals_f(33))


def test_costmodel_frozen_integers():
    """test_costmodel.cpp:10-53 against the host cost model the TrafficCounter uses."""
    from paper_2505_17701_b200 import costmodel as cm
    base = cm.llama3_8b_shape()
    assert [cm.shape_at_k(base, k).s_alive for k in (0.7, 0.8, 0.9)] == [4300, 2867, 1433]
    assert cm.flops_dense(base) == 352407552
    assert [cm.flops_mc(cm.shape_at_k(base, k)) for k in (0.7, 0.8, 0.9)] == [187946184, 164459314, 140956054]
    assert [cm.flops_dc(cm.shape_at_k(base, k)) for k in (0.7, 0.8, 0.9)] == [124591304, 89365298, 54114710]
    assert cm.traffic_dense_split(base).total() == 176287744
    assert [cm.traffic_mc_split(cm.shape_at_k(base, k)).total() for k in (0.7, 0.8, 0.9)] == \
        [94077132, 82336563, 70587801]
    assert [cm.traffic_dc_split(cm.shape_at_k(base, k)).total() for k in (0.7, 0.8, 0.9)] == \
        [62374912, 44766208, 27145216]
    d = cm.traffic_dense_split(base)
    assert (d.weight_reads, d.vector_reads, d.writes) == (176160768, 65536, 61440)
    # device byte model: bf16 DC@0.9 at the Llama shape (54.1 MB)
    b = cm.device_bytes("dc", 4096, 14336, 512, 1433, 2)["total_bytes"]
    assert abs(b / 1e6 - 54.1) < 0.2


def test_costmodel_matches_oracle_forms(oracle):
    from paper_2505_17701_b200 import costmodel as cm
    for d, F, r, s in ((16, 64, 6, 20), (4096, 14336, 512, 1433), (5120, 13824, 512, 2764)):
        t = cm.traffic_mc_split(cm.ShapeSpec(d, F, r, 5, s))
        assert (t.weight_reads, t.vector_reads, t.writes) == oracle.traffic_split("mc", d, F, 0, s)
        t = cm.traffic_dc_split(cm.ShapeSpec(d, F, r, 5, s))
        assert (t.weight_reads, t.vector_reads, t.writes) == oracle.traffic_split("dc", d, F, r, s)
