"""CPU ORACLE for the COUNTDOWN decode path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both loaded with ctypes:

* ``Oracle``: our plain-C restatement of the reference algorithm
  (``oracle/countdown_oracle.c``; every function cites the reference file:line it
  restates).  Builds anywhere with gcc (``make -C oracle oracle``).
* ``Reference``: the unmodified reference library compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref/libcountdown_ref.so`` by
  ``oracle/Makefile`` (only possible in the build container; the prebuilt .so
  travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2505_17701_b200`` never imports it; its CUDA path fails loudly when the
extension is missing.

Parity pinning: ``tests/test_oracle_pinning.py`` checks ``Oracle`` bit-for-bit
against ``Reference`` and against the committed golden fixtures in
``tests/golden/`` (made by ``tests/golden/make_golden.py`` from ``Reference``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcountdown_ref.so")
REF_SRC = "/root/reference/proj"

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_u64 = C.c_uint64


def _opt(arr):
    """ctypes argument for an optional (nullable) numpy buffer."""
    return None if arr is None else arr.ctypes.data_as(C.c_void_p)


def build(ref: bool = True) -> None:
    """Compile the C oracle (and, when the reference tree is present, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref", "ref-tests"], check=True)


class _RngState(C.Structure):
    _fields_ = [("state", C.c_uint64), ("has_spare", C.c_int), ("spare", C.c_double)]


class Oracle:
    """ctypes view of oracle/liboracle.so (the C restatement)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
        L = C.CDLL(path)
        self.L = L
        vp = C.c_void_p
        L.cdo_rng_init.argtypes = [C.POINTER(_RngState), _u64]
        L.cdo_rng_next_u64.argtypes = [C.POINTER(_RngState)]
        L.cdo_rng_next_u64.restype = _u64
        L.cdo_rng_normal.argtypes = [C.POINTER(_RngState)]
        L.cdo_rng_normal.restype = C.c_double
        L.cdo_rng_uniform.argtypes = [C.POINTER(_RngState)]
        L.cdo_rng_uniform.restype = C.c_double
        L.cdo_rng_fork_seed.argtypes = [C.POINTER(_RngState)]
        L.cdo_rng_fork_seed.restype = _u64
        L.cdo_fill_normal.argtypes = [C.POINTER(_RngState), _f32p, _i64]
        L.cdo_make_random_layer.argtypes = [C.POINTER(_RngState), _i64, _i64, _f32p, _f32p, _f32p]
        L.cdo_make_lowrank_predictor.argtypes = [C.POINTER(_RngState), _i64, _i64, _i64, _f32p, _f32p]
        L.cdo_act.argtypes = [C.c_int, C.c_float]
        L.cdo_act.restype = C.c_float
        L.cdo_gemv.argtypes = [_f32p, _i64, _i64, _f32p, _f32p]
        L.cdo_alive_count_for.argtypes = [C.c_double, _i64]
        L.cdo_alive_count_for.restype = _i64
        L.cdo_top_m_threshold.argtypes = [_f32p, _i64, _i64, C.POINTER(C.c_float), vp]
        L.cdo_forward_dense.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, vp, vp, vp, _f32p]
        L.cdo_weighted_sum.argtypes = [_i64, _i64, _f32p, _f32p, vp, _f32p]
        L.cdo_forward_sparse.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _u8p, _f32p]
        L.cdo_lowrank_logits.argtypes = [_i64, _i64, _i64, _f32p, _f32p, _f32p, vp, _f32p]
        L.cdo_threshold_abs.argtypes = [_f32p, _i64, C.c_float, _u8p]
        L.cdo_threshold_abs.restype = _i64
        L.cdo_threshold_signed.argtypes = [_f32p, _i64, C.c_float, _u8p]
        L.cdo_threshold_signed.restype = _i64
        L.cdo_pipeline_mc.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, C.c_float, _f32p, _u8p, vp]
        L.cdo_pipeline_mc.restype = _i64
        L.cdo_pipeline_dc.argtypes = [_i64, _i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p,
                                      _f32p, C.c_float, vp, _f32p, _u8p, vp]
        L.cdo_pipeline_dc.restype = _i64
        for n in ("cdo_traffic_dense_split",):
            getattr(L, n).argtypes = [_i64, _i64, _i64p]
        L.cdo_traffic_mc_split.argtypes = [_i64, _i64, _i64, _i64p]
        L.cdo_traffic_dc_split.argtypes = [_i64, _i64, _i64, _i64, _i64p]
        L.cdo_traffic_dc_oracle.argtypes = [_i64, _i64, _i64]
        L.cdo_traffic_dc_oracle.restype = _i64
        L.cdo_flops_dense.argtypes = [_i64, _i64, _i64]
        L.cdo_flops_dense.restype = _i64
        L.cdo_flops_mc.argtypes = [_i64, _i64, _i64, _i64]
        L.cdo_flops_mc.restype = _i64
        L.cdo_flops_dc.argtypes = [_i64, _i64, _i64, _i64, _i64]
        L.cdo_flops_dc.restype = _i64
        L.cdo_calibrate_mc.argtypes = [_i64, _i64, _f32p, _f32p, _i64, C.c_double, C.POINTER(C.c_double)]

    # --- RNG-driven generation (numerics.cpp:11-24, gated_mlp.cpp:61-75, predictor.cpp:52-69)
    class Rng:
        def __init__(self, oracle: "Oracle", seed: int):
            self.o = oracle
            self.st = _RngState()
            oracle.L.cdo_rng_init(C.byref(self.st), C.c_uint64(seed))

        def next_u64(self) -> int:
            return int(self.o.L.cdo_rng_next_u64(C.byref(self.st)))

        def uniform(self) -> float:
            return float(self.o.L.cdo_rng_uniform(C.byref(self.st)))

        def normal(self) -> float:
            return float(self.o.L.cdo_rng_normal(C.byref(self.st)))

        def fork(self) -> "Oracle.Rng":
            return Oracle.Rng(self.o, int(self.o.L.cdo_rng_fork_seed(C.byref(self.st))))

        def normals_f(self, n: int) -> np.ndarray:
            out = np.empty(n, np.float32)
            self.o.L.cdo_fill_normal(C.byref(self.st), out, n)
            return out

        def random_layer(self, d: int, F: int):
            up = np.empty((F, d), np.float32)
            gate = np.empty((F, d), np.float32)
            down = np.empty((F, d), np.float32)
            self.o.L.cdo_make_random_layer(C.byref(self.st), d, F, up, gate, down)
            return up, gate, down

        def lowrank_predictor(self, d: int, r: int, F: int):
            ta = np.empty((d, r), np.float32)
            tb = np.empty((r, F), np.float32)
            self.o.L.cdo_make_lowrank_predictor(C.byref(self.st), d, r, F, ta, tb)
            return ta, tb

    def rng(self, seed: int) -> "Oracle.Rng":
        return Oracle.Rng(self, seed)

    def generate(self, seed: int, d: int, F: int, r: int = 0):
        """bench() setup order (blocked_exec.cpp:396-415): layer, x, predictor from rng.fork()."""
        g = self.rng(seed)
        up, gate, down = g.random_layer(d, F)
        x = g.normals_f(d)
        ta = tb = None
        if r > 0:
            ta, tb = g.fork().lowrank_predictor(d, r, F)
        return dict(w_up=up, w_gate=gate, w_down=down, x=x, theta_a=ta, theta_b=tb)

    # --- numerics
    def act(self, act: int, x: float) -> float:
        return float(self.L.cdo_act(act, x))

    def gemv(self, w: np.ndarray, x: np.ndarray) -> np.ndarray:
        out = np.empty(w.shape[0], np.float32)
        self.L.cdo_gemv(np.ascontiguousarray(w), w.shape[0], w.shape[1], np.ascontiguousarray(x), out)
        return out

    def alive_count_for(self, k: float, F: int) -> int:
        return int(self.L.cdo_alive_count_for(k, F))

    def top_m_threshold(self, v: np.ndarray, m: int):
        v = np.ascontiguousarray(v, np.float32)
        tau = C.c_float()
        mask = np.empty(len(v), np.uint8)
        rc = self.L.cdo_top_m_threshold(v, len(v), m, C.byref(tau), _opt(mask))
        if rc != 0:
            raise ValueError("top_m_threshold: bad arguments")
        return float(tau.value), mask

    # --- layer semantics
    def forward_dense(self, L, x, act=0):
        F, d = L["w_up"].shape
        u, h, s = (np.empty(F, np.float32) for _ in range(3))
        y = np.empty(d, np.float32)
        self.L.cdo_forward_dense(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                 _opt(u), _opt(h), _opt(s), y)
        return dict(u=u, h=h, s=s, y=y)

    def forward_sparse(self, L, x, mask, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        self.L.cdo_forward_sparse(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                  np.ascontiguousarray(mask, np.uint8), y)
        return y

    def lowrank_logits(self, ta, tb, x):
        d, r = ta.shape
        F = tb.shape[1]
        lat = np.empty(r, np.float32)
        z = np.empty(F, np.float32)
        self.L.cdo_lowrank_logits(d, r, F, ta, tb, x, _opt(lat), z)
        return lat, z

    def pipeline_mc(self, L, x, tau, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        mask = np.empty(F, np.uint8)
        u = np.empty(F, np.float32)
        alive = self.L.cdo_pipeline_mc(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                       tau, y, mask, _opt(u))
        return dict(y=y, mask=mask, alive=int(alive), u=u)

    def pipeline_dc(self, L, x, tau_d=0.0, mask_override=None, act=0):
        F, d = L["w_up"].shape
        r = L["theta_a"].shape[1]
        y = np.empty(d, np.float32)
        mask = np.empty(F, np.uint8)
        z = np.empty(F, np.float32)
        mo = None if mask_override is None else np.ascontiguousarray(mask_override, np.uint8)
        alive = self.L.cdo_pipeline_dc(d, F, r, act, L["w_up"], L["w_gate"], L["w_down"],
                                       L["theta_a"], L["theta_b"], x, tau_d, _opt(mo), y, mask,
                                       _opt(z))
        return dict(y=y, mask=mask, alive=int(alive), logits=z)

    # --- cost model
    def traffic_split(self, method: str, d: int, F: int, r: int = 0, s: int = 0):
        out = np.zeros(3, np.int64)
        if method == "dense":
            rc = self.L.cdo_traffic_dense_split(d, F, out)
        elif method == "mc":
            rc = self.L.cdo_traffic_mc_split(d, F, s, out)
        elif method == "dc":
            rc = self.L.cdo_traffic_dc_split(d, F, r, s, out)
        else:
            raise ValueError(method)
        if rc != 0:
            raise ValueError("bad shape")
        return tuple(int(v) for v in out)

    def calibrate_mc(self, w_up, xs, k):
        F, d = w_up.shape
        xs = np.ascontiguousarray(xs, np.float32)
        out = C.c_double()
        rc = self.L.cdo_calibrate_mc(d, F, np.ascontiguousarray(w_up), xs, xs.shape[0], k, C.byref(out))
        if rc != 0:
            raise ValueError("calibrate: bad input")
        return float(out.value)


class ReferenceError_(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Reference:
    """ctypes view of oracle/_ref/libcountdown_ref.so (the unmodified reference library)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    f"/root/reference is mounted")
        L = C.CDLL(path)
        self.L = L
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate.argtypes = [_u64, _i64, _i64, _i64, C.c_int, vp, vp, vp, vp, vp, vp]
        L.ref_rng_normals.argtypes = [_u64, _i64, _f64p]
        L.ref_activation.argtypes = [C.c_int, _f32p, _i64, _f32p]
        L.ref_alive_count_for.argtypes = [C.c_double, _i64, C.POINTER(_i64)]
        L.ref_top_m_threshold.argtypes = [_f32p, _i64, _i64, C.POINTER(C.c_float), _u8p]
        L.ref_forward_dense.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, vp, vp, vp, vp]
        L.ref_forward_sparse.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _u8p, _f32p]
        L.ref_predict_logits.argtypes = [_i64, _i64, _i64, _f32p, _f32p, _f32p, _f32p]
        L.ref_forward_practical.argtypes = [C.c_int, _i64, _i64, _i64, C.c_int, _f32p, _f32p, _f32p,
                                            vp, vp, _f32p, C.c_float, _f32p, _u8p, C.POINTER(_i64)]
        L.ref_exec_dense.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _i64, _i64,
                                     C.c_int, _f32p, _i64p]
        L.ref_exec_mc.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p, _u8p,
                                  _i64, _i64, C.c_int, _f32p, _i64p]
        L.ref_exec_dc.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _u8p, _i64,
                                  _i64, C.c_int, _f32p, _i64p]
        L.ref_pipeline_mc.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, C.c_float,
                                      _i64, _i64, C.c_int, _f32p, _u8p, C.POINTER(_i64), _i64p]
        L.ref_pipeline_dc.argtypes = [_i64, _i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p,
                                      _f32p, vp, _i64, _i64, C.c_int, _f32p, _u8p, C.POINTER(_i64),
                                      _i64p]
        L.ref_model_new.argtypes = [_i64, _i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p,
                                    C.POINTER(vp)]
        L.ref_model_free.argtypes = [vp]
        L.ref_model_pipeline_dc.argtypes = [vp, _f32p, vp, _i64, _i64, C.c_int, _f32p, C.POINTER(_i64)]
        L.ref_bench.argtypes = [C.c_int, _i64, _i64, _i64, C.c_double, _i64, _i64, _i64, C.c_int,
                                _u64, _i64p, C.POINTER(C.c_double)]
        L.ref_bench_reference_dense.argtypes = [_i64, _i64, _i64, _u64, _i64p]
        L.ref_calibrate_mc.argtypes = [_i64, _i64, _f32p, _f32p, _i64, C.c_double, C.POINTER(C.c_double)]
        L.ref_traffic_split.argtypes = [C.c_int, _i64, _i64, _i64, _i64, _i64p]
        L.ref_flops.argtypes = [C.c_int, _i64, _i64, _i64, _i64, C.POINTER(_i64)]
        L.ref_write_model.argtypes = [C.c_char_p, _u64, _i64, _i64, _i64, C.c_int, C.c_double]
        L.ref_read_model.argtypes = [C.c_char_p, _i64p, vp, vp, vp, vp, vp]

    def _chk(self, rc: int):
        if rc != 0:
            raise ReferenceError_(rc, self.L.ref_last_error().decode())

    def max_threads(self) -> int:
        return int(self.L.ref_max_threads())

    def generate(self, seed, d, F, r=0, act=0):
        up = np.empty((F, d), np.float32)
        gate = np.empty((F, d), np.float32)
        down = np.empty((F, d), np.float32)
        x = np.empty(d, np.float32)
        ta = np.empty((d, r), np.float32) if r > 0 else None
        tb = np.empty((r, F), np.float32) if r > 0 else None
        self._chk(self.L.ref_generate(seed, d, F, r, act, _opt(up), _opt(gate), _opt(down),
                                      _opt(x), _opt(ta), _opt(tb)))
        return dict(w_up=up, w_gate=gate, w_down=down, x=x, theta_a=ta, theta_b=tb)

    def rng_normals(self, seed, n):
        out = np.empty(n, np.float64)
        self._chk(self.L.ref_rng_normals(seed, n, out))
        return out

    def activation(self, act, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self._chk(self.L.ref_activation(act, x, len(x), out))
        return out

    def alive_count_for(self, k, F):
        out = _i64()
        self._chk(self.L.ref_alive_count_for(k, F, C.byref(out)))
        return int(out.value)

    def top_m_threshold(self, v, m):
        v = np.ascontiguousarray(v, np.float32)
        tau = C.c_float()
        mask = np.empty(len(v), np.uint8)
        self._chk(self.L.ref_top_m_threshold(v, len(v), m, C.byref(tau), mask))
        return float(tau.value), mask

    def forward_dense(self, L, x, act=0):
        F, d = L["w_up"].shape
        u, h, s = (np.empty(F, np.float32) for _ in range(3))
        y = np.empty(d, np.float32)
        self._chk(self.L.ref_forward_dense(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                           _opt(u), _opt(h), _opt(s), _opt(y)))
        return dict(u=u, h=h, s=s, y=y)

    def forward_sparse(self, L, x, mask, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        self._chk(self.L.ref_forward_sparse(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                            np.ascontiguousarray(mask, np.uint8), y))
        return y

    def predict_logits(self, ta, tb, x):
        d, r = ta.shape
        F = tb.shape[1]
        z = np.empty(F, np.float32)
        self._chk(self.L.ref_predict_logits(d, r, F, ta, tb, x, z))
        return z

    def forward_practical(self, method, L, x, tau_hat=0.0, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        mask = np.empty(F, np.uint8)
        alive = _i64()
        ta, tb = L.get("theta_a"), L.get("theta_b")
        r = 0 if ta is None else ta.shape[1]
        self._chk(self.L.ref_forward_practical(0 if method == "mc" else 1, d, F, r, act, L["w_up"],
                                               L["w_gate"], L["w_down"], _opt(ta), _opt(tb), x,
                                               tau_hat, y, mask, C.byref(alive)))
        return dict(y=y, mask=mask, alive=int(alive.value))

    def exec_dense(self, L, x, blk=(16, 256), reduction=0, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        t = np.zeros(3, np.int64)
        self._chk(self.L.ref_exec_dense(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                        blk[0], blk[1], reduction, y, t))
        return y, tuple(int(v) for v in t)

    def exec_mc(self, L, x, u, mask, blk=(16, 256), reduction=0, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        t = np.zeros(3, np.int64)
        self._chk(self.L.ref_exec_mc(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                     np.ascontiguousarray(u, np.float32),
                                     np.ascontiguousarray(mask, np.uint8), blk[0], blk[1],
                                     reduction, y, t))
        return y, tuple(int(v) for v in t)

    def exec_dc(self, L, x, mask, blk=(16, 256), reduction=0, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        t = np.zeros(3, np.int64)
        self._chk(self.L.ref_exec_dc(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x,
                                     np.ascontiguousarray(mask, np.uint8), blk[0], blk[1],
                                     reduction, y, t))
        return y, tuple(int(v) for v in t)

    def pipeline_mc(self, L, x, tau, blk=(16, 256), reduction=0, act=0):
        F, d = L["w_up"].shape
        y = np.empty(d, np.float32)
        mask = np.empty(F, np.uint8)
        alive = _i64()
        t = np.zeros(3, np.int64)
        self._chk(self.L.ref_pipeline_mc(d, F, act, L["w_up"], L["w_gate"], L["w_down"], x, tau,
                                         blk[0], blk[1], reduction, y, mask, C.byref(alive), t))
        return dict(y=y, mask=mask, alive=int(alive.value), traffic=tuple(int(v) for v in t))

    def pipeline_dc(self, L, x, mask_override=None, blk=(16, 256), reduction=0, act=0):
        F, d = L["w_up"].shape
        r = L["theta_a"].shape[1]
        y = np.empty(d, np.float32)
        mask = np.empty(F, np.uint8)
        alive = _i64()
        t = np.zeros(3, np.int64)
        mo = None if mask_override is None else np.ascontiguousarray(mask_override, np.uint8)
        self._chk(self.L.ref_pipeline_dc(d, F, r, act, L["w_up"], L["w_gate"], L["w_down"],
                                         L["theta_a"], L["theta_b"], x, _opt(mo), blk[0], blk[1],
                                         reduction, y, mask, C.byref(alive), t))
        return dict(y=y, mask=mask, alive=int(alive.value), traffic=tuple(int(v) for v in t))

    def model(self, L, act=0):
        """A persistent reference GatedMlpLayer + low-rank Predictor (for timed loops)."""
        F, d = L["w_up"].shape
        r = L["theta_a"].shape[1]
        h = C.c_void_p()
        self._chk(self.L.ref_model_new(d, F, r, act, L["w_up"], L["w_gate"], L["w_down"], L["theta_a"],
                                       L["theta_b"], C.byref(h)))
        return h

    def model_free(self, h):
        self.L.ref_model_free(h)

    def model_pipeline_dc(self, h, x, d, mask_override=None, blk=(16, 256), reduction=0):
        y = np.empty(d, np.float32)
        alive = _i64()
        mo = None if mask_override is None else np.ascontiguousarray(mask_override, np.uint8)
        self._chk(self.L.ref_model_pipeline_dc(h, np.ascontiguousarray(x, np.float32), _opt(mo), blk[0], blk[1],
                                               reduction, y, C.byref(alive)))
        return dict(y=y, alive=int(alive.value))

    def bench(self, method: str, d, F, r, k, iters, seed=42, blk=(16, 256), reduction=0):
        m = {"dense": 0, "cats": 1, "mc": 2, "dc": 3}[method]
        out = np.zeros(3, np.int64)
        ratio = C.c_double()
        self._chk(self.L.ref_bench(m, d, F, r, k, iters, blk[0], blk[1], reduction, seed, out,
                                   C.byref(ratio)))
        return dict(p50_ns=int(out[0]), p95_ns=int(out[1]), traffic_elements=int(out[2]),
                    element_read_ratio=float(ratio.value))

    def bench_reference_dense(self, d, F, iters, seed=42):
        out = np.zeros(3, np.int64)
        self._chk(self.L.ref_bench_reference_dense(d, F, iters, seed, out))
        return dict(p50_ns=int(out[0]), p95_ns=int(out[1]), traffic_elements=int(out[2]))

    def calibrate_mc(self, w_up, xs, k):
        F, d = w_up.shape
        xs = np.ascontiguousarray(xs, np.float32)
        out = C.c_double()
        self._chk(self.L.ref_calibrate_mc(d, F, np.ascontiguousarray(w_up), xs, xs.shape[0], k,
                                          C.byref(out)))
        return float(out.value)

    def traffic_split(self, method, d, F, r=0, s=0):
        m = {"dense": 0, "cats": 1, "mc": 2, "dc": 3}[method]
        out = np.zeros(3, np.int64)
        self._chk(self.L.ref_traffic_split(m, d, F, r, s, out))
        return tuple(int(v) for v in out)

    def flops(self, method, d, F, r=0, s=0):
        m = {"dense": 0, "cats": 1, "mc": 2, "dc": 3}[method]
        out = _i64()
        self._chk(self.L.ref_flops(m, d, F, r, s, C.byref(out)))
        return int(out.value)


    def write_model(self, path, seed, d, F, r=0, act=0, k=0.0):
        """write_model (model_io.cpp:94-138) of the seeded bench() layer (+ predictor)."""
        self._chk(self.L.ref_write_model(str(path).encode(), seed, d, F, r, act, k))

    def read_model(self, path):
        """read_model (model_io.cpp:140-224).  Raises ReferenceError_ (code 2 = DataError)."""
        dims = np.zeros(5, np.int64)
        self._chk(self.L.ref_read_model(str(path).encode(), dims, None, None, None, None, None))
        d, F, r = int(dims[0]), int(dims[1]), int(dims[2])
        up, gate, down = (np.empty((F, d), np.float32) for _ in range(3))
        ta = np.empty((d, r), np.float32) if r > 0 else None
        tb = np.empty((r, F), np.float32) if r > 0 else None
        self._chk(self.L.ref_read_model(str(path).encode(), dims, _opt(up), _opt(gate), _opt(down), _opt(ta),
                                        _opt(tb)))
        return dict(d=d, F=F, r=r, act=int(dims[3]), seed=int(dims[4]), w_up=up, w_gate=gate, w_down=down,
                    theta_a=ta, theta_b=tb)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def rms_norm(y, eps=1e-5):
    """Input norm of the stacked layers (layer l+1's input is the
    RMS-normalised y_l, no gain, no residual): y / sqrt(mean(y^2) + eps), in double, rounded
    once to f32.  Test infrastructure: the product computes it on the device."""
    y = np.asarray(y, np.float64)
    return (y / np.sqrt(np.mean(y * y) + eps)).astype(np.float32)

