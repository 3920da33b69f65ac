"""The reference's operator API (proj/include/countdown/*.hpp), served by the B200 library.

Same names, argument meaning and error behaviour as the C++ API, so code (and tests)
written against ``exec_mc`` / ``exec_dc`` / ``pipeline_*`` / ``forward_practical`` /
``predict_logits`` read the same.  Every operator runs on the GPU through the C-ABI
(``include/countdown_b200.h``); there is no CPU compute path.

Mapping of the knobs that have no GPU meaning:
  * ``BlockConfig.blk_m / blk_n`` are accepted and ignored; results are invariant to them
    (acceptance.cpp:336-342), exactly as the reference's are.
  * ``BlockConfig.reduction``: DeterministicOrdered -> bit-exact kernels, UnorderedAccumulate
    -> the fused fast path (1e-4 relative L2 in f32, test_blocked_exec.cpp:87-99).
  * ``TrafficCounter`` is accumulated with the reference's per-stream element counts at the
    realized alive count (blocked_exec.cpp:63, 127-131, 145-169, 206-210, 283-287, 300-314,
    322-324, 362-376); they equal costmodel.cpp's closed forms term for term.

Extensions (C-ABI only in the reference's terms): a leading batch dimension on ``x``
(per-sample masks), ``tau_d`` for D-CountDown (Alg. 3's calibrated threshold,
PAPER.md:645; the reference hard-codes 0, predictor.cpp:145), and the layer's device
weight dtype (``device_dtype="bf16"`` for the perf path).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _capi
from ._capi import CudaError, DataError, NumericError, check, lib, ptr
from .costmodel import (ShapeSpec, alive_count_for, traffic_dense_split)

__all__ = [
    "Activation", "Reduction", "BlockConfig", "TrafficCounter", "ActivationMask",
    "GatedMlpLayer", "LowRankPredictor", "Predictor", "PredictorKind", "SparsityMethod",
    "SparsityMode", "SparsityConfig", "PracticalContext", "PracticalResult", "PipelineResult",
    "BenchStats", "DeviceLayer", "exec_dense", "exec_mc", "exec_cats", "exec_dc", "pipeline_dense",
    "pipeline_mc", "pipeline_cats", "pipeline_dc", "forward_sparse", "forward_practical", "predict_logits",
    "predict_mask", "calibrate", "top_m_threshold", "realized_sparsity", "bench", "synth_workload", "synth_normals",
    "DataError", "NumericError", "CudaError", "ModelFile", "read_model", "write_model", "checksum_hex",
]


class Activation(IntEnum):
    """numerics.hpp:78"""
    Silu = _capi.ACT_SILU
    GeluTanh = _capi.ACT_GELU_TANH


class Reduction(IntEnum):
    """blocked_exec.hpp:18"""
    DeterministicOrdered = _capi.REDUCTION_ORDERED
    UnorderedAccumulate = _capi.REDUCTION_UNORDERED


@dataclass
class BlockConfig:
    """blocked_exec.hpp:20-24 (blk_m / blk_n accepted, no GPU meaning)."""
    blk_m: int = 16
    blk_n: int = 256
    reduction: Reduction = Reduction.DeterministicOrdered


@dataclass
class TrafficCounter:
    """blocked_exec.hpp:26-31"""
    weight_reads: int = 0
    vector_reads: int = 0
    writes: int = 0

    def total(self) -> int:
        return self.weight_reads + self.vector_reads + self.writes

    def add(self, w: int, v: int, wr: int) -> None:
        self.weight_reads += int(w)
        self.vector_reads += int(v)
        self.writes += int(wr)


@dataclass
class ActivationMask:
    """numerics.hpp:64-76"""
    alive: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    alive_count: int = 0
    tau: float = 0.0

    def size(self) -> int:
        return int(self.alive.shape[0])

    def is_alive(self, i: int) -> bool:
        return bool(self.alive[i])

    def recount(self) -> None:
        self.alive_count = int(np.count_nonzero(self.alive))

    @staticmethod
    def all_alive(n: int) -> "ActivationMask":
        return ActivationMask(np.ones(n, np.uint8), n, float("-inf"))

    @staticmethod
    def none_alive(n: int) -> "ActivationMask":
        return ActivationMask(np.zeros(n, np.uint8), 0, float("inf"))


class SparsityMethod(IntEnum):
    """sparsity.hpp:17"""
    Cats = 0
    MCountdown = 1
    DCountdown = 2


class SparsityMode(IntEnum):
    Ideal = 0
    Practical = 1


@dataclass
class SparsityConfig:
    """sparsity.hpp:20-24"""
    method: SparsityMethod = SparsityMethod.DCountdown
    mode: SparsityMode = SparsityMode.Ideal
    k: float = 0.7


class PredictorKind(IntEnum):
    LowRank = 0
    Ternary = 1


@dataclass
class LowRankPredictor:
    """predictor.hpp:15-21: theta_a (d_model x d_rank), theta_b (d_rank x d_inter)."""
    d_model: int
    d_rank: int
    d_inter: int
    theta_a: np.ndarray
    theta_b: np.ndarray


class Predictor:
    """predictor.hpp:36-44 (the low-rank variant; the ternary predictor is out of scope)."""

    def __init__(self, impl: LowRankPredictor, device_dtype: str = "f32", device: int = 0):
        if not isinstance(impl, LowRankPredictor):
            raise DataError("predictor: only the low-rank predictor runs on the GPU path")
        self.impl = impl
        self.device_dtype = device_dtype
        self.device = device
        self._handle: DeviceLayer | None = None

    def kind(self) -> PredictorKind:
        return PredictorKind.LowRank

    def d_model(self) -> int:
        return self.impl.d_model

    def d_inter(self) -> int:
        return self.impl.d_inter

    def lowrank(self) -> LowRankPredictor:
        return self.impl

    def handle(self) -> "DeviceLayer":
        if self._handle is None:
            self._handle = DeviceLayer.predictor_only(self.impl, self.device_dtype, self.device)
        return self._handle


@dataclass
class PracticalContext:
    """sparsity.hpp:41-44"""
    tau_hat: float | None = None
    predictor: Predictor | None = None


@dataclass
class PracticalResult:
    y: np.ndarray
    mask: ActivationMask | list


@dataclass
class PipelineResult:
    """blocked_exec.hpp:52-56"""
    y: np.ndarray
    mask: ActivationMask | list
    traffic: TrafficCounter


@dataclass
class BenchStats:
    """blocked_exec.hpp:70-80"""
    method: str = ""
    k: float = 0.0
    d_model: int = 0
    d_inter: int = 0
    iters: int = 0
    p50_ns: int = 0
    p95_ns: int = 0
    traffic_elements: int = 0
    element_read_ratio: float = 0.0


_DTYPES = {"f32": _capi.DTYPE_F32, "bf16": _capi.DTYPE_BF16}


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class DeviceLayer:
    """Owns one cd_layer handle: the layer's weights (and predictor) resident in HBM."""

    def __init__(self, raw: C.c_void_p, d: int, F: int, r: int = 0):
        self.raw = raw
        self.d_model, self.d_inter, self.d_rank = d, F, r

    @staticmethod
    def create(w_up, w_gate, w_down, activation: int = 0, device_dtype: str = "f32",
               device: int = 0, row_range: tuple[int, int] | None = None) -> "DeviceLayer":
        w_up, w_gate, w_down = _f32(w_up), _f32(w_gate), _f32(w_down)
        F_total, d = w_up.shape
        out = C.c_void_p()
        if row_range is None:
            check(lib().cd_layer_create(device, d, F_total, int(activation), _DTYPES[device_dtype],
                                        ptr(w_up), ptr(w_gate), ptr(w_down), C.byref(out)))
            F = F_total
        else:
            rb, re_ = row_range
            check(lib().cd_layer_create_shard(device, d, F_total, rb, re_, int(activation),
                                              _DTYPES[device_dtype], ptr(w_up), ptr(w_gate),
                                              ptr(w_down), C.byref(out)))
            F = re_ - rb
        return DeviceLayer(out, d, F)

    @staticmethod
    def load(path: str, device_dtype: str = "bf16", device: int = 0) -> "DeviceLayer":
        """cd_layer_load_cdwn1: a CDWN1 model file (model_io.cpp:94-224) parsed, validated and
        uploaded by the library (no host copy of the weights is kept)."""
        out = C.c_void_p()
        dims = np.zeros(5, np.int64)
        check(lib().cd_layer_load_cdwn1(device, str(path).encode(), _DTYPES[device_dtype], C.byref(out),
                                        ptr(dims)))
        dl = DeviceLayer(out, int(dims[0]), int(dims[1]), max(0, int(dims[2])))
        dl.activation = Activation(int(dims[3]))
        dl.seed = int(dims[4]) & 0xFFFFFFFFFFFFFFFF  # the header's uint64 bit pattern
        dl.predictor_kind = "lowrank" if dims[2] > 0 else ("ternary" if dims[2] < 0 else None)
        return dl

    @staticmethod
    def predictor_only(p: LowRankPredictor, device_dtype: str = "f32", device: int = 0) -> "DeviceLayer":
        ta, tb = _f32(p.theta_a), _f32(p.theta_b)
        out = C.c_void_p()
        check(lib().cd_predictor_create(device, p.d_model, p.d_rank, p.d_inter, _DTYPES[device_dtype],
                                        ptr(ta), ptr(tb), C.byref(out)))
        return DeviceLayer(out, p.d_model, p.d_inter, p.d_rank)

    def set_predictor(self, p: LowRankPredictor) -> None:
        ta, tb = _f32(p.theta_a), _f32(p.theta_b)
        check(lib().cd_layer_set_predictor(self.raw, p.d_rank, ptr(ta), ptr(tb)))
        self.d_rank = p.d_rank

    def close(self) -> None:
        if self.raw:
            lib().cd_layer_destroy(self.raw)
            self.raw = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_bytes(self) -> int:
        v = C.c_int64()
        check(lib().cd_layer_device_bytes(self.raw, C.byref(v)))
        return int(v.value)

    def last_launches(self) -> int:
        v = C.c_int()
        check(lib().cd_layer_last_launches(self.raw, C.byref(v)))
        return int(v.value)

    def last_path(self) -> str:
        """Engine of the most recent forward call: "exact", "fast" or "tensor"."""
        v = C.c_int()
        check(lib().cd_layer_last_path(self.raw, C.byref(v)))
        return ("exact", "fast", "tensor")[v.value]

    # ---- host-buffer operators (batch-first arrays)
    def exec_dense(self, x, reduction) -> np.ndarray:
        x = _f32(x)
        y = np.empty_like(x)
        check(lib().cd_exec_dense(self.raw, x.shape[0], ptr(x), int(reduction), ptr(y)))
        return y

    def exec_mc(self, x, u, masks, reduction) -> np.ndarray:
        x, u = _f32(x), _f32(u)
        m = np.ascontiguousarray(masks, np.uint8)
        y = np.empty_like(x)
        check(lib().cd_exec_mc(self.raw, x.shape[0], ptr(x), ptr(u), ptr(m), int(reduction), ptr(y)))
        return y

    def exec_dc(self, x, masks, reduction) -> np.ndarray:
        x = _f32(x)
        m = np.ascontiguousarray(masks, np.uint8)
        y = np.empty_like(x)
        check(lib().cd_exec_dc(self.raw, x.shape[0], ptr(x), ptr(m), int(reduction), ptr(y)))
        return y

    def exec_cats(self, x, act_gate, masks, reduction) -> np.ndarray:
        x, h = _f32(x), _f32(act_gate)
        m = np.ascontiguousarray(masks, np.uint8)
        y = np.empty_like(x)
        check(lib().cd_exec_cats(self.raw, x.shape[0], ptr(x), ptr(h), ptr(m), int(reduction), ptr(y)))
        return y

    def pipeline_cats(self, x, tau, reduction, want_act=False):
        x = _f32(x)
        B = x.shape[0]
        y = np.empty_like(x)
        mask = np.empty((B, self.d_inter), np.uint8)
        alive = np.empty(B, np.int64)
        h = np.empty((B, self.d_inter), np.float32) if want_act else None
        check(lib().cd_pipeline_cats(self.raw, B, ptr(x), float(tau), int(reduction), ptr(y), ptr(mask),
                                     ptr(alive), ptr(h)))
        return y, mask, alive, h

    def pipeline_mc(self, x, tau, reduction, want_u=False):
        x = _f32(x)
        B = x.shape[0]
        y = np.empty_like(x)
        mask = np.empty((B, self.d_inter), np.uint8)
        alive = np.empty(B, np.int64)
        u = np.empty((B, self.d_inter), np.float32) if want_u else None
        check(lib().cd_pipeline_mc(self.raw, B, ptr(x), float(tau), int(reduction), ptr(y), ptr(mask),
                                   ptr(alive), ptr(u)))
        return y, mask, alive, u

    def pipeline_dc(self, x, tau_d, reduction, mask_override=None, want_logits=False):
        x = _f32(x)
        B = x.shape[0]
        y = np.empty_like(x)
        mask = np.empty((B, self.d_inter), np.uint8)
        alive = np.empty(B, np.int64)
        z = np.empty((B, self.d_inter), np.float32) if want_logits else None
        mo = None if mask_override is None else np.ascontiguousarray(mask_override, np.uint8)
        check(lib().cd_pipeline_dc(self.raw, B, ptr(x), float(tau_d), ptr(mo), int(reduction), ptr(y),
                                   ptr(mask), ptr(alive), ptr(z)))
        return y, mask, alive, z

    def predict_logits(self, x) -> np.ndarray:
        x = _f32(x)
        z = np.empty((x.shape[0], self.d_inter), np.float32)
        check(lib().cd_predict_logits(self.raw, x.shape[0], ptr(x), ptr(z)))
        return z

    # ---- device-pointer hot path (torch tensors or raw ints)
    def forward_device(self, method: int, x_dev, y_dev, tau: float = 0.0,
                       reduction: int = Reduction.UnorderedAccumulate, batch: int = 1,
                       mask_override=None, mask_out=None, indicator_out=None, alive_out=None,
                       stream=None, rms_eps: float | None = None) -> None:
        """cd_forward_device (rms_eps=None) or cd_forward_device_normed (input = RMSNorm(x))."""
        s = None if stream is None else C.c_void_p(stream)
        if rms_eps is not None:
            check(lib().cd_forward_device_normed(self.raw, int(method), int(batch), ptr(x_dev), float(rms_eps),
                                                 float(tau), int(reduction), ptr(mask_override), ptr(y_dev),
                                                 ptr(mask_out), ptr(indicator_out), ptr(alive_out), s))
            return
        check(lib().cd_forward_device(self.raw, int(method), int(batch), ptr(x_dev), float(tau),
                                      int(reduction), ptr(mask_override), ptr(y_dev), ptr(mask_out),
                                      ptr(indicator_out), ptr(alive_out), s))

    def bench_device(self, method: int, x, tau: float, reduction: int, warmup: int, iters: int) -> np.ndarray:
        x = _f32(np.atleast_2d(x))
        ns = np.empty(iters, np.int64)
        check(lib().cd_bench_device(self.raw, int(method), x.shape[0], ptr(x), float(tau), int(reduction),
                                    int(warmup), int(iters), ptr(ns)))
        return ns

    def sync(self) -> None:
        check(lib().cd_layer_sync(self.raw))

    def set_prefetch(self, nxt: "DeviceLayer | None") -> None:
        """cd_layer_set_prefetch: each fused D-CountDown step on this layer L2-prefetches the
        predictor of `nxt` (the layer that runs next; same shape), or nothing for None."""
        check(lib().cd_layer_set_prefetch(self.raw, None if nxt is None else nxt.raw))

    def set_engines(self, fused: bool = True, tensor: bool = True, host_graph: bool = True,
                    pdl_chain: bool = False) -> None:
        """cd_layer_set_engines: pick the engines this handle may use (A/B tests; all on by
        default).  Results stay within each reduction mode's contract whatever the choice.
        pdl_chain: the caller owns the device (no concurrent kernels), so the batch-1..4
        persistent kernels may be PDL-chained instead of launched cooperative."""
        flags = ((_capi.ENGINE_FUSED if fused else 0) | (_capi.ENGINE_TENSOR if tensor else 0) |
                 (_capi.ENGINE_HOST_GRAPH if host_graph else 0) | (_capi.ENGINE_PDL_CHAIN if pdl_chain else 0))
        check(lib().cd_layer_set_engines(self.raw, flags))

    @staticmethod
    def bench_stages(layers: "list[DeviceLayer]", method: int, x_dev, tau: float, warmup: int,
                     iters: int, batch: int = 1) -> list[float]:
        """Mean device ns of each kernel of the fused chain (PDL off, events between launches),
        rotating over `layers` so their rows fall out of L2 between uses."""
        arr = (C.c_void_p * len(layers))(*[l.raw for l in layers])
        ns = np.zeros(8, np.int64)
        n = C.c_int()
        check(lib().cd_bench_stages(arr, len(layers), int(method), int(batch), ptr(x_dev), float(tau),
                                    int(warmup), int(iters), ptr(ns), C.byref(n)))
        return [float(v) / iters for v in ns[: n.value]]


class GatedMlpLayer:
    """gated_mlp.hpp:12-23: all three matrices neuron-major (d_inter x d_model)."""

    def __init__(self, d_model: int, d_inter: int, activation: Activation, w_up, w_gate, w_down,
                 device_dtype: str = "f32", device: int = 0):
        self.d_model = int(d_model)
        self.d_inter = int(d_inter)
        self.activation = Activation(activation)
        self.w_up = np.asarray(w_up, np.float32)
        self.w_gate = np.asarray(w_gate, np.float32)
        self.w_down = np.asarray(w_down, np.float32)
        self.device_dtype = device_dtype
        self.device = device
        self._dev: DeviceLayer | None = None
        self._dev_predictor = None

    def validate(self) -> None:
        """gated_mlp.cpp:8-26"""
        if self.d_model <= 0 or self.d_inter <= 0:
            raise DataError(f"layer: bad dims d_model={self.d_model} d_inter={self.d_inter}")
        for m, name in ((self.w_up, "w_up"), (self.w_gate, "w_gate"), (self.w_down, "w_down")):
            if m.ndim != 2 or m.shape != (self.d_inter, self.d_model):
                rows, cols = (m.shape + (0, 0))[:2] if m.ndim else (0, 0)
                raise DataError(f"layer: {name} is {rows}x{cols}, expected "
                                f"{self.d_inter}x{self.d_model}")

    def device_layer(self, predictor: "Predictor | None" = None) -> DeviceLayer:
        """Upload once (cached); re-attach the predictor when a different one is used."""
        if self._dev is None:
            self.validate()
            self._dev = DeviceLayer.create(self.w_up, self.w_gate, self.w_down, self.activation,
                                           self.device_dtype, self.device)
        if predictor is not None and self._dev_predictor is not predictor:
            self._dev.set_predictor(predictor.lowrank())
            self._dev_predictor = predictor
        return self._dev

    def invalidate(self) -> None:
        """Drop the device copy (call after mutating the host weights)."""
        if self._dev is not None:
            self._dev.close()
        self._dev = None
        self._dev_predictor = None


# ---------------------------------------------------------------- helpers
def _batched(x, d: int, who: str):
    x = np.asarray(x, np.float32)
    single = x.ndim == 1
    xb = x.reshape(1, -1) if single else x
    if xb.ndim != 2 or xb.shape[1] != d:
        n = x.shape[0] if single else (x.shape[-1] if x.ndim else 0)
        raise DataError(f"{who}: x has length {n}, layer d_model {d}")
    return np.ascontiguousarray(xb), single


def _mask_rows(mask, B: int, F: int, who: str) -> np.ndarray:
    if isinstance(mask, ActivationMask):
        masks = [mask]
    elif isinstance(mask, (list, tuple)):
        masks = list(mask)
    else:
        arr = np.asarray(mask, np.uint8)
        masks = [arr] if arr.ndim == 1 else list(arr)
    rows = []
    for m in masks:
        a = m.alive if isinstance(m, ActivationMask) else np.asarray(m, np.uint8)
        if a.shape[0] != F:
            raise DataError(f"{who}: mask has {a.shape[0]} lanes, layer d_inter {F}")
        rows.append((a != 0).astype(np.uint8))
    if len(rows) == 1 and B > 1:
        rows = rows * B
    if len(rows) != B:
        raise DataError(f"{who}: {len(rows)} masks for a batch of {B}")
    return np.ascontiguousarray(np.stack(rows))


def _masks_out(m: np.ndarray, alive: np.ndarray, tau: float, single: bool):
    out = [ActivationMask(m[b].copy(), int(alive[b]), float(tau)) for b in range(m.shape[0])]
    return out[0] if single else out


def _reduction(cfg: BlockConfig | None) -> Reduction:
    return (cfg or BlockConfig()).reduction


# ---------------------------------------------------------------- operators
def exec_dense(layer: GatedMlpLayer, x, cfg: BlockConfig | None = None,
               tc: TrafficCounter | None = None) -> np.ndarray:
    """exec_dense (blocked_exec.hpp:34-35, blocked_exec.cpp:137-172)."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "exec_dense")
    y = layer.device_layer().exec_dense(xb, _reduction(cfg))
    if tc is not None:
        d, F, B = layer.d_model, layer.d_inter, xb.shape[0]
        t = traffic_dense_split(ShapeSpec(d, F))
        tc.add(B * t.weight_reads, B * t.vector_reads, B * t.writes)
    return y[0] if single else y


def _count_exec(tc, d, F, alive_counts, method: str):
    """Per-stream counts of exec_mc / exec_dc + down_projection (blocked_exec.cpp:127-131,
    206-210, 283-287)."""
    if tc is None:
        return
    for a in alive_counts:
        a = int(a)
        if method == "mc":
            tc.add(d * a + d * a, d + F + a + F, F + d)
        else:
            tc.add(2 * d * a + d * a, d + F + F, F + d)


def exec_mc(layer: GatedMlpLayer, x, u, mask, cfg: BlockConfig | None = None,
            tc: TrafficCounter | None = None) -> np.ndarray:
    """exec_mc (blocked_exec.hpp:39-40, blocked_exec.cpp:174-212).  Dead lanes' W rows and u
    entries are never read (they may hold NaN)."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "exec_mc")
    B, F = xb.shape[0], layer.d_inter
    masks = _mask_rows(mask, B, F, "exec_mc")
    ub = np.asarray(u, np.float32).reshape(B, -1) if np.asarray(u).ndim > 1 or B == 1 else np.tile(u, (B, 1))
    if ub.shape[1] != F:
        raise DataError("exec_mc: u length does not match d_inter")
    y = layer.device_layer().exec_mc(xb, np.ascontiguousarray(ub), masks, _reduction(cfg))
    _count_exec(tc, layer.d_model, F, masks.sum(axis=1), "mc")
    return y[0] if single else y


def exec_cats(layer: GatedMlpLayer, x, act_gate, mask, cfg: BlockConfig | None = None,
              tc: TrafficCounter | None = None) -> np.ndarray:
    """exec_cats (blocked_exec.hpp:43-44, blocked_exec.cpp:214-250): masked up GEMV times
    the caller's act(gate); dead lanes' rows and act_gate entries are never read."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "exec_cats")
    B, F = xb.shape[0], layer.d_inter
    masks = _mask_rows(mask, B, F, "exec_cats")
    hb = np.asarray(act_gate, np.float32)
    hb = hb.reshape(B, -1) if hb.ndim > 1 or B == 1 else np.tile(hb, (B, 1))
    if hb.shape[1] != F:
        raise DataError("exec_cats: act_gate length does not match d_inter")
    y = layer.device_layer().exec_cats(xb, np.ascontiguousarray(hb), masks, _reduction(cfg))
    _count_exec(tc, layer.d_model, F, masks.sum(axis=1), "mc")  # same streams as exec_mc
    return y[0] if single else y


def exec_dc(layer: GatedMlpLayer, x, mask, cfg: BlockConfig | None = None,
            tc: TrafficCounter | None = None) -> np.ndarray:
    """exec_dc (blocked_exec.hpp:47-48, blocked_exec.cpp:252-289)."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "exec_dc")
    B, F = xb.shape[0], layer.d_inter
    masks = _mask_rows(mask, B, F, "exec_dc")
    y = layer.device_layer().exec_dc(xb, masks, _reduction(cfg))
    _count_exec(tc, layer.d_model, F, masks.sum(axis=1), "dc")
    return y[0] if single else y


def pipeline_dense(layer: GatedMlpLayer, x, cfg: BlockConfig | None = None) -> PipelineResult:
    """pipeline_dense (blocked_exec.cpp:291-296)."""
    tc = TrafficCounter()
    y = exec_dense(layer, x, cfg, tc)
    return PipelineResult(y, ActivationMask.all_alive(layer.d_inter), tc)


def pipeline_mc(layer: GatedMlpLayer, x, tau: float, cfg: BlockConfig | None = None,
                want_u: bool = False) -> PipelineResult:
    """pipeline_mc (blocked_exec.cpp:316-328): dense up pass, |u| > tau, exec_mc."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "pipeline_mc")
    d, F = layer.d_model, layer.d_inter
    y, m, alive, u = layer.device_layer().pipeline_mc(xb, tau, _reduction(cfg), want_u)
    tc = TrafficCounter()
    for a in alive:
        tc.add(d * F, d, F)          # dense up pass (blocked_exec.cpp:322-324)
        tc.add(0, 2 * F, 2 * F)      # threshold_mask (blocked_exec.cpp:304-310)
    _count_exec(tc, d, F, alive, "mc")
    res = PipelineResult(y[0] if single else y, _masks_out(m, alive, tau, single), tc)
    if want_u:
        res.u = u[0] if single else u
    return res


def pipeline_cats(layer: GatedMlpLayer, x, tau: float, cfg: BlockConfig | None = None,
                  want_act: bool = False) -> PipelineResult:
    """pipeline_cats (blocked_exec.cpp:330-348): dense gate pass, act, |act| > tau, exec_cats."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "pipeline_cats")
    d, F = layer.d_model, layer.d_inter
    y, m, alive, h = layer.device_layer().pipeline_cats(xb, tau, _reduction(cfg), want_act)
    tc = TrafficCounter()
    for _ in alive:
        tc.add(d * F, d, F)          # dense gate pass (blocked_exec.cpp:336-337)
        tc.add(0, F, F)              # act (:338-342)
        tc.add(0, 2 * F, 2 * F)      # threshold_mask (:304-310)
    _count_exec(tc, d, F, alive, "mc")
    res = PipelineResult(y[0] if single else y, _masks_out(m, alive, tau, single), tc)
    if want_act:
        res.act = h[0] if single else h
    return res


def pipeline_dc(layer: GatedMlpLayer, x, p: Predictor, cfg: BlockConfig | None = None,
                mask_override=None, tau_d: float = 0.0, want_logits: bool = False) -> PipelineResult:
    """pipeline_dc (blocked_exec.cpp:350-379): low-rank predictor, mask = override or
    logits > tau_d, exec_dc.  The predictor runs (and is costed) even with an override."""
    layer.validate()
    xb, single = _batched(x, layer.d_model, "pipeline_dc")
    B, d, F = xb.shape[0], layer.d_model, layer.d_inter
    if mask_override is not None:
        mask_override = _mask_rows(mask_override, B, F, "pipeline_dc")
    if p.kind() != PredictorKind.LowRank:
        raise DataError("pipeline_dc: the blocked pipeline models the low-rank predictor")
    lp = p.lowrank()
    if lp.d_model != d or lp.d_inter != F:
        raise DataError("pipeline_dc: predictor shape does not match the layer")
    y, m, alive, z = layer.device_layer(p).pipeline_dc(xb, tau_d, _reduction(cfg), mask_override,
                                                       want_logits)
    tc = TrafficCounter()
    r = lp.d_rank
    for _ in range(B):
        tc.add(d * r + r * F, d + r, r + F)  # predictor (blocked_exec.cpp:362-364)
        tc.add(0, F, F)                      # logits read, mask write (:375-376)
    _count_exec(tc, d, F, alive, "dc")
    res = PipelineResult(y[0] if single else y, _masks_out(m, alive, tau_d, single), tc)
    if want_logits:
        res.logits = z[0] if single else z
    return res


def forward_sparse(layer: GatedMlpLayer, x, mask) -> np.ndarray:
    """forward_sparse (sparsity.cpp:44-71), bit-exact (ordered kernels)."""
    layer.validate()
    if isinstance(mask, ActivationMask) and mask.size() != layer.d_inter:
        raise DataError(f"forward_sparse: mask has {mask.size()} lanes, layer d_inter {layer.d_inter}")
    xb, single = _batched(x, layer.d_model, "forward_sparse")
    masks = _mask_rows(mask, xb.shape[0], layer.d_inter, "forward_sparse")
    y = layer.device_layer().exec_dc(xb, masks, Reduction.DeterministicOrdered)
    return y[0] if single else y


def predict_logits(p: Predictor, x) -> np.ndarray:
    """predict_logits (predictor.cpp:128-138), low-rank; bit-exact."""
    xb, single = _batched(x, p.d_model(), "predict_logits")
    z = p.handle().predict_logits(xb)
    return z[0] if single else z


def predict_mask(p: Predictor, x, tau_d: float = 0.0):
    """predict_mask (predictor.cpp:140-148): alive where logit > 0 (tau recorded 0)."""
    z = np.atleast_2d(predict_logits(p, x))
    masks = [ActivationMask((row > tau_d).astype(np.uint8), int(np.count_nonzero(row > tau_d)), float(tau_d))
             for row in z]
    return masks[0] if np.asarray(x).ndim == 1 else masks


def forward_practical(layer: GatedMlpLayer, x, cfg: SparsityConfig, ctx: PracticalContext,
                      reduction: Reduction = Reduction.DeterministicOrdered) -> PracticalResult:
    """forward_practical (sparsity.cpp:90-121): MC |W_up x| > tau_hat; DC predictor mask;
    then the sparse forward.  Default reduction is the bit-exact path (forward_sparse is the
    reference's serial semantic definition)."""
    bc = BlockConfig(reduction=reduction)
    if cfg.method == SparsityMethod.MCountdown:
        if ctx.tau_hat is None:
            raise DataError("forward_practical: mc needs a calibrated tau_hat")
        r = pipeline_mc(layer, x, float(np.float32(ctx.tau_hat)), bc)
        return PracticalResult(r.y, r.mask)
    if cfg.method == SparsityMethod.DCountdown:
        if ctx.predictor is None:
            raise DataError("forward_practical: dc needs a trained predictor")
        r = pipeline_dc(layer, x, ctx.predictor, bc)
        return PracticalResult(r.y, r.mask)
    if ctx.tau_hat is None:
        raise DataError("forward_practical: cats needs a calibrated tau_hat")
    r = pipeline_cats(layer, x, float(np.float32(ctx.tau_hat)), bc)
    return PracticalResult(r.y, r.mask)


def top_m_threshold(v, m: int, signed: bool = False, device: int = 0):
    """top_m_threshold (numerics.cpp:105-142) on the device (cd_top_m): the m lanes of largest
    magnitude (ties to the lower index) and tau = the (m+1)-th magnitude (+inf for m = 0, -inf
    for m = n).  A batch (B x n) gives B results.  signed=True orders by the value itself.
    Returns (tau, mask) -- arrays for a batch."""
    v = np.ascontiguousarray(v, np.float32)
    single = v.ndim == 1
    vb = np.atleast_2d(v)
    B, n = vb.shape
    tau = np.empty(B, np.float32)
    mask = np.empty((B, n), np.uint8)
    check(lib().cd_top_m(device, B, n, ptr(vb), int(m), 1 if signed else 0, ptr(tau), ptr(mask)))
    return (float(tau[0]), mask[0]) if single else (tau, mask)


def calibrate(layer: GatedMlpLayer, xs, k: float, method: SparsityMethod,
              predictor: Predictor | None = None, per_sample: bool = False):
    """calibrate (calibration.cpp:11-37) on the device (cd_calibrate): tau = mean over the T
    samples of each sample's exact top-m threshold, m = alive_count_for(k, d_inter), accumulated
    in double in sample order.  MC thresholds |u| (u = W_up x), CATS |act(W_gate x)| -- the
    exact kernels, bitwise the reference's.  DC extends it to the predictor logits s_hat
    (signed, Alg. 3's tau_D), for which the reference has no calibrator
    (predict_mask fixes 0).  per_sample=True also returns the T per-sample thresholds."""
    xb, _ = _batched(xs, layer.d_model, "calibrate")
    if xb.shape[0] == 0:
        raise DataError("calibrate: no calibration samples")
    mid = {SparsityMethod.MCountdown: _capi.METHOD_MC, SparsityMethod.Cats: _capi.METHOD_CATS,
           SparsityMethod.DCountdown: _capi.METHOD_DC}[SparsityMethod(method)]
    if mid == _capi.METHOD_DC and predictor is None:
        raise DataError("calibrate: dc needs a predictor")
    dev = layer.device_layer(predictor if mid == _capi.METHOD_DC else None)
    tau = C.c_double()
    taus = np.empty(xb.shape[0], np.float32)
    check(lib().cd_calibrate(dev.raw, mid, xb.shape[0], ptr(xb), float(k), C.byref(tau), ptr(taus)))
    return (float(tau.value), taus) if per_sample else float(tau.value)


def realized_sparsity(mask: ActivationMask) -> float:
    """sparsity.cpp:123-126"""
    if mask.size() == 0:
        raise DataError("realized_sparsity: empty mask")
    return 1.0 - mask.alive_count / mask.size()


# ---------------------------------------------------------------- model files (host side)
@dataclass
class ModelFile:
    """model_io.hpp ModelFile: the layer, seed provenance, optional predictor and its k."""
    layer: GatedMlpLayer
    seed: int = 0
    predictor: Predictor | None = None
    predictor_k: float = 0.0


_MAGIC = b"CDWN1"


def checksum_hex(a) -> str:
    """checksum_hex (model_io.cpp:82-92): FNV-1a 64 over the raw bytes, 16 hex digits."""
    h = 14695981039346656037
    for b in np.ascontiguousarray(a).tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def write_model(path: str, mf: ModelFile) -> None:
    """write_model (model_io.cpp:94-138): magic, u32 header length, compact JSON header with
    sorted keys (nlohmann's dump order), f32 blobs W_up, W_gate, W_down, theta_a, theta_b."""
    import json
    mf.layer.validate()
    pred = None
    if mf.predictor is not None:
        lp = mf.predictor.lowrank()
        pred = {"d_rank": lp.d_rank, "k": mf.predictor_k, "kind": "lowrank"}
    header = {"activation": "silu" if mf.layer.activation == Activation.Silu else "gelu",
              "d_inter": mf.layer.d_inter, "d_model": mf.layer.d_model, "predictor": pred,
              "schema": "v1", "seed": int(mf.seed)}
    hs = json.dumps(header, separators=(",", ":"), sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(_MAGIC)
        f.write(np.uint32(len(hs)).tobytes())
        f.write(hs)
        for m in (mf.layer.w_up, mf.layer.w_gate, mf.layer.w_down):
            f.write(np.ascontiguousarray(m, np.float32).tobytes())
        if mf.predictor is not None:
            f.write(np.ascontiguousarray(lp.theta_a, np.float32).tobytes())
            f.write(np.ascontiguousarray(lp.theta_b, np.float32).tobytes())


def read_model(path: str, device_dtype: str = "f32", device: int = 0) -> ModelFile:
    """read_model (model_io.cpp:140-224) on the host: same validation and error messages
    (DataError); the returned layer uploads to the device on first use."""
    import json
    try:
        buf = open(path, "rb").read()
    except OSError:
        raise DataError(f"cannot open '{path}' for reading")
    if len(buf) < 5 or buf[:5] != _MAGIC:
        raise DataError(f"{path}: not a model file (bad magic, expected CDWN1)")
    if len(buf) < 9:
        raise DataError(f"{path}: truncated header length")
    hlen = int(np.frombuffer(buf[5:9], np.uint32)[0])
    if len(buf) < 9 + hlen:
        raise DataError(f"{path}: truncated header")
    try:
        h = json.loads(buf[9:9 + hlen])
    except ValueError as e:
        raise DataError(f"{path}: bad header JSON: {e}")
    try:
        if h["schema"] != "v1":
            raise DataError(f"{path}: unsupported schema")
        d, F, seed = int(h["d_model"]), int(h["d_inter"]), int(h["seed"])
        act_name = h["activation"]
    except (KeyError, TypeError) as e:
        raise DataError(f"{path}: bad header field: {e}")
    if act_name not in ("silu", "gelu"):
        raise DataError(f"unknown activation '{act_name}' (expected silu|gelu)")
    if d <= 0 or F <= 0:
        raise DataError(f"{path}: non-positive dimensions in header")
    mat = d * F * 4
    expected = 3 * mat
    pd = h.get("predictor")
    r = 0
    if pd is not None:
        kind = pd.get("kind")
        if kind == "lowrank":
            r = int(pd["d_rank"])
            if r <= 0:
                raise DataError(f"{path}: non-positive predictor rank")
            expected += (d * r + r * F) * 4
        elif kind == "ternary":
            raise DataError(f"{path}: ternary predictor: the B200 path runs the low-rank predictor only")
        else:
            raise DataError(f"{path}: unknown predictor kind '{kind}'")
    payload = len(buf) - 9 - hlen
    if payload != expected:
        raise DataError(f"{path}: payload is {payload} bytes, expected {expected}")
    blob = np.frombuffer(buf, np.float32, count=expected // 4, offset=9 + hlen)
    names = ["w_up", "w_gate", "w_down"]
    mats = [blob[i * d * F:(i + 1) * d * F].reshape(F, d) for i in range(3)]
    for m, n in zip(mats, names):
        bad = np.flatnonzero(~np.isfinite(m))
        if bad.size:
            raise DataError(f"{path}: {n} contains a non-finite value at index {bad[0]}")
    act = Activation.Silu if act_name == "silu" else Activation.GeluTanh
    layer = GatedMlpLayer(d, F, act, mats[0].copy(), mats[1].copy(), mats[2].copy(), device_dtype, device)
    mf = ModelFile(layer, seed)
    if r > 0:
        ta = blob[3 * d * F:3 * d * F + d * r].reshape(d, r).copy()
        tb = blob[3 * d * F + d * r:].reshape(r, F).copy()
        for m, n in ((ta, "theta_a"), (tb, "theta_b")):
            bad = np.flatnonzero(~np.isfinite(m))
            if bad.size:
                raise DataError(f"{path}: {n} contains a non-finite value at index {bad[0]}")
        mf.predictor = Predictor(LowRankPredictor(d, r, F, ta, tb), device_dtype, device)
        mf.predictor_k = float(pd["k"])
    return mf


# ---------------------------------------------------------------- synthetic workloads
def synth_workload(seed: int, d_model: int, d_inter: int, d_rank: int = 0,
                   activation: Activation = Activation.Silu, device_dtype: str = "f32",
                   device: int = 0):
    """bench()'s seeded setup (blocked_exec.cpp:396-415): (layer, x, predictor-or-None)."""
    up = np.empty((d_inter, d_model), np.float32)
    gate = np.empty_like(up)
    down = np.empty_like(up)
    x = np.empty(d_model, np.float32)
    ta = np.empty((d_model, d_rank), np.float32) if d_rank > 0 else None
    tb = np.empty((d_rank, d_inter), np.float32) if d_rank > 0 else None
    check(lib().cd_synth_layer(seed, d_model, d_inter, d_rank, ptr(up), ptr(gate), ptr(down), ptr(x),
                               ptr(ta), ptr(tb)))
    layer = GatedMlpLayer(d_model, d_inter, activation, up, gate, down, device_dtype, device)
    pred = None
    if d_rank > 0:
        pred = Predictor(LowRankPredictor(d_model, d_rank, d_inter, ta, tb), device_dtype, device)
    return layer, x, pred


def synth_normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    check(lib().cd_synth_normals(seed, n, ptr(out)))
    return out


# ---------------------------------------------------------------- bench
_METHOD_IDS = {"dense": _capi.METHOD_DENSE, "mc": _capi.METHOD_MC, "dc": _capi.METHOD_DC,
               "cats": _capi.METHOD_CATS}


def bench(method: str, shape: ShapeSpec, k: float, iters: int, cfg: BlockConfig | None = None,
          seed: int = 42, device_dtype: str = "f32") -> BenchStats:
    """bench() (blocked_exec.cpp:391-455) on the device: seeded layer + input, exact-count
    alive sets via per-input ideal thresholds (tau_u = top-m |u| threshold for MC; for DC the
    ideal top-m |s| mask as an override, predictor cost kept), warmup max(10, iters/10),
    per-iteration CUDA-event times, p50/p95.  Traffic counts are the reference's."""
    if iters <= 0:
        raise DataError("bench: iters must be positive")
    if method not in _METHOD_IDS:
        raise DataError(f"unknown method '{method}' (expected dense|cats|mc|dc)")
    d, F = shape.d_model, shape.d_inter
    layer, x, pred = synth_workload(seed, d, F, shape.d_rank if method == "dc" else 0,
                                    device_dtype=device_dtype)
    red = _reduction(cfg)
    dev = layer.device_layer(pred)
    warmup = max(10, iters // 10)
    tau = 0.0
    if method != "dense":
        m = alive_count_for(k, F)
        if method == "mc":
            # per-input ideal threshold tau_u = (m+1)-th largest |u| (blocked_exec.cpp:408-409)
            u = np.abs(pipeline_mc(layer, x, float("inf"),
                                   BlockConfig(reduction=Reduction.DeterministicOrdered), want_u=True).u)
            ind = u
        elif method == "cats":
            # tau_h = (m+1)-th largest |act(gate)| (blocked_exec.cpp:410)
            ind = np.abs(pipeline_cats(layer, x, float("inf"),
                                       BlockConfig(reduction=Reduction.DeterministicOrdered), want_act=True).act)
        else:
            # exact-count DC mask: threshold the predictor's own logits at their (m+1)-th
            # largest value, so exactly m rows are alive (the reference instead overrides
            # with the ideal top-m |s| mask, blocked_exec.cpp:411,423: same count and bytes).
            ind = predict_logits(pred, x)
        tau, _ = top_m_threshold(ind, m, signed=(method == "dc"))
    ns = dev.bench_device(_METHOD_IDS[method], x, tau, red, warmup, iters)
    ns = np.sort(ns)
    p = lambda q: int(ns[int(round(q * (len(ns) - 1)))])
    tc = TrafficCounter()
    if method == "dense":
        tc = pipeline_dense(layer, x, cfg).traffic
    elif method == "mc":
        tc = pipeline_mc(layer, x, tau, cfg).traffic
    elif method == "cats":
        tc = pipeline_cats(layer, x, tau, cfg).traffic
    else:
        tc = pipeline_dc(layer, x, pred, cfg, tau_d=tau).traffic
    dense_total = traffic_dense_split(ShapeSpec(d, F)).total()
    return BenchStats(method, 0.0 if method == "dense" else k, d, F, iters, p(0.5), p(0.95), tc.total(),
                      tc.total() / dense_total)
