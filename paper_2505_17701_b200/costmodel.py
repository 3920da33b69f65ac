"""Closed-form FLOPs / traffic of one gated-MLP layer per method (host logic).

Restates /root/reference/proj/src/costmodel.cpp (Appendix D Tables 8-10 of the paper):
element counts at lane granularity, split into weight / vector / write streams.  The GPU
drop-in reports TrafficCounter values from these forms at the realized alive count,
which is exactly what the reference's instrumented executors count
(test_blocked_exec.cpp:125-212).  Also the B200 roofline byte model used by bench.py.
"""
from __future__ import annotations

from dataclasses import dataclass

from ._capi import DataError


@dataclass
class ShapeSpec:
    """costmodel.hpp:14-20"""
    d_model: int = 0
    d_inter: int = 0
    d_rank: int = 0
    c_act: int = 5
    s_alive: int = 0


def llama3_8b_shape() -> ShapeSpec:
    """costmodel.cpp:7"""
    return ShapeSpec(4096, 14336, 512, 5, 0)


def gemma2_9b_shape() -> ShapeSpec:
    """BASELINE.json configs[2]: d=3584, d_ff=14336 (GeLU-tanh)."""
    return ShapeSpec(3584, 14336, 512, 5, 0)


def qwen25_14b_shape() -> ShapeSpec:
    """BASELINE.json configs[4]: d=5120, d_ff=13824."""
    return ShapeSpec(5120, 13824, 512, 5, 0)


def alive_count_for(k: float, d_inter: int) -> int:
    """sparsity.cpp:19-27: floor((1-k) * d_inter), k in (0, 1)."""
    import math
    if not (k > 0.0 and k < 1.0):
        raise DataError(f"alive_count_for: k = {k} outside (0, 1)")
    if d_inter <= 0:
        raise DataError("alive_count_for: d_inter must be positive")
    return int(math.floor((1.0 - k) * float(d_inter)))


def shape_at_k(base: ShapeSpec, k: float) -> ShapeSpec:
    """costmodel.cpp:9-13"""
    return ShapeSpec(base.d_model, base.d_inter, base.d_rank, base.c_act,
                     alive_count_for(k, base.d_inter))


def _check(s: ShapeSpec, needs_rank: bool, needs_alive: bool, who: str) -> None:
    """costmodel.cpp:15-23"""
    if (s.d_model <= 0 or s.d_inter <= 0 or s.c_act < 0 or (needs_rank and s.d_rank <= 0)
            or (needs_alive and s.s_alive < 0)):
        raise DataError(f"{who}: bad shape d_model={s.d_model} d_inter={s.d_inter} "
                        f"d_rank={s.d_rank} s_alive={s.s_alive}")


@dataclass
class TrafficSplit:
    weight_reads: int = 0
    vector_reads: int = 0
    writes: int = 0

    def total(self) -> int:
        return self.weight_reads + self.vector_reads + self.writes


def flops_dense(s: ShapeSpec) -> int:
    _check(s, False, False, "flops_dense")
    return 6 * s.d_model * s.d_inter + s.c_act * s.d_inter + s.d_inter


def flops_mc(s: ShapeSpec) -> int:
    _check(s, False, True, "flops_mc")
    return (2 * s.d_model * s.d_inter + 2 * s.d_inter + 4 * s.d_model * s.s_alive
            + s.c_act * s.s_alive + s.s_alive)


def flops_dc(s: ShapeSpec) -> int:
    _check(s, True, True, "flops_dc")
    return (2 * s.d_model * s.d_rank + 2 * s.d_rank * s.d_inter + s.d_inter
            + 6 * s.d_model * s.s_alive + s.c_act * s.s_alive + s.s_alive)


def traffic_dense_split(s: ShapeSpec) -> TrafficSplit:
    """costmodel.cpp:59-66"""
    _check(s, False, False, "traffic_dense")
    return TrafficSplit(3 * s.d_model * s.d_inter, 2 * s.d_model + 4 * s.d_inter,
                        4 * s.d_inter + s.d_model)


def traffic_mc_split(s: ShapeSpec) -> TrafficSplit:
    """costmodel.cpp:77-84"""
    _check(s, False, True, "traffic_mc")
    return TrafficSplit(s.d_model * s.d_inter + 2 * s.d_model * s.s_alive,
                        2 * s.d_model + 4 * s.d_inter + s.s_alive, 4 * s.d_inter + s.d_model)


def traffic_dc_split(s: ShapeSpec) -> TrafficSplit:
    """costmodel.cpp:86-93"""
    _check(s, True, True, "traffic_dc")
    return TrafficSplit(s.d_model * s.d_rank + s.d_rank * s.d_inter + 3 * s.d_model * s.s_alive,
                        2 * s.d_model + s.d_rank + 3 * s.d_inter,
                        3 * s.d_inter + s.d_rank + s.d_model)


def elements_to_mb(elements: int) -> float:
    """costmodel.cpp:105-107 (MB = elements / 2^20)"""
    return elements / 1048576.0


# ---------------------------------------------------------------- B200 byte model
def device_bytes(method: str, d: int, F: int, r: int, alive: int, wbytes: int, batch: int = 1,
                 union_rows: int | None = None) -> dict:
    """Algorithmic HBM bytes of one decode step on the device.

    Weight rows actually streamed (union of per-sample alive rows for batch > 1) x d x dtype,
    the whole predictor for DC, plus the f32 vectors x (read) and y (written).  Masks and
    indicators never round-trip through HBM in the fused chain, so the reference's
    vector/write element terms (mask flags, |u|, logits) are not device traffic.
    """
    rows = alive if union_rows is None else union_rows
    vec = 4 * batch * 2 * d  # x in, y out (f32)
    if method == "dense":
        w = 3 * F * d * wbytes
    elif method == "mc":
        w = (F * d + 2 * rows * d) * wbytes
    elif method == "dc":
        w = (d * r + r * F + 3 * rows * d) * wbytes
    else:
        raise DataError(f"unknown method '{method}'")
    return {"weight_bytes": w, "vector_bytes": vec, "total_bytes": w + vec}
