"""d_ff tensor parallelism for the COUNTDOWN FFN.

The reference has no distribution at all; the north_star adds exactly
one strategy.  Rank g of G owns the contiguous neuron slice ``shard_range(F, G, g)`` of the
neuron-major W_up / W_gate / W_down (gated_mlp.hpp:16-19) and the matching rows of
theta_b^T; theta_a is replicated.  Practical-mode thresholds (tau_hat_M, tau_D) are per-layer
constants, so every rank thresholds and compacts its own neurons with no communication
(sparsity.cpp:90-121 is lane-local); each rank produces a partial y_g over its alive neurons
and ONE sum all-reduce of the d-wide output per layer combines them.  Sharded sums
re-associate the ascending-i fold of weighted_sum (gated_mlp.cpp:28-44), so TP parity is
tolerance-based (1e-4 f32 / 1e-2 bf16), never bitwise.

One process per GPU, ``torch.distributed`` (backend "nccl" on the GPU box, "gloo" in the
CPU tests) for the plumbing.  The per-layer kernel chain and its all-reduce are enqueued on
the same CUDA stream, so a whole decode step (chain + NCCL all-reduce, every layer) is
capturable in one CUDA graph.
"""
from __future__ import annotations

import numpy as np

from ._capi import DataError
from .api import DeviceLayer, GatedMlpLayer, Predictor, Reduction


def shard_range(d_inter: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced neuron slice [begin, end) of rank `rank` out of `world`."""
    if world <= 0 or not (0 <= rank < world):
        raise DataError(f"shard_range: rank {rank} of world {world}")
    if d_inter < world:
        raise DataError(f"shard_range: d_inter {d_inter} < world {world}")
    base, rem = divmod(d_inter, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def allreduce_sum_(y, group=None):
    """In-place sum of the ranks' partial outputs (a torch tensor; NCCL over NVLink on the
    device, gloo on CPU).  Enqueued on the caller's current stream context."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
    return y


class TPLayer:
    """One FFN layer's d_ff shard on this rank's GPU plus the output all-reduce."""

    def __init__(self, layer: GatedMlpLayer, predictor: Predictor | None, world: int, rank: int,
                 device: int = 0, device_dtype: str = "bf16", group=None):
        layer.validate()
        self.d_model, self.d_inter = layer.d_model, layer.d_inter
        self.world, self.rank, self.group = world, rank, group
        self.rows = shard_range(layer.d_inter, world, rank)
        self.dev = DeviceLayer.create(layer.w_up, layer.w_gate, layer.w_down, layer.activation,
                                      device_dtype, device, row_range=self.rows)
        if predictor is not None:
            lp = predictor.lowrank()
            if lp.d_model != layer.d_model or lp.d_inter != layer.d_inter:
                raise DataError("TPLayer: predictor shape does not match the layer")
            self.dev.set_predictor(lp)

    def forward_local(self, method: int, x_dev, y_dev, tau: float, stream: int, batch: int = 1,
                      alive_out=None) -> None:
        """This rank's partial y over its neuron slice (no communication)."""
        self.dev.forward_device(method, x_dev, y_dev, tau, Reduction.UnorderedAccumulate, batch,
                                alive_out=alive_out, stream=stream)

    def forward(self, method: int, x_dev, y_dev, tau: float, stream: int, batch: int = 1,
                alive_out=None) -> None:
        """Partial FFN on the shard, then the sum all-reduce: y_dev holds the full output."""
        self.forward_local(method, x_dev, y_dev, tau, stream, batch, alive_out)
        allreduce_sum_(y_dev, self.group)


def shard_partials_reference(partial_fn, d_inter: int, world: int) -> np.ndarray:
    """Host helper for tests: sum over ranks of partial_fn(begin, end) (what the all-reduce
    computes), in rank order."""
    acc = None
    for g in range(world):
        b, e = shard_range(d_inter, world, g)
        p = np.asarray(partial_fn(b, e), np.float64)
        acc = p if acc is None else acc + p
    return acc
