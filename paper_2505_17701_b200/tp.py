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

from . import _capi
from ._capi import DataError
from .api import DeviceLayer, GatedMlpLayer, Predictor, Reduction

RMS_EPS = 1e-5  # the stack's input-norm epsilon (Llama-3.1's rms_norm_eps)


def shard_range(d_inter: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced neuron slice [begin, end) of rank `rank` out of `world`."""
    if world <= 0 or not (0 <= rank < world):
        raise DataError(f"shard_range: rank {rank} of world {world}")
    if d_inter < world:
        raise DataError(f"shard_range: d_inter {d_inter} < world {world}")
    base, rem = divmod(d_inter, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


class nvtx_range:
    """NVTX range around host-side enqueueing (a no-op without CUDA / a profiler attached), so
    an nsys / ncu timeline shows each layer and each all-reduce."""

    def __init__(self, name: str):
        self.name = name
        self.on = False

    def __enter__(self):
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.nvtx.range_push(self.name)
                self.on = True
        except Exception:
            self.on = False
        return self

    def __exit__(self, *a):
        if self.on:
            import torch
            torch.cuda.nvtx.range_pop()


def allreduce_sum_(y, group=None):
    """In-place sum of the ranks' partial outputs (a torch tensor; NCCL over NVLink on the
    device, gloo on CPU).  Enqueued on the caller's current stream context."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        with nvtx_range("cd.allreduce"):
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
        with nvtx_range("cd.layer"):
            self.dev.forward_device(method, x_dev, y_dev, tau, Reduction.UnorderedAccumulate, batch,
                                    alive_out=alive_out, stream=stream)

    def forward(self, method: int, x_dev, y_dev, tau: float, stream: int, batch: int = 1,
                alive_out=None) -> None:
        """Partial FFN on the shard, then the sum all-reduce: y_dev holds the full output."""
        self.forward_local(method, x_dev, y_dev, tau, stream, batch, alive_out)
        allreduce_sum_(y_dev, self.group)


def stack_step(n_layers: int, x, ys, run_layer, allreduce) -> None:
    """One decode step through a layer stack (BASELINE.json configs[3]):
    layer 0 reads x; layer l+1 reads RMSNorm(y_l) -- the reference has no residual, so the
    stack is the layers chained through an input norm -- and every layer's partial output is
    summed over the ranks by one all-reduce before the next layer reads it.

    run_layer(l, x_in, y_out, normed) computes layer l's partial output on this rank's neurons
    into y_out, normalising x_in first when `normed`; allreduce(y) sums y over the ranks in
    place.  ys[l] keeps every layer's output (layer l+1's input)."""
    for l in range(n_layers):
        run_layer(l, x if l == 0 else ys[l - 1], ys[l], l > 0)
        allreduce(ys[l])


class TPStack:
    """A stack of d_ff-sharded layers on this rank's GPU (configs[3]).  Each layer is a
    TPLayer (its neuron slice + theta_b rows; theta_a replicated) with its own calibrated
    threshold; the step is one kernel per layer -- k_dc_fused normalises its input itself
    (cd_forward_device_normed) -- plus one NCCL all-reduce per layer, all on one stream, so the
    whole step is capturable in one CUDA graph."""

    def __init__(self, tps: "list[TPLayer]", taus, eps: float = RMS_EPS, group=None,
                 method: int = _capi.METHOD_DC, prefetch: bool = False):
        if not tps or len(tps) != len(taus):
            raise DataError("TPStack: need one threshold per layer")
        self.tps = list(tps)
        self.taus = [float(t) for t in taus]
        if method == _capi.METHOD_DC and prefetch:
            # a step runs the layers in order (then layer 0 of the next step): each layer
            # L2-prefetches the next one's predictor (measured slower on the B200 at the Llama
            # shape: the prefetch traffic delays the next step's latency-bound chain)
            for l, t in enumerate(self.tps):
                t.dev.set_prefetch(self.tps[(l + 1) % len(self.tps)].dev)
        self.eps, self.group, self.method = float(eps), group, method
        self.rows = self.tps[0].rows

    @staticmethod
    def synthetic(n_layers: int, d_model: int, d_inter: int, d_rank: int, k: float, world: int, rank: int,
                  seed0: int = 42, device: int = 0, device_dtype: str = "bf16", eps: float = RMS_EPS,
                  group=None, n_cal: int = 8, keep_host: bool = False) -> "TPStack":
        """configs[3]'s stack: layer l is the reference bench()'s seeded layer + low-rank
        predictor for seed seed0 + l; tau_D of layer l is calibrated on
        n_cal N(0, 1) inputs (unit-RMS, like the normalised inputs of layers >= 1) as the mean
        of the per-input exact top-m logit thresholds (calibration.cpp:11-37 on the logits).
        Host weights are dropped after each upload unless keep_host."""
        from .api import calibrate, synth_normals, synth_workload, SparsityMethod
        tps, taus, host = [], [], []
        xcal = np.stack([synth_normals(70_000 + i, d_model) for i in range(n_cal)])
        for l in range(n_layers):
            layer, _, pred = synth_workload(seed0 + l, d_model, d_inter, d_rank, device_dtype=device_dtype,
                                            device=device)
            taus.append(calibrate(layer, xcal, k, SparsityMethod.DCountdown, pred))
            tps.append(TPLayer(layer, pred, world, rank, device, device_dtype, group))
            layer.invalidate()
            if keep_host:
                host.append((layer, pred))
        st = TPStack(tps, taus, eps, group)
        st.host = host
        return st

    def __len__(self) -> int:
        return len(self.tps)

    def forward(self, x_dev, ys_dev, stream: int, batch: int = 1, comm: bool = True, masks_out=None,
                alive_out=None) -> None:
        """ys_dev[l] <- layer l's (all-reduced) output; ys_dev[-1] is the stack's output.
        masks_out[l] / alive_out[l] (optional device buffers): layer l's shard-local mask and
        alive count."""

        def run_layer(l, x_in, y_out, normed):
            with nvtx_range(f"cd.layer{l}"):
                self.tps[l].dev.forward_device(
                    self.method, x_in, y_out, self.taus[l], Reduction.UnorderedAccumulate, batch,
                    mask_out=None if masks_out is None else masks_out[l],
                    alive_out=None if alive_out is None else alive_out[l], stream=stream,
                    rms_eps=self.eps if normed else None)

        stack_step(len(self.tps), x_dev, ys_dev, run_layer,
                   (lambda y: allreduce_sum_(y, self.group)) if comm else (lambda y: None))


def shard_partials_reference(partial_fn, d_inter: int, world: int) -> np.ndarray:
    """Host helper for tests: sum over ranks of partial_fn(begin, end) (what the all-reduce
    computes), in rank order."""
    acc = None
    for g in range(world):
        b, e = shard_range(d_inter, world, g)
        p = np.asarray(partial_fn(b, e), np.float64)
        acc = p if acc is None else acc + p
    return acc
