"""d_ff tensor parallelism host logic on CPU: world_size 2 over gloo.

The device kernels need a B200; here each rank's partial output over its neuron slice comes
from the CPU oracle (test code only) and the product's shard partition + all-reduce
(paper_2505_17701_b200.tp) combine them.  The combined y must equal the single-device
forward_sparse within the f32 re-association tolerance (1e-5), and the shard-local masks of
practical mode must equal the slices of the global mask (thresholds are lane-local).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_17701_b200 import DataError
from paper_2505_17701_b200.tp import allreduce_sum_, shard_partials_reference, shard_range, stack_step, RMS_EPS


def test_shard_range_partitions():
    for F in (7, 48, 14336, 13824, 1001):
        for G in (1, 2, 3, 4, 8):
            if F < G:
                continue
            rs = [shard_range(F, G, g) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == F
            assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(14336, 8, 3) == (3 * 1792, 4 * 1792)
    with pytest.raises(DataError):
        shard_range(4, 8, 0)
    with pytest.raises(DataError):
        shard_range(16, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = O.Oracle()
        d, F, r = 48, 200, 8
        g = o.generate(31, d, F, r)
        x = g["x"]
        _, z = o.lowrank_logits(g["theta_a"], g["theta_b"], x)
        tau = float(np.quantile(z, 0.7))
        b, e = shard_range(F, world, rank)
        # shard-local practical mask: same lanes as the global one
        local_mask = (z[b:e] > np.float32(tau)).astype(np.uint8)
        shard = {k: g[k][b:e] for k in ("w_up", "w_gate", "w_down")}
        y = torch.from_numpy(o.forward_sparse(shard, x, local_mask).copy())
        allreduce_sum_(y)
        full = o.forward_sparse(g, x, (z > np.float32(tau)).astype(np.uint8))
        err = float(np.linalg.norm(y.numpy().astype(np.float64) - full) / np.linalg.norm(full))
        q.put((rank, err, int(local_mask.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tp_allreduce_matches_single_device(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for _, err, _ in res:
        assert err <= 1e-5
    # the shard alive counts add up to the global alive count
    import oracle as O
    o = O.Oracle()
    g = o.generate(31, 48, 200, 8)
    _, z = o.lowrank_logits(g["theta_a"], g["theta_b"], g["x"])
    assert sum(a for _, _, a in res) == int((z > np.float32(np.quantile(z, 0.7))).sum())


def test_shard_partials_reference_sums_in_rank_order(oracle):
    g = oracle.generate(5, 16, 40, 4)
    mask = np.ones(40, np.uint8)
    full = oracle.forward_sparse(g, g["x"], mask)

    def part(b, e):
        return oracle.forward_sparse({k: g[k][b:e] for k in ("w_up", "w_gate", "w_down")}, g["x"], mask[b:e])

    for G in (1, 2, 4, 8):
        y = shard_partials_reference(part, 40, G)
        assert np.linalg.norm(y - full) <= 1e-5 * np.linalg.norm(full)


def _stack_worker(rank, world, port, q):
    """configs[3] host logic: a 2-layer stack, each rank thresholding and computing its own
    neuron slice of every layer, the product's stack_step chaining the layers through the input
    RMS norm and one all-reduce per layer."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = O.Oracle()
        d, F, r, L = 48, 200, 8, 2
        gs = [o.generate(42 + l, d, F, r) for l in range(L)]
        taus = [float(np.quantile(o.lowrank_logits(g["theta_a"], g["theta_b"], g["x"])[1], 0.7)) for g in gs]
        b, e = shard_range(F, world, rank)
        x = torch.from_numpy(gs[0]["x"].copy())
        ys = [torch.zeros(d) for _ in range(L)]
        alive = [0] * L

        def run_layer(l, x_in, y_out, normed):
            g = gs[l]
            xi = O.rms_norm(x_in.numpy(), RMS_EPS) if normed else x_in.numpy()
            _, z = o.lowrank_logits(g["theta_a"], g["theta_b"], xi)
            m = (z[b:e] > np.float32(taus[l])).astype(np.uint8)
            alive[l] = int(m.sum())
            shard = {k: g[k][b:e] for k in ("w_up", "w_gate", "w_down")}
            y_out.copy_(torch.from_numpy(o.forward_sparse(shard, xi, m).copy()))

        stack_step(L, x, ys, run_layer, allreduce_sum_)
        # single device: the same stack without sharding
        xi = gs[0]["x"]
        for l in range(L):
            if l > 0:
                xi = O.rms_norm(y, RMS_EPS)
            _, z = o.lowrank_logits(gs[l]["theta_a"], gs[l]["theta_b"], xi)
            y = o.forward_sparse(gs[l], xi, (z > np.float32(taus[l])).astype(np.uint8))
        err = float(np.linalg.norm(ys[-1].numpy().astype(np.float64) - y) / np.linalg.norm(y))
        q.put((rank, err, alive))
    finally:
        dist.destroy_process_group()


def test_tp_two_layer_stack_matches_single_device():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stack_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for _, err, alive in res:
        assert err <= 1e-5
        assert all(a > 0 for a in alive)
