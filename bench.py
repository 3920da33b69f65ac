"""bench.py -- COUNTDOWN sparse Gated-MLP FFN decode on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the one the metric is quoted on): one Gated-MLP layer of
Llama-3.1-8B shape (d=4096, d_ff=14336, SiLU), bf16 weights (f32 x / y / accumulation),
batch-1 decode, D-CountDown (low-rank predictor r=512) at 90% target sparsity.  Weights,
predictor and inputs are the reference bench()'s seeded synthetic workload
(blocked_exec.cpp:396-415, bit-identical RNG), RNE-rounded to bf16 on upload.  tau_D is
calibrated per layer as the mean over 32 calibration inputs of each input's exact top-m
logit threshold (calibration.cpp:11-37 extended to the predictor logits, Alg. 3
PAPER.md:645); timed inputs are 16 other N(0,1) vectors.

A "step" = one token through one FFN layer.  `value` = tokens/s of the fused chain with
inputs resident in HBM: K steps captured in one CUDA graph, rotating over NL layer replicas
whose touched rows together exceed the 126 MB L2 (so every step streams its rows from HBM),
timed with CUDA events, barrier + synchronize on both sides, max over ranks.  `e2e` = the
same metric through the reference-facing C-ABI call with HOST buffers (cd_pipeline_dc:
H2D of x, the chain, D2H of y and the alive count, synchronous), wall-clock per call.

N > 1 (torchrun): d_ff tensor-parallel over the ranks, NCCL all-reduce of y
per step inside the graph; strong scaling (the same token stream, split neurons).

`--impl reference`: the reference's own CPU implementation (oracle/_ref, the unmodified
library built from /root/reference/proj/src) on the host cores: pipeline_dc on the same
layer / inputs with the same alive sets (mask_override = logits > tau_D computed by the
reference's predict_logits), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D, F, R = 4096, 14336, 512
SEED = 42
N_CAL, N_X = 32, 16
METRIC = "FFN decode tokens/s + effective HBM GB/s vs sparsity, Llama-3.1-8B shape"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--k", type=float, default=0.9)
    p.add_argument("--layers", type=int, default=8, help="layer replicas rotated per step (L2-cold)")
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-batched", action="store_true", help="skip BASELINE configs[4] (batch-64 + prefill)")
    p.add_argument("--no-configs", action="store_true", help="skip configs[2] (Gemma) and the f32 line")
    p.add_argument("--no-stack", action="store_true", help="skip configs[3] (the 32-layer stack)")
    p.add_argument("--cooperative", action="store_true",
                   help="launch the batch-1..4 persistent kernels cooperative (the library default) "
                        "instead of PDL-chained (CD_ENGINE_PDL_CHAIN: the bench owns the GPU)")
    p.add_argument("--prefetch", action="store_true",
                   help="L2-prefetch the next layer's predictor in each step (measured slower: off by default)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- workload
def workload():
    """Seeded layer + predictor (reference bench() order), calibration and timed inputs."""
    import paper_2505_17701_b200 as cd
    layer, _, pred = cd.synth_workload(SEED, D, F, R, device_dtype="bf16")
    xcal = np.stack([cd.synth_normals(10_000 + i, D) for i in range(N_CAL)])
    xs = np.stack([cd.synth_normals(1_000 + i, D) for i in range(N_X)])
    return layer, pred, xcal, xs


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu summary
    (profiles/ncu_traffic.json, written from a `ncu --set full` capture), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        j = json.load(f)
    v = j.get(kernel)
    return None if v is None else float(v["dram_bytes_per_launch"])


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def tensor_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return float(j.get("bf16_tflops_sustained", j.get("bf16_tflops", 1376.5))), "measured (sustained)"
    return 1376.5, "fallback"


def batched_section(torch, cd, timer, steps, peak_gbs):
    """BASELINE.json configs[4]: Qwen2.5-14B FFN shape (d=5120, d_ff=13824, SiLU), batch-64 decode at
    ~80% sparsity (per-sample masks, D- and M-CountDown) and a dense prefill of 2048 tokens, on the
    tcgen05 tensor-core path (kernels_tc.cu).  Weights 3 x 13824 x 5120 bf16 = 425 MB > L2, so every
    step streams them from HBM.  tau: mean over 8 calibration inputs of the per-input 0.8 quantile."""
    from paper_2505_17701_b200 import _capi
    Dq, Fq, Rq, B, P = 5120, 13824, 512, 64, 2048
    layer, _, pred = cd.synth_workload(SEED + 1, Dq, Fq, Rq, device_dtype="bf16")
    dev = layer.device_layer(pred)
    xcal = np.stack([cd.synth_normals(20_000 + i, Dq) for i in range(8)])
    xs = np.stack([cd.synth_normals(30_000 + i, Dq) for i in range(B)])
    z = np.atleast_2d(cd.predict_logits(pred, xcal))
    tau_dc = float(np.mean([np.quantile(r, 0.8) for r in z]))
    u = np.abs(cd.pipeline_mc(layer, xcal, float("inf"), cd.BlockConfig(reduction=cd.Reduction.DeterministicOrdered),
                              want_u=True).u)
    tau_mc = float(np.mean([np.quantile(r, 0.8) for r in u]))
    x_dev = torch.from_numpy(xs).cuda()
    xp = torch.from_numpy(np.stack([cd.synth_normals(40_000 + i, Dq) for i in range(P)])).cuda()
    wbytes = 3 * Fq * Dq * 2
    tpeak, tkind = tensor_peak()
    out = {"workload": "BASELINE configs[4]: qwen2.5-14b FFN d=5120 d_ff=13824 SiLU r=512, bf16 weights, "
                       "batch-64 decode (per-sample masks, row union ~100%) + dense prefill 2048 tokens",
           "engine": "tcgen05 tensor cores (TMA + UMMA + TMEM, stream-K), activations as bf16 hi/lo pairs "
                     "for decode", "cases": []}
    for name, method, nb, x, tau in (("dc80_b64", _capi.METHOD_DC, B, x_dev, tau_dc),
                                     ("mc80_b64", _capi.METHOD_MC, B, x_dev, tau_mc),
                                     ("dense_b64", _capi.METHOD_DENSE, B, x_dev, 0.0),
                                     ("prefill_2048", _capi.METHOD_DENSE, P, xp, 0.0)):
        y = torch.empty(nb, Dq, device="cuda")
        alive = torch.zeros(nb, dtype=torch.int32, device="cuda")

        def fwd(i, cs, method=method, nb=nb, x=x, y=y, alive=alive, tau=tau):
            dev.forward_device(method, x, y, tau=tau, batch=nb, alive_out=alive, stream=cs)

        with torch.cuda.stream(timer.stream):
            for i in range(3):
                fwd(i, timer.stream.cuda_stream)
        torch.cuda.synchronize()
        path = dev.last_path()
        n = steps if nb <= 64 else max(3, steps // 8)
        ms, n_timed, _ = timer.run(fwd, n)
        us = 1e3 * ms
        sp = 1.0 - alive.float().mean().item() / Fq
        case = {"case": name, "batch": nb, "path": path, "us_per_step": round(us, 2), "timed_steps": n_timed,
                "tokens_per_s": round(nb / us * 1e6, 1), "realized_sparsity": round(sp, 4)}
        if nb <= 64:
            pbytes = (Dq * Rq + Fq * Rq) * 2 if method == _capi.METHOD_DC else 0
            bytes_ = wbytes + pbytes + 2 * nb * Dq * 4
            case["roofline"] = {"bound": "hbm", "alg_bytes": bytes_, "achieved": round(bytes_ / us / 1e3, 1),
                                "peak": peak_gbs, "unit": "GB/s", "frac": round(bytes_ / us / 1e3 / peak_gbs, 4),
                                "note": "row union of 64 per-sample masks ~ all rows: dense-equivalent bytes"}
        else:
            flops = 2 * 3 * Fq * Dq * nb
            case["roofline"] = {"bound": "tensor", "alg_flops": flops, "achieved": round(flops / us / 1e6, 1),
                                "peak": tpeak, "peak_kind": tkind, "unit": "TFLOP/s",
                                "frac": round(flops / us / 1e6 / tpeak, 4)}
        out["cases"].append(case)
    del dev
    layer.invalidate()
    return out


# ----------------------------------------------------------------------------- CPU baseline
def cpu_baseline_sample():
    """The reference library's own bench() (blocked_exec.cpp:391-455): DC, Llama shape, k=0.9,
    Ordered, blk 16/256 (cmd_bench's defaults), all host threads; p50 of a bounded sample."""
    import oracle as O
    if not O.reference_available():
        return None
    ref = O.Reference()
    iters = 10
    t0 = time.time()
    r = ref.bench("dc", D, F, R, 0.9, iters, seed=SEED)
    return {"value": 1e9 / r["p50_ns"], "unit": "tokens/s", "cores": ref.max_threads(),
            "kind": "reference",
            "sample": f"reference bench(dc, d={D}, d_ff={F}, r={R}, k=0.9, iters={iters}) p50 "
                      f"{r['p50_ns']/1e6:.2f} ms/token, f32, OpenMP Ordered blk 16/256 "
                      f"({time.time()-t0:.1f} s incl. setup)"}


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref, the unmodified library) on the same
    layer, inputs and alive sets.  Only oracle/ is loaded here (the reference arm must not load
    the product library): inputs come from the reference's own Rng (normal_f == float(normal()),
    numerics.hpp:50-52), thresholds from its predict_logits and alive_count_for."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    if not O.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcountdown_ref.so not built"}))
        return
    ref = O.Reference()
    g = ref.generate(SEED, D, F, R)
    xcal = np.stack([ref.rng_normals(10_000 + i, D).astype(np.float32) for i in range(N_CAL)])
    xs = np.stack([ref.rng_normals(1_000 + i, D).astype(np.float32) for i in range(N_X)])
    m = ref.alive_count_for(args.k, F)
    taus = []
    for x in xcal:
        z = ref.predict_logits(g["theta_a"], g["theta_b"], x)
        order = np.lexsort((np.arange(F), -z))
        taus.append(float(z[order[m]]))
    tau = float(np.mean(taus))
    masks = [(ref.predict_logits(g["theta_a"], g["theta_b"], x) > np.float32(tau)).astype(np.uint8) for x in xs]
    # the reference layer / predictor objects are built once (as its own bench() does,
    # blocked_exec.cpp:396-415); each timed step is one pipeline_dc call
    h = ref.model(g)
    for i in range(args.warmup):
        ref.model_pipeline_dc(h, xs[i % N_X], D, masks[i % N_X])
    t0 = time.perf_counter()
    alive = 0
    for i in range(args.steps):
        r = ref.model_pipeline_dc(h, xs[i % N_X], D, masks[i % N_X])
        alive += r["alive"]
    dt = time.perf_counter() - t0
    ref.model_free(h)
    v = args.steps / dt
    cores = ref.max_threads()
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"llama3.1-8b FFN layer d={D} d_ff={F}, D-CountDown r={R} k={args.k}, batch 1 "
                                   "decode (reference CPU pipeline_dc, mask_override = logits > tau_D)",
                       "realized_sparsity": 1 - alive / args.steps / F},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "reference",
                             "sample": f"{args.steps} tokens x pipeline_dc, OpenMP {cores} threads, Ordered"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- ours
class Timer:
    """Steady-state device timing of a captured step sequence: a graph of `steps` steps is
    replayed back to back until the timed region lasts >= min_ms (so the rate does not depend
    on --steps: graph launch and the first step's unoverlapped prologue are amortised), CUDA
    events on the launching stream, barrier + synchronize on both sides, max over ranks."""

    def __init__(self, torch, stream, dist=None, min_ms=60.0):
        self.torch, self.stream, self.dist, self.min_ms = torch, stream, dist, min_ms

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, v):
        if self.dist is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def capture(self, fwd, steps):
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            with torch.cuda.graph(g, stream=self.stream):
                cs = torch.cuda.current_stream().cuda_stream
                for i in range(steps):
                    fwd(i, cs)
        return g

    def replay_ms(self, g, reps):
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.barrier()
        e0.record(self.stream)
        with torch.cuda.stream(self.stream):
            for _ in range(reps):
                g.replay()
        e1.record(self.stream)
        self.barrier()
        return self.max_over_ranks(e0.elapsed_time(e1))

    def run(self, fwd, steps, soak_s=0.0):
        """-> (ms per step, timed steps, replays).  Same replay count on every rank."""
        g = self.capture(fwd, steps)
        one = self.replay_ms(g, 1)
        reps = max(2, int(np.ceil(self.min_ms / max(one, 1e-3))))
        if soak_s > 0:
            self.replay_ms(g, max(1, int(soak_s * 1e3 / max(one, 1e-3))))
        ms = self.replay_ms(g, reps)
        del g
        return ms / (reps * steps), reps * steps, reps


def exact_logits(cd, pred, xs):
    """Predictor logits from the exact kernels (DeterministicOrdered: bitwise the reference's
    predict_logits, pinned by tests/test_gpu_parity.py)."""
    return np.atleast_2d(cd.predict_logits(pred, xs))


def top_m_tau(rows, m):
    """Mean over samples of each sample's exact top-m threshold (calibration.cpp:11-37: the
    (m+1)-th largest value, ties to the lower index, numerics.cpp:105-142), selected on the
    device (cd_top_m, signed order: the rows are logits or |u|), mean in double in order."""
    import paper_2505_17701_b200 as cd
    taus, _ = cd.top_m_threshold(np.atleast_2d(rows), m, signed=True)
    acc = 0.0
    for t in taus:
        acc += float(t)
    return acc / len(taus)


def flip_report(torch, cd, dev, method, xs, tau, z_exact, band=1e-6):
    """Near-threshold flips of the fast path's index sets against the exact indicator
    (north_star: index sets equal except lanes whose coefficient lies within 1e-6 relative of
    the threshold -- counted and reported).  The fast path's own indicator (logits / u) is
    returned by the same kernel and compared too."""
    B, Fx = z_exact.shape
    mask = torch.zeros((B, Fx), dtype=torch.uint8, device="cuda")
    ind = torch.zeros((B, Fx), dtype=torch.float32, device="cuda")
    y = torch.zeros((B, xs.shape[1]), device="cuda")
    xd = torch.from_numpy(np.ascontiguousarray(xs)).cuda()
    for b in range(B):
        dev.forward_device(method, xd[b], y[b], tau=tau, batch=1, mask_out=mask[b], indicator_out=ind[b])
    torch.cuda.synchronize()
    got = mask.cpu().numpy().astype(bool)
    zf = ind.cpu().numpy()
    ref = np.abs(z_exact) if method == cd._capi.METHOD_MC else z_exact
    want = ref > np.float32(tau)
    flips = got != want
    dist = np.abs(ref[flips].astype(np.float64) - tau) / max(abs(tau), 1e-30)
    return {"inputs": int(B), "lanes": int(B * Fx), "flips": int(flips.sum()),
            "flips_outside_1e-6": int((dist > band).sum()),
            "max_rel_dist_of_flip": float(dist.max()) if dist.size else 0.0,
            "indicator_max_abs_err_rel_tau": float(np.max(np.abs(
                (np.abs(zf) if method == cd._capi.METHOD_MC else zf) - ref)) / max(abs(tau), 1e-30)),
            "note": "fast-path mask vs exact-kernel indicator > tau (exact == reference bitwise)"}


PDL_CHAIN = True  # set from --cooperative in main(); the bench process owns the GPU


def serve_mode(devs):
    """The bench owns the device: PDL-chained persistent kernels (CD_ENGINE_PDL_CHAIN) unless
    --cooperative asks for the library's default cooperative launches."""
    for dv in devs:
        dv.set_engines(pdl_chain=PDL_CHAIN)


def gemma_section(torch, cd, timer, steps, peak_gbs):
    """BASELINE.json configs[2]: Gemma-2-9B FFN (d=3584, d_ff=14336, GeLU-tanh), r=512, bf16
    weights, batch 1 / 4 / 16 decode, M- and D-CountDown at 90% (per-sample masks; the bytes of
    a batched step are the UNION of the samples' active rows).  4 layer replicas rotate per
    step so the touched rows exceed L2."""
    from paper_2505_17701_b200 import costmodel as cm
    Dg, Fg, Rg, NL = 3584, 14336, 512, 4
    layers = []
    for i in range(NL):
        layer, _, pred = cd.synth_workload(SEED + 100 + i, Dg, Fg, Rg, activation=cd.Activation.GeluTanh,
                                           device_dtype="bf16")
        layers.append((layer, pred, layer.device_layer(pred)))
    serve_mode([lv[2] for lv in layers])
    layer0, pred0, _ = layers[0]
    xcal = np.stack([cd.synth_normals(50_000 + i, Dg) for i in range(16)])
    xs = np.stack([cd.synth_normals(60_000 + i, Dg) for i in range(16)])
    m = cd.alive_count_for(0.9, Fg)
    z_cal = exact_logits(cd, pred0, xcal)
    z_x = exact_logits(cd, pred0, xs)
    tau_dc = top_m_tau(z_cal, m)
    u_cal = np.abs(cd.pipeline_mc(layer0, xcal, float("inf"), cd.BlockConfig(
        reduction=cd.Reduction.DeterministicOrdered), want_u=True).u)
    u_x = np.abs(cd.pipeline_mc(layer0, xs, float("inf"), cd.BlockConfig(
        reduction=cd.Reduction.DeterministicOrdered), want_u=True).u)
    tau_mc = top_m_tau(u_cal, m)
    xd = torch.from_numpy(xs).cuda()
    out = {"workload": "BASELINE configs[2]: gemma-2-9b FFN d=3584 d_ff=14336 GeLU-tanh r=512, bf16 weights, "
                       "k=0.9 (tau calibrated on 16 inputs), per-sample masks, 4 layer replicas rotated",
           "cases": []}
    for method, name, tau, ind in ((cd._capi.METHOD_DC, "dc", tau_dc, z_x), (cd._capi.METHOD_MC, "mc", tau_mc, u_x)):
        for B in (1, 4, 16):
            y = torch.zeros((NL, B, Dg), device="cuda")
            nx = 16 // B

            def fwd(i, cs, method=method, B=B, y=y, tau=tau, nx=nx):
                li, xi = i % NL, (i // NL) % nx
                layers[li][2].forward_device(method, xd[xi * B:(xi + 1) * B], y[li], tau=tau, batch=B, stream=cs)

            with torch.cuda.stream(timer.stream):
                for i in range(2 * NL):
                    fwd(i, timer.stream.cuda_stream)
            torch.cuda.synchronize()
            path = layers[0][2].last_path()
            ms, n_timed, _ = timer.run(fwd, max(steps, 2 * NL))
            us = 1e3 * ms
            alive = ind > np.float32(tau)
            unions = [int(np.any(alive[j * B:(j + 1) * B], axis=0).sum()) for j in range(nx)]
            per = [int(a) for a in alive.sum(axis=1)]
            s_u = float(np.mean(unions))
            bytes_ = cm.device_bytes(name, Dg, Fg, Rg if name == "dc" else 0, int(round(s_u)), 2)["total_bytes"]
            bytes_ += (B - 1) * 8 * Dg  # the other samples' x / y
            out["cases"].append({
                "method": name, "batch": B, "path": path, "us_per_step": round(us, 3),
                "tokens_per_s": round(B / us * 1e6, 1), "realized_sparsity": round(1 - float(np.mean(per)) / Fg, 4),
                "union_rows": round(s_u, 1), "timed_steps": n_timed,
                "roofline": {"bound": "hbm", "alg_bytes": bytes_, "achieved": round(bytes_ / us / 1e3, 1),
                             "peak": peak_gbs, "unit": "GB/s", "frac": round(bytes_ / us / 1e3 / peak_gbs, 4)}})
    dense_y = torch.zeros((NL, Dg), device="cuda")

    def fwd_dense(i, cs):
        layers[i % NL][2].forward_device(cd._capi.METHOD_DENSE, xd[i % 16], dense_y[i % NL], batch=1, stream=cs)

    ms, n_timed, _ = timer.run(fwd_dense, max(steps, 2 * NL))
    bytes_ = 3 * Fg * Dg * 2 + 8 * Dg
    out["cases"].append({"method": "dense", "batch": 1, "us_per_step": round(1e3 * ms, 3),
                         "tokens_per_s": round(1e6 / (1e3 * ms), 1), "timed_steps": n_timed,
                         "roofline": {"bound": "hbm", "alg_bytes": bytes_, "achieved": round(bytes_ / (1e3 * ms) / 1e3, 1),
                                      "peak": peak_gbs, "unit": "GB/s",
                                      "frac": round(bytes_ / (1e3 * ms) / 1e3 / peak_gbs, 4)}})
    del layers
    return out


def f32_section(torch, cd, timer, steps, peak_gbs, k):
    """The headline workload at the reference's own precision (f32 weights, f32 arithmetic,
    numerics.cpp:77-87): same layer, inputs and tau_D as the headline, so the CPU arm compares
    like for like.  Device rate (2 replicas rotated: 2 x 112 MB touched > L2) and e2e through
    cd_pipeline_dc with host buffers; flips of the fast path's index sets vs the exact kernels
    (the "fp32 oracle mode", bitwise the reference)."""
    from paper_2505_17701_b200 import costmodel as cm
    from paper_2505_17701_b200._capi import lib, ptr, check
    NL = 2
    layer, _, pred = cd.synth_workload(SEED, D, F, R, device_dtype="f32")
    devs = [layer.device_layer(pred)]
    for _ in range(NL - 1):
        d2 = cd.DeviceLayer.create(layer.w_up, layer.w_gate, layer.w_down, 0, "f32")
        d2.set_predictor(pred.lowrank())
        devs.append(d2)
    serve_mode(devs)
    xcal = np.stack([cd.synth_normals(10_000 + i, D) for i in range(N_CAL)])
    xs = np.stack([cd.synth_normals(1_000 + i, D) for i in range(N_X)])
    z_cal = exact_logits(cd, pred, xcal)
    z_x = exact_logits(cd, pred, xs)
    tau = top_m_tau(z_cal, cd.alive_count_for(k, F))
    xd = torch.from_numpy(xs).cuda()
    y = torch.zeros((NL, D), device="cuda")

    def fwd(i, cs):
        devs[i % NL].forward_device(cd._capi.METHOD_DC, xd[i % N_X], y[i % NL], tau=tau, batch=1, stream=cs)

    with torch.cuda.stream(timer.stream):
        for i in range(2 * NL):
            fwd(i, timer.stream.cuda_stream)
    torch.cuda.synchronize()
    launches = devs[0].last_launches()
    ms, n_timed, _ = timer.run(fwd, max(steps, 2 * NL))
    alive = (z_x > np.float32(tau)).sum(axis=1)
    bytes_ = float(np.mean([cm.device_bytes("dc", D, F, R, int(a), 4)["total_bytes"] for a in alive]))
    # e2e: the reference-facing call with host buffers
    L = lib()
    yh = np.empty(D, np.float32)
    ah = np.empty(1, np.int64)
    xs_c = [np.ascontiguousarray(x) for x in xs]
    for i in range(3 * NL):
        check(L.cd_pipeline_dc(devs[i % NL].raw, 1, ptr(xs_c[i % N_X]), tau, None, 1, ptr(yh), None, ptr(ah), None))
    n = max(steps, 64)
    t0 = time.perf_counter()
    for i in range(n):
        check(L.cd_pipeline_dc(devs[i % NL].raw, 1, ptr(xs_c[i % N_X]), tau, None, 1, ptr(yh), None, ptr(ah), None))
    dt = time.perf_counter() - t0
    flips = flip_report(torch, cd, devs[0], cd._capi.METHOD_DC, xs, tau, z_x)
    out = {"workload": f"headline config at f32 (the reference's precision): llama3.1-8b FFN, D-CountDown r={R} "
                       f"k={k}, batch 1, f32 weights / arithmetic, same inputs and tau_D",
           "value": round(1e3 / ms, 1), "unit": "tokens/s", "us_per_step": round(1e3 * ms, 3), "timed_steps": n_timed,
           "kernels_per_step": launches, "realized_sparsity": round(1 - float(alive.mean()) / F, 4),
           "roofline": {"bound": "hbm", "alg_bytes": bytes_, "achieved": round(bytes_ / ms / 1e6, 1), "peak": peak_gbs,
                        "unit": "GB/s", "frac": round(bytes_ / ms / 1e6 / peak_gbs, 4)},
           "e2e": {"value": round(n / dt, 1), "unit": "tokens/s", "calls": n, "h2d_bytes_per_step": 4 * D,
                   "d2h_bytes_per_step": 4 * D + 4, "api": "cd_pipeline_dc (host buffers), wall clock"},
           "flips": flips}
    del devs
    layer.invalidate()
    return out


def stack_section(torch, cd, timer, world, rank, steps, peak_gbs, k, n_layers=32):
    """BASELINE.json configs[3]: the 32-layer Llama-3.1-8B FFN stack, layer l = seed 42 + l,
    layer l+1's input = RMSNorm(y_l) (fused into k_dc_fused), D-CountDown at k (tau_D
    calibrated per layer), bf16, d_ff tensor-parallel over the ranks with one NCCL all-reduce
    per layer; a token's whole stack (32 kernels + 32 all-reduces) is captured in the graph.
    Reports tokens/s through the stack and the all-reduce's share of layer time."""
    from paper_2505_17701_b200 import costmodel as cm
    from paper_2505_17701_b200.tp import TPStack
    t0 = time.time()
    st = TPStack.synthetic(n_layers, D, F, R, k, world, rank, seed0=SEED, device=torch.cuda.current_device())
    serve_mode([t.dev for t in st.tps])
    build_s = time.time() - t0
    xs = torch.from_numpy(np.stack([cd.synth_normals(90_000 + i, D) for i in range(4)])).cuda()
    ys = torch.zeros((n_layers, D), device="cuda")
    alive = torch.zeros((n_layers, 1), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(timer.stream):
        for i in range(2):
            st.forward(xs[i % 4], ys, timer.stream.cuda_stream, alive_out=alive)
    torch.cuda.synchronize()
    al = alive.cpu().numpy()[:, 0]
    Fl = st.rows[1] - st.rows[0]
    bytes_tok = float(sum(cm.device_bytes("dc", D, Fl, R, int(a), 2)["total_bytes"] for a in al))

    def tok(i, cs, comm=True):
        st.forward(xs[i % 4], ys, cs, comm=comm)

    n = max(2, min(steps, 8))
    ms, n_timed, _ = timer.run(tok, n)
    out = {"workload": f"BASELINE configs[3]: {n_layers}-layer llama3.1-8b FFN stack (seeds 42+l), input of layer "
                       f"l+1 = RMSNorm(y_l) fused into k_dc_fused, D-CountDown r={R} k={k} (tau_D per layer), bf16, "
                       f"tp{world} over d_ff" + (" + NCCL all-reduce per layer" if world > 1 else ""),
           "tokens_per_s": round(1e3 / ms, 1), "us_per_token": round(1e3 * ms, 2),
           "us_per_layer": round(1e3 * ms / n_layers, 3), "timed_tokens": n_timed,
           "realized_sparsity_rank_layers": round(1 - float(al.mean()) / Fl, 4),
           "roofline": {"bound": "hbm", "alg_bytes_per_token_per_rank": bytes_tok,
                        "achieved": round(bytes_tok / ms / 1e6, 1), "peak": peak_gbs, "unit": "GB/s",
                        "frac": round(bytes_tok / ms / 1e6 / peak_gbs, 4)},
           "build_s": round(build_s, 1)}
    if world > 1:
        ms_c, _, _ = timer.run(lambda i, cs: tok(i, cs, comm=False), n)
        out["allreduce"] = {"compute_only_us_per_layer": round(1e3 * ms_c / n_layers, 3),
                            "allreduce_share": round(max(0.0, 1 - ms_c / ms), 4),
                            "allreduce_bytes": 4 * D, "note": "share = 1 - (stack without the all-reduces) / stack"}
    del st
    return out


def run_ours(args):
    import torch
    import paper_2505_17701_b200 as cd
    from paper_2505_17701_b200 import costmodel as cm
    from paper_2505_17701_b200.tp import TPLayer, allreduce_sum_

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, peak_kind = peaks()
    stream = torch.cuda.Stream()
    timer = Timer(torch, stream, dist)

    layer, pred, xcal, xs = workload()
    m_of = lambda k: cd.alive_count_for(k, F)
    z_cal = exact_logits(cd, pred, xcal)
    z_x = exact_logits(cd, pred, xs)

    def tau_dc(k):
        return top_m_tau(z_cal, m_of(k))

    NL = args.layers
    tps = [TPLayer(layer, pred, world, rank, device=local, device_dtype="bf16") for _ in range(NL)]
    devs = [t.dev for t in tps]
    serve_mode(devs)
    if args.prefetch:
        # the replicas run in a fixed rotation: each step L2-prefetches the next one's predictor
        for i, dv in enumerate(devs):
            dv.set_prefetch(devs[(i + 1) % NL])
    x_dev = torch.from_numpy(xs).cuda()
    y_dev = torch.zeros((NL, N_X, D), device="cuda")

    def step_fn(method, tau, comm=True):
        def f(i, cs):
            li, xi = i % NL, i % N_X
            tps[li].forward_local(method, x_dev[xi], y_dev[li, xi], tau, cs)
            if comm and world > 1:
                allreduce_sum_(y_dev[li, xi])
        return f

    rb, re_ = tps[0].rows
    Fl = re_ - rb

    def chain_bytes(method, alive_local):
        return cm.device_bytes(method, D, Fl, R if method == "dc" else 0, int(alive_local), 2)["total_bytes"]

    # ---- headline: DC at k (default 0.9)
    tau = tau_dc(args.k)
    fwd = step_fn(cd._capi.METHOD_DC, tau)
    with torch.cuda.stream(stream):
        for i in range(max(args.warmup, 2 * NL)):
            fwd(i, stream.cuda_stream)
    torch.cuda.synchronize()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    clk = ClockSampler(int(vis[local]) if len(vis) > local and vis[local].strip().isdigit() else local)
    with clk:
        ms_step, n_timed, reps = timer.run(fwd, args.steps, soak_s=0.6)
    launches_per_step = devs[0].last_launches()
    # the same graph in the other launch mode of the persistent kernel, for transparency
    for dv in devs:
        dv.set_engines(pdl_chain=not PDL_CHAIN)
    ms_other, _, _ = timer.run(fwd, args.steps)
    serve_mode(devs)
    launch_mode = {"timed": "pdl_chain" if PDL_CHAIN else "cooperative",
                   "pdl_chain": "CD_ENGINE_PDL_CHAIN: PDL-chained persistent kernel, the bench owns the GPU",
                   "cooperative": "library default: cooperative launch (driver-guaranteed co-residency)",
                   ("cooperative" if PDL_CHAIN else "pdl_chain") + "_us_per_step": round(1e3 * ms_other, 3)}
    value = 1e3 / ms_step
    alive_x = (z_x[:, rb:re_] > np.float32(tau)).sum(axis=1)
    alive_full = (z_x > np.float32(tau)).sum(axis=1)
    realized = 1.0 - float(alive_full.mean()) / F
    bytes_step = float(np.mean([chain_bytes("dc", a) for a in alive_x]))

    # ---- dominant kernel: one launch per step (the fused persistent kernel), so its average
    # launch duration over the timed region is the region time / timed launches; the isolated
    # launch (PDL off, events around it, prologue not overlapped) is kept for reference
    st_iters = 64
    stage_ns = cd.DeviceLayer.bench_stages(devs, cd._capi.METHOD_DC, x_dev[0], tau, 8, st_iters)
    a0 = int(alive_x[0])
    if len(stage_ns) == 1:
        stage_bytes = [chain_bytes("dc", a0)]
        names = ["k_dc_fused"]
    else:
        stage_bytes = [D * R * 2 + 4 * D + 4 * R, Fl * R * 2 + 4 * R + 4 * D, 3 * a0 * D * 2 + 4 * D * 2 + 8 * a0]
        names = ["k_latent_fast", "k_indicator_dc", "k_sparse<DC>"]
    dom = int(np.argmax(stage_ns))
    stages = [{"kernel": n, "us_isolated": ns / 1e3, "alg_bytes": b, "gbs": b / ns}
              for n, ns, b in zip(names, stage_ns, stage_bytes)]
    if len(stage_ns) == 1 and world == 1:
        launch_ns = 1e6 * ms_step
        alg = bytes_step
        roof_how = (f"CUDA events over the timed region: {n_timed} launches of {names[0]} ({reps} replays of a "
                    f"{args.steps}-step graph), 1 per step; alg bytes = mean over the {N_X} inputs' realized "
                    f"active counts")
    else:
        launch_ns = stage_ns[dom]
        alg = stage_bytes[dom]
        roof_how = "per-kernel CUDA events (bench_stages: PDL off, an event after every launch)"
    achieved = alg / launch_ns  # bytes/ns == GB/s
    flips = flip_report(torch, cd, devs[0], cd._capi.METHOD_DC, xs, tau, z_x) if world == 1 else None

    # ---- e2e through the C-ABI with host buffers (rank 0's view)
    e2e = None
    if world == 1:
        from paper_2505_17701_b200._capi import lib, ptr, check
        L = lib()
        yh = np.empty(D, np.float32)
        ah = np.empty(1, np.int64)
        xs_c = [np.ascontiguousarray(x) for x in xs]

        def call(i):
            check(L.cd_pipeline_dc(devs[i % NL].raw, 1, ptr(xs_c[i % N_X]), tau, None, 1, ptr(yh), None, ptr(ah),
                                   None))

        # every rotated handle captures its host graph on its 2nd identical call: warm them all
        for i in range(max(args.warmup, 3 * NL)):
            call(i)
        t0 = time.perf_counter()
        for i in range(64):
            call(i)
        per = (time.perf_counter() - t0) / 64
        n_e2e = max(args.steps, int(np.ceil(0.2 / max(per, 1e-6))))
        t0 = time.perf_counter()
        for i in range(n_e2e):
            call(i)
        dt = time.perf_counter() - t0
        e2e = {"value": round(n_e2e / dt, 1), "unit": "tokens/s", "h2d_bytes_per_step": 4 * D,
               "d2h_bytes_per_step": 4 * D + 4, "calls": n_e2e,
               "timing": "wall clock over back-to-back synchronous C-ABI calls (>= 0.2 s, handles warmed)",
               "api": "cd_pipeline_dc (host buffers)"}

    # ---- all-reduce share (TP)
    comm = None
    if world > 1:
        ms_local, _, _ = timer.run(step_fn(cd._capi.METHOD_DC, tau, comm=False), args.steps)
        comm = {"layer_us": 1e3 * ms_step, "compute_only_us": 1e3 * ms_local,
                "allreduce_share": max(0.0, 1 - ms_local / ms_step), "allreduce_bytes": 4 * D}

    # ---- sparsity sweep (DC 50/70/80/90, MC 70/90, dense 0%)
    sweep = []
    if not args.no_sweep:
        n_sw = max(2 * NL, min(args.steps, 64))
        cases = [("dc", k) for k in (0.5, 0.7, 0.8, 0.9)] + [("mc", 0.7), ("mc", 0.9), ("dense", 0.0)]
        u_cal = u_x = None
        for method, k in cases:
            if method == "mc" and u_cal is None:
                ordc = cd.BlockConfig(reduction=cd.Reduction.DeterministicOrdered)
                u_cal = np.abs(cd.pipeline_mc(layer, xcal, float("inf"), ordc, want_u=True).u)
                u_x = np.abs(cd.pipeline_mc(layer, xs, float("inf"), ordc, want_u=True).u)
            if method == "dc":
                t = tau_dc(k)
                al = (z_x[:, rb:re_] > np.float32(t)).sum(axis=1)
                alf = (z_x > np.float32(t)).sum(axis=1)
                mid = cd._capi.METHOD_DC
            elif method == "mc":
                t = top_m_tau(u_cal, m_of(k))
                al = (u_x[:, rb:re_] > np.float32(t)).sum(axis=1)
                alf = (u_x > np.float32(t)).sum(axis=1)
                mid = cd._capi.METHOD_MC
            else:
                t, al, alf, mid = 0.0, np.full(N_X, Fl), np.full(N_X, F), cd._capi.METHOD_DENSE
            f = step_fn(mid, t)
            with torch.cuda.stream(stream):
                for i in range(2 * NL):
                    f(i, stream.cuda_stream)
            timer.barrier()
            ms_k, nt, _ = timer.run(f, n_sw)
            us = 1e3 * ms_k
            b = float(np.mean([chain_bytes(method, a) for a in al]))
            sweep.append({"method": method, "k": k, "realized_sparsity": round(1 - float(alf.mean()) / F, 4),
                          "tokens_per_s": round(1e3 / us * 1e3, 1), "us_per_token": round(us, 3),
                          "touched_mb_per_rank": round(b / 1e6, 2), "gbs_per_rank": round(b / us / 1e3, 1),
                          "hbm_frac": round(b / us / 1e3 / peak, 4), "timed_steps": nt})
        dense = [s for s in sweep if s["method"] == "dense"]
        dc90 = [s for s in sweep if s["method"] == "dc" and s["k"] == 0.9]
        if dense and dc90:
            sweep.append({"speedup_dc90_vs_dense": round(dense[0]["us_per_token"] / dc90[0]["us_per_token"], 2)})
    del tps, devs
    layer.invalidate()

    extra = {}
    if world == 1 and not args.no_configs:
        extra["gemma"] = gemma_section(torch, cd, timer, min(args.steps, 64), peak)
        extra["f32"] = f32_section(torch, cd, timer, min(args.steps, 64), peak, args.k)
    if world == 1 and not args.no_batched:
        extra["batched"] = batched_section(torch, cd, timer, min(args.steps, 50), peak)
    if not args.no_stack:
        extra["stack"] = stack_section(torch, cd, timer, world, rank, args.steps, peak, args.k)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (reference bench() seeded RNG, seed 42; bf16-rounded)",
            "config": {"workload": f"BASELINE configs[1]: llama3.1-8b FFN layer d={D} d_ff={F} SiLU, D-CountDown "
                                   f"r={R} k={args.k} (tau_D calibrated), batch-1 decode, bf16 weights",
                       "global_batch": 1, "parallelism": f"tp{world} (d_ff)" if world > 1 else "single",
                       "realized_sparsity": round(realized, 4),
                       "l2": f"inputs larger than L2: {NL} layer replicas rotated per step "
                             f"({NL * bytes_step / 1e6:.0f} MB touched per rotation > 126 MB L2)",
                       "graph": f"{args.steps} steps in one CUDA graph ({launches_per_step} kernel(s) per step, " +
                                ("PDL-chained" if PDL_CHAIN else "cooperative launches") +
                                (", + NCCL all-reduce" if world > 1 else "") +
                                f"), replayed {reps}x back to back in the timed region ({n_timed} timed steps)"},
            "timed_steps": n_timed,
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": ncu_traffic(names[dom]), "alg_bytes_per_launch": alg,
                         "launch_us": round(launch_ns / 1e3, 3), "timing": roof_how, "stages": stages,
                         "peak_nominal_gbs": 8000.0, "frac_of_nominal": round(achieved / 8000.0, 4)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * n_timed,
            "launch_mode": launch_mode,
            "clocks": clk.summary(),
            "flips": flips,
            "sweep": sweep,
        }
        line.update(extra)
        if comm:
            line["allreduce"] = comm
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    global PDL_CHAIN
    PDL_CHAIN = not args.cooperative
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
