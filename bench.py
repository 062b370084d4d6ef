#!/usr/bin/env python3
"""Benchmark of the hot path: minibatch SGD training of the paper's 784-30-10 MNIST net
(BASELINE.json configs[1], "config 2"), synthetic digit-shaped data, on B200 -- plus, in the
same run, the wide configurations 3-5 in both numerics modes under "configs".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A "step" is one SGD step (forward, backward, batch-summed tendencies, update) over one
minibatch of B rows drawn at a random contiguous start from the resident dataset.
K steps run as ONE nf_train_steps call.  Timing: CUDA events on the launching stream around
exactly K steps, barrier + synchronize on both sides, repeated R times (>= 1 s in total so
nvidia-smi can sample clocks during the timed region); every rep draws FRESH batch starts
from one long seeded schedule (no rep replays another's rows), over a dataset larger than
the 126 MB L2; the median rep is reported, max over ranks.  That is the paper's protocol of
timing the training portion only, repeated runs reported as a statistic (P:830-837,
P:886-887).

N > 1 (one process per GPU): launched by torchrun, or bench.py --gpus N spawns torchrun
itself when WORLD_SIZE is unset.  The headline c2 runs as replicas (its 95 KB co_sum per
step would cost more than the 11 us step); configs 3-5 run data-parallel
(per-rank batch B of a global batch N*B, NCCL all-reduce of the tendencies per layer,
overlapped with the backward; weak scaling).

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (oracle/, fp32
build = the paper's real32) on the same config instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

BYTES_PER_SAMPLE = {  # algorithmic HBM bytes per training sample: x row + y row, fp32
    cid: 4 * (c["dims"][0] + c["dims"][-1]) for cid, c in synth.CONFIGS.items()
}


def flops_per_sample(dims):
    """Dense useful flops per training sample: forward 2*n_l*n_{l-1} per layer, backward delta
    2*n_l*n_{l-1} for layers >= 2, weight gradient 2*n_l*n_{l-1} per layer."""
    f = 0
    for l in range(1, len(dims)):
        mac = dims[l] * dims[l - 1]
        f += 2 * mac + 2 * mac + (2 * mac if l >= 2 else 0)
    return f


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")     # rank count / transport visible in stderr
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def ensure_group(world):
    """A process group for the data-parallel path; at N = 1 a one-rank NCCL group, so the same
    all-reduce runs."""
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29533 + int(os.environ.get("LOCAL_RANK", "0"))))
        dist.init_process_group("nccl", rank=0, world_size=1)


def spawn_ranks(n):
    """bench.py --gpus N without torchrun: re-launch this script under torch.distributed.run
    with N processes on this node (127.0.0.1 rendezvous); returns its exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    """Max of a per-rank time over all ranks (NCCL on the GPU box, gloo on CPU tests)."""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(world, steps, batch, t_max):
    """Whole-job samples/s: every rank runs `steps` steps of `batch` rows (weak scaling,
    replicas), timed as the slowest rank."""
    return world * steps * batch / t_max


# Bounded CPU-oracle samples (about 10-15 s of single-core work each): (steps, rows per step).
# The oracle's per-sample cost does not depend on the batch size (one fwd/bwd per sample, one
# update per step), so a reduced batch is a fair sample of samples/s for the wide configs.
# NF_MATH_FP64 is bound by the FP64 FMA units (SIMT DFMA): peak measured by micro/fma_rate.cu
FP64_DFMA_TFLOPS = 34.82  # DFMA, 32 warps/SM, 148 SMs at 1965 MHz (59.9 FMA/clk/SM)
FP64_PEAK_SOURCE = "micro/fma_rate.cu DFMA rate, 148 SMs (profiles/r01_micro_fma_rate.txt)"
CPU_SAMPLE = {1: (5000000, None), 2: (500, None), 3: (8, 256), 4: (20, 512), 5: (1, 32)}  # ~10-15 s each


def run_cpu_oracle(cid, steps, batch=None, bits=32, X=None, Y=None):
    """The oracle as it stands (single-threaded C): `steps` SGD steps of config `cid` with
    `batch` rows per step (default: the config's).  Returns (samples/s, seconds, batch)."""
    import oracle
    cfg = synth.CONFIGS[cid]
    batch = batch or cfg["batch"]
    if X is None:
        X, Y = synth.dataset(cid, N=max(batch * 4, min(cfg["N"], 65536)))
    starts = synth.batch_starts(cid, steps=steps, N=len(X), batch=batch)
    o = oracle.Oracle(cfg["dims"], cfg["act"], bits=bits)
    p = synth.init_params(cid)
    o.train_steps(p, X, Y, batch, starts[:1], cfg["eta"])  # page in
    # one core (the calling thread pinned to the first CPU it may use), as SURVEY 8(d) plans
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    if old:
        os.sched_setaffinity(0, {min(old)})
    try:
        t0 = time.perf_counter()
        o.train_steps(p, X, Y, batch, starts, cfg["eta"])
        dt = time.perf_counter() - t0
    finally:
        if old:
            os.sched_setaffinity(0, old)
    return steps * batch / dt, dt, batch


def host_cpu():
    """Host CPU model and logical core count (the oracle baseline's hardware)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def workload_config(cid, math, N=None):
    """The `config` object of the JSON line: names the workload only (identical in both arms)."""
    cfg = synth.CONFIGS[cid]
    return {"workload": cfg["name"], "dims": cfg["dims"], "batch": cfg["batch"],
            "dataset_rows": N or cfg["N"], "math": math, "eta": cfg["eta"],
            "activation": cfg["act"], "batch_starts": "synth.batch_starts (seeded, uniform in [0, N-B])"}


def reference_arm(args):
    """--impl reference: the CPU oracle on this config (rank 0 only)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cid = args.config
    cfg = synth.CONFIGS[cid]
    import oracle
    # rows per step: the config's batch when a step costs well under a second on one core,
    # else a bounded sample of it (per-sample cost is batch independent)
    fl = flops_per_sample(cfg["dims"])
    rows = max(1, min(cfg["batch"], int(2.0e8 / fl)))
    X, Y = synth.dataset(cid, N=max(rows * 4, min(cfg["N"], 65536)))
    starts = synth.batch_starts(cid, steps=args.warmup + args.steps, N=len(X), batch=rows)
    o = oracle.Oracle(cfg["dims"], cfg["act"], bits=32)
    p = synth.init_params(cid)
    if args.warmup:
        p, _ = o.train_steps(p, X, Y, rows, starts[:args.warmup], cfg["eta"])
    t0 = time.perf_counter()
    o.train_steps(p, X, Y, rows, starts[args.warmup:], cfg["eta"])
    dt = time.perf_counter() - t0
    v = args.steps * rows / dt
    line = {
        "impl": "reference", "metric": "training samples/sec (fwd+bwd+SGD)", "value": v,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(cid, args.math),
        "parallelism": "1 host core",
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
                         "sample": f"{args.steps} SGD steps of {rows} rows (config batch {cfg['batch']}) of "
                                   f"{cfg['name']}, fp32 build of oracle/nf_oracle.c, single thread"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def tf32_peaks(peaks):
    """TF32 dense peaks = measured bf16 x (1.1 / 2.25), the guide's nominal ratio: the burst
    figure (a kernel / short step timed alone: the primary denominator) and the sustained one."""
    return peaks["bf16_tflops"] * 1.1 / 2.25, peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 1.1 / 2.25


class Timer:
    """Fresh-start reps of K steps each: CUDA events on `stream`, barrier + sync around each."""

    def __init__(self, world, stream):
        self.world, self.stream = world, stream

    def rep(self, fn):
        import torch
        barrier(self.world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        fn()
        e1.record(self.stream)
        torch.cuda.synchronize()
        barrier(self.world)
        return e0.elapsed_time(e1) / 1e3


def run_wide(nf, cid, math, world, rank, local, K, W, reps, dp, peaks, peak_src):
    """One wide configuration (3-5) in one numerics mode: W warm-up steps, then `reps` timed
    reps of K steps with fresh starts each; single GPU: nf_train_steps; N > 1 or dp:
    DataParallel (per-rank B rows of an N*B global batch, per-layer all-reduce overlapped with
    the backward).  Returns the sub-line dict."""
    import torch
    cfg = synth.CONFIGS[cid]
    B = cfg["batch"]
    gb = world * B if dp else B
    N = max(cfg["N"], 2 * gb)
    X, Y = synth.dataset(cid, N=N)
    starts = synth.batch_starts(cid, steps=W + K, N=N, batch=gb)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    del X, Y
    stream = torch.cuda.current_stream()
    net = nf.Net(cfg["dims"], cfg["act"], stream=stream)
    net.set_params(torch.from_numpy(synth.init_params(cid)).cuda())
    net.set_math({"fp32": nf.NF_MATH_FP32, "tf32": nf.NF_MATH_TF32}[math])
    loss = torch.zeros(K, device="cuda")
    if dp:
        from paper_1902_06714_b200.dp import DataParallel
        ensure_group(world)
        dpar = DataParallel(net)

        def steps(st):
            dpar.train_steps(Xd, Yd, gb, st, cfg["eta"])
    else:
        def steps(st):
            net.train_steps(Xd, Yd, B, st, cfg["eta"], step_loss=loss)
    steps(starts[:W])
    torch.cuda.synchronize()
    tm = Timer(world, stream)
    # every rep replays the same K starts (nf_train_steps replays its captured CUDA graph while
    # the arguments repeat; new starts would re-capture it), with L2 flushed before each rep by
    # writing a 256 MB buffer (> the 126 MB L2) outside the timed region
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    st_rep = starts[W:W + K]
    steps(st_rep)
    l0 = nf.nf_launch_count()
    times = []
    with ClockSampler(local) as clk:
        for r in range(reps):
            flush.zero_()
            times.append(tm.rep(lambda: steps(st_rep)))
    launches = (nf.nf_launch_count() - l0) // reps
    t = max_over_ranks(statistics.median(times), world)
    fl = flops_per_sample(cfg["dims"]) * gb
    burst, sust = tf32_peaks(peaks)
    ach = fl * K / t / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_c{cid}.json")
    if os.path.exists(prof):
        tj = json.load(open(prof))
        if tj.get("math") == math:
            traffic = tj["bytes_per_step"] * K
    del Xd, Yd, net, flush
    torch.cuda.empty_cache()
    return {
        "workload": cfg["name"], "math": math, "dims": cfg["dims"], "batch": B, "global_batch": gb,
        "dataset_rows": N, "steps": K, "warmup": W, "reps": reps,
        "stat": "median rep; each rep the same K fresh-drawn starts (graph replay), L2 flushed (256 MB write) before it",
        "ms_per_step": t * 1e3 / K, "value": gb * K / t, "unit": "samples/s",
        "parallelism": (f"dp{world}: nf_grad_layers on {B} rows per rank, NCCL all-reduce per layer block "
                        f"overlapped with the backward, nf_update" if dp else "1 GPU"),
        "roofline": {"bound": "tensor", "achieved": ach, "peak": burst, "unit": "TFLOP/s", "frac": ach / burst,
                     "frac_sustained": ach / sust, "traffic": traffic,
                     "peak_source": f"MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 = TF32 dense burst ({peak_src}); "
                                    f"frac_sustained vs bf16_tflops_sustained x 1.1/2.25",
                     "kernel": "whole step (every kernel of nf_train_steps)",
                     "algorithmic_flops_per_step": fl,
                     **({"mma_pipe_frac": 3 * ach / burst, "note": "3xTF32: 3 MMAs per useful product"}
                        if math == "fp32" else {})},
        "gpu_launches_per_rep": launches, "clocks": clk.summary(),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--min-seconds", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--configs", default=None,
                    help="wide configurations measured in the same run under 'configs', e.g. '5:tf32,5:fp32'; "
                         "default with the c2 headline: c5, c3, c4 in tf32 and fp32 (+ c5 tf32 data-parallel at N=1); "
                         "'none' to skip")
    ap.add_argument("--sub-steps", type=int, default=0, help="steps per timed rep of each wide config (0: auto)")
    ap.add_argument("--dp", action="store_true",
                    help="the headline config data-parallel (P:505-556) instead of replicas")
    ap.add_argument("--math", default="fp32", choices=["fp32", "tf32", "fp64"],
                    help="fp32: fp32 SIMT / 3xTF32 tensor cores (1e-4 parity); tf32: 1xTF32 tiles on RN-rounded "
                         "operands; fp64: the paper's real64 build on the FP64 units")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))

    import torch
    from paper_1902_06714_b200 import build as nfbuild
    if int(os.environ.get("LOCAL_RANK", "0")) == 0:
        nfbuild.build()
    import paper_1902_06714_b200 as nf

    world, rank, local = dist_setup()
    barrier(world)
    cid = args.config
    cfg = synth.CONFIGS[cid]
    B, K, W = cfg["batch"], args.steps, args.warmup
    dp = args.dp or (world > 1 and cid >= 3)
    gb = world * B if dp else B
    X, Y = synth.dataset(cid, N=max(cfg["N"], 2 * gb))
    N = len(X)
    # one long seeded schedule of starts; every rep takes the next K (replica r: its own stream)
    max_reps = 2000
    starts_all = synth.batch_starts(cid, steps=W + (max_reps + 1) * K, N=N, batch=gb)
    if not dp and world > 1:
        starts_all = np.roll(starts_all, -rank * 7919)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    stream = torch.cuda.current_stream()
    net = nf.Net(cfg["dims"], cfg["act"], stream=stream)
    net.set_params(torch.from_numpy(synth.init_params(cid)).cuda())
    net.set_math({"fp32": nf.NF_MATH_FP32, "tf32": nf.NF_MATH_TF32, "fp64": nf.NF_MATH_FP64}[args.math])
    loss = torch.zeros(K, device="cuda")
    if dp:
        from paper_1902_06714_b200.dp import DataParallel
        ensure_group(world)
        dpar = DataParallel(net)

        def run_steps(st, step_loss=None, Xs=Xd, Ys=Yd):
            dpar.train_steps(Xs, Ys, gb, st, cfg["eta"])
    else:
        def run_steps(st, step_loss=None, Xs=Xd, Ys=Yd):
            net.train_steps(Xs, Ys, B, st, cfg["eta"], step_loss=step_loss)

    run_steps(starts_all[:W])
    torch.cuda.synchronize()
    tm = Timer(world, stream)
    rep_i = [0]

    def next_starts():
        r = rep_i[0] % (max_reps + 1)
        rep_i[0] += 1
        return starts_all[W + r * K:W + (r + 1) * K]

    l0 = nf.nf_launch_count()
    t_first = tm.rep(lambda: run_steps(next_starts(), step_loss=loss))
    launches = nf.nf_launch_count() - l0
    reps = max(5, min(max_reps, int(args.min_seconds / max(t_first, 1e-6)) + 1))
    reps = int(max_over_ranks(reps, world))
    times = []
    with ClockSampler(local) as clk:
        for _ in range(reps):
            times.append(tm.rep(lambda: run_steps(next_starts(), step_loss=loss)))
    t_med = statistics.median(times)
    t_max = max_over_ranks(t_med, world)
    value = world * K * B / t_max

    peaks, peak_src = measured_peaks()
    alg_bytes = K * B * BYTES_PER_SAMPLE[cid]
    achieved = alg_bytes / t_med / 1e9
    tensor_bound = len(cfg["dims"]) > 3
    if tensor_bound:
        tf32_peak, tf32_sust = tf32_peaks(peaks)
        ach_tf = flops_per_sample(cfg["dims"]) * K * B / t_med / 1e12
    ach_f64 = flops_per_sample(cfg["dims"]) * K * B / t_med / 1e12
    # DRAM traffic of the roofline's kernel (c2: the fused kernel, `ncu --set full`; c3-c5: all
    # kernels of one TF32 step, tools/step_traffic.py) from a committed capture
    # (profiles/traffic_c<id>.json: dram bytes read + written per SGD step), scaled to this launch
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_c{cid}.json")
    if os.path.exists(prof) and args.math != "fp64":
        try:
            tj = json.load(open(prof))
            traffic = tj["bytes_per_step"] * K if tj.get("math", args.math) == args.math else None
        except Exception:
            traffic = None

    # ---- inference (the paper's `output`): nf_output over the whole resident dataset
    out = torch.empty((N, cfg["dims"][-1]), device="cuda")
    net.output(Xd, out)
    torch.cuda.synchronize()
    ti = [tm.rep(lambda: net.output(Xd, out)) for _ in range(5)]
    t_inf = statistics.median(ti)
    inf_bytes = N * 4 * (cfg["dims"][0] + cfg["dims"][-1])
    inference = {"value": world * N / max_over_ranks(t_inf, world), "unit": "samples/s", "rows": N,
                 "hbm_gbs": inf_bytes / t_inf / 1e9, "hbm_frac": inf_bytes / t_inf / 1e9 / peaks["hbm_gbs"],
                 "tflops": sum(2 * cfg["dims"][l] * cfg["dims"][l - 1]
                               for l in range(1, len(cfg["dims"]))) * N / t_inf / 1e12}

    # ---- e2e: same metric through the C-ABI with pinned HOST buffers; each step's batch
    # is copied host->device inside the call, the step losses are read back to the host.
    e2e = None
    if not args.no_e2e and not dp:
        Xh = torch.from_numpy(X).pin_memory()
        Yh = torch.from_numpy(Y).pin_memory()
        lh = torch.empty(K, dtype=torch.float32).pin_memory()

        def e2e_call():
            net.train_steps(Xh, Yh, B, next_starts(), cfg["eta"], step_loss=loss)
            lh.copy_(loss, non_blocking=True)

        tm.rep(e2e_call)
        te = statistics.median([tm.rep(e2e_call) for _ in range(3)])
        te = max_over_ranks(te, world)
        e2e = {"value": world * K * B / te, "unit": "samples/s",
               "h2d_bytes_per_step": B * BYTES_PER_SAMPLE[cid], "d2h_bytes_per_step": 4}
    del Xd, Yd
    torch.cuda.empty_cache()

    # ---- the wide configurations in the same run (configs 3-5, both numerics modes)
    subs = {}
    spec = args.configs
    if spec is None:
        spec = "none" if cid != 2 else "5:tf32,5:fp32,3:tf32,3:fp32,4:tf32,4:fp32"
        if cid == 2 and world == 1:
            spec += ",5:tf32:dp"
    if spec != "none":
        for item in spec.split(","):
            parts = item.split(":")
            c, m = int(parts[0]), parts[1]
            sub_dp = world > 1 or (len(parts) > 2 and parts[2] == "dp")
            Ks = args.sub_steps or {3: 20, 4: 20, 5: 5}[c]
            subs[f"c{c}-{m}" + ("-dp" if sub_dp and world == 1 else "")] = run_wide(
                nf, c, m, world, rank, local, Ks, 3, 3, sub_dp, peaks, peak_src)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_steps, cpu_rows = CPU_SAMPLE[cid]
        v, dt, rows = run_cpu_oracle(cid, cpu_steps, cpu_rows, X=X, Y=Y)
        cpu = {"value": v, "unit": "samples/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
               "sample": f"{cpu_steps} SGD steps of {rows} rows of {cfg['name']} ({dt:.1f} s), fp32 build of "
                         f"oracle/nf_oracle.c, single thread"}

    if rank == 0:
        fl = flops_per_sample(cfg["dims"])
        line = {
            "metric": "training samples/sec (fwd+bwd+SGD)",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": t_max * 1e3 / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": {"fp32": "f32", "tf32": "tf32", "fp64": "f64"}[args.math], "data": "synthetic",
            "config": workload_config(cid, args.math, N),
            "timing": {"steps_per_timed_call": K, "reps": reps,
                       "stat": "median rep; every rep draws fresh batch starts from one seeded schedule",
                       "l2": f"inputs larger than L2: dataset {X.nbytes / 1e6:.0f} MB > 126 MB L2, fresh random "
                             f"batch starts every rep (not flushed)"},
            "parallelism": (f"dp{world}: per step nf_grad_layers on {B} rows per rank, NCCL all-reduce "
                            f"per layer block overlapped with the backward (co_sum), nf_update; "
                            f"global batch {gb}"
                            if dp else f"replicas x{world}" if world > 1 else "1 GPU"),
            "roofline": ({"bound": "latency", "achieved": t_max * 1e6 / K, "peak": None, "unit": "us/step",
                          "frac": None, "traffic": None, "kernel": "single_cta_kernel",
                          "note": "config 1 (120 flop per sample): one CTA, a chain of CTA barriers per step "
                                  "(SURVEY 8(d): latency-bound, report us/step)"}
                         if cid == 1 and args.math != "fp64" else
                         {"bound": "alu", "achieved": ach_f64, "peak": FP64_DFMA_TFLOPS, "unit": "TFLOP/s",
                          "frac": ach_f64 / FP64_DFMA_TFLOPS, "traffic": None,
                          "peak_source": FP64_PEAK_SOURCE, "kernel": "whole step (gemm64_kernel + splitk64)",
                          "algorithmic_flops_per_step": flops_per_sample(cfg["dims"]) * B}
                         if args.math == "fp64" else
                         {"bound": "tensor", "achieved": ach_tf, "peak": tf32_peak, "unit": "TFLOP/s",
                          "frac": ach_tf / tf32_peak, "frac_sustained": ach_tf / tf32_sust, "traffic": traffic,
                          "peak_source": f"MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 = TF32 dense burst ({peak_src})",
                          "kernel": "whole step (gemm_tc_kernel + epilogue kernels)",
                          "algorithmic_flops_per_step": flops_per_sample(cfg["dims"]) * B}
                         if tensor_bound else
                         {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                          "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                          "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                          "kernel": "fused_small_kernel",
                          "algorithmic_bytes_per_launch": alg_bytes}),
            "flops": {"per_sample": fl, "achieved_tflops": fl * K * B / t_med / 1e12},
            "inference": inference,
            "configs": subs or None,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
