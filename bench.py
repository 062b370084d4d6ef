#!/usr/bin/env python3
"""Benchmark of the hot path: minibatch SGD training of the paper's 784-30-10 MNIST net
(BASELINE.json configs[1], "config 2"), synthetic digit-shaped data, on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A "step" is one SGD step (forward, backward, batch-summed tendencies, update) over one
minibatch of B=1000 rows drawn at a random contiguous start from the resident 50000-row
dataset.  K steps run as ONE nf_train_steps call (the fused persistent kernel
for this config).  Timing: CUDA events on the launching stream around exactly K steps,
barrier + synchronize on both sides, repeated R times (>= 1 s in total so nvidia-smi can
sample clocks during the timed region); the median rep is reported, max over ranks.
The dataset (157 MB) is larger than L2 (126 MB); L2 is not flushed between reps.

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


def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


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
        "config": {"workload": cfg["name"], "dims": cfg["dims"], "batch": cfg["batch"]},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
                         "sample": f"{args.steps} SGD steps of {rows} rows (config batch {cfg['batch']}) of "
                                   f"{cfg['name']}, fp32 build of oracle/nf_oracle.c, single thread"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--dp", action="store_true",
                    help="true data parallelism (P:505-556): every step, each rank's tendencies over its "
                         "B rows of a world*B global batch, NCCL all-reduce (co_sum), nf_update; default: "
                         "independent replicas (no collective)")
    ap.add_argument("--math", default="fp32", choices=["fp32", "tf32", "fp64"],
                    help="fp32: fp32 SIMT / 3xTF32 tensor cores (1e-4 parity); tf32: 1xTF32 tiles; "
                         "fp64: the paper's real64 build on the FP64 units")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    from paper_1902_06714_b200 import build as nfbuild
    nfbuild.build()
    import paper_1902_06714_b200 as nf

    world, rank, local = dist_setup(args.gpus)
    cid = args.config
    cfg = synth.CONFIGS[cid]
    B, K, W = cfg["batch"], args.steps, args.warmup
    X, Y = synth.dataset(cid)
    N = len(X)
    # --dp: the global batch of a step is world * B rows, rank r owns the r-th block of B
    starts = synth.batch_starts(cid, steps=W + K, N=N - ((world - 1) * B if args.dp else 0))
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    stream = torch.cuda.current_stream()
    net = nf.Net(cfg["dims"], cfg["act"], stream=stream)
    net.set_params(torch.from_numpy(synth.init_params(cid)).cuda())
    net.set_math({"fp32": nf.NF_MATH_FP32, "tf32": nf.NF_MATH_TF32, "fp64": nf.NF_MATH_FP64}[args.math])
    loss = torch.zeros(K, device="cuda")
    if args.dp:
        from paper_1902_06714_b200.dp import DataParallel
        if world == 1:   # a one-rank NCCL group, so the all-reduce runs at N = 1 too
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1)
        dp = DataParallel(net)

        def run_steps(st, step_loss=None, Xs=Xd, Ys=Yd):
            dp.train_steps(Xs, Ys, world * B, st, cfg["eta"])
    else:
        def run_steps(st, step_loss=None, Xs=Xd, Ys=Yd):
            net.train_steps(Xs, Ys, B, st, cfg["eta"], step_loss=step_loss)

    # warm-up (W untimed steps)
    run_steps(starts[:W])
    torch.cuda.synchronize()

    def timed_rep():
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_steps(starts[W:], step_loss=loss)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        return e0.elapsed_time(e1) / 1e3

    l0 = nf.nf_launch_count()
    t_first = timed_rep()
    launches = nf.nf_launch_count() - l0
    reps = max(5, min(2000, int(args.min_seconds / max(t_first, 1e-6)) + 1))
    times = []
    with ClockSampler(local) as clk:
        for _ in range(reps):
            times.append(timed_rep())
    t_med = statistics.median(times)
    t_max = max_over_ranks(t_med, world)
    value = job_throughput(world, K, B, t_max)

    peaks, peak_src = measured_peaks()
    alg_bytes = K * B * BYTES_PER_SAMPLE[cid]
    achieved = alg_bytes / t_med / 1e9
    tensor_bound = len(cfg["dims"]) > 3
    if tensor_bound:
        # TF32 dense peak = measured bf16 x (1.1 / 2.25), the guide's nominal ratio.  The
        # profiling recipe: the burst figure for a kernel timed alone, the sustained one for
        # kernels under sustained load.  Which one applies is read off this run's clocks: the
        # sustained figure when the SM clock under load sat below max (power cap: c5 runs at
        # ~1.55 GHz), the burst one when it held the maximum clock (c3, c4).
        ck = clk.summary()
        sustained = ("bf16_tflops_sustained" in peaks and ck.get("sm_mhz") and ck.get("sm_max_mhz")
                     and ck["sm_mhz"] < 0.95 * ck["sm_max_mhz"])
        bf16 = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
        tf32_peak = bf16 * 1.1 / 2.25
        tf32_burst = peaks["bf16_tflops"] * 1.1 / 2.25
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
    ti = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        net.output(Xd, out)
        e1.record(stream)
        torch.cuda.synchronize()
        ti.append(e0.elapsed_time(e1) / 1e3)
    t_inf = statistics.median(ti)
    inf_bytes = N * 4 * (cfg["dims"][0] + cfg["dims"][-1])
    inference = {"value": world * N / max_over_ranks(t_inf, world), "unit": "samples/s", "rows": N,
                 "hbm_gbs": inf_bytes / t_inf / 1e9, "hbm_frac": inf_bytes / t_inf / 1e9 / peaks["hbm_gbs"],
                 "tflops": sum(2 * cfg["dims"][l] * cfg["dims"][l - 1]
                               for l in range(1, len(cfg["dims"]))) * N / t_inf / 1e12}

    # ---- e2e: same metric through the C-ABI with pinned HOST buffers; each step's batch
    # is copied host->device inside the call, the step losses are read back to the host.
    e2e = None
    if not args.no_e2e and not args.dp:
        Xh = torch.from_numpy(X).pin_memory()
        Yh = torch.from_numpy(Y).pin_memory()
        lh = torch.empty(K, dtype=torch.float32).pin_memory()

        def e2e_rep():
            barrier(world)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            net.train_steps(Xh, Yh, B, starts[W:], cfg["eta"], step_loss=loss)
            lh.copy_(loss, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier(world)
            return e0.elapsed_time(e1) / 1e3

        e2e_rep()
        te = statistics.median([e2e_rep() for _ in range(3)])
        te = max_over_ranks(te, world)
        e2e = {"value": world * K * B / te, "unit": "samples/s",
               "h2d_bytes_per_step": B * BYTES_PER_SAMPLE[cid], "d2h_bytes_per_step": 4}

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
            "config": {"workload": cfg["name"], "dims": cfg["dims"], "batch": B, "dataset_rows": N,
                       "math": args.math,
                       "eta": cfg["eta"], "steps_per_timed_call": K, "reps": reps, "stat": "median rep",
                       "l2": f"dataset {X.nbytes / 1e6:.0f} MB > 126 MB L2, not flushed",
                       "parallelism": (f"dp{world}: per step nf_grad on {B} rows per rank, NCCL all-reduce "
                                       f"of the tendencies (co_sum), nf_update; global batch {world * B}"
                                       if args.dp else f"replicas x{world}" if world > 1 else "1 GPU")},
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
                          "frac": ach_tf / tf32_peak, "traffic": traffic,
                          "peak_source": (f"MEASURED_PEAKS.json bf16_tflops{'_sustained' if sustained else ''}"
                                          f" x 1.1/2.25 = TF32 dense, {'sustained: SM clock under load below max (power cap)' if sustained else 'burst: SM clock at max'}"
                                          f" ({peak_src})"),
                          "frac_vs_burst_peak": ach_tf / tf32_burst,
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
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1 or args.dp:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
