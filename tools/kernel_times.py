"""Warm per-kernel device times of the training step (torch.profiler / CUPTI activity records;
kernels run back to back as in the bench, unlike ncu's serialised cold-cache replays).
A kernel's duration includes its PDL wait (it launches while its predecessor runs) and the
side-stream backward overlaps the main stream, so the per-kernel times sum to more than the
step.  Usage: python tools/kernel_times.py 3,4,5 [tf32|fp32] [steps]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402


def run(cid, math, steps):
    cfg = synth.CONFIGS[cid]
    B = cfg["batch"]
    X, Y = synth.dataset(cid, N=B)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    net = nf.Net(cfg["dims"], cfg["act"])
    net.set_math(math)
    net.set_params(torch.from_numpy(synth.init_params(cid)).cuda())
    for _ in range(5):
        net.train_batch(Xd, Yd, cfg["eta"])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        net.train_batch(Xd, Yd, cfg["eta"])
    e1.record()
    torch.cuda.synchronize()
    step_us = e0.elapsed_time(e1) * 1e3 / steps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            net.train_batch(Xd, Yd, cfg["eta"])
        torch.cuda.synchronize()
    per = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.replace("(anonymous namespace)::", "").split("(")[0][:80]
            per[k][0] += 1
            per[k][1] += ev.device_time
    tot = sum(t for _, t in per.values())
    print(f"c{cid} {sys.argv[2] if len(sys.argv) > 2 else 'tf32'}: {step_us:.1f} us/step (events, unprofiled); "
          f"kernel time {tot / steps:.1f} us/step")
    for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"  {n / steps:5.1f} x/step {t / steps:9.1f} us/step  {100 * t / tot:5.1f} %  {k}")


if __name__ == "__main__":
    math = nf.NF_MATH_FP32 if (len(sys.argv) > 2 and sys.argv[2] == "fp32") else nf.NF_MATH_TF32
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    for c in sys.argv[1].split(","):
        run(int(c), math, steps)
