"""DRAM traffic of ONE warm SGD step (all kernels of nf_train_batch) for a config, for the
bench's roofline `traffic` key when the roofline covers the whole step (c3-c5).
Run under ncu with the profiler range (only the bracketed step is captured):
  ncu --profile-from-start off --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      --log-file gpurun_out/steps.csv python tools/step_traffic.py 3,4,5 tf32
then: python tools/step_traffic.py --sum gpurun_out/steps.csv
Each config's step is preceded, inside the captured range, by one torch fill kernel that
separates the configs in the launch list."""
import csv
import os
import sys
from collections import defaultdict


def summarise(path):
    rows = list(csv.DictReader(line for line in open(path) if line.startswith('"')))
    groups, cur = [], None
    for r in rows:
        if "FillFunctor" in r["Kernel Name"]:
            if r["Metric Name"] == "gpu__time_duration.sum":
                cur = []
                groups.append(cur)
            continue
        cur.append(r)
    for g in groups:
        summarise_group(g)


def summarise_group(rows):
    per = defaultdict(lambda: [0, 0.0, 0.0])   # launches, bytes, us
    tot_b = tot_t = 0.0
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        k = r["Kernel Name"].split("(")[0][:90]
        if r["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[unit]
            per[k][1] += v
            tot_b += v
        elif r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[unit]
            per[k][0] += 1
            per[k][2] += v
            tot_t += v
    for k, (n, b, t) in sorted(per.items(), key=lambda kv: -kv[1][2]):
        print(f"{n:3d} x {t:10.1f} us {b / 1e6:10.1f} MB  {k}")
    print(f"{len(rows) // 3} launches; step total: {tot_t:.1f} us (cold-cache, serialised), {tot_b / 1e6:.1f} MB DRAM "
          f"(read + write) -> bytes_per_step {int(tot_b)}")


def main():
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import synth
    import paper_1902_06714_b200 as nf

    math = {"tf32": nf.NF_MATH_TF32, "fp32": nf.NF_MATH_FP32}[sys.argv[2] if len(sys.argv) > 2 else "tf32"]
    for cid in [int(c) for c in sys.argv[1].split(",")]:
        one_step(torch, synth, nf, cid, math)


def one_step(torch, synth, nf, cid, math):
    cfg = synth.CONFIGS[cid]
    B = cfg["batch"]
    X, Y = synth.dataset(cid, N=B)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    net = nf.Net(cfg["dims"], cfg["act"])
    net.set_math(math)
    net.set_params(torch.from_numpy(synth.init_params(cid)).cuda())
    for _ in range(3):
        net.train_batch(Xd, Yd, cfg["eta"])
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    torch.zeros(1, device="cuda")       # separator
    net.train_batch(Xd, Yd, cfg["eta"])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    if sys.argv[1] == "--sum":
        summarise(sys.argv[2])
    else:
        main()
