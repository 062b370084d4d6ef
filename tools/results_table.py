"""README results table from a default bench line: python tools/results_table.py <bench.json>"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
rows = []
rows.append(("c2 `[784,30,10]` B=1000 (default bench)",
             f"{d['value'] / 1e6:.1f} M samples/s ({d['ms_per_step'] * 1e3:.2f} us/step); e2e from host "
             f"{d['e2e']['value'] / 1e6:.1f} M/s (PCIe-bound)",
             f"{100 * d['roofline']['frac']:.1f} % of HBM (latency-bound: one GPU-wide co_sum + barrier per step; DESIGN.md §6)"))
inf = d["inference"]
rows.append(("c2 inference (`nf_output`)", f"{inf['value'] / 1e6:.0f} M samples/s ({inf['hbm_gbs'] / 1e3:.2f} TB/s)",
             f"{100 * inf['hbm_frac']:.0f} % of HBM"))
names = {"c5": "c5 `[4096x4, 1024]` B=16384", "c3": "c3 `[784,1024,1024,10]` B=4096", "c4": "c4 `[784,256x8,10]` B=2048"}
for k, v in d["configs"].items():
    c, m = k.split("-")[0], "-".join(k.split("-")[1:])
    r = v["roofline"]
    mode = {"tf32": "TF32 tiles", "fp32": "fp32 (3xTF32)", "tf32-dp": "TF32, data-parallel step on a 1-rank NCCL group"}[m]
    rows.append((f"{names[c]}, {mode}", f"{v['value'] / 1e6:.2f} M samples/s ({v['ms_per_step'] * 1e3:.1f} us/step, "
                 f"{r['achieved']:.0f} TFLOP/s useful)", f"{100 * r['frac']:.1f} % of the burst TF32 peak"))
print("| Config | Training | Roofline |\n|---|---|---|")
for a, b, c in rows:
    print(f"| {a} | {b} | {c} |")
print(f"\ncpu oracle: {d['cpu_baseline']['value'] / 1e3:.1f} k samples/s ({d['cpu_baseline']['cores']} core)")
