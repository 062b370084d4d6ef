"""Sweep the K6 decomposition (cluster size C, cluster count G) on config 2: us/step."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
import synth, paper_1902_06714_b200 as nf
cfg = synth.CONFIGS[2]
X, Y = synth.dataset(2)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
net = nf.Net(cfg["dims"], cfg["act"])
net.set_params(torch.from_numpy(synth.init_params(2)).cuda())
st = synth.batch_starts(2, steps=300)
net.train_steps(Xd, Yd, 1000, st[:50], 3.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record(); net.train_steps(Xd, Yd, 1000, st, 3.0); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / len(st) * 1e3)
print(sorted(ts)[2])
'''
grid = [(8, [15, 12]), (4, [33, 30]), (6, [22])]
if len(sys.argv) > 1 and sys.argv[1] == "2cta":
    grid = [(8, [30, 36, 24]), (4, [60, 66, 50]), (2, [120])]
for C, Gs in grid:
    for G in Gs:
        env = dict(os.environ, ROOT=ROOT, NF_FUSED_C=str(C), NF_FUSED_G=str(G))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        print(f"C={C} G={G}: {r.stdout.strip() or r.stderr.strip()[-200:]} us/step", flush=True)
