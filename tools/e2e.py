"""End-to-end c2 training from pinned host memory (nf_train_steps, per-step H2D copies):
samples/s over 500 steps, median of 5 (CUDA events on the net's stream)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402

cfg = synth.CONFIGS[2]
X, Y = synth.dataset(2)
Xh, Yh = torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory()
starts = synth.batch_starts(2, steps=500, N=len(X))
net = nf.Net(cfg["dims"], cfg["act"])
net.set_params(torch.from_numpy(synth.init_params(2)).cuda())
net.train_steps(Xh, Yh, 1000, starts[:20], 3.0)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    net.train_steps(Xh, Yh, 1000, starts, 3.0)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
t = statistics.median(ts)
print(f"{os.environ.get('TAG', '')}: {500 * 1000 / t / 1e6:.2f} M samples/s, {500 * 3176000 / t / 1e9:.1f} GB/s H2D")
