"""nf_output over config 2's resident 50,000-row dataset, timed with CUDA events (median of reps);
for ncu captures of the inference kernel.  Usage: python tools/infer_probe.py [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cfg = synth.CONFIGS[2]
X, _ = synth.dataset(2)
Xd = torch.from_numpy(X).cuda()
net = nf.Net(cfg["dims"], cfg["act"], stream=torch.cuda.current_stream())
net.set_params(torch.from_numpy(synth.init_params(2)).cuda())
out = torch.empty(X.shape[0], 10, device="cuda")
ts = []
for r in range(reps + 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nf.nf_output(net.h, Xd, X.shape[0], out)
    e1.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
t = statistics.median(ts)
print(f"nf_output 50000 rows: {t:.1f} us  {50000 / t:.1f} M rows/s  {50000 * 3176 / t / 1e3:.0f} GB/s")
