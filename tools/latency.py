"""Per-step device time of small-batch training (the paper's train_single regime):
nf_train_steps over many steps on c1 and on the c2 net with batch 1..32 (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402


def per_step(dims, act, p, X, Y, batch, steps, eta):
    net = nf.Net(dims, act)
    net.set_params(torch.from_numpy(p).cuda())
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    rng = np.random.default_rng(0)
    starts = rng.integers(0, len(X) - batch + 1, size=steps)
    net.train_steps(Xd, Yd, batch, starts[:10], eta)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    net.train_steps(Xd, Yd, batch, starts, eta)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


only = sys.argv[1:]  # e.g. "c2:1" = the c2 net at batch 1 only (for ncu)
if only:
    c2 = synth.CONFIGS[2]
    X2, Y2 = synth.dataset(2, N=20000)
    for spec in only:
        if spec == "c1":
            c1 = synth.CONFIGS[1]
            X1, Y1 = synth.dataset(1)
            print(f"c1: {per_step(c1['dims'], c1['act'], synth.init_params(1), X1, Y1, 8, 2000, 1.0):.2f} us/step")
            continue
        b = int(spec.split(":")[1])
        print(f"c2 B={b}: {per_step(c2['dims'], c2['act'], synth.init_params(2), X2, Y2, b, 500, 0.1):.2f} us/step")
    sys.exit(0)
c1 = synth.CONFIGS[1]
X1, Y1 = synth.dataset(1)
print(f"c1 {c1['dims']} B=8: {per_step(c1['dims'], c1['act'], synth.init_params(1), X1, Y1, 8, 2000, 1.0):.2f} us/step")
c2 = synth.CONFIGS[2]
X2, Y2 = synth.dataset(2, N=20000)
for b in (1, 2, 4, 8, 16, 32, 100):
    print(f"c2 {c2['dims']} B={b}: {per_step(c2['dims'], c2['act'], synth.init_params(2), X2, Y2, b, 2000, 0.1):.2f} us/step")
