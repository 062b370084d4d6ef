"""Task-level profile of the deep-net megakernel (NF_DMK_PROF=1: per task type, the mean
dependency wait and run time over the first 64 tasks of each CTA), config 4 in TF32.
    python tools/deep_mk_profile.py [steps]"""
import os
import sys

os.environ["NF_DMK_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[4]
X, Y = synth.dataset(4, N=8 * cfg["batch"])
net = nf.Net(cfg["dims"], cfg["act"])
net.set_math(nf.NF_MATH_TF32)
net.set_params(torch.from_numpy(synth.init_params(4)).cuda())
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
starts = synth.batch_starts(4, steps=steps, N=len(X))
for _ in range(2):
    net.train_steps(Xd, Yd, cfg["batch"], starts, cfg["eta"])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
net.train_steps(Xd, Yd, cfg["batch"], starts, cfg["eta"])
e1.record()
torch.cuda.synchronize()
print(f"{steps} steps: {e0.elapsed_time(e1) * 1e3 / steps:.1f} us/step (with the profiler's host copy)")
