"""Warm device time of the C-ABI operations on a config's full batch (CUDA events):
nf_output (forward chain), nf_grad (forward + backward + tendencies), nf_train_batch (step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
math = nf.NF_MATH_TF32 if (len(sys.argv) > 2 and sys.argv[2] == "tf32") else nf.NF_MATH_FP32
cfg = synth.CONFIGS[cid]
B = cfg["batch"]
X, Y = synth.dataset(cid, N=B)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
net = nf.Net(cfg["dims"], cfg["act"])
net.set_math(math)
net.set_params(torch.from_numpy(synth.init_params(cid)).cuda())
out = torch.empty((B, cfg["dims"][-1]), device="cuda")
g = torch.empty(net.n_params, device="cuda")


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print(f"config {cid} math {'tf32' if math else 'fp32'} B={B}")
only_train = len(sys.argv) > 3 and sys.argv[3] == "train"   # (for ncu launch lists of one step)
if not only_train:
    print(f"  nf_output      {t(lambda: net.output(Xd, out)):9.1f} us")
    print(f"  nf_grad        {t(lambda: net.grad(Xd, Yd, g)):9.1f} us")
print(f"  nf_train_batch {t(lambda: net.train_batch(Xd, Yd, 0.01)):9.1f} us")
