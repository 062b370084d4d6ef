import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1902_06714_b200 as nf
cfg = synth.CONFIGS[3]
X, Y = synth.dataset(3, N=4096)
net = nf.Net(cfg["dims"], cfg["act"]); net.set_math(nf.NF_MATH_TF32)
net.set_params(torch.from_numpy(synth.init_params(3)).cuda())
Xd = torch.from_numpy(X).cuda(); out = torch.empty((4096, 10), device="cuda")
for _ in range(3): net.output(Xd, out)
torch.cuda.synchronize()
