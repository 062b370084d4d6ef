"""Per-phase timing of the fused small-net kernel (NF_FUSED_PROF=1): globaltimer stamps per
CTA per step, printed by the library to stderr.  Usage: python tools/phase_profile.py [steps]"""
import os
import sys

os.environ["NF_FUSED_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
cfg = synth.CONFIGS[2]
X, Y = synth.dataset(2)
net = nf.Net(cfg["dims"], cfg["act"])
net.set_params(torch.from_numpy(synth.init_params(2)).cuda())
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
starts = synth.batch_starts(2, steps=steps)
for _ in range(2):
    net.train_steps(Xd, Yd, cfg["batch"], starts, cfg["eta"])
torch.cuda.synchronize()
if os.environ.get("PP_FRESH"):  # a third call on fresh batch starts after an L2 flush: x from HBM, as in bench.py
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush.fill_(1.0)
    torch.cuda.synchronize()
    print("---- fresh starts, L2 flushed", file=sys.stderr, flush=True)
    net.train_steps(Xd, Yd, cfg["batch"], synth.batch_starts(2, steps=2 * steps)[steps:], cfg["eta"])
    torch.cuda.synchronize()
