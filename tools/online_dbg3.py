import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, synth, oracle
import paper_1902_06714_b200 as nf
from parity import rel_err
dims, act = [200, 136, 72, 5], "tanh"
p = synth.random_params(41, dims, 0.3)
X, Y = synth.random_batch(42, 64, dims[0], dims[-1], "uniform")
o = oracle.Oracle(dims, act)
st = list(range(0, 64, 3))
mode = sys.argv[1]
net = nf.Net(dims, act); net.set_params(torch.from_numpy(p).cuda())
q = p.astype(np.float64)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
for k in range(8):
    s0 = st[k]
    if mode == "steps":
        net.train_steps(Xd, Yd, 1, [s0], 0.7)
    else:
        net.train_batch(torch.from_numpy(X[s0:s0+1]).cuda(), torch.from_numpy(Y[s0:s0+1]).cuda(), 0.7)
    q, _ = o.train_batch(q, X[s0:s0+1], Y[s0:s0+1], 0.7)
    gp = net.get_params()
    print(mode, "step", k, "sample", s0, "param err", f"{rel_err(gp, q):.2e}", "max|p|", f"{np.abs(gp).max():.3f}",
          "finite", bool(np.isfinite(gp).all()))
