import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, synth, oracle
import paper_1902_06714_b200 as nf
from parity import rel_err
dims, act = [200, 136, 72, 5], "tanh"
p = synth.random_params(41, dims, 0.3)
X, Y = synth.random_batch(42, 64, dims[0], dims[-1], "uniform")
for eta, st in [(0.7, list(range(0, 64, 3))), (0.1, list(range(0, 64, 6)))]:
    for k in [1, 2, 5, len(st)]:
        net = nf.Net(dims, act); net.set_params(torch.from_numpy(p).cuda())
        net.train_steps(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), 1, st[:k], eta)
        ref, _ = oracle.Oracle(dims, act).train_steps(p, X, Y, 1, st[:k], eta)
        print("eta", eta, "steps", k, "err", rel_err(net.get_params(), ref), "upd", rel_err(net.get_params() - p, ref - p))
# locate the largest discrepancy after 5 steps at eta 0.7, and step-by-step single-sample grads
st = list(range(0, 64, 3))
net = nf.Net(dims, act); net.set_params(torch.from_numpy(p).cuda())
o = oracle.Oracle(dims, act)
q = p.copy()
for k in range(6):
    s0 = st[k]
    g = net.grad(torch.from_numpy(X[s0:s0+1]).cuda(), torch.from_numpy(Y[s0:s0+1]).cuda()).cpu().numpy()
    gr = o.grad(net.get_params(), X[s0:s0+1], Y[s0:s0+1])
    errs = [(rel_err(a, b), rel_err(c, d)) for (a, c), (b, d) in zip(o.layers(g), o.layers(gr))]
    print("step", k, "sample", s0, "grad err per layer W/b", " ".join(f"{e1:.1e}/{e2:.1e}" for e1, e2 in errs))
    net.train_steps(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), 1, [s0], 0.7)
