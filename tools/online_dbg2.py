import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, synth, oracle
import paper_1902_06714_b200 as nf
from parity import rel_err
dims, act = [200, 136, 72, 5], "tanh"
p = synth.random_params(41, dims, 0.3)
X, Y = synth.random_batch(42, 64, dims[0], dims[-1], "uniform")
o = oracle.Oracle(dims, act)
net = nf.Net(dims, act); net.set_params(torch.from_numpy(p).cuda())
bad = []
for s0 in range(64):
    g = net.grad(torch.from_numpy(X[s0:s0+1]).cuda(), torch.from_numpy(Y[s0:s0+1]).cuda()).cpu().numpy()
    gr = o.grad(p, X[s0:s0+1], Y[s0:s0+1])
    e = rel_err(g, gr)
    if e > 1e-4: bad.append((s0, e))
print("bad samples (grad at the initial params):", bad)
# the same with host arrays (staging path)
bad2 = []
for s0 in range(64):
    g = net.grad(np.ascontiguousarray(X[s0:s0+1]), np.ascontiguousarray(Y[s0:s0+1]))
    e = rel_err(g, o.grad(p, X[s0:s0+1], Y[s0:s0+1]))
    if e > 1e-4: bad2.append((s0, e))
print("bad samples (host buffers):", bad2)
# full batch of 64
g = net.grad(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()).cpu().numpy()
print("batch-64 grad err", rel_err(g, o.grad(p, X, Y)))
