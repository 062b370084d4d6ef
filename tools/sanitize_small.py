"""Small invocations of every kernel family for compute-sanitizer (one tool per run):
fused K6 (c1 and a short c2), fused inference, generic SIMT + skinny kernels, tcgen05 GEMMs
(per-tile 3xTF32 and 1xTF32), loss/accuracy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# c1 fused
X, Y = synth.dataset(1)
net = nf.Net([3, 5, 2], "sigmoid")
net.train_steps(dev(X), dev(Y), 8, synth.batch_starts(1, steps=5), 1.0)
# c2 fused, 3 steps; inference; loss/accuracy
X, Y = synth.dataset(2, N=3000)
net = nf.Net([784, 30, 10], "sigmoid")
net.set_params(dev(synth.init_params(2)))
net.train_steps(dev(X), dev(Y), 1000, [0, 1000, 2000], 3.0)
net.output(dev(X))
net.loss(dev(X), dev(Y)); net.accuracy(dev(X), dev(Y))
# generic: tc (fp32 3x and tf32 1x), skinny output layer, SIMT
for math in (0, 1):
    dims = [256, 192, 136, 10]
    x, y = synth.random_batch(1, 640, dims[0], dims[-1])
    net = nf.Net(dims, "tanh,sigmoid")
    net.set_math(math)
    net.train_batch(dev(x), dev(y), 0.1)
    net.grad(dev(x), dev(y))
    net.output(dev(x))
x, y = synth.random_batch(2, 50, 37, 13)
net = nf.Net([37, 45, 13], "relu")
net.train_batch(dev(x), dev(y), 0.1)
torch.cuda.synchronize()
print("sanitize_small ok")
