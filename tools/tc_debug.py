"""Per-layer error report of the tensor-core path vs the fp64 oracle (debug aid, GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402
from parity import rel_err  # noqa: E402

for dims, act, n in [([200, 136, 72, 5], "tanh", 300), ([256, 128, 64], "sigmoid", 4096),
                     ([516, 260, 132, 3], "gaussian,sigmoid", 333)]:
    p = synth.random_params(1, dims, 1.0 / np.sqrt(max(dims)))
    x, y = synth.random_batch(2, n, dims[0], dims[-1], "uniform")
    o = oracle.Oracle(dims, act)
    ref_out, ref_g = o.output(p, x), o.grad(p, x, y)
    for math in (0, 1):
        net = nf.Net(dims, act)
        net.set_math(math)
        net.set_params(torch.from_numpy(p).cuda())
        out = net.output(torch.from_numpy(x).cuda()).cpu().numpy()
        g = net.grad(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()).cpu().numpy()
        errs = [(rel_err(a, b), rel_err(c, d)) for (a, c), (b, d) in zip(o.layers(g), o.layers(ref_g))]
        print(dims, act, n, "math", math, "out", f"{rel_err(out, ref_out):.2e}",
              "grad W/b per layer", " ".join(f"{e1:.2e}/{e2:.2e}" for e1, e2 in errs), flush=True)
