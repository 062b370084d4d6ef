import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, synth, oracle
from parity import rel_err
dims, act = [200, 136, 72, 5], "tanh"
p = synth.random_params(41, dims, 0.3)
X, Y = synth.random_batch(42, 64, dims[0], dims[-1], "uniform")
st = list(range(0, 64, 3))[:8]
o64 = oracle.Oracle(dims, act, bits=64)
o32 = oracle.Oracle(dims, act, bits=32)
q64, _ = o64.train_steps(p, X, Y, 1, st, 0.7)
q32, _ = o32.train_steps(p, X, Y, 1, st, 0.7)
print("fp32 oracle vs fp64 oracle after 8 online steps (eta 0.7):", rel_err(q32, q64))
i = int(np.argmax(np.abs(q32 - q64)))
print("worst index", i, q32[i], q64[i])
q64b, _ = o64.train_steps(p, X, Y, 1, list(range(0, 64, 6)), 0.1)
q32b, _ = o32.train_steps(p, X, Y, 1, list(range(0, 64, 6)), 0.1)
print("fp32 oracle vs fp64 oracle after 11 online steps (eta 0.1):", rel_err(q32b, q64b))
