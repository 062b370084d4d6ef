"""Per-call fixed cost of nf_train_steps on config 2 (K6): device time (CUDA events around the
call, as bench.py times it) and host time of the call, for several step counts; the slope is
the per-step cost, the intercept the per-call overhead.
    python tools/k6_call_overhead.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1902_06714_b200 as nf  # noqa: E402

cfg = synth.CONFIGS[2]
X, Y = synth.dataset(2)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
net = nf.Net(cfg["dims"], cfg["act"], stream=torch.cuda.current_stream())
net.set_params(torch.from_numpy(synth.init_params(2)).cuda())
loss = torch.zeros(1000, device="cuda")
starts = synth.batch_starts(2, steps=200000)
pos = [0]


def nxt(k):
    s = starts[pos[0]:pos[0] + k]
    pos[0] = (pos[0] + k) % (len(starts) - 1000)
    return s


for k in (1, 2, 5, 20, 100, 500):
    for _ in range(3):
        net.train_steps(Xd, Yd, 1000, nxt(k), 3.0, step_loss=loss)
    dev, host = [], []
    for _ in range(50 if k < 100 else 10):
        st = nxt(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        net.train_steps(Xd, Yd, 1000, st, 3.0, step_loss=loss)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        dev.append(e0.elapsed_time(e1) * 1e3)
        host.append((t1 - t0) * 1e6)
    d, h = statistics.median(dev), statistics.median(host)
    print(f"steps {k:4d}: device {d:9.1f} us ({d / k:6.2f} us/step)   host call {h:7.1f} us", flush=True)

# host-side breakdown of one call (NF_TRACE_HOST=1 stamps from the library) and the Python wrapper
if os.environ.get("NF_TRACE_HOST"):
    st = nxt(20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    net.train_steps(Xd, Yd, 1000, st, 3.0, step_loss=loss)
    t1 = time.perf_counter()
    print(f"python wrapper total {1e6 * (t1 - t0):.1f} us", flush=True)
    lib = nf.lib()
    import ctypes
    args = (net.h, nf._ptr(Xd), nf._ptr(Yd), Xd.shape[0], 1000, nf._ptr(np.ascontiguousarray(st), np.int64), len(st),
            ctypes.c_float(3.0), nf._ptr(loss))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lib.nf_train_steps(*args)
    t1 = time.perf_counter()
    print(f"raw ctypes call {1e6 * (t1 - t0):.1f} us", flush=True)
