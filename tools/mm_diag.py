"""Multi-vector product timing / profiling helper (dev tool).
usage: mm_diag.py NLOG [k]  (config-5 generator: copy model, degree 16)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n = 1 << nlog
g = P.CsrGraph.copy_model(n, 16.0, 0.7, 0.8, seed=0x170807271 + 5)
dg = P.BvGraph(P.BvStream.encode(g, P.BvParams()))
X = torch.rand(n, k, dtype=torch.float32, device="cuda")
Y = torch.empty_like(X)
for _ in range(3):
    dg.matmat(X, Y)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dg.matmat(X, Y)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"n=2^{nlog} m={g.m} k={k} ms={np.median(ts):.3f} Gedge-vectors/s={g.m * k / np.median(ts) / 1e6:.1f}")
