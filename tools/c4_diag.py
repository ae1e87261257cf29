"""C4 (social graph, R = inf) gather timing helper (dev tool). usage: c4_diag.py NLOG [window]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 23
W = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
n = 1 << nlog
g = P.CsrGraph.social(n, seed=0x170807271 + 4)
s = P.BvStream.encode(g, P.BvParams(max_ref=0))
dg = P.BvGraph(s, P.CreateOptions(window=W))
inf = dg.info()
x = torch.rand(n, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    dg.matvec(x, y)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dg.matvec(x, y)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"n=2^{nlog} m={g.m} W={W} ms={np.median(ts):.3f} Gedges/s={g.m / np.median(ts) / 1e6:.1f} "
      f"coverage={inf['window_coverage']:.3f} heavy={inf['bvs_heavy_rows']} slices={inf['bvs_slices']} "
      f"util={inf['bvs_lane_iters_used'] / max(1, inf['bvs_lane_iters']):.2f}")
