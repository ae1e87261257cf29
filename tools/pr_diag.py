"""PageRank timing helper (dev tool): config-3 generator (A^T of a copy model).
usage: pr_diag.py NLOG [iters]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.environ.get("CMVG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = 1 << nlog
g = P.CsrGraph.copy_model(n, 24.0, 0.7, 0.8, seed=0x170807271 + 3)
at = g.transpose()
t0 = time.time()
dg = P.BvGraph(P.BvStream.encode(at, P.BvParams()))
tb = time.time() - t0
deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
dg.pagerank(deg, alpha=0.15, iterations=3)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = float("inf")
for _ in range(int(os.environ.get("PR_DIAG_REPS", "1"))):  # min over repetitions
    a.record()
    p, it = dg.pagerank(deg, alpha=0.15, iterations=iters)
    b.record()
    torch.cuda.synchronize()
    ms = min(ms, a.elapsed_time(b))
    print(f"  rep: {a.elapsed_time(b) / it:.3f} ms/iter")
print(f"n=2^{nlog} m={g.m} iters={it} ms/iter={ms / it:.3f} iter/s={it / ms * 1e3:.1f} build_s={tb:.1f} "
      f"Gedges/s={g.m * it / ms / 1e6:.1f}")
if os.environ.get("PR_DIAG_INFO"):
    inf = dg.info()
    print({k: v for k, v in inf.items() if k.startswith(("bvs", "window", "max_depth", "nblocks"))})
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        dg.matvec(x, y)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        dg.matvec(x, y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"gather A^T (x resident, L2 warm-ish): ms={ms:.3f} Gedges/s={g.m / ms / 1e6:.1f}")
