import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1708_07271_b200 as P
n = 1 << 24
g = P.CsrGraph.copy_model(n, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
dg = P.BvGraph(P.BvStream.encode(g, P.BvParams()))
x = torch.rand(n, dtype=torch.float64).pin_memory().numpy()
y = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
for _ in range(3):
    dg.matvec(x, y)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); dg.matvec(x, y); ts.append(time.perf_counter() - t0)
print(os.environ.get("CMVG_EXP_CHUNKS"), os.environ.get("CMVG_EXP_XFAR_DEV"), "e2e ms", min(ts) * 1e3, np.median(ts) * 1e3)
