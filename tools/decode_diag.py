"""GPU BV decode timing (dev tool): usage decode_diag.py NLOG [cfg]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 24
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 1 << nlog
if cfg == 4:
    g = P.CsrGraph.social(n, seed=0x170807271 + 4)
    s = P.BvStream.encode(g, P.BvParams(max_ref=0))
else:
    g = P.CsrGraph.copy_model(n, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
    s = P.BvStream.encode(g, P.BvParams())
dg = P.BvGraph(s)
ro = torch.empty(n + 1, dtype=torch.int64, device="cuda")
co = torch.empty(max(g.m, 1), dtype=torch.int32, device="cuda")
dg.decode_csr_device(ro, co)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    dg.decode_csr_device(ro, co)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
ok = np.array_equal(co[:g.m].cpu().numpy().view(np.uint32), g.columns)
print(f"cfg{cfg} n=2^{nlog} m={g.m} decode ms={min(ts) * 1e3:.2f} Gedges/s={g.m / min(ts) / 1e9:.2f} exact={ok} "
      f"serial={os.environ.get('CMVG_SERIAL_DECODE')}")
