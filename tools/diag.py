"""Diagnostics (dev tool): worst-row parity analysis and a single-size timing.
usage: diag.py NLOG [mode] [threads] [window] [block_rows] [dtype]"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1708_07271_b200 as P

try:  # measured HBM GB/s (driver-written), else the profiling recipe's fallback
    import json as _json
    PEAK_GBS = float(_json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'MEASURED_PEAKS.json')))['hbm_gbs'])
except Exception:
    PEAK_GBS = 6650.0
from oracle import pyoracle as O

a = sys.argv + [None] * 8
nlog = int(a[1] or 20); mode = a[2] or "prefix"; thr = int(a[3] or 128); W = int(a[4] or 2048)
B = int(a[5] or 1024); dt = a[6] or "f64"; cap = int(a[7] or 0)
n = 1 << nlog
g = P.CsrGraph.copy_model(n, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
s = P.BvStream.encode(g, P.BvParams())
dg = P.BvGraph(s, P.CreateOptions(interval_mode=mode, lanes=thr, window=W, block_rows=B, stream_cap_words=cap))
rng = np.random.default_rng(11)
x = (rng.integers(0, 2**64, size=n, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0**-53
if dt == "f32":
    x = x.astype(np.float32)
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)
flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
for _ in range(3):
    dg.matvec(xd, yd)
torch.cuda.synchronize()
ts = []
for _ in range(8):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dg.matvec(xd, yd); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
info = dg.info()
alg = s.stats()["stream_bits"] / 8 + n * x.itemsize * 2
print(f"n=2^{nlog} m={g.m} mode={mode} thr={thr} W={W} B={B} {dt} ms={np.median(ts):.4f} "
      f"Gedges/s={g.m / np.median(ts) / 1e6:.1f} frac={alg / (np.median(ts) * 1e-3) / (PEAK_GBS * 1e9):.3f} cap={info['bvs_stream_cap_words']}")
y = yd.double().cpu().numpy()
want = O.matvec_csr_raw(g.n, g.row_offsets, g.columns, x.astype(np.float64), O.threads())
nz = want != 0
rel = np.zeros(n)
rel[nz] = np.abs(y[nz] - want[nz]) / want[nz]
print("  zero rows exact:", bool(np.all(y[~nz] == 0)), "max rel", rel.max())
