"""Host-pointer gather timeline (dev tool): the pipelined pinned path's chunk
timeline (CMVG_PIPE_TRACE) next to the raw PCIe copy rates of the same bytes.
usage: e2e_trace.py [NLOG]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n = 1 << nlog
g = P.CsrGraph.copy_model(n, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
dg = P.BvGraph(P.BvStream.encode(g, P.BvParams()))
xh = np.random.default_rng(1).random(n)
xp = torch.from_numpy(xh).pin_memory()
yp = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.empty(n, dtype=torch.float64, device="cuda")


def t(f, k=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3


s2 = torch.cuda.Stream()


def both():
    xd.copy_(xp, non_blocking=True)
    with torch.cuda.stream(s2):
        yp.copy_(yd, non_blocking=True)
    s2.synchronize()


mb = n * 8 / 1e6
h2d = t(lambda: xd.copy_(xp, non_blocking=True))
d2h = t(lambda: yp.copy_(yd, non_blocking=True))
bi = t(both)
print(f"{mb:.0f} MB: H2D {h2d:.3f} ms ({mb / h2d:.1f} GB/s)  D2H {d2h:.3f} ms ({mb / d2h:.1f} GB/s)  "
      f"both at once {bi:.3f} ms")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def chunked(C=16):  # the pipeline's copy pattern without kernels: D2H chunk c after H2D chunk c
    step = (n + C - 1) // C
    for c in range(C):
        lo, hi = c * step, min(n, (c + 1) * step)
        with torch.cuda.stream(sa):
            xd[lo:hi].copy_(xp[lo:hi], non_blocking=True)
            e = torch.cuda.Event()
            e.record(sa)
        with torch.cuda.stream(sb):
            sb.wait_event(e)
            yp[lo:hi].copy_(yd[lo:hi], non_blocking=True)
    sb.synchronize()
    sa.synchronize()


print(f"chunked copy pattern (16 chunks, D2H c after H2D c): {t(chunked):.3f} ms; 8 chunks {t(lambda: chunked(8)):.3f}")
xn, yn = xp.numpy(), yp.numpy()
e = t(lambda: dg.matvec(xn, yn))
dev = t(lambda: dg.matvec(xd, yd))
print(f"host-pointer gather {e:.3f} ms ({g.m / e / 1e6:.1f} Gedges/s); device-pointer gather {dev:.3f} ms")
