"""Biclique-cover product on the GPU beside the BV gather and the CSR kernel
on the same copy-model graph (dev/measurement tool).
Prints one JSON object: cover sizes (compressed_size vs m vs the BV stream),
extraction time, and per-product device times (L2 flushed before each).
usage: biclique_bench.py [NLOG] [DEG]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 20
deg = float(sys.argv[2]) if len(sys.argv) > 2 else 12.0
n = 1 << nlog
g = P.CsrGraph.copy_model(n, deg, seed=0x170807271 + 1)
t0 = time.time()
cov = P.BicliqueCover.extract_greedy(g, per_round=0)
t_ext = time.time() - t0
assert cov.verify(g)
s = P.BvStream.encode(g, P.BvParams())
bv = P.BvGraph(s)
x = torch.from_numpy((np.random.default_rng(1).random(n))).cuda()
y = torch.empty_like(x)
ro = torch.from_numpy(g.row_offsets.astype(np.int64)).cuda()
co = torch.from_numpy(g.columns.view(np.int32)).cuda()
flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


t_bic = timed(lambda: cov.matvec(x, y))
yb = y.clone()
t_bv = timed(lambda: bv.matvec(x, y))
t_csr = timed(lambda: P.csr_matvec_device(ro, co, x, y))
err = float(((yb - y).abs() / y.abs().clamp_min(1e-300)).max())
bl, res = cov.lists()
print(json.dumps({
    "graph": f"copy model n=2^{nlog} mean degree {deg:g}", "n": n, "m": g.m,
    "bicliques": len(bl), "residual": int(len(res)), "compressed_size": cov.compressed_size,
    "compressed_over_m": cov.compressed_size / g.m, "bv_bits_per_edge": s.stats()["stream_bits"] / g.m,
    "extract_s": t_ext, "ms": {"biclique": t_bic, "bv_gather": t_bv, "csr": t_csr},
    "gedges_s": {"biclique": g.m / t_bic / 1e6, "bv_gather": g.m / t_bv / 1e6, "csr": g.m / t_csr / 1e6},
    "biclique_vs_csr_max_rel_err": err}))
