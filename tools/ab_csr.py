"""A/B timing of the CSR comparison kernel at C2 (dev tool).
usage: ab_csr.py LIB [LIB ...]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1708_07271_b200 as P
g = P.CsrGraph.copy_model(1 << 24, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
x = torch.rand(g.n, dtype=torch.float64, device="cuda")
ro = torch.from_numpy(g.row_offsets.astype(np.int64)).cuda(); co = torch.from_numpy(g.columns.view(np.int32)).cuda()
y = torch.empty_like(x); fl = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
for _ in range(3): P.csr_matvec_device(ro, co, x, y)
ts = []
for _ in range(10):
    fl.zero_(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); P.csr_matvec_device(ro, co, x, y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(f"{np.median(ts):.4f} ms  {(4*g.m + 24*g.n) / np.median(ts) / 1e6:.0f} GB/s")
'''.replace("ROOT", repr(ROOT))
for lib in sys.argv[1:]:
    out = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, CMVG_LIBRARY=os.path.abspath(lib)),
                         capture_output=True, text=True)
    print(lib, out.stdout.strip() or out.stderr[-1500:], flush=True)
