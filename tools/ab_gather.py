"""A/B timing of the gather at C2 (dev tool): median kernel time of y = A x^T
for each library given (CMVG_LIBRARY-style paths), L2 flushed before every
launch; parity vs the oracle on the first.
usage: ab_gather.py [--dtype f64|f32] [--nlog 24] LIB [LIB ...]"""
import argparse, os, subprocess, sys, json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, os, json, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1708_07271_b200 as P
nlog, dt, form, reps = int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4])
n = 1 << nlog
g = P.CsrGraph.copy_model(n, 20.0, 0.7, 0.8, seed=0x170807271 + 2)
s = P.BvStream.encode(g, P.BvParams())
dg = P.BvGraph(s, P.CreateOptions())
rng = np.random.default_rng(11)
x = (rng.integers(0, 2**64, size=n, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0**-53
if dt == "f32":
    x = x.astype(np.float32)
xd = torch.from_numpy(x).cuda(); yd = torch.empty_like(xd)
flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
for _ in range(3): dg.matvec(xd, yd, form=form)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dg.matvec(xd, yd, form=form); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
y = yd.double().cpu().numpy()
from oracle import pyoracle as O
gg = g if form == "gather" else g.transpose()
want = O.matvec_csr_raw(gg.n, gg.row_offsets, gg.columns, x.astype(np.float64), O.threads())
nz = want != 0
rel = float(np.max(np.abs(y[nz] - want[nz]) / want[nz])) if nz.any() else 0.0
print(json.dumps({"ms": float(np.median(ts)), "min": float(np.min(ts)), "m": g.m, "rel": rel,
                  "zeros_exact": bool(np.all(y[~nz] == 0))}))
'''.replace("ROOT", repr(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--form", default="gather")
    ap.add_argument("--nlog", type=int, default=24)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    res = {}
    for r in range(a.rounds):  # alternate to average out box drift
        for lib in a.libs:
            env = dict(os.environ, CMVG_LIBRARY=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD, str(a.nlog), a.dtype, a.form, str(a.reps)],
                                 env=env, capture_output=True, text=True)
            if out.returncode:
                print(lib, "FAILED", out.stderr[-2000:])
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res.setdefault(lib, []).append(d)
            print(f"round {r} {lib}: {d['ms']:.4f} ms (min {d['min']:.4f}) "
                  f"{d['m'] / d['ms'] / 1e6:.1f} Gedges/s rel {d['rel']:.2e} zeros {d['zeros_exact']}", flush=True)


if __name__ == "__main__":
    main()
