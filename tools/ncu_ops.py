"""Per-opcode aggregation of an ncu source page (dev tool): warp instructions,
shared-memory wavefronts and stall samples per SASS opcode (loads/stores split
by address form).  usage: ncu_ops.py REPORT KERNEL_REGEX [TOP]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0, 0.0])
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        inst = float(r[ix["Instructions Executed"]] or 0)
        samp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        th = float(r[ix["Predicated-On Thread Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r'(@!?U?P\w+\s+)?(\S+)\s*(.*)', src)
    if not m:
        continue
    op, args = m.group(2), m.group(3)
    key = op
    if op.startswith(('LDS', 'STS')):
        a = args.split(',')[-1] if op.startswith('LDS') else args.split(',')[0]
        key = op + " " + re.sub(r'R\d+', 'R', a)
    g = agg[key]
    g[0] += wf
    g[1] += inst
    g[2] += samp
    g[3] += 1
    g[4] += th
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"warp inst {ti:.4g}  smem wf {tw:.4g}  samples {ts:.0f}  avg threads {sum(v[4] for v in agg.values()) / ti:.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][1] / ti + kv[1][0] / tw))[:top]:
    print(f"{k:36s} inst {v[1] / ti * 100:5.1f}%  wf {v[0] / tw * 100:5.1f}%  samp {v[2] / ts * 100:5.1f}%  n={v[3]}")
