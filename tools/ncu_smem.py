"""Shared-memory wavefronts per SASS instruction from an ncu report (dev tool).

    python tools/ncu_smem.py REPORT.ncu-rep [KERNEL_REGEX] [TOP]

Prints the instructions with the most shared-memory wavefronts (actual vs
ideal) and the warp-level instruction count, to attribute LSU load.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else "bvf_gather"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--kernel-name",
                          f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    recs = []
    tot_wf = tot_inst = 0.0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
            ideal = float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
            inst = float(r[ix["Instructions Executed"]] or 0)
            samp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        tot_wf += wf
        tot_inst += inst
        recs.append((wf, ideal, inst, samp, r[ix["Address"]], r[ix["Source"]]))
    print(f"total smem wavefronts {tot_wf:.4g}, warp instructions {tot_inst:.4g}")
    for wf, ideal, inst, samp, addr, src in sorted(recs, reverse=True)[:top]:
        print(f"{wf:12.4g} ideal {ideal:12.4g} inst {inst:10.4g} samples {samp:8.0f}  {addr}  {src[:70]}")
    print("--- top instructions by stall samples")
    for wf, ideal, inst, samp, addr, src in sorted(recs, key=lambda t: -t[3])[:top]:
        print(f"samples {samp:8.0f} inst {inst:10.4g} wf {wf:10.4g}  {addr}  {src[:70]}")


if __name__ == "__main__":
    main()
