"""Per-CUDA-source-line attribution from an ncu report (dev tool).

    python tools/ncu_lines.py REPORT.ncu-rep [KERNEL_REGEX] [TOP]

Uses `ncu --page source --print-source=cuda,sass --csv`, whose rows with a
line number carry the per-line aggregates (warp-stall samples, warp-level
instructions executed).  Prints the top lines by stall samples with their
share of samples and instructions, plus per-file totals.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else "bvd_gather_kernel"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                          "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    fpath = "?"
    hdr = None
    rows = []
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fpath = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("", "Function Name"):
            continue
        try:
            samp = int(rec[4])
            inst = int(rec[7])
        except (ValueError, IndexError):
            continue
        rows.append((fpath, int(rec[0]), rec[1].strip(), samp, inst))
    ts = sum(r[3] for r in rows) or 1
    ti = sum(r[4] for r in rows) or 1
    print(f"total samples {ts}  warp instructions {ti}")
    files = {}
    for f, _, _, s, i in rows:
        a = files.setdefault(f, [0, 0])
        a[0] += s
        a[1] += i
    for f, (s, i) in sorted(files.items(), key=lambda kv: -kv[1][0]):
        print(f"  {f:24s} samples {100 * s / ts:5.1f}%  instr {100 * i / ti:5.1f}%")
    print()
    for f, ln, src, s, i in sorted(rows, key=lambda r: -r[3])[:top]:
        print(f"{100 * s / ts:5.1f}% {100 * i / ti:5.1f}%  {f}:{ln:<4d} {src[:110]}")


if __name__ == "__main__":
    main()
