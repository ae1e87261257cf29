"""SASS regions of a kernel from an ncu report (dev tool): runs of consecutive
instructions with equal execution counts, ranked by executed instructions.

    python tools/ncu_sass.py REPORT.ncu-rep KERNEL_REGEX [TOP] [--dump A B]
"""
import csv
import io
import subprocess
import sys


def load(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                          "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[h]
    ia, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    data = []
    for r in rows[h + 1:]:
        if len(r) > ia and r[ia].isdigit():
            data.append((r[src].strip(), int(r[ia]), int(r[ss] or 0)))
    return data


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
    data = load(rep, kern)
    if "--dump" in sys.argv:
        i = sys.argv.index("--dump")
        a, b = int(sys.argv[i + 1]), int(sys.argv[i + 2])
        for k in range(a, b + 1):
            print(f"{k:5d} {data[k][1]:10d} {data[k][2]:6d}  {data[k][0]}")
        return
    tot = sum(d[1] for d in data) or 1
    tss = sum(d[2] for d in data) or 1
    regions, start = [], 0
    for i in range(1, len(data) + 1):
        if i == len(data) or data[i][1] != data[start][1]:
            regions.append((start, i - 1))
            start = i
    print(f"{len(data)} instructions, {tot} executed, {tss} samples")
    big = sorted(regions, key=lambda ab: -sum(d[1] for d in data[ab[0]:ab[1] + 1]))[:top]
    for a, b in sorted(big):
        ex = sum(d[1] for d in data[a:b + 1])
        sm = sum(d[2] for d in data[a:b + 1])
        print(f"{a:5d}-{b:5d} n={b - a + 1:4d} exec/instr={data[a][1]:10d} instr {100 * ex / tot:5.1f}%  "
              f"samples {100 * sm / tss:5.1f}%  {data[a][0][:60]}")


if __name__ == "__main__":
    main()
