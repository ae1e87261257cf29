"""Summarise an ncu report (or a launch-list CSV) into JSON for profiles/.

usage:
  python tools/ncu_summary.py report.ncu-rep out.json [key]      # --set full capture
  python tools/ncu_summary.py --launches launches.csv out.json   # gpu__time_duration list
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__inst_executed.sum": "warp_instructions",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_per_block",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_rate_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_lsu_wavefronts_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def full(rep, out, key=None):
    hdr, units, rows = raw_rows(rep)
    res = []
    for r in rows:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", "")}
        for k, name in WANT.items():
            if k in d and d[k] not in ("", None):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                e[name] = v * SCALE.get(u.get(k, ""), 1)
        stalls = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        e["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        if "dram_read" in e and "dram_write" in e:
            e["dram_bytes_per_launch"] = e["dram_read"] + e["dram_write"]
        res.append(e)
    blob = {"report": rep, "kernels": res}
    if key:
        prev = {}
        try:
            prev = json.load(open(out))
        except Exception:
            pass
        prev[key] = res[0] if len(res) == 1 else res
        blob = prev
    json.dump(blob, open(out, "w"), indent=1)
    print(json.dumps(blob, indent=1)[:3000])


def launches(csv_path, out):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]]
        unit = r[idx["Metric Unit"]]
        v = float(r[idx["Metric Value"]].replace(",", "")) * SCALE.get(unit, 1)
        per[name][0] += 1
        per[name][1] += v
    # handle creation (the device build: decode + block transcode) and the
    # oracle / torch set-up run before the timed steps: listed apart, the
    # shares are of the per-step kernels only
    oneoff = ("bvf_build_blocks", "bvf_block_sizes", "bvf_pack_", "bv_decode_tiles", "bv_sync_index",
              "bv_index_groups", "bv_scan_segments")
    step = {k: v for k, v in per.items() if not any(o in k for o in oneoff)}
    once = {k: v for k, v in per.items() if k not in step}
    total = sum(v[1] for v in step.values())
    res = sorted(({"kernel": k, "launches": v[0], "total_s": v[1], "share": v[1] / total if total else 0}
                  for k, v in step.items()), key=lambda e: -e["total_s"])
    res1 = sorted(({"kernel": k, "launches": v[0], "total_s": v[1]} for k, v in once.items()),
                  key=lambda e: -e["total_s"])
    json.dump({"source": csv_path, "total_s": total, "kernels": res,
               "handle_creation_kernels (not in the step)": res1}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
