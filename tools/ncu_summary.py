"""Summarise `ncu --set full` reports into committed profile files (dev tool).

usage: ncu_summary.py out_prefix report.ncu-rep [report2.ncu-rep ...]

Writes
  <out_prefix>_summary.csv : one row per captured launch -- duration, DRAM
      bytes, SM / tensor / fp64 / shared-memory utilisation, top stalls;
  <out_prefix>_traffic.json : {profiler tag: DRAM bytes per launch}, the
      `roofline.traffic` figure bench.py reports (mean over the captured
      launches of each kernel).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}

# kernel-name fragment -> profiler tag used by bench.py (csrc ProfScope names)
TAGS = {
    "resident_omp": "resident_step1",
    "resident_mma": "resident_step1",
    "gram_omp": "gram_step2",
    "alpha0_warp": "route_alpha0",
    "alpha0_mma": "route_alpha0",
    "downsample": "downsample",
    "corr_topk": "corr_topk",
    "ls_group": "ls_step",
    "rescan_kernel": "rescan",
    "ls_final": "ls_final",
}


SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
         "nsecond": 1e-6, "second": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw_rows(rep):
    """Rows of the raw page with durations in ms and byte counts in bytes."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        for i, h in enumerate(hdr):
            if h in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
                v = num(r[i])
                if v is not None and units[i] in SCALE:
                    d[h] = v * SCALE[units[i]]
        res.append(d)
    return res


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    lines, traffic = [], defaultdict(list)
    for rep in reps:
        for r in raw_rows(rep):
            name = r.get("Kernel Name", "")
            row = {"report": rep.split("/")[-1], "kernel": name.split("(")[0][-70:]}
            for k, m in METRICS.items():
                row[k] = r.get(m, "")
            stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v)
                      for k, v in r.items()
                      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
                      not k.endswith("not_issued") and num(v)}
            tot = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
            row["top_stalls"] = "; ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top)
            lines.append(row)
            for frag, tag in TAGS.items():
                if frag in name:
                    rd, wr = num(r.get(METRICS["dram_read_bytes"])), num(r.get(METRICS["dram_write_bytes"]))
                    ms = num(r.get(METRICS["duration_ms"])) or 0.0
                    if rd is not None and wr is not None:
                        traffic[tag].append((ms, rd + wr))
    with open(prefix + "_summary.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(lines[0].keys()))
        w.writeheader()
        w.writerows(lines)
    # main launches only: the rescan-resume passes of ls_step touch a handful of signals
    t = {}
    for k, v in traffic.items():
        top = max(ms for ms, _ in v)
        main_ = [b for ms, b in v if ms >= 0.25 * top]
        t[k] = sum(main_) / len(main_)
    t["_source"] = "ncu --set full --clock-control none, dram__bytes_read.sum + dram__bytes_write.sum " \
                   "per launch (mean over captured launches): " + ", ".join(x.split("/")[-1] for x in reps)
    with open(prefix + "_traffic.json", "w") as f:
        json.dump(t, f, indent=1)
    for row in lines:
        print(row["kernel"][-40:], row["duration_ms"], row["dram_read_bytes"], row["dram_write_bytes"],
              row["tensor_pipe_pct"], row["fp64_pipe_pct"], row["smem_wavefronts_pct"], row["top_stalls"])


if __name__ == "__main__":
    main()
