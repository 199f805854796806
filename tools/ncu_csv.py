"""Top stall reasons and key counters from `ncu --page raw --csv` exports (dev tool).
usage: ncu_csv.py gpurun_out/r2_<name>_raw.csv [...]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("==", path, d.get("Kernel Name", "")[:80])
    for k in KEYS:
        if k in d:
            print(f"  {k} = {d[k]} {u.get(k, '')}")
    st = [(k, float(v.replace(',', ''))) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
          and v.replace(',', '').replace('.', '').isdigit()]
    tot = sum(v for _, v in st) or 1
    for k, v in sorted(st, key=lambda kv: -kv[1])[:7]:
        print(f"  stall {k[33:]}: {100 * v / tot:.1f}%")
