"""Summarise the round-2 `ncu --set full` captures (raw-page CSV exports in
gpurun_out/r2_<name>_raw.csv) into profiles/r2_ncu_summary.csv and the
per-unit DRAM traffic bench.py reports (profiles/r2_ncu_traffic.json).
usage: ncu_summary_r2.py"""
import csv
import json
import os

CAPTURES = {  # name -> (profiler tag or None, units in the captured launch, unit, what)
    "gram": ("gram_step2", 65536, "signal", "cfg 4 zero-tree step 2, on-chip-H kernel gram_reg2 (default: 24 register + 40 shared rows)"),
    "alpha0": ("route_alpha0", 65536, "signal", "cfg 4 routed alpha0 on fp64 tensor-core tiles"),
    "down": ("downsample", 65536, "signal", "cfg 4 block-mean downsample"),
    "corr": ("corr_topk", 65536, "signal", "cfg 4 step 1 tcgen05 fp16 scan + top-8 (iteration 40)"),
    "lswide": ("ls_step", 65536, "signal", "cfg 4 step 1 least squares (iteration 40)"),
    "resid": ("ls_resid", 65536, "signal", "cfg 4 step 1 scan operand r = y - D32_S x (iteration 40)"),
    "rescan": ("rescan", 65536, "signal", "cfg 4 step 1 tiled fp64 rescan (launch 20: queue nearly empty under the fp16 scan)"),
    "corrfull": ("corr_topk_full", 65536, "signal", "cfg 4 full OMP tcgen05 fp16 scan, dictionary in 4 parts (iteration 40)"),
    "lswidefull": ("ls_step_full", 65536, "signal", "cfg 4 full OMP least squares (iteration 40)"),
    "residfull": ("ls_resid_full", 65536, "signal", "cfg 4 full OMP scan operand, bulk-copy ring (iteration 40)"),
    "pipe_extract": ("extract_patches", 1034289, "patch", "f2 extraction, 1024^2 image, 8x8 stride 1, remove_dc"),
    "pipe_reconstruct": (None, 1034289, "patch", "f2 reconstruction D_S x + dc"),
    "pipe_aggregate": (None, 1034289, "patch", "f2 overlap-add"),
    "ksvdc": ("ksvd_update", 256, "atom", "f1 K-SVD update stage, 16-CTA cluster (N=64, T=256, M=20k)"),
}
KEYS = [("duration_ms", "gpu__time_duration.sum"), ("dram_read", "dram__bytes_read.sum"),
        ("dram_write", "dram__bytes_write.sum"), ("inst", "smsp__inst_executed.sum"),
        ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("smem_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        ("dram_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed")]
SCALE = {"ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def num(v, u):
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)
    except ValueError:
        return None


rows, traffic = [], {"_source": "ncu --set full --clock-control none (round 2): dram__bytes_read.sum + "
                                 "dram__bytes_write.sum of one captured launch / the units it processed; "
                                 "bench.py multiplies by the units of its own launch"}
for name, (tag, units, unit, what) in CAPTURES.items():
    path = os.path.join("gpurun_out", f"r2_{name}_raw.csv")
    if not os.path.exists(path):
        continue
    r = list(csv.reader(open(path)))
    if len(r) < 3:
        continue
    d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))
    row = {"capture": name, "kernel": d.get("Kernel Name", "")[:70], "what": what, "units": units,
           "unit": unit}
    for k, m in KEYS:
        row[k] = num(d.get(m, ""), u.get(m, ""))
    stalls = [(k[33:], num(v, "")) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
    stalls = [(k, v) for k, v in stalls if v]
    tot = sum(v for _, v in stalls) or 1.0
    row["top_stalls"] = "; ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(stalls, key=lambda kv: -kv[1])[:3])
    b = (row["dram_read"] or 0) + (row["dram_write"] or 0)
    row["dram_bytes_per_unit"] = b / units
    rows.append(row)
    if tag:
        traffic[tag] = {"bytes_per_unit": b / units, "unit": unit, "capture": f"r2_{name}"}
os.makedirs("profiles", exist_ok=True)
with open("profiles/r2_ncu_summary.csv", "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
    w.writeheader()
    w.writerows(rows)
with open("profiles/r2_ncu_traffic.json", "w") as f:
    json.dump(traffic, f, indent=1)
for r in rows:
    print(f"{r['capture']:16s} {r['duration_ms']:9.3f} ms  {r['dram_bytes_per_unit']/1e3:9.1f} KB/{r['unit']}  "
          f"issue {r['issue_active_pct'] or 0:5.1f}%  tensor {r['tensor_pipe_pct'] or 0:5.1f}%  fp64 {r['fp64_pipe_pct'] or 0:5.1f}%  {r['top_stalls']}")
