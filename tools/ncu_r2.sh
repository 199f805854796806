#!/bin/bash
# Round-2 evidence (run under gpurun): the ncu launch list of the bench command
# (after it exited 0 without ncu), then one `--set full` capture per cfg-4
# kernel via tools/ncu_one.sh (65,536 device-generated configs[4] signals).
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-api --no-extras > gpurun_out/r2_ncu_launch.log 2>&1
echo "launch list rc=$?"
for spec in "gram gram_cta 0 zt" "lswide ls_wide 40 zt" "resid resid_split 40 zt" "alpha0 alpha0_mma 0 zt" \
            "down downsample 0 zt" "corr corr_topk 40 zt" "rescan rescan_tile 20 zt" \
            "corrfull corr_topk 40 full" "residfull resid_split 40 full" "lswidefull ls_wide 40 full"; do
  bash tools/ncu_one.sh $spec
  echo "$spec done"
done
