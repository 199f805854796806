#!/bin/bash
# Round-2 final evidence (run under gpurun, after the bench exited 0 without ncu):
# one `--set full` capture per kernel of the current cfg-4 defaults
# (tools/ncu_one.sh: 65,536 device-generated configs[4] signals), then the
# f-row kernels.  Summarise with tools/ncu_summary_r2.py.
set -u
mkdir -p gpurun_out
for spec in "gram gram_reg2 0 zt" "lswide ls_wide 40 zt" "resid resid_f32 40 zt" "alpha0 alpha0_mma 0 zt" \
            "down downsample_direct 0 zt" "corr corr_topk 40 zt" "rescan rescan_tile 20 zt" \
            "corrfull corr_topk 40 full" "residfull resid_bulk 40 full" "lswidefull ls_wide 40 full"; do
  bash tools/ncu_one.sh $spec
  echo "$spec done"
done
bash tools/ncu_pipe.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ksvd -c 1 -f -o /tmp/ks python tools/ksvd_one.py > gpurun_out/ks.log 2>&1
ncu -i /tmp/ks.ncu-rep --page raw --csv > gpurun_out/r2_ksvdc_raw.csv
