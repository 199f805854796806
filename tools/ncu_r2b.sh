#!/bin/bash
# Round-2 captures of kernels changed / missed by tools/ncu_r2.sh
set -u
bash tools/ncu_one.sh down downsample_direct 0 zt
bash tools/ncu_one.sh resid resid_f32 40 zt
bash tools/ncu_pipe.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ksvd -c 1 -f -o /tmp/ks python tools/ksvd_one.py > gpurun_out/ks.log 2>&1
ncu -i /tmp/ks.ncu-rep --page raw --csv > gpurun_out/r2_ksvdc_raw.csv
ncu -i /tmp/ks.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_ksvdc_source.csv; gzip -f gpurun_out/r2_ksvdc_source.csv
