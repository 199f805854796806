#!/bin/bash
# ncu --set full captures of the cfg 4 zero-tree / full-OMP kernels (one launch
# each, 65,536 device-generated signals).  Output: gpurun_out/r2_*.ncu-rep
set -x
P=${P:-65536}
run() {  # name, kernel regex, skip, what
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s "$3" -c 1 \
    -f -o gpurun_out/r2_$1 python tools/probe_big.py 4 $P $4 1 > gpurun_out/r2_$1.log 2>&1
}
run gram gram_omp 0 zt
run lswide ls_wide 40 zt
run resid resid_split 40 zt
run alpha0 alpha0_mma 0 zt
run down downsample 0 zt
run corr corr_topk 40 zt
run corrfull corr_topk 40 full
run residfull resid_split 40 full
run lswidefull ls_wide 40 full
# bring back CSV pages (the reports themselves exceed gpurun's 64 MiB merge limit)
for f in gpurun_out/r2_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > ${b}_source.csv 2>/dev/null
  gzip -f ${b}_source.csv
done
mkdir -p /tmp/ncu_keep && mv gpurun_out/r2_*.ncu-rep /tmp/ncu_keep/
