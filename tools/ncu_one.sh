#!/bin/bash
# one ncu --set full capture: ncu_one.sh name kernel_regex skip what [P] -> gpurun_out/r2_<name>_{raw,details}.csv, _source.csv.gz
name=$1; kre=$2; skip=$3; what=$4; P=${5:-65536}
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kre" -s "$skip" -c 1 \
  -f -o /tmp/r2_$name python tools/probe_big.py 4 $P $what 1 > gpurun_out/r2_$name.log 2>&1
ncu -i /tmp/r2_$name.ncu-rep --page raw --csv > gpurun_out/r2_${name}_raw.csv 2>/dev/null
ncu -i /tmp/r2_$name.ncu-rep --page details --csv > gpurun_out/r2_${name}_details.csv 2>/dev/null
ncu -i /tmp/r2_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_${name}_source.csv 2>/dev/null
gzip -f gpurun_out/r2_${name}_source.csv
