#!/bin/bash
# ncu --set full of the patch-pipeline kernels (bench pipeline_ends leg)
for k in extract reconstruct aggregate; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o /tmp/r2_pipe_$k \
    python tools/pipe_ends.py > gpurun_out/r2_pipe_$k.log 2>&1
  ncu -i /tmp/r2_pipe_$k.ncu-rep --page raw --csv > gpurun_out/r2_pipe_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/r2_pipe_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_pipe_${k}_source.csv 2>/dev/null
  gzip -f gpurun_out/r2_pipe_${k}_source.csv
done
python tools/pipe_ends.py > gpurun_out/pipe_ends.json 2>&1
