#!/bin/bash
# Round-end evidence refresh (run under gpurun): GPU tests, the default bench,
# then -- only after the bench exited 0 -- the ncu launch list of the same
# command and one `--set full` capture per top kernel.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || { echo "bench failed"; tail -5 gpurun_out/bench.err; exit 1; }
tail -1 gpurun_out/bench.json | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
for k in resident_mma gram_omp alpha0_mma downsample corr_topk ls_group; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/full_$k \
      python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$k.log 2>&1
done
ls gpurun_out/*.ncu-rep
