#!/bin/bash
# Round-2 evidence refresh (run under gpurun): GPU tests, the default bench,
# then -- only after the bench exited 0 -- the ncu launch list of the same
# command (our kernels only) for the per-step shares.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || { echo "bench failed"; tail -5 gpurun_out/bench.err; exit 1; }
tail -1 gpurun_out/bench.json | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:3cdb -c 6000 --csv \
    --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-api --no-extras > gpurun_out/r2_ncu_launch.log 2>&1
echo "launch list rc=$?"
