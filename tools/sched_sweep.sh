#!/bin/bash
# e2e pipeline schedule sweep (dev tool, run under gpurun): zero-tree host-buffer
# call time for several CDB_PIPE_SCHEDULE chunk weightings.
for s in "" "9.47,42.62,37.89,10.02" "8,44,40,8" "7,31,31,24,7" "10,45,45" "6,30,30,26,8" "8,46,38,8" "11,42,37,10"; do
  echo "schedule [$s]: $(CDB_PIPE_SCHEDULE=$s python tools/probe_e2e.py 2>&1 | tail -3 | tr '\n' ' ')"
done
