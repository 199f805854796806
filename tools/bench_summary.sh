#!/bin/bash
# usage: tools/bench_summary.sh out.json  -- print the key numbers of a bench line
python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('zt', round(d['value']), 'ms', round(d['ms_per_step'], 3), '| full', round(d['full_omp']['value']),
      'ms', round(d['full_omp']['ms_per_step'], 3), '| e2e', round(d['e2e']['value']))
print({k: round(v, 3) for k, v in d['kernels_ms_per_step'].items()})
print({k: round(v, 3) for k, v in d['kernels_full_ms_per_step'].items()})
PY
