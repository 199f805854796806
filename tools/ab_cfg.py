"""Zero-tree per-kernel times on one BASELINE config under two env settings (dev tool).
usage: ab_cfg.py ci P "ENV=a" ..."""
import os, subprocess, sys
ci, P = sys.argv[1], sys.argv[2]
for spec in sys.argv[3:]:
    env = dict(os.environ)
    env.update(dict(kv.split('=') for kv in spec.split(',') if kv))
    out = subprocess.run([sys.executable, "tools/probe_big.py", ci, P, "zt", "2"], env=env, capture_output=True, text=True)
    print(spec or "default", out.stdout.strip().splitlines()[-1][:400], flush=True)
