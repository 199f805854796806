"""Full-OMP per-kernel times on configs[4] (dev tool).  usage: ab_full.py P "ENV=a" ..."""
import os, subprocess, sys
P = sys.argv[1]
for spec in sys.argv[2:]:
    env = dict(os.environ)
    env.update(dict(kv.split('=') for kv in spec.split(',') if kv))
    out = subprocess.run([sys.executable, "tools/probe_big.py", "4", P, "full", "2"], env=env, capture_output=True, text=True)
    print(spec or "default", out.stdout.strip().splitlines()[-1][:400], flush=True)
