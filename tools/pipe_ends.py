"""The bench's pipeline_ends leg alone (dev tool, for ncu captures of the
patch kernels).  usage: pipe_ends.py"""
import json, sys
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.bench_pipeline_ends(bench.load_peaks()[0])))
