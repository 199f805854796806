"""One K-SVD update stage on the device (dev tool, for ncu).  usage: ksvd_one.py [n t m k]"""
import sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import ksvd_oracle as KO
from paper_1511_05174_b200.learn import update_stage
a = [int(v) for v in sys.argv[1:5]] if len(sys.argv) > 4 else [64, 256, 20000, 8]
y, d, x = KO.problem(a[0], a[1], a[2], a[3], 7, (3, 4))
update_stage(y, d.copy(), x.copy(), 2)
