import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import ksvd_oracle as KO
from paper_1511_05174_b200.learn import update_stage
y, d, x = KO.problem(64, 256, 20000, 8, 7, (3, 4))
update_stage(y, d.copy(), x.copy(), 2)
