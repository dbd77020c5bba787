import os, sys
sys.path.insert(0, '/root/repo')
os.environ["ADP_STEP"] = "1"
import paper_2502_09758_b200 as adp
from paper_2502_09758_b200 import _native as nat, configs
up = configs.config3(0, size=256)
p = up.lower_problem(up.b0)
print("flags", p.op.plan().flags(), p.op.plan().geometry())
