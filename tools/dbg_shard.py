import os, sys; sys.path.insert(0, '.')
os.environ["QTT_DEBUG"] = "1"
import torch
from qtt_workload import random_case
from paper_1511_06029_b200 import parallel as par
import paper_1511_06029_b200 as q
_, cores, x = random_case(1400 + 11 + 2, 11, 33, 1)
print([c.shape for c in cores])
for g in range(4):
    try:
        sh = par.QttShard(cores, 2, g); print(g, sh.stages()); sh.close()
    except Exception as e:
        print("ERR", g, e)
