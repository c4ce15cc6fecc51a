import sys, os; sys.path.insert(0,'.')
os.environ["QTT_DEBUG"]="1"
import torch, numpy as np
from qtt_workload import random_case
import paper_1511_06029_b200 as q
import oracle
r,c,x=random_case(23,15,24,1)
for maxL in (6,10):
    op=q.QttOperator(c,max_stage_levels=maxL)
    print(op.stages())
    try:
        y=op.apply(torch.from_numpy(x).cuda()); torch.cuda.synchronize()
        print(oracle.compare(y.cpu().numpy(), oracle.apply_alg2(c,x)))
    except Exception as e: print("ERR", e)
