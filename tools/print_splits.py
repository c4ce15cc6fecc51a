import torch, paper_1511_06029_b200 as q
from qtt_workload import generate, random_case
for name in ("c1","c2","c3","c3x16","c4","c5"):
    cfg, cores, _ = generate(name, with_x=False)
    with q.QttOperator(cores) as op:
        print(name, [(s["k_first"], s["k_last"], s["variant"]) for s in op.stages()], op.stage_splits(cfg.nrhs))
for d, r in ((12,256),(14,128),(16,64),(13,96),(18,256),(20,128),(11,256),(11,128),(12,48),(14,32)):
    ranks=[1]+[r]*(d-1)+[1]
    _, cores, _ = random_case(1, d, r, 1, ranks=ranks)
    with q.QttOperator(cores) as op:
        print(d, r, [(s["k_first"], s["k_last"], s["variant"]) for s in op.stages()], op.stage_splits(1), op.stage_splits(3))
