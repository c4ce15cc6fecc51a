"""Randomised parity sweep over all kernel variants: random d, rank profiles,
nrhs, stage caps, and random runs of diagonal (block-diagonal) levels, against
the oracle.  Prints the variants exercised."""
import collections
import sys

import numpy as np
import torch

import oracle
import paper_1511_06029_b200 as q
from qtt_workload import random_case

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(2024)
seen = collections.Counter()
fails = 0
for c in range(n_cases):
    d = int(rng.integers(1, 19))
    maxr = int(rng.choice([2, 5, 8, 16, 24, 33, 48, 64]))
    nrhs = int(rng.choice([1, 1, 2, 3]))
    ranks, cores, x = random_case(7000 + c, d, maxr, nrhs)
    if rng.random() < 0.5 and d >= 2:           # a run of diagonal levels
        a = int(rng.integers(0, d))
        b = int(rng.integers(a, d)) + 1
        eye = np.eye(2).reshape(1, 2, 2, 1)
        for k in range(a, b):
            cores[k] = np.ascontiguousarray(cores[k] * eye)
    maxL = None if rng.random() < 0.6 else int(rng.integers(1, 11))
    with q.QttOperator(cores, max_stage_levels=maxL) as op:
        st = op.stages()
        for s in st:
            seen[(s["variant"], s["ksplit"] > 1)] += 1
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    try:
        oracle.assert_close(y, oracle.apply_alg2(cores, x))
    except AssertionError as e:
        fails += 1
        print("FAIL case", c, d, maxr, nrhs, maxL, [(s["k_first"], s["k_last"], s["variant"]) for s in st], str(e)[:200])
print("variants exercised:", dict(seen))
print("cases", n_cases, "failures", fails)
sys.exit(1 if fails else 0)
