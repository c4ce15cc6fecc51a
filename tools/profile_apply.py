"""Run a few QTT applies of one BASELINE config (for ncu / compute-sanitizer).

    python tools/profile_apply.py --config c4 --reps 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--rank", type=int, default=0, help="constant interior rank (bench's large-rank rows)")
    ap.add_argument("--d", type=int, default=18)
    ap.add_argument("--stage-times", action="store_true")
    ap.add_argument("--bie", choices=["M", "Y"], default=None, help="a factor of qtt_workload.bie_case")
    args = ap.parse_args()
    import torch
    import paper_1511_06029_b200 as q
    from qtt_workload import generate
    if args.bie:
        from qtt_workload import bie_case
        _, cM, _, cY, x = bie_case(0, 21, 9, 95, 50, 1)
        cores = cM if args.bie == "M" else cY
    elif args.rank:
        from qtt_workload import random_case
        ranks = [1] + [args.rank] * (args.d - 1) + [1]
        _, cores, x = random_case(4242, args.d, args.rank, 1, ranks=ranks)
    else:
        cfg, cores, x = generate(args.config)
    op = q.QttOperator(cores)
    xt = torch.from_numpy(x).cuda()
    y = torch.empty_like(xt)
    for _ in range(args.reps):
        op.apply(xt, out=y)
    torch.cuda.synchronize()
    print("stages:", [(s["k_first"], s["k_last"], s["variant"]) for s in op.stages()])
    if args.stage_times:
        op.set_stage_timing(True)
        op.stage_times()
        for _ in range(3):
            op.apply(xt, out=y)
        torch.cuda.synchronize()
        ms, n = op.stage_times()
        print("stage ms:", [round(m / n, 4) for m in ms])
    print("ok", float(y.abs().sum()))
    op.close()


if __name__ == "__main__":
    main()
