#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, the launch list and one
# `ncu --set full` capture of the dominant kernel.  Usage (from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh <tag> [ncu-kernel-regex] [launch-skip]'
# Everything lands in gpurun_out/<tag>_*.
set -u
TAG=${1:-run}
KRE=${2:-level_dmma_kernel}
SKIP=${3:-6}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> $O/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
tail -3 $O/${TAG}_pytest.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?"
cat $O/${TAG}_bench.json | head -c 600; echo
# launch list (same command as the bench, no cpu baseline so it stays short)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > $O/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
echo "launches exit $?"
PCMD="python tools/profile_apply.py --config c4 --reps 1"
timeout 600 $PCMD > $O/${TAG}_plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 \
    -o $O/${TAG}_prof -f $PCMD > $O/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
ls -la $O | tail -20
