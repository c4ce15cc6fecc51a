#!/bin/bash
# Profiling call: bench line (with cpu_baseline), launch list, ncu --set full of
# kernels matching a regex.  gpurun -- 'bash tools/gpu_profile.sh <tag> <regex> <skip> <count> [config]'
set -u
TAG=$1; KRE=$2; SKIP=${3:-0}; CNT=${4:-1}; CFG=${5:-c4}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > $O/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
echo "launches exit $?"
PCMD="python tools/profile_apply.py --config $CFG --reps 1"
timeout 600 $PCMD > $O/${TAG}_plain2.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c $CNT \
    -o $O/${TAG}_prof -f $PCMD > $O/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
