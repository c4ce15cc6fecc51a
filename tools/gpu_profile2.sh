#!/bin/bash
# Round profiling call: bench line (+cpu_baseline), launch list of the bench
# command, ncu --set full of the c4 wide stages, one r=48 level, and the Morton pack.
set -u
TAG=$1
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1"
timeout 600 $CMD > $O/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
echo "launches exit $?"
PCMD="python tools/profile_apply.py --config c4 --reps 1"
timeout 600 $PCMD > $O/${TAG}_plain2.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dmma -s 0 -c 2 \
    -o $O/${TAG}_prof_c4a -f $PCMD > $O/${TAG}_ncu_full_a.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:wide -s 1 -c 1 \
    -o $O/${TAG}_prof_c4b -f $PCMD > $O/${TAG}_ncu_full_b.log 2>&1
echo "ncu full exit $?"
MCMD="python tools/profile_morton.py"
timeout 300 $MCMD > $O/${TAG}_plain3.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:morton -c 2 \
    -o $O/${TAG}_prof_morton -f $MCMD > $O/${TAG}_ncu_full_m.log 2>&1
echo "ncu morton exit $?"
