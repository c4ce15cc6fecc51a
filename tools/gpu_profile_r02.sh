#!/bin/bash
# Round-2 profiling call: default bench line, the ncu launch list of the same
# command, and ncu --set full captures of the dominant c4 kernel, the fused
# apply (c1, c2) and the streaming diagonal stage (BIE factor M).
#   gpurun -- 'bash tools/gpu_profile_r02.sh <tag>'
set -u
TAG=${1:-r02p}
O=gpurun_out
mkdir -p $O
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1"
timeout 600 $CMD > $O/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches_c4.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
echo "launches exit $?"
full() {   # name regex skip count driver-args
  timeout 600 python tools/profile_apply.py $5 > $O/${TAG}_$1_plain.log 2>&1 && \
    timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 \
      -o $O/${TAG}_$1 -f python tools/profile_apply.py $5 > $O/${TAG}_$1_ncu.log 2>&1
  echo "ncu $1 exit $?"
}
full c4_level8 level_dmma_kernel 4 1 "--config c4 --reps 1"
full c4_wide wide_dmma_kernel 2 2 "--config c4 --reps 2"
full bieM_diag diag_stream 1 1 "--bie M --reps 2"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_small -s 2 -c 1 \
  -o $O/${TAG}_c1_fused -f python tools/profile_fused.py c1 > $O/${TAG}_c1_fused_ncu.log 2>&1; echo "ncu c1 fused $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_small -s 2 -c 1 \
  -o $O/${TAG}_c2_fused -f python tools/profile_fused.py c2 > $O/${TAG}_c2_fused_ncu.log 2>&1; echo "ncu c2 fused $?"
