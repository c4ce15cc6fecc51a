#!/bin/bash
# Round profiling call (r01bo+): gpu_profile2.sh plus ncu --set full of the
# split-K last stage of the constant r = 256, d = 18 profile.
set -u
TAG=$1
bash tools/gpu_profile2.sh $TAG
O=gpurun_out
RCMD="python tools/profile_apply.py --rank 256 --d 18 --reps 1"
timeout 600 $RCMD > $O/${TAG}_plain4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide -s 3 -c 1 \
    -o $O/${TAG}_prof_r256split -f $RCMD > $O/${TAG}_ncu_full_r.log 2>&1
echo "ncu split exit $?"
