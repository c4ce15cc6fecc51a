#!/bin/bash
# bench (no cpu baseline, no extras unless EXTRA=1) under several env settings:
#   gpurun -- 'bash tools/ab_env_multi.sh <tag> "VAR=a" "VAR=b" ...'   (first run: no setting)
TAG=$1; shift
X="--no-extra"; [ "${EXTRA:-0}" = "1" ] && X=""
python bench.py --no-cpu-baseline --steps 5 $X > gpurun_out/${TAG}_0.json 2>/dev/null; echo "base $?"
i=1
for kv in "$@"; do
  env $kv python bench.py --no-cpu-baseline --steps 5 $X > gpurun_out/${TAG}_$i.json 2>/dev/null; echo "$kv $?"
  i=$((i+1))
done
