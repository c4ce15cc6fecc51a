#!/bin/bash
# A/B: bench with and without an environment setting.  gpurun -- 'bash tools/ab_env.sh <tag> VAR=value'
TAG=$1; shift
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_A.json 2> gpurun_out/${TAG}_A.err
echo "A exit $?"
env "$@" python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_B.json 2> gpurun_out/${TAG}_B.err
echo "B exit $?"
