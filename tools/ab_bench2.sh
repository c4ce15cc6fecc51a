#!/bin/bash
# A/B with extra bench args: gpurun -- 'bash tools/ab_bench2.sh <tag> <alt .so> [bench args...]'
TAG=$1; ALT=$2; shift 2
python bench.py --no-cpu-baseline --steps 5 "$@" > gpurun_out/${TAG}_A.json 2> gpurun_out/${TAG}_A.err
echo "A exit $?"
QTT_LIB_PATH=$PWD/$ALT python bench.py --no-cpu-baseline --steps 5 "$@" > gpurun_out/${TAG}_B.json 2> gpurun_out/${TAG}_B.err
echo "B exit $?"
