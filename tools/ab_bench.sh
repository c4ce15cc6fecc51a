#!/bin/bash
# A/B: bench (no cpu baseline) with the default library and with an alternative build.
#   gpurun -- 'bash tools/ab_bench.sh <tag> <alt .so path relative to repo>'
TAG=$1; ALT=$2
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_A.json 2> gpurun_out/${TAG}_A.err
echo "A exit $?"
QTT_LIB_PATH=$PWD/$ALT python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_B.json 2> gpurun_out/${TAG}_B.err
echo "B exit $?"
