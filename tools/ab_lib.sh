#!/bin/bash
# A/B of two builds, interleaved (A B A B) on one box, on c4 and c3:
#   gpurun -- 'bash tools/ab_lib.sh <tag> <alt .so path relative to repo>'
TAG=$1; ALT=$2
for rep in 1 2; do
  for cfg in c4 c3; do
    python bench.py --no-cpu-baseline --no-extra --steps 10 --config $cfg > gpurun_out/${TAG}_${cfg}_A${rep}.json 2> gpurun_out/${TAG}_${cfg}_A${rep}.err
    QTT_LIB_PATH=$PWD/$ALT python bench.py --no-cpu-baseline --no-extra --steps 10 --config $cfg > gpurun_out/${TAG}_${cfg}_B${rep}.json 2> gpurun_out/${TAG}_${cfg}_B${rep}.err
  done
done
python - <<PY
import json, glob
for f in sorted(glob.glob("gpurun_out/${TAG}_c*_[AB]?.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
