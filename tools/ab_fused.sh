#!/bin/bash
# A/B of fused-plan splits (QTT_FUSED_FORCE_STAGES) for c1 and c2, us per apply.
export PYTHONPATH=$PWD
for spec in "1-8,9-12" "1-6,7-9,10-12" "1-7,8-12" "1-4,5-8,9-12" "1-8,9-10,11-12"; do
  echo "c1 $spec: $(QTT_FORCE_FUSED=1 QTT_FUSED_FORCE_STAGES=$spec python tools/time_small.py c1 | python -c 'import json,sys; d=json.load(sys.stdin)["c1"]; print(d["cached_us_batched"], d["plan"])')"
done
for spec in "1-7,8-10,11-15" "1-6,7-8,9-10,11-15" "1-6,7-9,10-12,13-15" "1-5,6-8,9-11,12-15" "1-7,8-11,12-15" "1-7,8-9,10-11,12-15"; do
  echo "c2 $spec: $(QTT_FORCE_FUSED=1 QTT_FUSED_FORCE_STAGES=$spec python tools/time_small.py c2 | python -c 'import json,sys; d=json.load(sys.stdin)["c2"]; print(d["cached_us_batched"], d["plan"])')"
done
