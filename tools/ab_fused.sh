#!/bin/bash
# A/B of fused-plan splits (QTT_FUSED_FORCE_STAGES) for c1 and c2, us per apply
# (back-to-back stream applies and in-graph device time, tools/time_small_graph.py).
export PYTHONPATH=$PWD
run() {  # name spec
  QTT_FORCE_FUSED=1 QTT_FUSED_FORCE_STAGES=$2 python tools/time_small_graph.py $1 | python -c "import json,sys; d=json.load(sys.stdin)['$1']; print(d['stream_us'], d['graph_us'], d['plan'])"
}
for spec in "1-8,9-12" "1-6,7-12" "1-7,8-12" "1-5,6-12" "1-6,7-9,10-12" "1-4,5-8,9-12" "1-8,9-10,11-12"; do
  echo "c1 $spec: $(run c1 $spec)"
done
for spec in "1-7,8-10,11-15" "1-7,8-15" "1-8,9-15" "1-6,7-8,9-10,11-15" "1-6,7-9,10-15" "1-5,6-8,9-11,12-15" "1-7,8-11,12-15" "1-7,8-9,10-11,12-15" "1-6,7-10,11-15"; do
  echo "c2 $spec: $(run c2 $spec)"
done
