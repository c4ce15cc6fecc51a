#!/bin/bash
# Quick GPU iteration: build, smoke, GPU tests (optional filter), bench.
#   gpurun -- 'bash tools/gpu_quick.sh <tag> [pytest -k expr] [extra bench args]'
set -u
TAG=${1:-q}
KEXPR=${2:-}
set -- "${@:3}"
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1
echo "smoke exit $?"; tail -2 $O/${TAG}_smoke.log
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$KEXPR" > $O/${TAG}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1
fi
echo "pytest exit $?"; tail -15 $O/${TAG}_pytest.log
timeout 900 python bench.py --no-cpu-baseline "$@" > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?"; tail -5 $O/${TAG}_bench.err
python - <<PY
import json
d=json.load(open("$O/${TAG}_bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "per-stage", d["per_stage_roofline"]["frac"], "alg", d["per_stage_roofline"]["algorithmic_frac"])
for s in d["per_stage_roofline"]["stages"]:
    print(s["levels"], s["ranks"], s["variant"], "%.3f ms"%s["ms"], "frac %.3f"%s["roofline_frac"], "exec %.3f"%s["roofline_frac_executed"])
PY
