#!/bin/bash
# Bounds-checked build (compute-sanitizer is closed on this pool): every epilogue
# store traps outside its output buffer (-DQTT_BOUNDS_CHECK, LevelArgs.out_limit).
# Builds it, then runs the variant fuzz and the GPU suite against it.
#   gpurun -- 'bash tools/gpu_bounds_check.sh'
set -u
mkdir -p paper_1511_06029_b200/dbg
QTT_EXTRA_NVFLAGS="-DQTT_BOUNDS_CHECK" QTT_LIB_OUT=paper_1511_06029_b200/dbg/libqtt_b200_checked.so \
  QTT_OBJ_DIR=/tmp/obj_chk python -m paper_1511_06029_b200.build --force
export QTT_LIB_PATH=paper_1511_06029_b200/dbg/libqtt_b200_checked.so
PYTHONPATH=. timeout 900 python tools/fuzz_variants.py 300 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not bench and not plain_c and not perf_regression" | tail -3
