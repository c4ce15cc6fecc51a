export PYTHONPATH=$PWD
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_dmma_kernel -s 1 -c 1 -o gpurun_out/r02zy_c3pair -f python tools/profile_apply.py --config c3 --reps 1 > gpurun_out/r02zy_ncu.log 2>&1
echo "ncu exit $?"
