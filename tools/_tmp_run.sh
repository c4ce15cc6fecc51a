export PYTHONPATH=$PWD
timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_dmma_kernel -s 4 -c 1 -o gpurun_out/r02zu_c4_level -f python tools/profile_apply.py --config c4 --reps 1 > gpurun_out/r02zu_ncu1.log 2>&1
echo "ncu exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_small -s 2 -c 1 -o gpurun_out/r02zu_c2_fused -f python tools/profile_fused.py c2 > gpurun_out/r02zu_ncu2.log 2>&1
echo "ncu exit $?"
