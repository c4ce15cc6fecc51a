nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks/fp64_peaks > gpurun_out/peaks.json 2>&1
kill $SMI
cat gpurun_out/peaks.json
nvidia-smi -q | grep -i -A3 "power\|clocks" | head -60 > gpurun_out/smi_q.txt
free -g; nproc; lscpu | head -20
