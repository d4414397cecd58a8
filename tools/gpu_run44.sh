set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -k "dsub4 or fallback_split" > gpurun_out/gpu_tests_a.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_a.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lm_count|lm_scan_|lm_scatter|lut_tiles|lm_tensor|lm_select|refine_stage" -s 0 -c 14 -o gpurun_out/traffic_c5 python tools/profile_c5_scan.py 2 > gpurun_out/ncu_c5traffic.log 2>&1
echo done
