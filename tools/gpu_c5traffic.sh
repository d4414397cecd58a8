set -x
mkdir -p gpurun_out
timeout 900 python tools/profile_c5_scan.py 1 > gpurun_out/plain_c5scan.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lm_count|lm_scan_|lm_scatter|lut_tiles|lm_tensor|lm_select|refine_stage" -s 0 -c 14 -o gpurun_out/traffic_c5 python tools/profile_c5_scan.py 2 > gpurun_out/ncu_c5traffic.log 2>&1
echo done
