# ncu DRAM bytes + launch times of one c5 (100M x 128, nprobe 64) search
set -x
mkdir -p gpurun_out
timeout 900 python tools/profile_c5_scan.py 1 > gpurun_out/plain_c5scan.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "search/" -o gpurun_out/traffic_c5 python tools/profile_c5_scan.py 2 > gpurun_out/ncu_c5traffic.log 2>&1
echo done
