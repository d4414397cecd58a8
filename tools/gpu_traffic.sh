# ncu evidence for one c2pl search: DRAM traffic per kernel + the launch list (cold, serialised)
set -x
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "search/" -o gpurun_out/traffic_c2pl_r2 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/launches_c2pl_r2.csv python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_launch.log 2>&1
echo done
