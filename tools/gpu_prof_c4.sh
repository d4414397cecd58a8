set -x
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py c4 2 auto 2 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "search/" -o gpurun_out/prof_c4 python tools/profile_step.py c4 2 auto 2 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/plain_c4.log
echo done
