set -x
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "search/" -k regex:"lm_select|refine_stage|coarse_topw|coarse_certify|lm_tensor|lut_tiles" -o gpurun_out/prof_r2a python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
echo done
