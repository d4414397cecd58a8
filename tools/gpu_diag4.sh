set -x
mkdir -p gpurun_out
RAIRS_LM_DIAG=64 timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/lmprof_64.log 2>&1
RAIRS_LM_DIAG=95 timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/lmprof_95.log 2>&1
echo done
