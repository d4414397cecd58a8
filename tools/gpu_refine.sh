set -x
mkdir -p gpurun_out
for v in 0 1 2; do RAIRS_REFINE_VARIANT=$v timeout 300 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain_$v.log 2>&1; done
RAIRS_REFINE_VARIANT=2 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
for v in 0 1 2; do RAIRS_REFINE_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"refine|lm_tensor" -s 0 -c 2 -o gpurun_out/prof_ref$v python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/ncu_ref$v.log 2>&1; done
echo done
