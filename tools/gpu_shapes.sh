# tensor-kernel pipeline shapes (RAIRS_LM_SHAPE) + one full capture of the search kernels
set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -k "search_parity or many_queries or full_size_sampled" > gpurun_out/gpu_tests_a.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_a.log
for sh in 0 1 2 3; do
  RAIRS_LM_SHAPE=$sh timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain_s$sh.log 2>&1 && \
  RAIRS_LM_SHAPE=$sh timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lm_tensor" -c 20 --csv --log-file gpurun_out/launch_s$sh.csv python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/ncu_s$sh.log 2>&1
done
RAIRS_LM_SHAPE=1 timeout 300 python -m pytest tests -m gpu -x -q -k "search_parity or many_queries" > gpurun_out/gpu_tests_s1.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_s1.log
timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"coarse_topw|coarse_certify|lm_tensor|lm_select|refine_stage" -s 52 -c 5 -o gpurun_out/prof_lm7 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/ncu_full.log 2>&1
echo done
