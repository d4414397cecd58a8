set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "search_parity or many_queries or full_size_sampled" > gpurun_out/gpu_tests_a.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_a.log
RAIRS_LM_DIAG=64 timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/lmprof_64.log 2>&1
RAIRS_LM_DIAG=95 timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/lmprof_95.log 2>&1
timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lm_tensor" -c 6 --csv --log-file gpurun_out/diag6.csv python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_diag6.log 2>&1
echo done
