set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "search_parity or many_queries or full_size or ties" > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 200 python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lut_|lm_|refine|coarse" -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/ncu_launch.log 2>&1
echo done
