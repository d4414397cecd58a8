set -x
mkdir -p gpurun_out
timeout 300 python tools/profile_c5_coarse.py > gpurun_out/plain_c5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"coarse|probe_exact|lm_|lut_|refine" -c 500 --csv --log-file gpurun_out/launches_c5.csv python tools/profile_c5_coarse.py > gpurun_out/ncu_c5.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 200 python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lut_|lm_|refine|coarse" -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/ncu_launch.log 2>&1
echo done
