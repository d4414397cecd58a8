set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/ncu_launch.log 2>&1 ; \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lm_tensor|lm_select|refine_kernel|coarse_select" -s 0 -c 8 -o gpurun_out/prof_lm python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_full.log 2>&1
echo done
