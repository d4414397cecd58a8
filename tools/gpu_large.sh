# GPU: parity smoke of the changed kernels, then the large BJ configs (c3: 1M x 1536, c4: 10M x 96)
set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -k "many_queries or full_size or search_parity" > gpurun_out/gpu_tests_a.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_a.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c3.log
echo done
