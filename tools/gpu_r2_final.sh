# full GPU suite + default bench (c4) + c4pl bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_default.err
timeout 900 python bench.py --config c4pl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4pl.json 2> gpurun_out/bench_c4pl.err; echo "c4pl rc=$?"; tail -2 gpurun_out/bench_c4pl.err
