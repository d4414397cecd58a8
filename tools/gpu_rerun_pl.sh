mkdir -p gpurun_out
python bench.py --config c4pl --steps 10 --warmup 3 --gt-queries 2000 > gpurun_out/bench_c4pl.json 2> gpurun_out/bench_c4pl.err; echo "c4pl rc=$?"
python bench.py --config c5 --nprobe 64 --steps 5 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --latency-queries 50 --k1 0 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python bench.py --config c5pl --steps 5 --warmup 3 --gt-queries 1000 --compare-single 0 --latency-queries 50 --no-cpu-baseline > gpurun_out/bench_c5pl.json 2> gpurun_out/bench_c5pl.err; echo "c5pl rc=$?"
