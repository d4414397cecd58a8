# bench lines: c4 (default), c4pl, c3pl, c5pl
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
python bench.py --config c4pl --steps 10 --warmup 3 --gt-queries 2000 > gpurun_out/bench_c4pl.json 2> gpurun_out/bench_c4pl.err; echo "c4pl rc=$?"
python bench.py --config c3pl --steps 5 --warmup 3 --gt-queries 1000 --latency-queries 50 > gpurun_out/bench_c3pl.json 2> gpurun_out/bench_c3pl.err; echo "c3pl rc=$?"
python bench.py --config c5pl --steps 5 --warmup 3 --gt-queries 1000 --compare-single 0 --latency-queries 50 > gpurun_out/bench_c5pl.json 2> gpurun_out/bench_c5pl.err; echo "c5pl rc=$?"
tail -n 2 gpurun_out/bench_c*.err
