# final round-2 measurements: GPU suite, every config's bench line, reference arm,
# launch list of the default command, c4 DRAM traffic, fs_scan ncu summary
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_c4_reference.json 2> gpurun_out/bench_c4_ref.err; echo "ref rc=$?"
python bench.py --config c4pl --steps 10 --warmup 3 --gt-queries 2000 --no-cpu-baseline > gpurun_out/bench_c4pl.json 2> gpurun_out/bench_c4pl.err; echo "c4pl rc=$?"
python bench.py --config c2pl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2pl.json 2> gpurun_out/bench_c2pl.err; echo "c2pl rc=$?"
python bench.py --config c3pl --steps 5 --warmup 3 --gt-queries 1000 --latency-queries 50 --no-cpu-baseline > gpurun_out/bench_c3pl.json 2> gpurun_out/bench_c3pl.err; echo "c3pl rc=$?"
python bench.py --config c5pl --steps 5 --warmup 3 --gt-queries 1000 --compare-single 0 --latency-queries 50 --no-cpu-baseline > gpurun_out/bench_c5pl.json 2> gpurun_out/bench_c5pl.err; echo "c5pl rc=$?"
python bench.py --config c5 --nprobe 64 --steps 5 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --latency-queries 50 --k1 0 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
bash tools/gpu_bench_launches.sh; python tools/ncu_launches.py gpurun_out/launches_bench_c4.csv > gpurun_out/launches_summary.txt 2>&1
timeout 300 python tools/profile_step.py c4 2 auto 2 > gpurun_out/plain_c4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/ncu_traffic_c4_search.csv \
  python tools/profile_step.py c4 2 auto 2 > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?"
bash tools/gpu_prof_fs.sh c4 2 > /dev/null 2>&1; python tools/ncu_brief.py gpurun_out/prof_fs_c4.ncu-rep fs_scan > gpurun_out/ncu_fs_c4_brief.txt; echo "prof rc=$?"
