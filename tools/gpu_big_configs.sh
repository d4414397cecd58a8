# c5 (100M x 128, nprobe 64) and c3 (1M x 1536) bench lines + c5 scan-path comparison
mkdir -p gpurun_out
python bench.py --config c5 --nprobe 64 --steps 5 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --latency-queries 50 --k1 0 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "c5 rc=$?"; tail -2 gpurun_out/bench_c5.err
for m in simt listmajor; do SCAN_MODE=$m python tools/time_fs.py c5 64 5 2>&1 | tail -1; done
python bench.py --config c3 --steps 5 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --latency-queries 50 --k1 0 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "c3 rc=$?"; tail -2 gpurun_out/bench_c3.err
