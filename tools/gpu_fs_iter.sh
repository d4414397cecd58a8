# one fast-scan iteration on the GPU: parity tests of the scan, c4 bench line, ncu of fs_scan
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "simt or massive or padded or c4 or insert or delete" 2>&1 | tail -3 > gpurun_out/t.log
cat gpurun_out/t.log
python bench.py --config c4 --steps 10 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --no-cpu-baseline --latency-queries 0 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
print('c4', d['value'], d['config']['nprobe'], d['recall10@10'], d['stage_ms_per_step'], d['roofline']['frac'], d['dco_per_query'])"
if [ "$1" = "ncu" ]; then bash tools/gpu_prof_fs.sh c4 2; fi
