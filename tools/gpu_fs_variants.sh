for v in 0 1; do
RAIRS_FS_VARIANT=$v python bench.py --config c4 --steps 10 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --no-cpu-baseline --latency-queries 0 > gpurun_out/bench_c4_v$v.json 2> gpurun_out/bench_c4_v$v.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench_c4_v$v.json').read().strip().splitlines()[-1])
print('c4 v$v', d['value'], d['config']['nprobe'], d['recall10@10'], d['stage_ms_per_step'], d['roofline']['frac'])"
done
