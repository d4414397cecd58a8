# GPU suite + short bench lines (side lines off) for the given configs: bash tools/gpu_check.sh "c4 c2pl"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
for cfg in ${1:-c4}; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --compare-single 0 --updates 0 --latency-queries 0 --k1 0 --seil-paper 0 --no-cpu-baseline > gpurun_out/chk_$cfg.json 2> gpurun_out/chk_$cfg.err
  python -c "
import json
d=json.loads(open('gpurun_out/chk_$cfg.json').read().strip().split('\n')[-1])
print('$cfg', d['value'], d['ms_per_step'], d['stage_ms_per_step'], 'scan', d['roofline']['avg_launch_ms'], 'frac', d['roofline']['frac'], 'recall', d.get('recall10@10'), 'unc', d.get('coarse_uncertified_per_step'))
"
done
