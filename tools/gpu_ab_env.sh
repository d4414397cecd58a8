# A/B of an environment switch on the default c4 bench line (side lines off):
#   bash tools/gpu_ab_env.sh VAR "v1 v2 ..." [config] [reps]
VAR=$1; VALS=$2; CFG=${3:-c4}; REPS=${4:-1}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 10 --warmup 3 --compare-single 0 --updates 0 --latency-queries 0 --k1 0 --seil-paper 0 --no-cpu-baseline"
for r in $(seq $REPS); do
for v in $VALS; do
  env $VAR=$v timeout 600 $CMD > gpurun_out/ab_${VAR}_$v.json 2> gpurun_out/ab_${VAR}_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/ab_${VAR}_$v.json').read().strip().split('\n')[-1])
print('$VAR=$v', d['value'], d['ms_per_step'], d['stage_ms_per_step'], 'scan', d['roofline']['avg_launch_ms'], 'recall', d.get('recall10@10'))
"
done; done
