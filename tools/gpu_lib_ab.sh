# A/B of prebuilt library variants (ablibs/librairs_<tag>.so) on the default c4 line (side lines off):
#   LIB_TAGS="a b" bash tools/gpu_lib_ab.sh
mkdir -p gpurun_out
cp paper_2601_07183_b200/librairs.so /tmp/librairs_orig.so
for t in $LIB_TAGS; do
  cp ablibs/librairs_$t.so paper_2601_07183_b200/librairs.so
  timeout 600 python bench.py --steps 10 --warmup 3 --compare-single 0 --updates 0 --latency-queries 0 --k1 0 --seil-paper 0 --no-cpu-baseline > gpurun_out/lib_$t.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/lib_$t.json').read().strip().split('\n')[-1])
print('LIB=$t', d['value'], d['ms_per_step'], d['stage_ms_per_step'], 'scan', d['roofline']['avg_launch_ms'])
"
done
cp /tmp/librairs_orig.so paper_2601_07183_b200/librairs.so
