# coarse A/B: parity of the coarse paths, then c4 / c4pl / c2pl stage times per variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse or full_size or build_assignment or exact_fallback or search_parity" > gpurun_out/cab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/cab_tests.log
Q="--steps 10 --warmup 3 --gt-queries 1000 --no-cpu-baseline --compare-single 0 --latency-queries 0 --k1 0 --updates 0 --seil-paper 0"
for c in c4 c4pl c2pl; do
for v in "" "RAIRS_COARSE_HALFLISTS=0" "RAIRS_COARSE_DBG=2"; do
  env $v timeout 600 python bench.py --config $c $Q > gpurun_out/cab.json 2> gpurun_out/cab.err || { echo "$c $v FAILED"; tail -3 gpurun_out/cab.err; continue; }
  python - "$c" "$v" <<'P'
import json,sys; d=json.load(open('gpurun_out/cab.json'))
print(sys.argv[1], sys.argv[2] or "default", round(d['value']/1e6,3), d['stage_ms_per_step'], 'uncert', d.get('coarse_uncertified_per_step'), 'recall', d.get('recall10@10'))
P
done; done
