# single-query / small-batch latency A/B over environment settings
mkdir -p gpurun_out
for e in ${LAT_ENVS:-"X=0"}; do
  echo "== $e"; env $e timeout 300 python tools/lat_1q.py ${LAT_CFG:-c4} ${LAT_NPROBE:-2} 200 2>&1 | tail -3
done
