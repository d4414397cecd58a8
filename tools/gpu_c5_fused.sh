# c5 (100M x 128, nprobe 64) scan stage: list-major with score rows vs fused (no score rows)
for f in 0 1; do RAIRS_LM_FUSED=$f timeout 600 python tools/time_fs.py c5 64 5 2>&1 | tail -1 | sed "s/^/fused $f: /"; done
