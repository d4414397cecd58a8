for ns in 1 2 4 8; do RAIRS_COARSE_NSPLIT=$ns python tools/time_fs.py c4 2 10 2>&1 | tail -1 | sed "s/^/nsplit $ns: /"; done
