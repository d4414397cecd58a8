for e in "TAG=default" "RAIRS_FS_PACK=0" "RAIRS_FS_ORDER=0" "RAIRS_FS_RING=4" "RAIRS_FS_VARIANT=1"; do env $e TAG=$e timeout 300 python tools/dbg/small17b.py 2>&1 | tail -1; done
