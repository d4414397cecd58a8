set -x
mkdir -p gpurun_out
RAIRS_DEBUG_SYNC=1 timeout 600 python tools/repro_train_c5.py 8000000 > gpurun_out/repro3.log 2>&1; echo "exit $?" >> gpurun_out/repro3.log
RAIRS_DEBUG_SYNC=1 timeout 600 python tools/repro_train_c5.py 100000000 > gpurun_out/repro4.log 2>&1; echo "exit $?" >> gpurun_out/repro4.log
echo done
