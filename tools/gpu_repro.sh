set -x
mkdir -p gpurun_out
timeout 300 python tools/repro_train.py 65536 300000 > gpurun_out/repro1.log 2>&1; echo "exit $?" >> gpurun_out/repro1.log
timeout 300 python tools/repro_train.py 65536 2100000 > gpurun_out/repro2.log 2>&1; echo "exit $?" >> gpurun_out/repro2.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/repro_train.py 65536 300000 > gpurun_out/repro_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/repro_memcheck.log
echo done
