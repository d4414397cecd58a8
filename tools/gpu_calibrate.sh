# calibration of the -pl generators on 1M-row samples (profiles/calibration_<cfg>.jsonl)
mkdir -p gpurun_out
python tools/calibrate_pl.py c4pl '[[0.5,1024],[1.0,1024],[2.0,1024],[3.0,1024]]' > gpurun_out/calibration_c4pl.jsonl 2> gpurun_out/cal_c4pl.err
python tools/calibrate_pl.py c5pl '[[0.5,4096],[1.0,4096],[1.5,4096],[2.5,4096]]' > gpurun_out/calibration_c5pl.jsonl 2> gpurun_out/cal_c5pl.err
python tools/calibrate_pl.py c3pl '[[0.01,256],[0.016,256],[0.025,256],[0.04,256]]' > gpurun_out/calibration_c3pl.jsonl 2> gpurun_out/cal_c3pl.err
tail -2 gpurun_out/cal_*.err
