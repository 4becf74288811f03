python tools/l2_probe.py 30 3 > gpurun_out/probe.log 2>&1
python tools/l2_probe.py 30 3 >> gpurun_out/probe.log 2>&1
