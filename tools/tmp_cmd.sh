python tools/ab_cfg.py 5 5 > gpurun_out/ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "matrix or random_small or two_hundred or config_parity and 5" > gpurun_out/pytest_gpu.log 2>&1
echo rc=$? >> gpurun_out/pytest_gpu.log
