timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02c.log 2>&1; tail -n 8 gpurun_out/gpu_tests_r02c.log
timeout 900 python tools/gpu/exp_hot_sweep.py 2 > gpurun_out/hot_sweep2.log 2>&1
timeout 900 python tools/gpu/exp_hot_sweep.py 3 > gpurun_out/hot_sweep3.log 2>&1
timeout 900 python tools/gpu/exp_hot_sweep.py 4 > gpurun_out/hot_sweep4.log 2>&1
timeout 900 python tools/gpu/exp_batch_B.py > gpurun_out/batch_B.log 2>&1
