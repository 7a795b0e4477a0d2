timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r02a.log 2>&1
tail -n 30 gpurun_out/gpu_tests_r02a.log
