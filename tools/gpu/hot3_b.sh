# hot3 second pass: tests, A/B vs hot2 on configs 2/3/4
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_acceptance.py -x -q -p no:cacheprovider > gpurun_out/h3_tests.log 2>&1; tail -3 gpurun_out/h3_tests.log
timeout 600 python tools/exp_flags.py 2 30 0,8388608 > gpurun_out/h3_ab2.log 2>&1; tail -1 gpurun_out/h3_ab2.log
timeout 900 python tools/exp_flags.py 3 10 0,8388608 > gpurun_out/h3_ab3.log 2>&1; tail -1 gpurun_out/h3_ab3.log
timeout 900 python tools/exp_flags.py 4 5 0,8388608 > gpurun_out/h3_ab4.log 2>&1; tail -1 gpurun_out/h3_ab4.log
