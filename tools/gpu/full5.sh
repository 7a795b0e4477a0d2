bash tools/gpu/prof_final.sh > gpurun_out/prof_final.log 2>&1
timeout 900 python tools/gpu/exp_period_ttt.py 2 > gpurun_out/period2.log 2>&1
timeout 1200 python tools/gpu/exp_period_ttt.py 3 > gpurun_out/period3.log 2>&1
timeout 1200 python tools/gpu/exp_period_ttt.py 4 > gpurun_out/period4.log 2>&1
du -sh gpurun_out
