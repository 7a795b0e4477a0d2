# round-2 evidence: launch list of a short bench + ncu --set full of the hot kernel (config 2, 3) and the batched kernel
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --no-path --no-big --no-io --no-extra > gpurun_out/ncu_launch_r02.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_hot_kernel --launch-skip 1 -c 1 -o gpurun_out/prof_hot_r02_c2 -f python tools/prof_async.py --batch 0 --wpc 32 --hp 24 --c 4 --per_launch 30 --hot_max 512 --warm 1 --epochs 1 > gpurun_out/prof_hot_r02_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_hot_kernel --launch-skip 1 -c 1 -o gpurun_out/prof_hot_r02_c3 -f python tools/prof_big.py 3 0.25 > gpurun_out/prof_hot_r02_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_hot_kernel --launch-skip 1 -c 1 -o gpurun_out/prof_hot_r02_c4 -f python tools/prof_big.py 4 0.25 > gpurun_out/prof_hot_r02_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_group_batch --launch-skip 1 -c 1 -o gpurun_out/prof_batch_r02 -f python tools/gpu/prof_batch.py 0 > gpurun_out/prof_batch_r02.log 2>&1
