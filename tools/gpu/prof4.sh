python tools/gpu/prof_batch.py 0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_group_batch --launch-skip 1 -c 1 -o gpurun_out/prof_batch_a -f python tools/gpu/prof_batch.py 0 > gpurun_out/prof_batch_a.log 2>&1
