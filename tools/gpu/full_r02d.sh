# round-2 pass after the spread batched path: GPU suite + full bench line
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r02d.log 2>&1
tail -n 3 gpurun_out/gpu_tests_r02d.log
timeout 2400 python bench.py --steps 10 --warmup 3 --detail-out gpurun_out/bench_detail_r02d.json > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
tail -c 1500 gpurun_out/bench_r02d.json
