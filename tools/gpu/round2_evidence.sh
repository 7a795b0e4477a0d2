# round-2 evidence pass: GPU suite, full bench line, launch list + ncu captures (tools/gpu/prof_final.sh)
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r02.log 2>&1
tail -n 5 gpurun_out/gpu_tests_r02.log
timeout 2400 python bench.py --steps 10 --warmup 3 --detail-out gpurun_out/bench_detail_r02.json > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
tail -c 3000 gpurun_out/bench_r02.json
bash tools/gpu/prof_final.sh > gpurun_out/prof_final.log 2>&1
du -sh gpurun_out
