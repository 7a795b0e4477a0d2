timeout 600 python tools/gpu/exp_literal.py > gpurun_out/literal.log 2>&1
timeout 2400 python bench.py --steps 10 --warmup 3 --detail-out gpurun_out/bench_detail_r02a.json > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
