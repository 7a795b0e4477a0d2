# functional dry run of the N=2 path (both ranks on the one GPU: the numbers are NOT a scaling measurement)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu --no-big --no-io --no-extra --e2e-steps 1 > gpurun_out/bench_n2_dry.json 2> gpurun_out/bench_n2_dry.err
echo "rc=$?"; tail -c 600 gpurun_out/bench_n2_dry.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?"; tail -c 800 gpurun_out/bench_ref.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
