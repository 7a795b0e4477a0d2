python -m pytest tests/test_gpu_batch.py tests/test_gpu_lambda_path.py -x -q 2>&1 | tail -3
python bench.py --no-cpu --no-big --no-io --no-extra --detail-out gpurun_out/bench_detail_sc4.json > gpurun_out/bench_sc4.json 2> gpurun_out/bench_sc4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_sc4.json").read().strip().splitlines()[-1])
lp = d["lambda_path"]
print(json.dumps({k: v for k, v in lp.items() if k not in ("per_lambda_time_to_1e-6",)}, indent=None)[:6000])
PY
timeout 600 python tools/gpu/exp_batch_B.py 2>&1 | tail -8
