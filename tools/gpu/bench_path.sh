# the bench line restricted to config 2 and the lambda path (config 5), with the per-lambda summary printed
python bench.py --no-cpu --no-big --no-io --no-extra --detail-out gpurun_out/bench_detail_path.json > gpurun_out/bench_path.json 2> gpurun_out/bench_path.err
tail -3 gpurun_out/bench_path.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_path.json").read().strip().splitlines()[-1])
lp = d["lambda_path"]
print(lp.get("batched_path_to_1e-6"), lp["value"], lp["max_rank_ms"])
for r in lp["per_lambda_time_to_1e-6"]:
    print(round(r["lambda_over_max"], 4), r["reached"], r["seconds_to_1e-6"], r["epochs_to_1e-6"], r["batched"])
PY
