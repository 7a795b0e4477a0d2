export PS_BATCH_HSHARE=4
python bench.py --no-cpu --no-big --no-io --no-extra --detail-out gpurun_out/bench_detail_sc15.json > gpurun_out/bench_sc15.json 2> gpurun_out/bench_sc15.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_sc15.json").read().strip().splitlines()[-1])
lp = d["lambda_path"]
print({k: lp[k] for k in ("value", "max_rank_ms", "roofline_frac_per_gpu", "rank0_ms_reps", "max_rel_objective_diff_batched_vs_serial", "batched_path_to_1e-6")})
print([(r["n_gpus"], round(r["rank0_ms"], 2)) for r in lp["rank_shares_measured_on_this_gpu"]])
det = json.load(open("gpurun_out/bench_detail_sc15.json"))
print("gaps batched", det["lambda_path.rank0_certified_rel_gap_per_lambda"] if "lambda_path.rank0_certified_rel_gap_per_lambda" in det else [k for k in det][:20])
for r in lp["per_lambda_time_to_1e-6"]:
    print(round(r["lambda_over_max"], 4), r["batched"]["reached"], r["batched"]["epochs_to_1e-6"], r["batched"]["final_rel_gap"])
PY
python -m pytest tests/test_gpu_batch.py tests/test_gpu_lambda_path.py -x -q 2>&1 | tail -2
