timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -p no:cacheprovider 2>&1 | tail -5
python tools/gpu/prof_batch.py 0; python tools/gpu/prof_batch.py 8; python tools/gpu/prof_batch.py 4
timeout 1200 python tools/gpu/exp_batch_path.py 30 2>&1 | tail -6
