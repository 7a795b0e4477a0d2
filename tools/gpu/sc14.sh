for R in 0 2 4 8; do
  echo "== hshare $R"; PS_BATCH_HSHARE=$R timeout 900 python tools/gpu/exp_batch_scatter.py "16:-1:128,8:-1:128,4:-1:128,2:-1:128,1:-1:128" 2>&1 | tail -5
done
