for v in A B C; do
  echo "== $v"; PROXSAGA_LIB=$GRAFT_REPO_ROOT/paper_1707_06468_b200/libproxsaga_$v.so timeout 600 python tools/gpu/exp_batch_scatter.py "16:-1:128,8:-1:128:0,4:-1:128:0,2:-1:128:0" 2>&1 | tail -4
done
