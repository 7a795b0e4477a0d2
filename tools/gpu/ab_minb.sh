# A/B: batched kernel register cap (B: __launch_bounds__(512, 2), 64 registers, spills) vs A (default)
for v in A B A B; do
  echo "== $v"; PROXSAGA_LIB=$GRAFT_REPO_ROOT/paper_1707_06468_b200/libproxsaga_$v.so timeout 600 python tools/gpu/exp_batch_rep.py 0 32 2>&1 | grep '"B"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['B'], round(d['Mrows'], 1), round(d['Mlam_updates'], 1))"
done
