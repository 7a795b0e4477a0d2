#!/bin/bash
# A/B: the same experiment against two builds (paper_1707_06468_b200/libproxsaga_{A,B}.so)
for v in A B A B; do
  echo "== $v"; PROXSAGA_LIB=$GRAFT_REPO_ROOT/paper_1707_06468_b200/libproxsaga_$v.so "$@" 2>&1 | tail -3
done
