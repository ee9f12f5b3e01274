#!/bin/bash
# A/B of k_gur's 16-byte pair accesses (FEMI_GUR_VEC) at C5 + the graph-mode GPU tests
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/gurvec; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
for rep in 1 2; do for v in 0 1; do
  FEMI_GUR_VEC=$v timeout 300 $B > $O/bench_v${v}_$rep.json 2> $O/bench_v${v}_$rep.err
done; done
for v in 0 1; do FEMI_GUR_VEC=$v FEMI_LOOP_PROF=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > $O/loop_v$v.json 2> $O/loop_v$v.err; done
timeout 900 python -m pytest tests -m gpu -q -x -k "graph or c5 or switches or colour or tonal or max_image" > $O/pytest_sub.log 2>&1; echo "pytest rc $?" >> $O/pytest_sub.log
echo done
