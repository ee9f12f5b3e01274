#!/bin/bash
# k_gt paired tiles vs single: C5 bench + loop timeline
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4f; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
for p in 1 0 1 0; do FEMI_GT_PAIR=$p timeout 600 $B >> $O/bench_pair$p.json 2>> $O/bench_pair$p.err; done
for p in 1 0; do FEMI_GT_PAIR=$p FEMI_LOOP_PROF=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> $O/loop_pair$p.err; done
timeout 1500 python -m pytest tests -m gpu -q -x -k "c5 or 2880 or 8192 or graph or notma or tonal" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
echo done
