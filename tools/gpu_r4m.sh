#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4m; mkdir -p $O
FEMI_PCG_TIMERS=1 timeout 300 python tools/diag_cgr.py 1,2,4 5 > $O/timers.txt 2>&1
timeout 300 python tools/diag_cgr.py 1,2,3,4 > $O/cgs.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "config1 or config2 or x0 or constant or full_mask or small or ragged or degenerate or shared or tonal_small" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
echo done
