#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4k; mkdir -p $O
FEMI_PCG_TIMERS=1 timeout 300 python tools/diag_cgr.py 1,2,3,4 5 > $O/timers.txt 2>&1
timeout 300 python tools/diag_cgr.py 1,2,3,4 > $O/cgs.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; done
FEMI_LIB=libfemi_check.so timeout 1500 python -m pytest tests -m gpu -q -x -k "config1 or config2 or config3 or config4 or tonal or x0 or shared" > $O/pytest_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_checked.log
echo done
