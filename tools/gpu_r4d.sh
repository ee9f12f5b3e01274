#!/bin/bash
# k_cgs with halo push: timing, timers, GPU parity (default + device-checked), C1/C2/C4 bench
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4d; mkdir -p $O
timeout 300 python tools/diag_cgr.py > $O/cgs.txt 2>&1
FEMI_PCG_TIMERS=1 timeout 300 python tools/diag_cgr.py > $O/cgs_timers.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 1 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
FEMI_LIB=libfemi_check.so timeout 1500 python -m pytest tests -m gpu -q -x -k "config1 or config2 or config4 or tonal or densify" > $O/pytest_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_checked.log
echo done
