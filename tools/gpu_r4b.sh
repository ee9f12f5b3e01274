#!/bin/bash
# k_cgp (pipelined resident CG) vs k_cgr: per-solve timing, phase timers, GPU parity, C1/C2/C4 bench
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4b; mkdir -p $O
for p in 0 1; do
  FEMI_CG_PIPE=$p timeout 300 python tools/diag_cgr.py > $O/cgr_pipe$p.txt 2>&1
  FEMI_CG_PIPE=$p FEMI_PCG_TIMERS=1 timeout 300 python tools/diag_cgr.py > $O/cgr_timers_pipe$p.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 1 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; done
echo done
