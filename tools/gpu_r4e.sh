#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4e; mkdir -p $O
timeout 300 python tools/diag_cgr.py 1,2,3,4 > $O/cgs.txt 2>&1
FEMI_CG_PIPE=0 timeout 300 python tools/diag_cgr.py 3 > $O/cgr_c3.txt 2>&1
for p in 1 0; do FEMI_CG_PIPE=$p timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3_p$p.json 2> $O/bench_c3_p$p.err; done
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
echo done
