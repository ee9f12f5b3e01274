#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4h; mkdir -p $O
for fm in 8192 0; do
FEMI_FILL_MIN=$fm timeout 300 python tools/diag_cgr.py 1,2,3,4 > $O/cgs_fill$fm.txt 2>&1
for c in 1 2 3 4; do FEMI_FILL_MIN=$fm timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c${c}_fill$fm.json 2> $O/bench_c${c}_fill$fm.err; done
done
echo done
