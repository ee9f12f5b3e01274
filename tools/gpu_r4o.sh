#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4o; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
FEMI_LIB=libfemi_check.so timeout 1500 python -m pytest tests -m gpu -q -x -k "config1 or config3 or densify or colour or band or inpaint" > $O/pytest_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_checked.log
FEMI_ASM_PROF=1 timeout 300 python tools/diag_c3_stages.py 3 > $O/stages.txt 2>&1
timeout 300 python tools/diag_c3_host.py 5 > $O/c3_split.txt 2>&1
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-tonal > $O/bench_c5.json 2> $O/bench_c5.err
echo done
