#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4r; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "device_layouts" > $O/pytest_lay.log 2>&1; echo "pytest rc $?" >> $O/pytest_lay.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
FEMI_LIB=libfemi_check.so timeout 1500 python -m pytest tests -m gpu -q -x -k "config1 or config2 or config3 or config4 or densify or x0 or shared or failure" > $O/pytest_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_checked.log
FEMI_ASM_PROF=1 timeout 300 python tools/diag_c3_stages.py 3 > $O/stages.txt 2>&1
timeout 300 python tools/diag_c3_host.py 5 > $O/c3_split.txt 2>&1
for c in 2 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; done
echo done
