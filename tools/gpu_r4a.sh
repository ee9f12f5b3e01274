#!/bin/bash
# Session-3 re-entry check of HEAD: GPU suite, smoke, C5 / C4 / C2 / C1 bench lines
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
for c in 1 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; done
FEMI_TONAL_PROF=1 timeout 600 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_c4_prof.json 2> $O/bench_c4_prof.err
echo done
