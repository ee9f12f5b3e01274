#!/bin/bash
# Final-tree check after the solver pruning: GPU suite, smoke, the driver's C5 bench line, C2/C4,
# and the C5 launch list (gpu__time_duration, recipe pass) of the same bench command.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/${EVDIR:-fin}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err
for c in 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_c$c.json 2> $O/bench_c$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_c5_recipe.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > $O/ncu_recipe.log 2>&1
echo done
