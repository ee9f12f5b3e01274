#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4g; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "shared_across" > $O/pytest_shared.log 2>&1; echo "pytest rc $?" >> $O/pytest_shared.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 1 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; done
echo done
