#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4u; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -k "tonal or config4 or smoke or apply or c5_legs" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
for k in 1 2; do timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-cpu-baseline >> $O/bench_c4.json 2>> $O/bench_c4.err; done
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
echo done
