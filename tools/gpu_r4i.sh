#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "x0 or config1 or config2 or config3 or constant or full_mask or shared" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 --log-file $O/launches_c4tonal.csv python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu2.log 2>&1
FEMI_TONAL_PROF=1 timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
echo done
