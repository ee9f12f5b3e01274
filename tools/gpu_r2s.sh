#!/bin/bash
# k_gt two-tile consumers (FEMI_GT_PAIR) A/B, branch-free raster classification; GPU suite
mkdir -p gpurun_out
for p in 1 0 1; do FEMI_GT_PAIR=$p timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/pair$p.json 2>/dev/null; python tools/show_bench.py gpurun_out/pair$p.json; done
FEMI_LOOP_PROF=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-tonal --steps 2 --warmup 3 > /dev/null 2> gpurun_out/loop_pair.err
grep "femi loop" gpurun_out/loop_pair.err | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_s.log 2>&1; tail -2 gpurun_out/pytest_s.log
