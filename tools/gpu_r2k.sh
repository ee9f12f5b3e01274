#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_x1.json 2> gpurun_out/bench_x1.err
FEMI_BENCH_X0=3 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_x3.json 2> gpurun_out/bench_x3.err
FEMI_RASTER_MINB=5 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_m5.json 2> gpurun_out/bench_m5.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_x.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_x.log
echo done
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-tonal"
FEMI_PCG_KBENCH=1 timeout 300 $CMD > /dev/null 2> gpurun_out/kb_warm.log
FEMI_PCG_KBENCH=1 FEMI_KBENCH_FLUSH=1 timeout 300 $CMD > /dev/null 2> gpurun_out/kb_flush.log
FEMI_PCG_KBENCH=1 FEMI_KBENCH_NOGU=1 timeout 300 $CMD > /dev/null 2> gpurun_out/kb_nogu.log
FEMI_PCG_KBENCH=1 FEMI_KBENCH_NOGU=1 FEMI_KBENCH_FLUSH=1 timeout 300 $CMD > /dev/null 2> gpurun_out/kb_nogu_flush.log
echo done2
