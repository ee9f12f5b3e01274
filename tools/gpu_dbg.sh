#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do
FEMI_RASTER_PF=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_pf1_$rep.json 2>/dev/null
FEMI_RASTER_PF=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_pf0_$rep.json 2>/dev/null
done
timeout 300 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/bench_c6pf.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "inpaint or colour or config or mask or constant or ragged or max" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
echo done
