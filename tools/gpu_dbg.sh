#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FEMI_RASTER_2P=1 timeout 900 python -m pytest tests -m gpu -x -q -k "inpaint or config1 or config3 or config5 or mask or constant or ragged or max or densify or incremental" > gpurun_out/pytest_2p.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_2p.log
for rep in 1 2; do
FEMI_RASTER_2P=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_2p_$rep.json 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_1p_$rep.json 2>/dev/null
done
echo done
