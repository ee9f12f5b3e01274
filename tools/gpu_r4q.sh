#!/bin/bash
# raster A/B: f prefetched one window ahead (FEMI_RASTER_PF=1, 3 CTAs/SM) vs default
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4q; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
for k in 1 2 3; do
  FEMI_RASTER_PF=1 timeout 600 $B >> $O/pf.json 2>> $O/pf.err
  timeout 600 $B >> $O/base.json 2>> $O/base.err
done
FEMI_RASTER_PF=1 timeout 900 python -m pytest tests -m gpu -q -x -k "inpaint or config5 or densify or band or config3" > $O/pytest_pf.log 2>&1; echo "pytest rc $?" >> $O/pytest_pf.log
echo done
