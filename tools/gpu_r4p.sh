#!/bin/bash
# raster A/B: per-round deduplicated vertex-value gathers (libfemi.so) vs previous (libfemi_old.so)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4p; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
for k in 1 2 3; do
  timeout 600 $B >> $O/new.json 2>> $O/new.err
  FEMI_LIB=libfemi_old.so timeout 600 $B >> $O/old.json 2>> $O/old.err
done
timeout 900 python -m pytest tests -m gpu -q -x -k "inpaint or raster or colour or config5 or densify or band" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
echo done
