#!/bin/bash
# k_gt two-tile consumer: chunk 4 / 6 / 8 diagonals, against the one-tile consumer
mkdir -p gpurun_out
for v in jpc4 jpc8; do FEMI_LIB=$PWD/tmp_old/libfemi_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/$v.json 2>/dev/null; echo $v; python tools/show_bench.py gpurun_out/$v.json; done
for p in 1 0; do FEMI_GT_PAIR=$p timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/jpc6_p$p.json 2>/dev/null; echo jpc6 pair $p; python tools/show_bench.py gpurun_out/jpc6_p$p.json; done
