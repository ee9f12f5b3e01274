#!/bin/bash
mkdir -p gpurun_out
for c in 0 1 0 1; do FEMI_GU_CARVE=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/carve$c.json 2>/dev/null; echo "carve $c"; python tools/show_bench.py gpurun_out/carve$c.json; done
for c in 0 1; do FEMI_GU_CARVE=$c FEMI_LOOP_PROF=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/loopc$c.err; grep "femi loop" gpurun_out/loopc$c.err | tail -1; done
for c in 0 1; do FEMI_GU_CARVE=$c FEMI_GT_PAIR=4 FEMI_PCG_KBENCH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/kbc$c.err; echo "carve $c pair 4 (launch+tail)"; grep "femi kbench" gpurun_out/kbc$c.err | tail -1; done
