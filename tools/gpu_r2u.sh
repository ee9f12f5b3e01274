#!/bin/bash
mkdir -p gpurun_out
for p in 0 2 4; do FEMI_GT_PAIR=$p FEMI_PCG_KBENCH=1 FEMI_KBENCH_NOGU=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/kbn$p.err; echo "nogu pair $p"; grep "femi kbench" gpurun_out/kbn$p.err | tail -2; done
for p in 0 2; do FEMI_PDL_PRE=0 FEMI_GT_PAIR=$p FEMI_PCG_KBENCH=1 FEMI_KBENCH_NOGU=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/kbp$p.err; echo "pre0 nogu pair $p"; grep "femi kbench" gpurun_out/kbp$p.err | tail -2; done
for L in 1 2; do FEMI_L2POL=$L FEMI_GT_PAIR=2 FEMI_PCG_KBENCH=1 FEMI_KBENCH_NOGU=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/kbl$L.err; echo "l2pol $L nogu pair 2"; grep "femi kbench" gpurun_out/kbl$L.err | tail -2; done
