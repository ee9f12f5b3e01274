#!/bin/bash
# prologue rework: A/B against the previous library, kernel times, GPU suite, bench; C3 host split
mkdir -p gpurun_out
FEMI_LIB=$PWD/tmp_old/libfemi_old.so timeout 600 python tools/ab_bits.py dump gpurun_out/ab_old.npz > gpurun_out/ab.log 2>&1
timeout 600 python tools/ab_bits.py dump gpurun_out/ab_new.npz >> gpurun_out/ab.log 2>&1
python tools/ab_bits.py compare gpurun_out/ab_old.npz gpurun_out/ab_new.npz >> gpurun_out/ab.log 2>&1
rm -f gpurun_out/ab_old.npz gpurun_out/ab_new.npz
FEMI_PROLOGUE_BENCH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/pb3.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
FEMI_MESH_PROF=1 FEMI_ASM_PROF=1 timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3q.json 2> gpurun_out/c3q.err
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3q2.json 2> /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1
tail -3 gpurun_out/pytest_q.log
