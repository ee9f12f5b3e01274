#!/bin/bash
# A/B bit identity of the fused prologue, its kernel times, the GPU suite and a bench line
mkdir -p gpurun_out
FEMI_LIB=$PWD/tmp_old/libfemi_old.so timeout 600 python tools/ab_bits.py dump gpurun_out/ab_old.npz > gpurun_out/ab.log 2>&1
timeout 600 python tools/ab_bits.py dump gpurun_out/ab_new.npz >> gpurun_out/ab.log 2>&1
python tools/ab_bits.py compare gpurun_out/ab_old.npz gpurun_out/ab_new.npz >> gpurun_out/ab.log 2>&1
rm -f gpurun_out/ab_old.npz gpurun_out/ab_new.npz
FEMI_PROLOGUE_BENCH=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tonal > /dev/null 2> gpurun_out/pb2.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_p.log 2>&1
tail -3 gpurun_out/pytest_p.log
