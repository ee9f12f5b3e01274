#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FEMI_DEBUG=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
FEMI_DEBUG=1 FEMI_JNS=8 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_q8.json 2> gpurun_out/bench_q8.err
FEMI_PDL_PRE=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_qp0.json 2> gpurun_out/bench_qp0.err
FEMI_GU_CTAS=296 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_qg2.json 2> gpurun_out/bench_qg2.err
FEMI_GU_CTAS=888 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_qg6.json 2> gpurun_out/bench_qg6.err
echo done
