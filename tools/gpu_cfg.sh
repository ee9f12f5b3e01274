#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in 2 3 4; do timeout 600 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c5t.json 2> gpurun_out/bench_c5t.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
