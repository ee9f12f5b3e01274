#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/bench_v_*.json
for rep in 1 2; do
FEMI_NO_HALO=1 FEMI_L2PF=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_v_base_$rep.json 2>/dev/null
FEMI_NO_HALO=1 FEMI_L2PF=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_v_pf_$rep.json 2>/dev/null
FEMI_L2PF=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_v_halopf_$rep.json 2>/dev/null
done
FEMI_NO_HALO=1 FEMI_LOOP_PROF=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e > /dev/null 2> gpurun_out/loopprof.err
echo done
