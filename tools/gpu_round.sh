#!/bin/bash
# Round evidence: GPU parity tests, smoke, bench lines (C5 default, C1-C4, C6 colour, C3 warm,
# reference arm), loop timeline, launch list of the C5 timed region (graph-level), ncu --set
# full captures of the SpMV (k_gt<FIRST>, a graph node outside the WHILE body), the raster and
# the resident solver (C2).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --warm > gpurun_out/bench_c3w.json 2> gpurun_out/bench_c3w.err
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --n 30 --warm > gpurun_out/bench_c3nw.json 2> gpurun_out/bench_c3nw.err
timeout 300 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err
FEMI_LOOP_PROF=1 timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tonal --steps 2 --warmup 3 > gpurun_out/loop.json 2> gpurun_out/loop.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --graph-profiling graph --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum \
  --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
FEMI_PCG_KBENCH=1 timeout 900 $NCU -k regex:"k_gu|k_gt" -s 8 -c 2 -o gpurun_out/prof_body $CMD > gpurun_out/prof_body.log 2>&1
timeout 900 $NCU -k regex:"k_raster_tri" -s 3 -c 1 -o gpurun_out/prof_raster $CMD > gpurun_out/prof_raster.log 2>&1
timeout 900 $NCU -k regex:"k_cgr" -s 1 -c 1 -o gpurun_out/prof_cgr python bench.py --config 2 --steps 1 --warmup 1 > gpurun_out/prof_cgr.log 2>&1
echo done
