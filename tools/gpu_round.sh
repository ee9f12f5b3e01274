#!/bin/bash
# Round evidence: GPU parity tests, smoke, bench lines (C5 default, C1), launch list of the
# C5 timed region (graph-level), and ncu --set full captures of the top kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --graph-profiling graph --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum \
  --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:"k_raster_tri" -s 3 -c 1 -o gpurun_out/prof_raster $CMD > gpurun_out/prof_raster.log 2>&1
KB="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
FEMI_PCG_KBENCH=1 timeout 600 $KB > gpurun_out/kb_plain.log 2>&1 && \
FEMI_PCG_KBENCH=1 timeout 900 $NCU -k regex:"k_gt|k_gu" -s 40 -c 2 -o gpurun_out/prof_solver $KB > gpurun_out/prof_solver.log 2>&1
echo done
