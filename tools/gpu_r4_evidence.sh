#!/bin/bash
# Round-2 final evidence (session 3): GPU parity suite (default + device-checked builds), smoke,
# the driver's C5 bench line, the reference arm, C1-C4 / C6 / C3 variants, C5 loop timeline, the
# graph-level launch list of the C5 timed region with DRAM bytes, the resident solver's phase
# timers, and ncu --set full of k_raster_grp, k_gur/k_gt (standalone) and k_cgs (C4, C2).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/${EVDIR:-ev}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
nproc >> $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
FEMI_LIB=libfemi_check.so timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu_checked.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
for c in 2 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_c$c.json 2> $O/bench_c$c.err; done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --warm > $O/bench_c3w.json 2> $O/bench_c3w.err
timeout 900 python bench.py --config 3 --n 100 --warm --steps 2 --warmup 1 > $O/bench_c3_n100w.json 2> $O/bench_c3_n100w.err
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 > $O/bench_c6.json 2> $O/bench_c6.err
timeout 300 python tools/diag_c3_host.py 5 > $O/c3_host_split.txt 2>&1
FEMI_PCG_TIMERS=1 timeout 300 python tools/diag_cgr.py 1,2,3,4 5 > $O/cgs_timers.txt 2>&1
timeout 300 python tools/diag_cgr.py 1,2,3,4 > $O/cgs_solve_times.txt 2>&1
FEMI_LOOP_PROF=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-tonal --steps 2 --warmup 3 > $O/loop.json 2> $O/loop.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
timeout 900 ncu --graph-profiling graph --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum \
  --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:"k_raster_grp" -s 3 -c 1 -o $O/prof_raster $CMD > $O/prof_raster.log 2>&1
FEMI_PCG_KBENCH=1 timeout 900 $NCU -k regex:"k_gur|k_gt" -s 8 -c 2 -o $O/prof_body $CMD > $O/prof_body.log 2>&1
timeout 900 $NCU -k regex:"k_cgs" -s 2 -c 1 -o $O/prof_cgs_c4 python tools/diag_cgr.py 4 1 > $O/prof_cgs_c4.log 2>&1
timeout 900 $NCU -k regex:"k_cgs" -s 2 -c 1 -o $O/prof_cgs_c2 python tools/diag_cgr.py 2 1 > $O/prof_cgs_c2.log 2>&1
echo done
