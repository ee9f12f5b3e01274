#!/bin/bash
# row-band path: GPU band tests (default + device-checked build), band bench (R = 1, 4 lockstep), whole GPU suite, smoke
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/r3h
timeout 900 python -m pytest tests/test_band.py -m gpu -q -x -rA > gpurun_out/r3h/pytest_band.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3h/pytest_band.log
FEMI_LIB=libfemi_check.so timeout 900 python -m pytest tests/test_band.py -m gpu -q -x > gpurun_out/r3h/pytest_band_chk.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3h/pytest_band_chk.log
timeout 600 python bench.py --band --steps 3 --warmup 1 > gpurun_out/r3h/bench_band1.json 2> gpurun_out/r3h/bench_band1.err
timeout 600 python bench.py --band --bands 4 --steps 3 --warmup 1 > gpurun_out/r3h/bench_band4.json 2> gpurun_out/r3h/bench_band4.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3h/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3h/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/r3h/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r3h/smoke.log
echo done
