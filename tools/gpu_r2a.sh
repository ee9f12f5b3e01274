#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rA -s -k "c5_legs or config2 or config3" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_sanitize.sh
echo done
