#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
(timeout 120 python tools/asm_bench.py 3; FEMI_ASM_PROF=1 timeout 120 python tools/asm_bench.py 3 2>/dev/null; timeout 120 python tools/asm_bench.py 4; timeout 120 python tools/asm_bench.py 1) > gpurun_out/asm.log 2>&1
echo done
