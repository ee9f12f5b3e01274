#!/bin/bash
# C3 host path: stage split after the mesh-table rework (vt without atomics, one-pass CSR, corner-local neighbour test)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/r3k2
timeout 300 python tools/diag_c3_host.py 5 > gpurun_out/r3k2/c3_split.txt 2>&1
FEMI_ASM_PROF=2 timeout 300 python tools/diag_c3_stages.py 3 > gpurun_out/r3k2/stages_host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "config3 or densify or mesh or inpaint or config1 or band" > gpurun_out/r3k2/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3k2/pytest.log
echo done
