#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4v; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "cluster_size_switch" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
FEMI_LIB=libfemi_check.so timeout 900 python -m pytest tests -m gpu -q -k "cluster_size_switch" > $O/pytest_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_checked.log
echo done
