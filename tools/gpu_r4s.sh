#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4s; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "size_classes or empty_ctas" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
FEMI_LIB=libfemi_check.so timeout 900 python -m pytest tests -m gpu -q -k "size_classes or empty_ctas" > $O/pytest_checked.log 2>&1; echo "pytest rc $?" >> $O/pytest_checked.log
FEMI_PCG_TIMERS=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2105_01586_b200 import femi, pipeline
from synth import make_config
from synth.generate import draw_mask, draw_unknowns
W=1024; rng=np.random.default_rng(W); c=make_config(4,W=W,H=W,seed=W)
mk=draw_mask(rng,W*W,84000); un=draw_unknowns(rng,W,W,mk,45000)
M=femi.Mesh(W,W,mk,un); S=femi.System(M)
g=pipeline.mask_values(torch.as_tensor(c['f'],device='cuda').reshape(-1),M.export()['vert_px'],S.n_u)
u=torch.empty(S.nv,dtype=torch.float64,device='cuda')
print(femi.inpaint_solve_batched([S],[g],[u],femi.cg_opts(rtol=1e-10)), S.n_u)
" > $O/rp6.txt 2>&1
echo done
