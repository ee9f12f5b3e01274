"""Per-stage host split of C3 runs (FEMI_MESH_PROF / FEMI_ASM_PROF stamps aggregated): runs
tools/diag_c3_host.py in a child with the stamps on and sums each stage's increments.
    python tools/diag_c3_stages.py [reps]"""
import collections
import os
import re
import subprocess
import sys

reps = sys.argv[1] if len(sys.argv) > 1 else "3"
env = dict(os.environ, FEMI_MESH_PROF="1", FEMI_ASM_PROF=os.environ.get("FEMI_ASM_PROF", "1"))
p = subprocess.run([sys.executable, "tools/diag_c3_host.py", reps], env=env, capture_output=True, text=True)
print(p.stdout)
tot = collections.OrderedDict()
prev = {}
calls = collections.Counter()
for line in p.stderr.splitlines():
    m = re.match(r"(mesh_insert|mesh_build|assemble)\s+(\S+)\s+([\d.]+) (ms|s)", line)
    if not m:
        continue
    kind, stage, v, unit = m.groups()
    v = float(v) * (1e3 if unit == "s" else 1.0)
    key = (kind, stage)
    first = stage in ("renumber", "order", "uploads") if kind != "mesh_build" else stage == "order"
    d = v if first else v - prev.get(kind, 0.0)
    prev[kind] = v
    tot[key] = tot.get(key, 0.0) + d
    calls[key] += 1
runs = int(reps) + 2
for (kind, stage), v in tot.items():
    print(f"{kind:12s} {stage:12s} {v / runs:8.3f} ms/run  ({calls[(kind, stage)] // runs} calls/run)")
