"""profiles/traffic.json from an ncu launch list of the C5 timed region (--graph-profiling graph,
dram__bytes_read.sum / dram__bytes_write.sum): the mean DRAM bytes of one solve-graph launch
and of one raster launch. Usage: python tools/update_traffic.py <launches.csv> <iters>"""
import csv
import json
import os
import sys

src, iters = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
h, data = rows[0], rows[1:]
iN, iM, iV, iI = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launches = {}
for r in data:
    launches.setdefault((int(r[iI]), r[iN]), {})[r[iM]] = float(r[iV].replace(",", ""))
graph = [v for (i, k), v in launches.items() if k == "graph"]
raster = [v for (i, k), v in launches.items() if "k_raster" in k]
gb = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in graph) / len(graph)
rb = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in raster) / len(raster)
out = {"C5": {"solve_graph_bytes_per_launch": int(gb), "solve_graph_bytes_per_iter": int(gb / iters),
              "raster_bytes_per_launch": int(rb), "iters": iters,
              "source": f"ncu --graph-profiling graph --metrics dram__bytes_read.sum,dram__bytes_write.sum over the "
                        f"bench.py C5 timed region ({os.path.relpath(src)}), mean of {len(graph)} solve-graph and "
                        f"{len(raster)} raster launches"}}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                 "traffic.json"), "w"), indent=1)
print(out)
