import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    det = d.get("detail", {})
    print(f, round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 4),
          {k: det.get(k) for k in ("solve_ms", "raster_ms", "cg_iters", "us_per_cg_iter") if k in det},
          "frac", round(d.get("roofline", {}).get("frac", 0), 3))
