import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith("{"):
        d=json.loads(l); print(d["config"]["workload"], round(d["ms_per_step"],4), {k[:8]:round(v,4) for k,v in (d.get("kernels_ms") or {}).items()}, round(d["roofline"]["frac"],3))
