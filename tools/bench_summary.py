import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    r=d["roofline"]
    print(f, "ms", round(d["ms_per_step"],3), "TF", round(d["value"],2), "top", r["kernel"], round(r["launch_ms"],3), "frac", round(r["frac"],3), d["config"]["breakdown_ms"], "e2e", d["e2e"] and round(d["e2e"]["ms_per_step"],2))
