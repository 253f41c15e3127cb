"""Print the headline fields of a bench.py JSON line (log file argument)."""
import json
import sys

s = open(sys.argv[1]).read()
i = s.find('{"metric"')
d = json.loads(s[i:].split("\n")[0])
c = d["config"]
print(f"value {d['value']:.3f} {d['unit']}  ms/step {d['ms_per_step']:.1f}  roofline frac {d['roofline']['frac']:.3f} "
      f"(exec {d['roofline'].get('executed_frac', 0):.3f})  clocks {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
if d.get("e2e"):
    print(f"e2e {d['e2e']['value']:.3f}  ms {d['e2e']['ms_per_step']:.1f}")
for k in ("breakdown_ms_summed", "breakdown_ms"):
    if k in c:
        print(k, json.dumps(c[k]))
if "per_kind_level" in c:
    print(" ".join(f"{k}:{v['ms']:.0f}ms/{v['tflops_exec']:.1f}TF" for k, v in c["per_kind_level"].items() if v["ms"] > 5))
