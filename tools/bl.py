"""Print the key fields of a bench JSON line (last line of a log)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline", {})
    pk = {k: (round(v["ms_per_step"], 3), round(v.get("frac") or 0, 3)) for k, v in r.get("per_kernel", {}).items()
          if v.get("ms_per_step")}
    print(path, "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "comp",
          round(d.get("compress_GBps", 0), 1), "decomp", round(d.get("decompress_GBps", 0), 1),
          "hbm_step", round(d.get("hbm_frac_step", 0), 3), pk, d.get("clocks", {}).get("reasons"))
