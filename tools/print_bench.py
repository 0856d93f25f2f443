"""Print the headline fields of bench.py JSON lines: python tools/print_bench.py FILE ..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        e = d.get("e2e") or {}
        r = d.get("roofline") or {}
        c5 = d.get("config5") or {}
        print(f, "value", round(d.get("value", 0), 1), "e2e", round(e.get("value", 0), 1),
              "samples", e.get("samples_s"), "frac", round(r.get("frac", 0) or 0, 3),
              "parity", (d.get("parity") or {}).get("pass"),
              "c5", round(c5.get("value", 0), 1), "c5frac",
              round((c5.get("roofline") or {}).get("frac", 0) or 0, 3),
              "clocks", (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
