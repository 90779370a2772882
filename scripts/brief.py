"""Summarise bench.py JSON lines from stdin: value, e2e, per-kernel avg us."""
import json, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    k = {n: (v["avg_us"], v["launches"], v["achieved_gbs"]) for n, v in d.get("kernels", {}).items()}
    print(tag, "value", d["value"], "e2e", (d.get("e2e") or {}).get("value"), "solve", d.get("solve"))
    print(tag, "roofline", d.get("roofline"))
    print(tag, "kernels", k, flush=True)
