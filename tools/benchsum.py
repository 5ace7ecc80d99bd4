"""Print the headline fields of a bench.py JSON line (last line of a log)."""
import json, signal, sys
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
e2e = d.get("e2e") or {}
print("value %.4g shots/s  ms/step %.2f  e2e %.4g  flagged %s  events %s" % (
    d["value"], d["ms_per_step"], e2e.get("value", 0), d.get("flagged_work_items"), d.get("stage_events")))
for k, v in d["kernel_ms_per_step"].items():
    print("  %-14s %s" % (k, [round(x, 2) for x in v] if isinstance(v, list) else round(v, 2)))
r = d["roofline"]
print("  roofline:", r["kernel"], "frac %.4f" % r["frac"], "fma frac %.4f" % r["fma"]["frac"], "share %.2f" % r["share_of_step"])
print("  e2e:", {k: v for k, v in e2e.items() if k not in ("timing", "unit")})
