import json, sys
for f in sys.argv[1:]:
    for ln in open(f):
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        print(f, "ms %.2f" % d["ms_per_step"], "GF/s %.0f" % d.get("gflops_tile", 0),
              "roof %.3f" % d.get("fp64_roofline", {}).get("frac", 0), "e2e ms %.1f" % d.get("e2e", {}).get("ms_per_step", 0), "kernel TF/s %.2f" % d.get("roofline", {}).get("achieved", 0))
        for k, v in (d.get("profile") or d.get("profile_direct") or {}).items():
            print("   %-14s %8.2f ms %6d launches %7.1f us/launch %8.2f GF  %6.2f TF/s" % (
                k, v["ms"], v["launches"], 1e3 * v["ms"] / v["launches"], v["gflop"], v["gflop"] / max(v["ms"], 1e-9)))
