import json, sys
for c in sys.argv[1:]:
    d = json.load(open(c))
    print(c, "value %.1f ms %.3f" % (d["value"], d["ms_per_step"]), "roof frac %.3f achieved %.0f" % (d["roofline"]["frac"], d["roofline"]["achieved"]),
          "e2e", round(d["e2e"]["value"], 1) if d.get("e2e") else None, "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    for k, v in d["kernels"].items():
        print("   %-11s n=%2d ms=%.3f share=%.2f GBps=%.0f" % (k, v["launches_per_step"], v["ms_per_step"], v["share"], v["algorithmic_GBps"]))
    if "-v" in sys.argv[0:1]:
        pass
    pl = d["per_launch_ms"]; print("   per launch:", " ".join("%s:%.3f" % (p[:2], x) for p, x in zip(d["plan"], pl) if p in ("level", "last_level", "pair", "hist")))
