import json, sys
for c in (3, 4, 5):
    for pre in sys.argv[1:]:
        try:
            d = json.load(open(f"gpurun_out/{pre}_cfg{c}.json"))
        except Exception as e:  # noqa: BLE001
            print(c, pre, "ERR", e)
            continue
        print(c, pre, round(d["value"], 1), round(d["ms_per_step"], 3),
              {k: (round(v["ms_per_step"], 3), v["launches_per_step"]) for k, v in d["kernels"].items()})
