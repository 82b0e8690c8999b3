"""Print one line per bench JSON log: value, step, clocks, per-kernel ms."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unparsable:", e)
        continue
    ks = [(k["name"], round(k["ms"], 4)) for k in d["roofline"]["kernels"]]
    print(d["config"]["graph"], round(d["value"], 1), "TFLOP/s", round(d["ms_per_step"], 4), "ms",
          "frac", round(d["config"]["frac_of_peak"], 3), "gemm", round(d["roofline"]["achieved"], 1),
          "e2e", round(d["e2e"]["value"], 1), "clk", d["clocks"].get("sm_mhz"), ks[:8])
