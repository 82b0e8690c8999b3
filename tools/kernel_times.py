"""Per-launch-class device times of a plan on one GPU (profile mode).

usage: python tools/kernel_times.py PLAN [runs] [precision]   (ED_LIB_PATH selects a variant build)
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_plan
from paper_2410_02682_b200.executor import Context, PreparedPlan

name = sys.argv[1]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = Context(0)
plan = load_plan(name)
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
pp = PreparedPlan(ctx, plan, precision=prec, profile=True)
pp.generate_inputs(1)
for _ in range(3):
    pp.run()
tot = {}
for _ in range(runs):
    pp.run()
    for k in pp.kernel_stats():
        tot[k["name"]] = tot.get(k["name"], 0.0) + k["ms"] / runs
print(name, os.path.basename(os.environ.get("ED_LIB_PATH", "libed_gpu.so")),
      f"total={sum(tot.values()):.4f}",
      " ".join(f"{n}={v:.4f}" for n, v in sorted(tot.items(), key=lambda x: -x[1])[:int(os.environ.get('KT_TOP', '4'))]))
pp.close()
