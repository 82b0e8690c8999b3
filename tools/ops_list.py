import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import load_plan
from oracle import bridge as B
from paper_2410_02682_b200.executor import Context, PreparedPlan
ctx = Context(0)
for name in sys.argv[1:]:
    plan = load_plan(name)
    pp = PreparedPlan(ctx, plan, precision="bf16", profile=True)
    pp.upload(B.generate_inputs(plan, 1))
    pp.run()
    print(name, [s["name"] for s in pp.kernel_stats()])
    pp.close()
