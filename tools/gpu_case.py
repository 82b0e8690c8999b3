"""Run one parity case in isolation (debug helper): python tools/gpu_case.py <plan> <prec> [seed]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bridge as B
from paper_2410_02682_b200.plan import Plan
from paper_2410_02682_b200.executor import execute, Context

name, prec = sys.argv[1], sys.argv[2]
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 7
plan = Plan.load(f"plans/{name}.json")
ins = B.generate_inputs(plan, seed)
want, _, _, _ = B.oracle_execute(plan, ins)
ctx = Context(0)
try:
    rep = execute(plan, ins, precision=prec, ctx=ctx)
except Exception as e:
    print(f"CASE {name} {prec}: ERROR {e}")
    sys.exit(1)
errs = {v: B.max_rel_err(rep.outputs[v], want[v]) for v in want}
exact = all(np.array_equal(rep.outputs[v], want[v]) for v in want)
print(f"CASE {name} {prec}: exact={exact} err={max(errs.values()):.3e} launches={rep.gpu_launches}")
