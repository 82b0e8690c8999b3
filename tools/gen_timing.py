"""Time ed_generate_inputs (device) against the host generate_inputs restatement
on a config's inputs (host timed on a bounded sample, extrapolated)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bridge as B
from paper_2410_02682_b200.executor import Context, PreparedPlan
from paper_2410_02682_b200.plan import Plan

ctx = Context(0)
for name in sys.argv[1:]:
    plan = Plan.load(f"plans/{name}_p8_L1.json")
    n = sum(plan.numel(v) for v in plan.input_vertices())
    pp = PreparedPlan(ctx, plan, precision="bf16")
    pp.generate_inputs(1)
    t0 = time.perf_counter()
    pp.generate_inputs(2)
    dev = time.perf_counter() - t0
    pp.close()
    k = 20_000_000
    t0 = time.perf_counter()
    B.oracle_generate_input(k, plan.integer_valued(), 2, 0)
    host = (time.perf_counter() - t0) * n / k
    print(f"{name}: {n / 1e6:.0f} M values; device {dev:.3f} s ({n / dev / 1e9:.2f} G values/s); "
          f"host (1 thread, libstdc++) ~{host:.1f} s extrapolated; speed-up {host / dev:.0f}x")
