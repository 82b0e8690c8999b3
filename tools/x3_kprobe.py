"""fp32x3 error growth with K (tools/probe_plans/kprobe_K.json: 256 x K x 256,
one join): linear growth in K of the error relative to sum|x||y| points at
truncating accumulation inside the tensor core, sqrt(K) at round-to-nearest."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_02682_b200.executor import Context, execute
from paper_2410_02682_b200.plan import Plan

ctx = Context(0)
rng = np.random.default_rng(3)
for K in (32, 256, 2048, 16384):
    plan = Plan.load(os.path.join(ROOT, "tools", "probe_plans", f"kprobe_{K}.json"))
    x = rng.uniform(-1, 1, (256, K))
    y = rng.uniform(-1, 1, (K, 256))
    ins = {plan.find("X"): x, plan.find("Y"): y}
    want = x @ y
    S = np.abs(x) @ np.abs(y)
    x32, y32 = x.astype(np.float32).astype(np.float64), y.astype(np.float32).astype(np.float64)
    want32 = x32 @ y32
    # sequential fp32 RN accumulation (what the reference's f32 mode does), 32 rows
    seq = np.zeros((32, 256), dtype=np.float32)
    for j in range(K):
        seq = (seq + (x32[:32, j:j + 1].astype(np.float32) * y32[j:j + 1, :].astype(np.float32))).astype(np.float32)
    for prec in ("fp32x3", "tf32"):
        got = execute(plan, ins, precision=prec, ctx=ctx).outputs[plan.outputs[0]]
        e = np.abs(got - want32)
        print(f"K={K:6d} {prec:7s} max|err|/S {np.max(e / S):.3e} mean(err/S) {np.mean(e / S):.3e} "
              f"mean signed (got-want)/S {np.mean((got - want32) / S):+.3e} max_rel_err {np.max(e / np.maximum(1, np.abs(want32))):.3e}",
              flush=True)
    es = np.abs(seq - want32[:32])
    print(f"K={K:6d} seqfp32 max|err|/S {np.max(es / S[:32]):.3e} mean(err/S) {np.mean(es / S[:32]):.3e} "
          f"max_rel_err {np.max(es / np.maximum(1, np.abs(want32[:32]))):.3e}", flush=True)
