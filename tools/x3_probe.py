"""fp32x3 accuracy probe: real-valued U[-1,1) inputs through GEMM-shaped plans,
max_rel_err / normwise vs fp64 for tf32 and fp32x3 (kCta 1 / 2, K-major /
MN-major operands)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_plan
from paper_2410_02682_b200.executor import Context, execute
import tolerance as T

ctx = Context(0)
rng = np.random.default_rng(5)
for name in ["gemm_nn_p1_L1", "gemm_tn_p1_L1", "gemm_nt_p1_L1", "gemm_batch_p1_L1", "gemm_ragged_p1_L1",
             "chain3_s_p8_L1", "bmm2_s_p8_L1", "hoc_s_p8_L1"]:
    plan = load_plan(name)
    ins = {vid: rng.uniform(-1, 1, size=plan.vertices[vid].bound) for vid in plan.input_vertices()}
    want = execute(plan, ins, precision="fp64", ctx=ctx).outputs
    line = [name]
    for prec in ("tf32", "fp32x3"):
        got = execute(plan, ins, precision=prec, ctx=ctx).outputs
        e = max(T.max_rel_err(got[v], want[v]) for v in want)
        n = max(T.normwise(got[v], want[v]) for v in want)
        line.append(f"{prec}: mre {e:.2e} nw {n:.2e}")
    print("  ".join(line), flush=True)
