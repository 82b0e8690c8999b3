"""Kernels each case of tests/test_gpu_fusion_fuzz.py launches (bf16): which fused."""
import sys, random; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import test_gpu_fusion_fuzz as T
from oracle import bridge as B
from paper_2410_02682_b200.plan import Plan
from paper_2410_02682_b200.executor import Context, PreparedPlan
ctx=Context(0)
for i,kind,p,L in T.CASES:
    rng=random.Random(1000+i)
    text,f=T.attention_text(rng) if kind=="attention" else T.ffnn_text(rng)
    doc=B.ref_plan_json(text,p,L); plan=Plan.from_json(doc)
    pp=PreparedPlan(ctx,plan,precision="bf16",profile=True)
    pp.generate_inputs(1); pp.run()
    names=[k["name"].split(":")[0] for k in pp.kernel_stats()]
    pp.close()
    print(i,kind,p,L,"fused" if f in names else "UNFUSED", sorted(set(names)))
