"""Per-exec-vertex comparison of a bf16 run against the fp64 dense graph:
python tools/debug_vertices.py <plan> [prec]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from test_gpu_fullsize import _inputs, _dense_fp64
from paper_2410_02682_b200.plan import Plan
from paper_2410_02682_b200.executor import Context, PreparedPlan, EdError
name = sys.argv[1]; prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
plan = Plan.load(f"plans/{name}.json")
ins = _inputs(plan)
ctx = Context(0)
pp = PreparedPlan(ctx, plan, precision=prec)
pp.upload(ins); pp.run()
vals = _dense_fp64(plan, ins, torch)
seen = set()
for u in plan.exec:
    if u.kind == 0: continue
    v = plan.vertices[u.producer]
    try:
        got = torch.from_numpy(pp.download_chunk(u.id)).cuda()
    except EdError as e:
        continue
    full = vals[u.producer]
    if u.kind == 2:
        # region of the consumer partition
        part = [b // c for b, c in zip(v.bound, u.chunk_bound)]
    else:
        part = None
    if u.kind == 1:
        e = v.expr
        dls = e.distinct_labels()
        zk = [u.key[dls.index(l)] for l in e.out]
        key = zk
    else:
        key = u.key
    sl = tuple(slice(k * c, (k + 1) * c) for k, c in zip(key, u.chunk_bound))
    want = full[sl]
    if u.kind == 1 and e.agg is not None and any(dls.index(l) >= 0 and l not in e.out for l in dls):
        # join partial of an aggregation: skip exact compare
        tag = "partial"
    else:
        tag = ""
    err = float(((got - want).abs().max() / want.abs().max().clamp(min=1e-30)).item())
    if (u.producer, u.kind) not in seen or err > 1e-2:
        print(f"{v.name:8s} id={u.id:4d} kind={u.kind} key={u.key} err={err:.3e} {tag}", flush=True)
        seen.add((u.producer, u.kind))
