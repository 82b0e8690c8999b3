"""Comm / compute overlap of the peer transport, one process driving WORLD
ranks on one GPU (ed_ctx_create_multi with the device repeated): per rank,
the receive copies (on the comm stream) against what the compute stream
waited for them, and the step time. A functional view of the N > 1 path on a
single B200 — the ranks share its SMs and HBM, so times are not throughput.

usage: python tools/peer_overlap.py PLAN WORLD [precision] [runs]
       (ED_PEER_PREFETCH=0: each receive at its consumer, the previous schedule)
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_plan
from paper_2410_02682_b200.executor import Context, PreparedPlan

name, world = sys.argv[1], int(sys.argv[2])
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 5
plan = load_plan(name)
ctx = Context.multi([0] * world)
out = {"plan": name, "world": world, "precision": prec, "prefetch": os.environ.get("ED_PEER_PREFETCH", "1") != "0"}
pp = PreparedPlan(ctx, plan, precision=prec, transport="peer")
pp.generate_inputs(1)
for _ in range(2):
    pp.run()
ms = []
for _ in range(runs):
    ms.append(pp.run().device_ms)
rep = pp.run()
out["step_ms"] = sorted(ms)[len(ms) // 2]
out["peer_bytes_per_step"] = rep.peer_bytes
pp.close()
pp = PreparedPlan(ctx, plan, precision=prec, transport="peer", profile=True)
pp.generate_inputs(1)
for _ in range(2):
    pp.run()
pp.run()
ranks = {}
for k in pp.kernel_stats():
    r, sep, n = k["name"].partition("/")
    if not sep:
        continue  # summed over ranks
    d = ranks.setdefault(r, {"copy_ms": 0.0, "copy_bytes": 0.0, "exposed_ms": 0.0, "compute_ms": 0.0})
    if n == "peer_recv_copy":
        d["copy_ms"] += k["ms"]
        d["copy_bytes"] += k["bytes"]
    elif n.startswith("nccl_recv"):
        d["exposed_ms"] += k["ms"]
    elif not n.startswith("nccl_send"):
        d["compute_ms"] += k["ms"]
for d in ranks.values():
    d["hidden_frac"] = 1 - d["exposed_ms"] / d["copy_ms"] if d["copy_ms"] > 0 else None
out["ranks"] = ranks
pp.close()
ctx.close()
print(json.dumps(out))
