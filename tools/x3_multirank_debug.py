"""fp32x3 across L in-process ranks on one GPU vs the f64 golden, per output
and per env variant (debug aid for the multi-rank lo-shadow paths)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
from conftest import load_golden, load_plan
import tolerance as T
from paper_2410_02682_b200.executor import Context, PreparedPlan
case, world, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
import os
name, ins, o64, o32, orc, counters, total = load_golden(case)
plan = load_plan(name)
ctx = Context.multi([0] * world) if world > 1 else Context(0)
import os
pp = PreparedPlan(ctx, plan, precision=prec, profile=os.environ.get("XMR_PROF") == "1",
                  graph=os.environ.get("XMR_NOGRAPH") != "1")
pp.upload(ins); pp.run(); outs = pp.download()
bad = []
for vid, w in o64.items():
    m, e, b = T.error(prec, outs[vid], w)
    if e > b: bad.append((vid, e))
print("BAD", len(bad), "of", len(o64), bad[:6])
pp.close(); ctx.close()
''' % (ROOT, os.path.join(ROOT, "tests"))

for case, world in [("attention_p8_L4_s1084", 4), ("softmax_p8_L4_s1084", 4), ("chain8_pinned_L8_s7", 8),
                    ("ffnn_p4_L2_s23", 2), ("mix_p4_L2_s41", 2)]:
    for tag, env in [("base", {}), ("w1", None), ("lo_epi0", {"ED_X3_LO_EPI": "0"}),
                     ("direct0", {"ED_PEER_DIRECT": "0"}), ("prefetch0", {"ED_PEER_PREFETCH": "0"}),
                     ("nograph", {"XMR_NOGRAPH": "1"}), ("profile", {"XMR_PROF": "1"})]:
        e = dict(os.environ, **(env or {}))
        try:
            r = subprocess.run([sys.executable, "-c", CHILD, case, "1" if env is None else str(world), "fp32x3"],
                               env=e, capture_output=True, text=True, timeout=120)
        except subprocess.TimeoutExpired:
            print(f"{case} L{world} {tag}: TIMEOUT", flush=True)
            continue
        out = (r.stdout + r.stderr[-600:]).strip().replace("\n", " | ")
        print(f"{case} L{world} {tag}: {out}", flush=True)
