"""Fused attention kernel time on attn_big with two input distributions:
the reference's integer stream (logits ~1e5: rescales of O nearly every
block) and unit-variance activations (logits O(1), as in a trained model;
rescales rare). Profile mode, CUDA events, mean of `runs`.

    python tools/attn_data_probe.py [runs]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_plan  # noqa: E402
from paper_2410_02682_b200.executor import Context, PreparedPlan  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx = Context(0)
plan = load_plan("attn_big_p8_L1")
pp = PreparedPlan(ctx, plan, precision="bf16", profile=True)


def timed(label):
    for _ in range(3):
        pp.run()
    tot = {}
    for _ in range(runs):
        pp.run()
        for k in pp.kernel_stats():
            tot[k["name"]] = tot.get(k["name"], 0.0) + k["ms"] / runs
    att = {k: v for k, v in tot.items() if k.startswith("attention")}
    print(label, " ".join(f"{k}={v:.4f}" for k, v in att.items()), flush=True)


pp.generate_inputs(1)
timed("reference-stream")
rng = np.random.default_rng(0)
ins = {}
for name in ("Q", "K", "V"):
    ins[plan.find(name)] = rng.standard_normal((4096, 4096), dtype=np.float32)
for name in ("WQ", "WK", "WV", "WO"):
    ins[plan.find(name)] = (rng.standard_normal((4096, 32, 128), dtype=np.float32) / 64.0).astype(np.float32)
pp.upload(ins)
timed("unit-variance")
pp.close()
