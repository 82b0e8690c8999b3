"""Generate tests/golden/ from the UNMODIFIED reference (oracle/_ref).

Fixtures:
  kat.json            known-answer vectors quoted from the reference's own tests
                      (test_relation.cc:36-61, 98-124; test_einsum.cc:78-106)
  <graph>_p<p>_L<L>_s<seed>.npz
                      inputs (generate_inputs), reference execute() outputs in
                      f64 and f32 mode, per-machine counters, total transferred

    python oracle/gen_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import bridge as B  # noqa: E402
from paper_2410_02682_b200.plan import Plan  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# (plan file, seed): the acceptance matrix's seed rule 1000+10p+L
# (acceptance.cc:207) plus test_runtime.cc's seeds
CASES = []
for g in ["matmul", "ffnn", "softmax", "attention"]:
    for p in (1, 4, 8):
        for L in (1, 2, 4):
            CASES.append((f"{g}_p{p}_L{L}", 1000 + 10 * p + L))
CASES += [("matmul8_pinned_L16", 5), ("chain8_pinned_L2", 7), ("chain8_pinned_L4", 7), ("chain8_pinned_L8", 7)]
for g in ["sqdiff", "absmax", "mix"]:
    for p in (1, 2, 4):
        CASES.append((f"{g}_p{p}_L2", 41))
CASES += [("attention_p8_L4", 17), ("ffnn_p4_L2", 23), ("matmul_p4_L2", 29)]


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, seed in CASES:
        doc = json.load(open(os.path.join(ROOT, "plans", name + ".json")))
        plan = Plan.from_json(doc)
        g = doc["graph_text"]
        ins = {vid: B.ref_generate_input(g, seed, vid, plan.vertices[vid].bound) for vid in plan.input_vertices()}
        o64, _, cnt, tot = B.ref_execute(doc, ins, threaded=False, f32=False)
        o32, _, _, _ = B.ref_execute(doc, ins, threaded=False, f32=True)
        ev = B.ref_eval_reference(doc, ins)
        arrs = {}
        for vid, a in ins.items():
            arrs[f"in_{vid}"] = a
        for vid, a in o64.items():
            arrs[f"out64_{vid}"] = a
            arrs[f"oracle_{vid}"] = ev[vid]
        for vid, a in o32.items():
            arrs[f"out32_{vid}"] = a
        arrs["counters"] = np.array(cnt, dtype=np.int64)
        arrs["total"] = np.array(tot, dtype=np.int64)
        arrs["seed"] = np.array(seed)
        np.savez_compressed(os.path.join(OUT, f"{name}_s{seed}.npz"), **arrs)
    kat = {
        "source": "reference tests, quoted",
        "kernel_eval_matmul": {"cite": "test_relation.cc:98-106", "x": [1, 2, 3, 4], "y": [5, 6, 7, 8],
                               "out": [19, 22, 43, 50], "fp": 8},
        "kernel_eval_relu": {"cite": "test_relation.cc:108-115", "x": [-1, 2], "out": [0, 2]},
        "kernel_eval_elementwise_mul": {"cite": "test_relation.cc:117-124", "x": [2], "y": [3], "out": [6]},
        "matmul_1x1": {"cite": "test_einsum.cc:78-87", "x": [3], "y": [4], "out": 12},
        "sqdiff_sum": {"cite": "test_einsum.cc:89-99", "x": [1, 2, 3, 4], "y": [5, 6, 7, 8],
                       "out": [41, 61, 13, 25]},
        "absdiff_max": {"cite": "test_einsum.cc:101-106", "x": [1, 2, 3, 4], "y": [5, 6, 7, 8],
                        "out": [5, 6, 3, 4]},
        "matrix_u": {"cite": "test_relation.cc:13-19",
                     "values": [1, 2, 5, 6, 3, 4, 7, 8, 9, 10, 13, 14, 11, 12, 15, 16]},
        "chunk_u_2x4": {"cite": "test_relation.cc:36-47",
                        "keys": {"0,0": [1, 3], "0,1": [2, 4], "0,2": [5, 7], "1,3": [14, 16]}},
        "chunk_u_2x2": {"cite": "test_relation.cc:49-55",
                        "keys": {"0,0": [1, 2, 3, 4], "0,1": [5, 6, 7, 8], "1,0": [9, 10, 11, 12],
                                 "1,1": [13, 14, 15, 16]}},
    }
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    print(f"wrote {len(CASES)} fixtures + kat.json to {OUT}")


if __name__ == "__main__":
    main()


def artifacts():
    """tests/golden/artifacts/: the reference's own taskgraph/1 + execgraph/1
    (json_io.cc) for plan-ingestion tests."""
    out = os.path.join(OUT, "artifacts")
    os.makedirs(out, exist_ok=True)
    for name in ["attention_p8_L4", "ffnn_p4_L2", "chain8_pinned_L4", "attn_big_p8_L8", "bmm2_repart_p8_L2"]:
        doc = json.load(open(os.path.join(ROOT, "plans", name + ".json")))
        tg, eg = B.ref_artifacts(doc["graph_text"], doc["p"], doc["n_machines"], doc["alpha"], doc.get("pinned"))
        json.dump(tg, open(os.path.join(out, name + ".taskgraph.json"), "w"))
        json.dump(eg, open(os.path.join(out, name + ".execgraph.json"), "w"))


if __name__ == "__main__" and "--artifacts" in sys.argv:
    artifacts()
