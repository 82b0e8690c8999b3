"""Generate tests/golden/fuzz/: random EinSum graphs planned, placed and
executed by the UNMODIFIED reference (oracle/_ref), as parity fixtures.

Each case is a small random DAG over labels of size 8-32 mixing the forms the
graph grammar (parse.h:5-22) has: contractions (sum/max over mul, add, sqdiff,
absdiff), broadcast element-wise joins (add, sub, mul), maps (relu, neg,
scale, exp on inputs), and unary reductions (sum/max). The reference planner
(optimize_dag + explode + place_all) picks the partitions for p in {1, 2, 4,
8} and L in {1, 2, 4}; inputs come from the reference's generate_inputs; the
fixture holds the plan, inputs, f64 and f32 outputs and transfer counters.

    python oracle/gen_fuzz.py [n_cases]
"""
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import bridge as B  # noqa: E402
from paper_2410_02682_b200.plan import Plan  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fuzz")
LABELS = "ijklmn"


def rand_graph(rng: random.Random, sizes=(8, 16, 32), max_elems=4096) -> str:
    size = {l: rng.choice(list(sizes)) for l in LABELS}
    tensors = []  # (name, labels, is_input)
    lines = []

    def elems(ls):
        n = 1
        for l in ls:
            n *= size[l]
        return n

    def pick_labels(k):
        while True:
            ls = rng.sample(LABELS, k)
            if elems(ls) <= max_elems:
                return ls

    for n in range(rng.randint(2, 3)):
        ls = pick_labels(rng.randint(1, 3))
        name = f"X{n}"
        tensors.append((name, ls, True))
        lines.append(f"input {name}:[{','.join(str(size[l]) for l in ls)}]")

    def ref(t):
        return f"{t[0]}[{','.join(t[1])}]"

    made = 0
    tries = 0
    while made < rng.randint(2, 5) and tries < 200:
        tries += 1
        kind = rng.choice(["contract", "contract", "ewise", "map", "reduce"])
        name = f"V{made}"
        if kind == "contract":
            a, b = rng.choice(tensors), rng.choice(tensors)
            shared = [l for l in a[1] if l in b[1]]
            union = list(dict.fromkeys(a[1] + b[1]))
            if not shared or len(union) > 4:
                continue
            agg = [l for l in shared if rng.random() < 0.8] or shared[:1]
            out = [l for l in union if l not in agg]
            if not out or elems(out) > max_elems:
                continue
            rng.shuffle(out)
            aggop, join = rng.choice([("sum", "mul"), ("sum", "mul"), ("sum", "add"), ("sum", "sqdiff"),
                                      ("max", "absdiff"), ("max", "mul")])
            lines.append(f"{name}[{','.join(out)}] = {aggop}[{','.join(agg)}] {join}({ref(a)}, {ref(b)})")
            tensors.append((name, out, False))
        elif kind == "ewise":
            a = rng.choice(tensors)
            subs = [t for t in tensors if t is not a and set(t[1]) <= set(a[1]) and t[1]]
            if not subs:
                continue
            b = rng.choice(subs)
            join = rng.choice(["add", "sub", "mul"])
            x, y = (a, b) if rng.random() < 0.7 else (b, a)
            out = list(a[1])
            lines.append(f"{name}[{','.join(out)}] = {join}({ref(x)}, {ref(y)})")
            tensors.append((name, out, False))
        elif kind == "map":
            a = rng.choice(tensors)
            op = rng.choice(["relu", "neg", "scale(0.5)"] + (["exp"] if a[2] else []))
            lines.append(f"{name}[{','.join(a[1])}] = map {op}({ref(a)})")
            tensors.append((name, list(a[1]), False))
        else:
            a = rng.choice([t for t in tensors if len(t[1]) >= 2] or [None])
            if a is None:
                continue
            k = rng.randint(1, len(a[1]) - 1)
            agg = rng.sample(a[1], k)
            out = [l for l in a[1] if l not in agg]
            op = rng.choice(["sum", "max"])
            lines.append(f"{name}[{','.join(out)}] = {op}[{','.join(agg)}] map identity({ref(a)})")
            tensors.append((name, out, False))
        made += 1
    if made == 0:
        return None
    outs = [tensors[-1][0]]
    others = [t[0] for t in tensors[:-1] if not t[2]]
    if others and rng.random() < 0.4:
        outs.append(rng.choice(others))
    for o in outs:
        lines.append(f"output {o}")
    return "\n".join(lines) + "\n"


def main():
    n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    os.makedirs(OUT, exist_ok=True)
    rng = random.Random(20261017)
    k = made = 0
    while made < n_cases and k < 20 * n_cases:
        k += 1
        text = rand_graph(rng)
        if text is None:
            continue
        p = rng.choice([1, 2, 4, 8])
        L = rng.choice([1, 2, 4])
        try:
            doc = B.ref_plan_json(text, p, L)
        except Exception:
            continue
        plan = Plan.from_json(doc)
        seed = 100 + made
        g = doc["graph_text"]
        ins = {vid: B.ref_generate_input(g, seed, vid, plan.vertices[vid].bound) for vid in plan.input_vertices()}
        try:
            o64, _, cnt, tot = B.ref_execute(doc, ins, threaded=False, f32=False)
            o32, _, _, _ = B.ref_execute(doc, ins, threaded=False, f32=True)
        except Exception:
            continue
        if any(not np.all(np.isfinite(a)) for a in list(o64.values()) + list(o32.values())):
            continue
        name = f"fuzz{made:02d}_p{p}_L{L}"
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        arrs = {f"in_{vid}": a for vid, a in ins.items()}
        arrs.update({f"out64_{vid}": a for vid, a in o64.items()})
        arrs.update({f"out32_{vid}": a for vid, a in o32.items()})
        arrs["counters"] = np.array(cnt, dtype=np.int64)
        arrs["total"] = np.array(tot, dtype=np.int64)
        np.savez_compressed(os.path.join(OUT, f"{name}_s{seed}.npz"), **arrs)
        made += 1
    print(f"{made} cases from {k} graphs")


if __name__ == "__main__":
    main()
