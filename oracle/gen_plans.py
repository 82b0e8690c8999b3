"""Emit plans/ from the UNMODIFIED reference planner (oracle/_ref).

The reference's parser, optimize_dag, explode and place_all
(runtime.cc:511-516) stay the planner; this script runs them once, here,
and stores their output as "edplan/1" JSON under plans/. The executor
(paper_2410_02682_b200) only ever reads those files — the product never
links or calls the reference.

    python oracle/gen_plans.py            # all plans
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import bridge as B  # noqa: E402

REF_GRAPHS = "/root/reference/proj/graphs"
OUT = os.path.join(ROOT, "plans")

# config graphs (graphs/*.eg); p = 8 throughout
CONFIGS = ["chain3", "bmm2", "ffnn_big", "attn_big", "hoc"]
TWINS = ["chain3_s", "bmm2_s", "ffnn_s", "attn_s", "hoc_s", "hoc_m"]  # hoc_m: bench.py's CPU-baseline sample
# C2's repartition variant: batch-sharded Z1 feeding row-sharded Z2
# (pinning precedent test_runtime.cc:58-72)
BMM2_REPART = {"Z1": [8, 1, 1, 8, 1, 1], "Z2": [1, 8, 1, 1, 1, 1]}

# test_runtime.cc's hand-pinned cases (:25-56, :58-93)
MATMUL8 = ("input X:[8,8]\ninput Y:[8,8]\n"
           "Z[i,k] = sum[j] mul(X[i,j], Y[j,k])\noutput Z\n")
CHAIN8 = ("input X:[8,8]\ninput Y:[8,8]\ninput W:[8,8]\n"
          "Z[i,k] = sum[j] mul(X[i,j], Y[j,k])\n"
          "Z2[i,k] = sum[j] mul(Z[i,j], W[j,k])\noutput Z2\n")


# small graphs for the other operator families (test_einsum.cc:89-106,
# test_einsum.cc:137-150) and for the tensor-core layout paths: K-major /
# MN-major operands, swapped roles, batch labels, ragged extents
SMALL = {
    "sqdiff": "input X:[2,2]\ninput Y:[2,2]\nZ[i,k] = sum[j] sqdiff(X[i,j], Y[j,k])\noutput Z\n",
    "absmax": "input X:[2,2]\ninput Y:[2,2]\nZ[i,k] = max[j] absdiff(X[i,j], Y[j,k])\noutput Z\n",
    "divzero": "input X:[4,4]\ninput Y:[4,4]\nZ[i,j] = div(X[i,j], Y[i,j])\noutput Z\n",
    # a wide exp map: device exp vs the host's std::exp over every range (tests/test_gpu_parity.py)
    "expmap": "input X:[1024,4096]\nY[i,j] = map exp(X[i,j])\noutput Y\n",
    "mix": ("input X:[16,24]\ninput Y:[24,8]\n"
            "A[i,k] = sum[j] sqdiff(X[i,j], Y[j,k])\nB[i] = max[k] map neg(A[i,k])\n"
            "C[i,k] = add(A[i,k], B[i])\nD[k,i] = map scale(0.5)(C[i,k])\noutput D\n"),
}
LAYOUT = {
    "gemm_nn": "input X:[256,192]\ninput Y:[192,320]\nZ[i,k] = sum[j] mul(X[i,j], Y[j,k])\noutput Z\n",
    "gemm_tn": "input X:[192,256]\ninput Y:[192,320]\nZ[i,k] = sum[j] mul(X[j,i], Y[j,k])\noutput Z\n",
    "gemm_nt": "input X:[256,192]\ninput Y:[320,192]\nZ[i,k] = sum[j] mul(X[i,j], Y[k,j])\noutput Z\n",
    "gemm_swap": "input X:[256,192]\ninput Y:[192,320]\nZ[k,i] = sum[j] mul(X[i,j], Y[j,k])\noutput Z\n",
    "gemm_ragged": "input X:[200,72]\ninput Y:[72,296]\nZ[i,k] = sum[j] mul(X[i,j], Y[j,k])\noutput Z\n",
    "gemm_batch": ("input X:[4,128,96]\ninput Y:[4,96,160]\n"
                   "Z[b,i,k] = sum[j] mul(X[b,i,j], Y[b,j,k])\noutput Z\n"),
    "gemm_heads": ("input Q:[128,4,32]\ninput K:[96,4,32]\n"
                   "T[h,s,t] = sum[d] mul(Q[s,h,d], K[t,h,d])\noutput T\n"),
    "gemm_merge": ("input A:[8,16,8,16]\ninput B:[8,16,8,16]\n"
                   "Z[a,b,e,f] = sum[c,d] mul(A[a,b,c,d], B[c,d,e,f])\noutput Z\n"),
}


def write(name, doc):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(doc, f, separators=(",", ":"))


def main():
    n = 0
    for g in ["matmul", "ffnn", "softmax", "attention"]:
        text = open(os.path.join(REF_GRAPHS, g + ".eg")).read()
        for p in (1, 4, 8):
            for L in (1, 2, 4, 8):
                write(f"{g}_p{p}_L{L}", B.ref_plan_json(text, p, L))
                n += 1
    write("matmul8_pinned_L16", B.ref_plan_json(MATMUL8, 8, 16, pinned={"Z": [2, 2, 2, 4]}))
    for L in (2, 4, 8):
        write(f"chain8_pinned_L{L}", B.ref_plan_json(CHAIN8, 8, L, pinned={"Z": [2, 2, 2, 4], "Z2": [4, 1, 1, 4]}))
        n += 1
    for g, text in SMALL.items():
        for p in (1, 2, 4):
            for L in (1, 2):
                write(f"{g}_p{p}_L{L}", B.ref_plan_json(text, p, L))
                n += 1
    for g, text in LAYOUT.items():
        for p in (1, 8):
            write(f"{g}_p{p}_L1", B.ref_plan_json(text, p, 1))
            n += 1
    for g in CONFIGS + TWINS:
        text = open(os.path.join(ROOT, "graphs", g + ".eg")).read()
        for L in (1, 2, 4, 8):
            write(f"{g}_p8_L{L}", B.ref_plan_json(text, 8, L))
            n += 1
    for g in ("bmm2", "bmm2_s"):
        text = open(os.path.join(ROOT, "graphs", g + ".eg")).read()
        for L in (1, 2, 4, 8):
            write(f"{g}_repart_p8_L{L}", B.ref_plan_json(text, 8, L, pinned=BMM2_REPART))
            n += 1
    print(f"wrote {n + 1} plans to {OUT}")


if __name__ == "__main__":
    main()
