"""ed_generate_inputs: generate_inputs(graph, seed) (runtime.cc:552-571) on the
device must equal the host's std::mt19937_64 + libstdc++ distributions (the
oracle, pinned to the reference's own generate_inputs in test_oracle.py) bit
for bit, integer [-4, 4] and U[-1, 1) graphs alike, then chunk exactly like
an upload of the same tensors."""
import numpy as np
import pytest

from conftest import load_plan
from oracle import bridge as B

pytestmark = pytest.mark.gpu

CASES = [("matmul_p4_L2", "fp64"), ("ffnn_p4_L2", "fp64"), ("attention_p8_L4", "fp64"), ("chain3_s_p8_L1", "fp64"),
         ("attn_s_p8_L1", "fp32"), ("hoc_s_p8_L1", "bf16"), ("chain3_p8_L1", "fp64")]


@pytest.mark.parametrize("name,prec", CASES)
def test_device_generate_inputs_bitexact(gpu_ctx, name, prec):
    from paper_2410_02682_b200.executor import PreparedPlan
    plan = load_plan(name)
    seed = 5
    want = B.generate_inputs(plan, seed)
    pp = PreparedPlan(gpu_ctx, plan, precision=prec)
    pp.generate_inputs(seed)
    got = pp.download(dtype=np.float64, vertices=plan.input_vertices())
    for vid, w in want.items():
        w = w if prec == "fp64" else w.astype(np.float32).astype(np.float64)
        assert np.array_equal(got[vid], w), (name, plan.vertices[vid].name)
    # and the run on generated inputs equals the run on uploaded ones
    rep_gen = pp.run()
    out_gen = pp.download(dtype=np.float64)
    pp.upload(want)
    pp.run()
    out_up = pp.download(dtype=np.float64)
    pp.close()
    for vid in plan.outputs:
        assert np.array_equal(out_gen[vid], out_up[vid])
    assert rep_gen.total_transferred >= 0
