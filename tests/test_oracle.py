"""The CPU oracle (oracle/oracle.cc) pinned against the reference's own
known-answer tests and against fixtures produced by the compiled reference
(oracle/gen_golden.py). CPU only."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_cases, load_golden, load_plan
from oracle import bridge as B
from paper_2410_02682_b200 import abi


def _vertex(lz, lx, ly, join=None, map_=None, agg=None, c=0.0):
    keep = []
    ids = {}
    def lab(ls):
        a = (C.c_int32 * max(1, len(ls)))(*[ids.setdefault(l, len(ids)) for l in ls])
        keep.append(a)
        return C.cast(a, abi.i32p)
    v = abi.ed_vertex_c()
    v.arity = 2 if ly is not None else 1
    v.join_op = abi.JOIN[join] if join else -1
    v.map_op = abi.MAP[map_] if map_ else -1
    v.agg_op = abi.AGG[agg] if agg else -1
    v.scale_c = c
    v.rank_z, v.lz = len(lz), lab(lz)
    v.rank_x, v.lx = len(lx), lab(lx)
    v.rank_y, v.ly = (len(ly), lab(ly)) if ly is not None else (0, lab([]))
    return v, keep


def _kernel_eval(v, local_xy, x, y=None, f32=False, nout=None):
    lxy = np.array(local_xy, dtype=np.int64)
    out = np.zeros(nout, dtype=np.float64)
    err = C.create_string_buffer(256)
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64) if y is not None else None
    code = B.orc().oracle_kernel_eval(C.byref(v), lxy.ctypes.data, x.ctypes.data,
                                      y.ctypes.data if y is not None else None, out.ctypes.data, int(f32), err, 256)
    return code, out


KAT = json.load(open(os.path.join(GOLDEN, "kat.json")))


def test_kat_kernel_eval_matmul():
    # test_relation.cc:98-106
    v, keep = _vertex(["i", "k"], ["i", "j"], ["j", "k"], join="mul", agg="sum")
    k = KAT["kernel_eval_matmul"]
    code, out = _kernel_eval(v, [2, 2, 2, 2], k["x"], k["y"], nout=4)
    assert code == 0 and out.tolist() == k["out"]


def test_kat_relu_and_elementwise():
    v, keep = _vertex(["i", "j"], ["i", "j"], None, map_="relu")
    k = KAT["kernel_eval_relu"]
    assert _kernel_eval(v, [1, 2], k["x"], nout=2)[1].tolist() == k["out"]
    v, keep = _vertex(["i"], ["i"], ["i"], join="mul")
    k = KAT["kernel_eval_elementwise_mul"]
    assert _kernel_eval(v, [1, 1], k["x"], k["y"], nout=1)[1].tolist() == k["out"]


def test_kat_semiring_joins():
    # test_einsum.cc:89-106 — the dense oracle
    for key, join, agg in (("sqdiff_sum", "sqdiff", "sum"), ("absdiff_max", "absdiff", "max")):
        v, keep = _vertex(["i", "k"], ["i", "j"], ["j", "k"], join=join, agg=agg)
        k = KAT[key]
        x = np.array(k["x"], dtype=np.float64)
        y = np.array(k["y"], dtype=np.float64)
        out = np.zeros(4)
        bxy = np.array([2, 2, 2, 2], dtype=np.int64)
        err = C.create_string_buffer(256)
        assert B.orc().oracle_eval_expr(C.byref(v), bxy.ctypes.data, x.ctypes.data, y.ctypes.data,
                                        out.ctypes.data, err, 256) == 0
        assert out.tolist() == k["out"]


def test_kat_1x1():
    v, keep = _vertex(["i", "k"], ["i", "j"], ["j", "k"], join="mul", agg="sum")
    k = KAT["matmul_1x1"]
    assert _kernel_eval(v, [1, 1, 1, 1], k["x"], k["y"], nout=1)[1][0] == k["out"]


def test_div_by_zero_is_eval_error():
    v, keep = _vertex(["i"], ["i"], ["i"], join="div")
    code, _ = _kernel_eval(v, [2, 2], [1, 2], [1, 0], nout=2)
    assert code == abi.ED_ERR_EVAL


@pytest.mark.parametrize("d,key", [((2, 4), "chunk_u_2x4"), ((2, 2), "chunk_u_2x2")])
def test_kat_chunk_walkthrough(d, key):
    # test_relation.cc:36-55: block-index layout of the 4x4 matrix U
    u = np.array(KAT["matrix_u"]["values"], dtype=np.float64)
    bound = np.array([4, 4], dtype=np.int64)
    dd = np.array(d, dtype=np.int64)
    out = np.zeros(16)
    B.orc().oracle_chunk(2, bound.ctypes.data, dd.ctypes.data, u.ctypes.data, out.ctypes.data)
    csz = 16 // (d[0] * d[1])
    for k, vals in KAT[key]["keys"].items():
        k0, k1 = map(int, k.split(","))
        lin = k0 * d[1] + k1
        assert out[lin * csz:(lin + 1) * csz].tolist() == vals
    back = np.zeros(16)
    B.orc().oracle_assemble(2, bound.ctypes.data, dd.ctypes.data, out.ctypes.data, back.ctypes.data)
    assert np.array_equal(back, u)


def test_chunk_assemble_round_trips():
    # test_relation.cc:305-339: every divisor vector up to rank 4
    rng = np.random.default_rng(123)
    for bound in [(5,), (8,), (4, 6), (2, 3, 4), (4, 2, 3, 2)]:
        t = rng.uniform(-1, 1, size=bound)
        divs = [[v for v in range(1, b + 1) if b % v == 0] for b in bound]
        for d in np.array(np.meshgrid(*divs)).T.reshape(-1, len(bound)):
            bd = np.array(bound, dtype=np.int64)
            dd = np.ascontiguousarray(d, dtype=np.int64)
            ch = np.zeros(t.size)
            B.orc().oracle_chunk(len(bound), bd.ctypes.data, dd.ctypes.data, t.ctypes.data, ch.ctypes.data)
            back = np.zeros(t.size)
            B.orc().oracle_assemble(len(bound), bd.ctypes.data, dd.ctypes.data, ch.ctypes.data, back.ctypes.data)
            assert np.array_equal(back, t.ravel())


def test_max_rel_err():
    got = np.array([1.0, 2.0, 100.0])
    exp = np.array([1.5, 2.0, 101.0])
    ref = max(0.5 / 1.5, 0.0, 1.0 / 101.0)
    assert B.orc().oracle_max_rel_err(got.ctypes.data, exp.ctypes.data, 3) == pytest.approx(ref)
    assert B.max_rel_err(got, exp) == pytest.approx(ref)


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_matches_reference_fixture(case):
    """Restated executor == compiled reference execute(), bit for bit, in f64
    and f32 mode, with identical transfer counters; inputs == generate_inputs."""
    name, ins, o64, o32, orc, counters, total = load_golden(case)
    plan = load_plan(name)
    seed = int(case.rsplit("_s", 1)[1])
    gen = B.generate_inputs(plan, seed)
    for vid, a in ins.items():
        assert np.array_equal(gen[vid], a), "generate_inputs restatement differs"
    out, _, cnt, tot = B.oracle_execute(plan, ins, f32=False)
    for vid, a in o64.items():
        assert np.array_equal(out[vid], a)
    assert cnt == counters and tot == total
    out, _, _, _ = B.oracle_execute(plan, ins, f32=True)
    for vid, a in o32.items():
        assert np.array_equal(out[vid], a)
    # the reference's own f64 executor agrees with its dense oracle (acceptance criterion 5)
    for vid, a in o64.items():
        assert B.max_rel_err(a, orc[vid]) <= 1e-10


@pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_on_pinned_plans():
    for name in ["chain8_pinned_L4", "matmul8_pinned_L16", "mix_p4_L2"]:
        plan = load_plan(name)
        doc = plan.source
        ins = B.generate_inputs(plan, 3)
        ro, _, cnt, tot = B.ref_execute(doc, ins, threaded=True)
        oo, _, ocnt, otot = B.oracle_execute(plan, ins)
        assert all(np.array_equal(ro[k], oo[k]) for k in ro)
        assert cnt == ocnt and tot == otot


def test_device_exp_restatement_matches_host_libm(tmp_path):
    """csrc/libm_exp.cuh (the device's map exp) compiled for the host equals
    the host's std::exp (ops.cc:24) bit for bit on 8M random doubles over
    every range and on the overflow / underflow / subnormal edges."""
    import subprocess
    exe = tmp_path / "exp_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", os.path.join(ROOT, "oracle", "exp_check.cc"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "2000000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:]
    assert r.stdout.strip().endswith("0 / 8000022 differ")
