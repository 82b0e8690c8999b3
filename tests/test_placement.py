"""GPU-aware re-placement (ed_gpu_placement), host-only.

The re-placer may move memory-bound exec vertices between machines; it must
never touch input chunks or contraction joins (except, with fuse_chains, the
QK^T joins of an attention block, which follow their block onto one GPU),
never make the estimate worse,
and — because results are placement-independent (acceptance.cc:241-250) —
the re-placed plan must give bitwise the reference's outputs, while its
transfer counters must equal what the UNMODIFIED reference execute()
(runtime.cc:119-172) reports under the same machine_of.
"""
import numpy as np
import pytest

from conftest import load_plan
from oracle import bridge as B
from paper_2410_02682_b200 import build
from paper_2410_02682_b200.executor import gpu_placement

build.build()

# small plans the re-placer actually changes (2-28 vertices moved)
SMALL = ["attention_p8_L4", "mix_p4_L2", "chain8_pinned_L4", "ffnn_p8_L8", "attention_p8_L8", "ffnn_p4_L4",
         "matmul_p8_L8"]
BIG = ["ffnn_big_p8_L8", "attn_big_p8_L8", "attn_big_p8_L4", "bmm2_repart_p8_L8", "chain3_p8_L8", "hoc_p8_L8"]


def _contraction(plan, u):
    e = plan.vertices[u.producer].expr
    return u.kind == 1 and e.join == "mul" and e.agg == "sum"


@pytest.mark.parametrize("name", SMALL + BIG)
def test_replacement_moves_only_memory_bound_vertices(name):
    plan = load_plan(name)
    new, before, after = gpu_placement(plan, fuse_chains=False)
    assert after <= before + 1e-12
    for u, v in zip(plan.exec, new.exec):
        assert (u.kind, u.key, u.deps, u.fp, u.sz) == (v.kind, v.key, v.deps, v.fp, v.sz)
        assert 0 <= v.machine < plan.n_machines
        if u.kind == 0 or _contraction(plan, u):
            assert v.machine == u.machine, (name, u.id)


def test_replacement_balances_the_ffnn_softmax():
    """The reference piles FFNN's softmax vertices on GPUs 0-1;
    the re-placer spreads them and cuts the estimated busiest-GPU time."""
    plan = load_plan("ffnn_big_p8_L8")
    new, before, after = gpu_placement(plan)
    assert after < 0.85 * before
    sm = plan.find("SM.max")
    used = {new.exec[j].machine for j in plan.joins_of(sm)}
    assert len(used) > 2


def test_replacement_is_deterministic():
    plan = load_plan("attn_big_p8_L8")
    a = gpu_placement(plan)[0]
    b = gpu_placement(plan)[0]
    assert [u.machine for u in a.exec] == [u.machine for u in b.exec]


@pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", SMALL)
def test_replaced_plan_matches_reference(name):
    plan = load_plan(name)
    new, _, _ = gpu_placement(plan)
    assert any(u.machine != v.machine for u, v in zip(plan.exec, new.exec))
    ins = B.generate_inputs(plan, 11)
    machines = [u.machine for u in new.exec]
    want, _, ref_cnt, ref_total = B.ref_execute(plan.source, ins, threaded=False, machine_of=machines)
    base, _, _, _ = B.ref_execute(plan.source, ins, threaded=False)
    got, _, cnt, total = B.oracle_execute(new, ins)
    for vid in plan.outputs:
        assert np.array_equal(want[vid], base[vid]), "reference outputs depend on placement"
        assert np.array_equal(got[vid], want[vid])
    assert cnt == ref_cnt and total == ref_total


def _attention_t1(plan):
    """QK^T vertices of attention blocks: contractions read (maybe through a
    map) by a row softmax whose output feeds another contraction."""
    t1 = set()
    for y in plan.vertices:
        e = y.expr
        if e is None or e.join != "div":
            continue
        ex = plan.vertices[y.inputs[0]]
        sv = plan.vertices[ex.inputs[0]]
        xid = sv.inputs[0]
        x = plan.vertices[xid]
        if x.expr is not None and x.expr.join == "mul":
            t1.add(xid)
        elif x.expr is not None and len(x.inputs) == 1:
            t1.add(x.inputs[0])
    return t1


@pytest.mark.parametrize("name", SMALL + BIG + ["attn_big_p8_L2", "ffnn_big_p8_L4", "attn_s_p8_L4"])
def test_fusion_aware_replacement(name):
    """fuse_chains: the estimate never gets worse, only attention QK^T joins
    among the contractions move, and every region of a co-located chain ends
    on one GPU with the join that consumes it."""
    plan = load_plan(name)
    new, before, after = gpu_placement(plan, fuse_chains=True)
    assert after <= before + 1e-12
    t1 = _attention_t1(plan)
    for u, v in zip(plan.exec, new.exec):
        assert (u.kind, u.key, u.deps, u.fp, u.sz) == (v.kind, v.key, v.deps, v.fp, v.sz)
        if u.kind == 0 or (_contraction(plan, u) and u.producer not in t1):
            assert v.machine == u.machine, (name, u.id)


@pytest.mark.parametrize("name,chain", [("attn_big_p8_L2", ["T1", "T3", "O"]), ("attn_big_p8_L4", ["T1", "T3", "O"]),
                                        ("ffnn_big_p8_L4", ["SM.max", "SM.sub", "SM.exp", "SM.sum", "Y"])])
def test_fusion_aware_replacement_colocates_chains(name, chain):
    """Each chain region's joins share a GPU after the fusion-aware re-placement
    (the reference's placement splits them)."""
    plan = load_plan(name)
    new, before, after = gpu_placement(plan, fuse_chains=True)
    assert after < before
    ids = {plan.find(n) for n in chain}

    def split(p):
        bad = 0
        for u in p.exec:
            if u.kind == 1 and u.producer == plan.find(chain[-1]):
                stack, seen = [u.id], set()
                while stack:
                    i = stack.pop()
                    for d in p.exec[i].deps:
                        if p.exec[d].producer in ids and d not in seen:
                            seen.add(d)
                            stack.append(d)
                bad += any(p.exec[d].machine != u.machine for d in seen)
        return bad
    assert split(new) == 0 and split(plan) > 0
