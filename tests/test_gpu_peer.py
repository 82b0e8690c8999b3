"""Multi-rank execution with real device-to-device transfers on ONE GPU.

World 2 / 4: one process per rank, all on cuda:0 (NCCL refuses two ranks on
one device, so these runs use the peer transport: a consumer copies the
producer's chunk straight out of the producer's HBM through a CUDA IPC
mapping once the producer's ready flag carries the run's epoch — on an 8-GPU
box the same copies travel over NVLink). Each rank runs its share of the
placed ExecGraph through the C ABI, rank 0 assembles the outputs (collective
ed_download), and they must equal the reference executor's outputs bit for bit
(FP64) with the reference's transfer counters; two consecutive runs exercise
the epoch / write-after-read barriers.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, load_golden, load_plan
import tolerance as T

pytestmark = pytest.mark.gpu

CASES = [("attention_p8_L4_s1084", 4), ("attention_p8_L4_s1084", 2), ("ffnn_p4_L2_s23", 2),
         ("chain8_pinned_L4_s7", 4), ("mix_p4_L2_s41", 2), ("softmax_p8_L4_s1084", 4),
         ("chain8_pinned_L8_s7", 8)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, case, port, q, precision, replaced, want_kernels=False, reupload=False):
    import sys
    from datetime import timedelta
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        import torch.distributed as dist
        from paper_2410_02682_b200.executor import Context, PreparedPlan, gpu_placement
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=timedelta(seconds=120))
        if case.startswith("fuzz:"):  # a randomised fixture (tests/test_gpu_fuzz.py)
            from test_gpu_fuzz import _load
            plan, ins, o64, o32, counters, total = _load(case[5:])
        elif case.endswith(".plan"):  # a plan without a golden fixture: seeded host inputs
            from oracle import bridge as B
            name = case[:-5]
            plan = load_plan(name)
            ins = B.generate_inputs(plan, 3)
        else:
            name, ins, o64, o32, orc, counters, total = load_golden(case)
            plan = load_plan(name)
        if replaced:
            plan = gpu_placement(plan)[0]
        ctx = Context(0, rank, world, None)
        pp = PreparedPlan(ctx, plan, precision=precision, transport="peer", profile=want_kernels)
        blobs = [None] * world
        dist.all_gather_object(blobs, pp.peer_export())
        pp.peer_import(blobs)
        results = []
        if reupload:
            # upload -> run -> upload -> run with no download in between: a rank
            # must not overwrite input chunks a slower peer is still pulling
            from oracle import bridge as B
            for seed in (3, 4):
                pp.upload(B.generate_inputs(plan, seed))
                rep = pp.run()
            outs = pp.download()
            results.append((rep.machines, rep.total_transferred, outs if rank == 0 else None))
        else:
            pp.upload(ins)
        for _ in range(0 if reupload else 2):
            rep = pp.run()
            outs = pp.download()
            results.append((rep.machines, rep.total_transferred, outs if rank == 0 else None))
        kernels = [k["name"] for k in pp.kernel_stats()] if want_kernels else None
        pp.close()
        if rank == 0 and want_kernels:  # the same plan on one rank, for comparison
            c1 = Context(0)
            p1 = PreparedPlan(c1, plan, precision=precision)
            p1.upload(ins)
            p1.run()
            results.append(p1.download())
            p1.close()
            c1.close()
        ctx.close()
        dist.barrier()
        q.put((rank, "ok", (results, kernels) if want_kernels else (results if rank == 0 else None)))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        import traceback
        q.put((rank, f"{type(e).__name__}: {e}\n{traceback.format_exc()[-1500:]}", None))


def _run(case, world, precision="fp64", replaced=False, want_kernels=False, reupload=False):
    import torch.multiprocessing as mp
    from paper_2410_02682_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, case, port, q, precision, replaced, want_kernels, reupload))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=280) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, _ in res:
        assert status == "ok", f"rank {rank}: {status}"
    if want_kernels:
        return {rank: r for rank, s, r in res}
    return next(r for rank, s, r in res if rank == 0)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case,world", CASES)
def test_peer_transport_fp64_bitexact(case, world):
    from oracle import bridge as B
    name, ins, o64, o32, orc, counters, total = load_golden(case)
    plan = load_plan(name)
    for machines, tt, outs in _run(case, world):
        for vid, want in o64.items():
            assert np.array_equal(outs[vid], want), (case, vid, B.max_rel_err(outs[vid], want))
        assert tt == total and [tuple(m) for m in machines] == [tuple(c) for c in counters]


@pytest.mark.timeout(300)
def test_peer_transport_replaced_plan_bf16():
    """The GPU-aware re-placement run on 4 ranks in the tensor-core mode."""
    case = "attention_p8_L4_s1084"
    name, ins, o64, o32, orc, counters, total = load_golden(case)
    from oracle import bridge as B
    for machines, tt, outs in _run(case, 4, precision="bf16", replaced=True):
        for vid, want in o64.items():
            assert T.within("bf16", outs[vid], want), vid


@pytest.mark.timeout(300)
@pytest.mark.parametrize("name,fused,world,replaced", [
    ("attn_s_p8_L2", "attention_fused", 2, False), ("ffnn_s_p8_L2", "softmax_rows", 2, False),
    ("attn_s_p8_L4", "attention_fused", 4, True), ("ffnn_s_p8_L4", "softmax_rows", 4, True)])
def test_peer_transport_fuses_per_rank(name, fused, world, replaced):
    """Cross-vertex fusions are decided per rank: with the reduced twins on
    2 / 4 ranks (the 4-rank plans re-placed with fuse_chains, which keeps each
    chain region on one GPU) every rank runs the fused kernel for its
    co-located regions, and the outputs agree with the single-rank run."""
    got = _run(name + ".plan", world, precision="bf16", replaced=replaced, want_kernels=True)
    for rank in range(world):
        assert any(k.startswith(fused) for k in got[rank][1]), (rank, got[rank][1])
    results = got[0][0]
    single = results[-1]
    for machines, tt, outs in results[:-1]:
        for vid, want in single.items():
            # both runs round to bf16, with different sibling fold orders
            # (tests/tolerance.py: the normwise bar of the tensor-core modes)
            assert T.normwise(outs[vid], want) <= 1e-2, vid


def _fuzz_multirank():
    import glob
    from test_gpu_fuzz import CASES
    out = []
    for c in CASES:
        L = int(c.split("_L")[1].split("_")[0])
        if L > 1:
            out.append((c, L))
    return out[:8]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case,world", _fuzz_multirank())
def test_peer_transport_fuzz_fp64_bitexact(case, world):
    """Random graphs (tests/test_gpu_fuzz.py) on L ranks of one GPU through
    the peer transport: bit-exact f64 and the reference's counters."""
    from test_gpu_fuzz import _load, _same
    plan, ins, o64, o32, counters, total = _load(case)
    for machines, tt, outs in _run("fuzz:" + case, world):
        for vid, want in o64.items():
            assert _same(outs[vid], want, plan, 1e-14), (case, vid)
        assert tt == total and [tuple(m) for m in machines] == [tuple(c) for c in counters]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("name,world", [("attention_p8_L4", 4), ("chain8_pinned_L4", 4)])
def test_peer_transport_reupload_between_runs(name, world):
    """new inputs uploaded between two runs without a download in
    between wait for every peer to finish the first run (write-after-read on
    the exported input chunks); the second run's outputs are those of the
    second inputs, bit for bit (f64) against the CPU oracle."""
    from oracle import bridge as B
    plan = load_plan(name)
    want, _, counters, total = B.oracle_execute(plan, B.generate_inputs(plan, 4))
    for machines, tt, outs in _run(name + ".plan", world, reupload=True):
        for vid, w in want.items():
            assert np.array_equal(outs[vid], w), vid
        assert tt == total


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case,world", [("attention_p8_L4_s1084", 4), ("ffnn_p4_L2_s23", 2),
                                        ("chain8_pinned_L4_s7", 4), ("mix_p4_L2_s41", 2),
                                        ("softmax_p8_L4_s1084", 4), ("chain8_pinned_L8_s7", 8)])
def test_single_process_multi_rank(case, world):
    """ed_ctx_create_multi: ONE process drives all L ranks (the reference's
    single execute() over L machines, runtime.cc:301-355) — here all on
    cuda:0 — exchanging chunks through the in-process peer transport:
    bit-exact f64 / f32 and the reference's counters, twice in a row, and
    re-uploads between runs without a download."""
    from oracle import bridge as B
    from paper_2410_02682_b200.executor import Context, PreparedPlan
    name, ins, o64, o32, orc, counters, total = load_golden(case)
    plan = load_plan(name)
    ctx = Context.multi([0] * world)
    try:
        for prec, want in (("fp64", o64), ("fp32", o32)):
            pp = PreparedPlan(ctx, plan, precision=prec)
            pp.upload(ins)
            for _ in range(2):
                rep = pp.run()
                outs = pp.download()
                for vid, w in want.items():
                    assert np.array_equal(outs[vid], w), (case, prec, vid, B.max_rel_err(outs[vid], w))
                assert [tuple(m) for m in rep.machines] == [tuple(c) for c in counters]
                assert rep.total_transferred == total and rep.device_ms > 0
            pp.upload(B.generate_inputs(plan, 9))
            pp.run()
            pp.upload(ins)
            pp.run()
            outs = pp.download()
            for vid, w in want.items():
                assert np.array_equal(outs[vid], w), (case, prec, vid)
            pp.close()
    finally:
        ctx.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case,world", [("attention_p8_L4_s1084", 4), ("chain8_pinned_L8_s7", 8),
                                        ("softmax_p8_L4_s1084", 4)])
def test_single_process_multi_rank_tensor_modes(case, world):
    """The tensor-core modes across L in-process ranks on one GPU (8 ranks
    share cuda:0's hardware queues: CUDA_DEVICE_MAX_CONNECTIONS): fp32x3
    within the reference's own max_rel_err bar of the f64 outputs, bf16
    within its normwise bar, the reference's counters, twice in a row."""
    from paper_2410_02682_b200.executor import Context, PreparedPlan
    name, ins, o64, o32, orc, counters, total = load_golden(case)
    plan = load_plan(name)
    ctx = Context.multi([0] * world)
    try:
        for prec in ("fp32x3", "bf16"):
            pp = PreparedPlan(ctx, plan, precision=prec)
            pp.upload(ins)
            for _ in range(2):
                rep = pp.run()
                outs = pp.download()
                for vid, w in o64.items():
                    metric, err, bar = T.error(prec, outs[vid], w)
                    assert err <= bar, (case, prec, vid, metric, err)
                assert [tuple(m) for m in rep.machines] == [tuple(c) for c in counters]
                assert rep.total_transferred == total
            pp.close()
    finally:
        ctx.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case,world", [("ffnn_p4_L2_s23", 2), ("attention_p8_L4_s1084", 4),
                                        ("chain8_pinned_L8_s7", 8)])
def test_single_process_multi_rank_op_by_op(case, world):
    """In-process ranks launched op by op (no CUDA graph; profile mode times
    every op): each rank's kernels are loaded before its first run, so a
    first launch cannot wait on a rank's receive spinning for a chunk whose
    producer has not been launched yet. Bit-exact f64, per-rank kernel stats."""
    from paper_2410_02682_b200.executor import Context, PreparedPlan
    name, ins, o64, o32, orc, counters, total = load_golden(case)
    plan = load_plan(name)
    ctx = Context.multi([0] * world)
    try:
        for kw in ({"graph": False}, {"profile": True}):
            pp = PreparedPlan(ctx, plan, precision="fp64", **kw)
            pp.upload(ins)
            for _ in range(2):
                rep = pp.run()
                outs = pp.download()
                for vid, w in o64.items():
                    assert np.array_equal(outs[vid], w), (case, kw, vid)
                assert rep.total_transferred == total
            if kw.get("profile"):
                import re
                ranks = {m.group(1) for k in pp.kernel_stats() for m in [re.match(r"r(\d+)/", k["name"])] if m}
                assert ranks == {str(r) for r in range(world)}, ranks
            pp.close()
    finally:
        ctx.close()


def _fuzz_multirank_all():
    from test_gpu_fuzz import CASES
    return [(c, int(c.split("_L")[1].split("_")[0])) for c in CASES if int(c.split("_L")[1].split("_")[0]) > 1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case,world", _fuzz_multirank_all())
def test_single_process_multi_rank_fuzz_tensor_modes(case, world):
    """Every randomised graph with L > 1 (tests/test_gpu_fuzz.py) on L
    in-process ranks of one GPU in each tensor-core mode: the received
    operands (inputs included) carry what the mode needs — a bf16 copy, a
    TF32 lo shadow — so each mode meets its bar (tests/tolerance.py) exactly
    as on one rank."""
    from test_gpu_fuzz import _load
    from paper_2410_02682_b200.executor import Context, PreparedPlan
    plan, ins, o64, o32, counters, total = _load(case)
    ctx = Context.multi([0] * world)
    try:
        for prec in ("tf32", "bf16", "fp32x3"):
            pp = PreparedPlan(ctx, plan, precision=prec)
            pp.upload(ins)
            rep = pp.run()
            outs = pp.download()
            for vid, w in o64.items():
                metric, err, bar = T.error(prec, outs[vid], w)
                assert err <= bar, (case, prec, vid, metric, err)
            assert rep.total_transferred == total
            pp.close()
    finally:
        ctx.close()
