"""Parity at BASELINE.json's full sizes, on the B200.

The CPU oracle cannot run these (hours); instead:
  * integer known answers: generate_inputs-style integers in [-4,4] keep the
    first contraction of chain3 / bmm2 and all of hoc exact in every mode
    (partial sums < 2^24), checked against an fp64 GEMM;
  * the rest against the dense graph evaluated in fp64 (torch.einsum on the
    GPU as the checker), with the bf16 bound written below.
"""
import numpy as np
import pytest

from conftest import load_plan

pytestmark = pytest.mark.gpu

BF16_BOUND = 3e-2   # max_rel_err (tensor.cc:9-19) vs the fp64 dense graph, bf16 mode


def _inputs(plan, seed=1):
    rng = np.random.default_rng(seed)
    out = {}
    for vid in plan.input_vertices():
        shape = plan.vertices[vid].bound
        if plan.integer_valued():
            out[vid] = rng.integers(-4, 5, size=shape, dtype=np.int8).astype(np.float32)
        else:
            out[vid] = (rng.random(size=shape, dtype=np.float32) * 2 - 1).astype(np.float32)
    return out


def _dense_fp64(plan, ins, torch, upto=None, bf16_operands=False):
    """eval_reference (reference.cc:62-82) restated with torch.einsum in fp64.
    bf16_operands rounds every contraction operand to bf16 first (the
    executor's bf16 mode), isolating accumulation error."""
    vals = {vid: torch.from_numpy(np.asarray(a, dtype=np.float64)).cuda() for vid, a in ins.items()}
    for v in plan.vertices:
        if v.expr is None:
            continue
        e = v.expr
        letters = {}
        for ls in e.ins + [e.out]:
            for l in ls:
                letters.setdefault(l, chr(ord("a") + len(letters)))
        spec_in = ["".join(letters[l] for l in ls) for ls in e.ins]
        spec_out = "".join(letters[l] for l in e.out)
        x = vals[v.inputs[0]]
        y = vals[v.inputs[1]] if e.is_binary else None
        if e.join == "mul" and e.agg == "sum":
            if bf16_operands:
                x, y = x.to(torch.bfloat16).double(), y.to(torch.bfloat16).double()
            r = torch.einsum(f"{spec_in[0]},{spec_in[1]}->{spec_out}", x, y)
        elif e.is_binary:
            # broadcast y over x's layout
            yy = torch.einsum(f"{spec_in[1]}->{spec_in[1]}", y)
            shape = [x.shape[spec_in[0].index(c)] if c in spec_in[1] else 1 for c in spec_in[0]]
            yb = yy.permute(*[spec_in[1].index(c) for c in spec_in[0] if c in spec_in[1]]).reshape(shape)
            r = {"sub": x - yb, "div": x / yb, "add": x + yb, "mul": x * yb}[e.join]
        else:
            m = {"relu": torch.relu, "exp": torch.exp, "neg": torch.neg, "identity": lambda t: t,
                 "scale": lambda t: t * e.scale_c}[e.map](x)
            if e.agg is None:
                r = m
            else:
                red = [spec_in[0].index(c) for c in spec_in[0] if c not in spec_out]
                r = m.amax(dim=red) if e.agg == "max" else m.sum(dim=red)
        vals[v.vid] = r
        if upto is not None and v.name == upto:
            return r
    return vals


def _run(gpu_ctx, plan, ins, prec="bf16"):
    from paper_2410_02682_b200.executor import PreparedPlan
    pp = PreparedPlan(gpu_ctx, plan, precision=prec)
    pp.upload(ins)
    pp.run()
    return pp


def _rel(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))))


def test_hoc_full_size_exact(gpu_ctx):
    """C5 128^4: one contraction, K = 16384 split over 2 siblings folded in
    TMEM; integer partial sums < 2^24, so the output is exact."""
    torch = pytest.importorskip("torch")
    plan = load_plan("hoc_p8_L1")
    ins = _inputs(plan)
    pp = _run(gpu_ctx, plan, ins)
    got = pp.download(dtype=np.float32)[plan.outputs[0]]
    pp.close()
    a = torch.from_numpy(ins[plan.find("A")]).cuda().double().reshape(128 * 128, 128 * 128)
    b = torch.from_numpy(ins[plan.find("B")]).cuda().double().reshape(128 * 128, 128 * 128)
    want = (a @ b).reshape(128, 128, 128, 128).cpu().numpy()
    assert np.array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("name", ["bmm2", "bmm2_repart"])
def test_integer_chain_full_size(gpu_ctx, name):
    """First contraction exact (its partial sums < 2^24); the final output
    within 1e-5 of fp64 on the same bf16-rounded operands (accumulation is
    the only error left)."""
    torch = pytest.importorskip("torch")
    plan = load_plan(f"{name}_p8_L1")
    ins = _inputs(plan)
    pp = _run(gpu_ctx, plan, ins)
    got = pp.download(dtype=np.float32)[plan.outputs[0]]
    # first contraction: exact integers (partial sums < 2^24). Chunks that only
    # feed the next bf16 GEMM exist only as bf16, so compare those with the
    # exact values rounded once.
    first = next(v for v in plan.vertices if v.expr is not None)
    z1 = _dense_fp64(plan, ins, torch, upto=first.name)
    assert float(z1.abs().max()) < 2 ** 24
    for u in plan.exec:
        if u.kind != 2 or u.producer != first.vid:
            continue
        sl = tuple(slice(k * c, (k + 1) * c) for k, c in zip(u.key, u.chunk_bound))
        exact = z1[sl]
        chunk = torch.from_numpy(pp.download_chunk(u.id)).cuda()
        assert torch.equal(chunk, exact) or torch.equal(chunk, exact.float().bfloat16().double()), u.id
    pp.close()
    del z1
    want_q = _dense_fp64(plan, ins, torch, bf16_operands=True)[plan.outputs[0]].cpu().numpy()
    assert _rel(got, want_q) <= 1e-5


def _vertex_tensor(pp, plan, w, torch):
    """The GPU's value of graph vertex w, assembled from any materialised
    refinement layer of w (None if w was fused away)."""
    layers = {}
    for u in plan.exec:
        if u.kind == 2 and u.producer == w:
            layers.setdefault((u.consumer, u.slot), []).append(u)
    v = plan.vertices[w]
    for lay in layers.values():
        out = torch.empty(v.bound, dtype=torch.float64, device="cuda")
        try:
            for u in lay:
                sl = tuple(slice(k * c, (k + 1) * c) for k, c in zip(u.key, u.chunk_bound))
                out[sl] = torch.from_numpy(pp.download_chunk(u.id)).cuda()
            return out
        except Exception:
            continue
    # no materialised refinement layer (consumers read the producer's regions
    # in place): assemble from the region accumulators (region-head joins)
    if v.expr is not None:
        dls = v.expr.distinct_labels()
        out = torch.empty(v.bound, dtype=torch.float64, device="cuda")
        seen = torch.zeros(v.bound, dtype=torch.bool, device="cuda")
        for u in plan.exec:
            if u.kind != 1 or u.producer != w:
                continue
            try:
                chunk = torch.from_numpy(pp.download_chunk(u.id)).cuda()
            except Exception:
                continue
            key = [u.key[dls.index(l)] for l in v.expr.out]
            sl = tuple(slice(k * c, (k + 1) * c) for k, c in zip(key, u.chunk_bound))
            out[sl] = chunk
            seen[sl] = True
        if bool(seen.all()):
            return out
    return None


def _op_fp64(plan, v, args, torch):
    """One vertex of eval_expr (reference.cc:3-60) in fp64."""
    sub = type(plan)(plan.p, plan.n_machines, plan.alpha, plan.vertices, [v.vid], plan.exec)
    ins = {i: a for i, a in zip(v.inputs, args)}
    # evaluate only this vertex: reuse _dense_fp64 on a one-vertex view
    vals = {vid: a for vid, a in ins.items()}
    e = v.expr
    letters = {}
    for ls in e.ins + [e.out]:
        for l in ls:
            letters.setdefault(l, chr(ord("a") + len(letters)))
    si = ["".join(letters[l] for l in ls) for ls in e.ins]
    so = "".join(letters[l] for l in e.out)
    x = args[0]
    y = args[1] if e.is_binary else None
    if e.join == "mul" and e.agg == "sum":
        return torch.einsum(f"{si[0]},{si[1]}->{so}", x, y)
    if e.is_binary:
        shape = [x.shape[si[0].index(c)] if c in si[1] else 1 for c in si[0]]
        yb = y.permute(*[si[1].index(c) for c in si[0] if c in si[1]]).reshape(shape)
        return {"sub": x - yb, "div": x / yb, "add": x + yb, "mul": x * yb}[e.join]
    m = {"relu": torch.relu, "exp": torch.exp, "neg": torch.neg, "identity": lambda t: t,
         "scale": lambda t: t * e.scale_c}[e.map](x)
    if e.agg is None:
        return m
    red = [si[0].index(c) for c in si[0] if c not in so]
    return m.amax(dim=red) if e.agg == "max" else m.sum(dim=red)


PER_VERTEX_BOUND = 2e-2  # max|got - want| / max|want|, bf16 operands, fp32 accumulation


@pytest.mark.parametrize("name", ["ffnn_big", "attn_big", "chain3", "attn_s"])
def test_per_vertex_full_size(gpu_ctx, name):
    """Per-vertex parity at full size: every materialised vertex
    against fp64 evaluated on the GPU's OWN inputs to it, so conditioning of
    earlier vertices (softmax logits reach ~1e3 here) cannot mask or fake an
    error. Vertices fused into a consumer's kernel are checked as the
    composition they became (e.g. relu(A) from X, W1; the softmax chain from
    its input)."""
    torch = pytest.importorskip("torch")
    plan = load_plan(f"{name}_p8_L1")
    ins = _inputs(plan)
    pp = _run(gpu_ctx, plan, ins)
    got = {vid: torch.from_numpy(np.asarray(a, dtype=np.float64)).cuda() for vid, a in ins.items()}
    for v in plan.vertices:
        if v.expr is not None:
            g = _vertex_tensor(pp, plan, v.vid, torch)
            if g is not None:
                got[v.vid] = g
    checked = 0
    memo = {}

    def value(w):
        """GPU value if materialised, else fp64 composition from materialised inputs."""
        if w in got:
            return got[w]
        if w not in memo:
            memo[w] = _op_fp64(plan, plan.vertices[w], [value(i) for i in plan.vertices[w].inputs], torch)
        return memo[w]

    for v in plan.vertices:
        if v.expr is None or v.vid not in got:
            continue
        want = _op_fp64(plan, v, [value(i) for i in v.inputs], torch)
        err = float(((got[v.vid] - want).abs().max() / want.abs().max().clamp(min=1e-30)).item())
        assert err <= PER_VERTEX_BOUND, (v.name, err)
        checked += 1
    pp.close()
    assert checked >= 3


@pytest.mark.parametrize("name", ["attn_big", "attn_s"])
def test_attention_block_runs_fused(gpu_ctx, name):
    """The T1 -> scale -> softmax -> O chain runs as one fused kernel (bf16),
    and the logits are never materialised."""
    from paper_2410_02682_b200.executor import PreparedPlan, EdError
    plan = load_plan(f"{name}_p8_L1")
    pp = PreparedPlan(gpu_ctx, plan, precision="bf16", profile=True)
    pp.upload(_inputs(plan))
    pp.run()
    names = [k["name"] for k in pp.kernel_stats()]
    assert any(n.startswith("attention_fused") for n in names), names
    assert not any(n.startswith("softmax_rows") for n in names), names
    t1 = plan.find("T1")
    ref = next(u.id for u in plan.exec if u.kind == 2 and u.producer == t1)
    with pytest.raises(EdError):
        pp.download_chunk(ref)
    pp.close()


@pytest.mark.parametrize("name", ["bmm2_s_p8_L1", "ffnn_s_p8_L1", "matmul_p8_L1"])
def test_run_steps_pipeline_matches_blocking_calls(gpu_ctx, name):
    """ed_run_steps (pipelined serving loop) gives, step for step, the outputs
    of the blocking upload / run / download sequence on the same inputs."""
    from paper_2410_02682_b200.executor import PreparedPlan
    plan = load_plan(name)
    steps = [_inputs(plan, seed=s) for s in (1, 2, 3)]
    pp = PreparedPlan(gpu_ctx, plan, precision="bf16")
    want = []
    for ins in steps:
        pp.upload(ins)
        pp.run()
        want.append(pp.download(dtype=np.float32))
    got = [{vid: np.empty(plan.vertices[vid].bound, dtype=np.float32) for vid in plan.outputs} for _ in steps]
    rep = pp.run_steps(steps, got)
    pp.close()
    assert rep.device_ms > 0
    for w, g in zip(want, got):
        for vid in plan.outputs:
            assert np.array_equal(w[vid], g[vid])
