"""Checkers for the full-size parity tests (test infrastructure only).

* `op_fp64`: one vertex of eval_expr (reference.cc:3-60) restated with
  torch in fp64 on the GPU — fast enough for 10^12-flop vertices;
* `ref_slice`: the reference's OWN eval_expr (oracle/_ref, the unmodified
  sources) on a row slice of one vertex, fed the same inputs — pins the
  torch restatement to the reference where the reference can afford it;
* `max_rel_err`: tensor.cc:9-19, the reference's parity metric.
"""
import numpy as np

from oracle import bridge as B

U32 = 2.0 ** -24   # fp32 unit roundoff
U16 = 2.0 ** -9    # bf16 unit roundoff (8 significant bits)


def letters(e):
    m = {}
    for ls in e.ins + [e.out]:
        for l in ls:
            m.setdefault(l, chr(ord("a") + len(m)))
    return m


def op_fp64(v, args, torch, absolute=False):
    """eval_expr of graph vertex v on fp64 torch tensors. absolute=True gives
    sum |x|*|y| for a mul/sum contraction (the magnitude every partial sum
    is bounded by, whatever the summation order)."""
    e = v.expr
    lt = letters(e)
    si = ["".join(lt[l] for l in ls) for ls in e.ins]
    so = "".join(lt[l] for l in e.out)
    x = args[0]
    y = args[1] if e.is_binary else None
    if e.join == "mul" and e.agg == "sum":
        if absolute:
            x, y = x.abs(), y.abs()
        return torch.einsum(f"{si[0]},{si[1]}->{so}", x, y)
    if e.is_binary:
        shape = [x.shape[si[0].index(c)] if c in si[1] else 1 for c in si[0]]
        yb = y.permute(*[si[1].index(c) for c in si[0] if c in si[1]]).reshape(shape)
        r = {"sub": x - yb, "div": x / yb, "add": x + yb, "mul": x * yb}[e.join]
        if e.agg is None:
            return r
        red = [si[0].index(c) for c in si[0] if c not in so]
        return r.amax(dim=red) if e.agg == "max" else r.sum(dim=red)
    m = {"relu": torch.relu, "exp": torch.exp, "neg": torch.neg, "identity": lambda t: t,
         "scale": lambda t: t * e.scale_c}[e.map](x)
    if e.agg is None:
        return m
    red = [si[0].index(c) for c in si[0] if c not in so]
    return m.amax(dim=red) if e.agg == "max" else m.sum(dim=red)


def contraction_k(plan, v):
    """Length of each dot product of a mul/sum vertex (product of the
    aggregated labels' extents)."""
    e = v.expr
    ext = {}
    for ls, b in zip(e.ins, [plan.vertices[w].bound for w in v.inputs]):
        for l, n in zip(ls, b):
            ext[l] = n
    k = 1
    for l in e.agg_labels():
        k *= ext[l]
    return k


def max_rel_err(got, want, torch):
    """tensor.cc:9-19: max |got - want| / max(1, |want|)."""
    return float(((got - want).abs() / want.abs().clamp(min=1.0)).max().item())


def normwise(got, want):
    return float(((got - want).abs().max() / want.abs().max().clamp(min=1e-300)).item())


def vertex_tensor(pp, plan, w, torch):
    """The GPU's value of graph vertex w (fp64 on the GPU), assembled from a
    materialised refinement layer of w, or from its region accumulators
    (region-head joins); None if w was fused into a consumer's kernel."""
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


def slice_picks(plan, v, which, budget=3e7):
    """Which rows of v's output a reference slice evaluates: output labels,
    largest extent first, are cut to 2 values (at the start for which = 0,
    5/7 of the way in for which = 1) until the slice's scalar products
    (output elements x aggregated extent) fit the budget — about a second of
    the reference's interpretive eval_expr. Returns {label: (start, count)}."""
    e = v.expr
    ext = {}
    for ls, w in zip(e.ins, v.inputs):
        for l, n in zip(ls, plan.vertices[w].bound):
            ext[l] = n
    k = 1
    for l in e.agg_labels():
        k *= ext[l]
    picks = {}
    size = 1
    for l in e.out:
        size *= ext[l]
    for l in sorted(e.out, key=lambda l: -ext[l]):
        if size * k <= budget:
            break
        n = ext[l]
        cnt = min(2, n)
        picks[l] = (0 if which == 0 else (n * 5) // 7 // cnt * cnt, cnt)
        size = size // n * cnt
    return picks


def _vertex_line(graph_text, name):
    for line in graph_text.splitlines():
        s = line.strip()
        if s.startswith(name + "[") and "=" in s:
            return s
    raise KeyError(name)


def ref_slice(plan, graph_text, v, args, picks, torch, f32=None):
    """The reference's eval_expr (reference.cc:3-60, through oracle/_ref's
    edref_eval_vertex) on a slice of v (picks: {label: (start, count)}): a
    one-vertex graph whose inputs are the given tensors cut to those ranges.
    f32=False / True evaluates through the reference's kernel_eval (kernel.cc)
    in f64 / in its f32 mode instead of eval_expr.
    Returns (reference slice, index tuple of that slice in v's output)."""
    e = v.expr
    decl, arrs = [], []
    if len(set(v.inputs)) != len(v.inputs):
        raise ValueError("a vertex reading one tensor twice")

    def cut(ls):
        return tuple(slice(picks[l][0], picks[l][0] + picks[l][1]) if l in picks else slice(None) for l in ls)

    for ls, w, a in zip(e.ins, v.inputs, args):
        t = a[cut(ls)]
        arrs.append(np.ascontiguousarray(t.cpu().numpy(), dtype=np.float64))
        decl.append(f"input {plan.vertices[w].name}:[{','.join(str(n) for n in t.shape)}]")
    text = "\n".join(decl + [_vertex_line(graph_text, v.name), f"output {v.name}"]) + "\n"
    oshape = [picks[l][1] if l in picks else n for l, n in zip(e.out, v.bound)]
    out = np.empty(oshape, dtype=np.float64)
    err = B.C.create_string_buffer(1024)
    vid = len(decl)  # the expression vertex follows its input declarations
    y = arrs[1] if len(arrs) > 1 else None
    if f32 is None:
        B._check(B.ref().edref_eval_vertex(text.encode(), vid, B._ptr(arrs[0]), B._ptr(y), B._ptr(out), err, 1024),
                 err)
    else:
        B._check(B.ref().edref_kernel_vertex(text.encode(), vid, int(bool(f32)), B._ptr(arrs[0]), B._ptr(y),
                                             B._ptr(out), err, 1024), err)
    return torch.from_numpy(out).to(args[0].device), cut(e.out)


def fused_chain(plan, v, got):
    """The vertices a fused kernel computed on the way to v (graph vertices
    between v and its materialised ancestors, in topological order), or []
    when every input of v is materialised."""
    if all(i in got for i in v.inputs):
        return []
    chain, seen = [], set()

    def visit(w):
        if w in got or w in seen:
            return
        seen.add(w)
        for i in plan.vertices[w].inputs:
            visit(i)
        chain.append(w)

    for i in v.inputs:
        visit(i)
    return chain


def chain_rows(plan, graph_text, v, chain, got, want_full, which, torch):
    """v and the fused chain before it evaluated by the reference's f32 mode
    (kernel_eval with f32 = true, kernel.cc:43-44) vertex by vertex on two rows
    of v's first output label, from the materialised inputs. Returns
    (ours, theirs): max_rel_err (tensor.cc:9-19) of the GPU's v and of the
    reference's f32 chain against want_full (v composed in fp64) on those rows."""
    lab = v.expr.out[0]
    n = v.bound[0]
    start = 0 if which == 0 else (n * 5) // 7 // 2 * 2
    f32 = {}
    for w in chain + [v.vid]:
        vw = plan.vertices[w]
        args, picks = [], {}
        for ls, i in zip(vw.expr.ins, vw.inputs):
            if i in f32:
                args.append(f32[i])  # already cut to the rows
            else:
                a = got[i]
                if lab in ls:
                    d = ls.index(lab)
                    a = a.narrow(d, start, 2)
                args.append(a)
        if lab in vw.expr.out:
            picks[lab] = (0, 2)
        ref, _ = ref_slice(plan, graph_text, vw, args, picks, torch, f32=True)
        f32[w] = ref
    d = v.expr.out.index(lab)
    want = want_full.narrow(d, start, 2)
    ours = max_rel_err(got[v.vid].narrow(d, start, 2), want, torch)
    theirs = max_rel_err(f32[v.vid], want, torch)
    return ours, theirs
