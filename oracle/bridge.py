"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

  liboracle.so      C++ restatement of the reference executor (oracle.cc)
  _ref/libedref.so  the unmodified reference sources + ref_shim.cc

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module. The product (paper_2410_02682_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libedref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

_ref = None
_orc = None


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        err = [C.c_char_p, C.c_size_t]
        lib.edref_plan.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_double, C.c_char_p,
                                   C.POINTER(C.c_void_p)] + err
        lib.edref_free.argtypes = [C.c_void_p]
        lib.edref_artifacts.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_double, C.c_char_p,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)] + err
        lib.edref_generate_input.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_void_p, C.c_int64] + err
        lib.edref_execute.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_double, C.c_char_p,
                                      C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)] + err
        lib.edref_execute_placed.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_double, C.c_char_p,
                                             C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                             C.POINTER(C.c_int32), C.c_int32,
                                             C.POINTER(C.c_void_p), C.POINTER(C.c_double),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int64)] + err
        lib.edref_eval_reference.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)] + err
        lib.edref_eval_vertex.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p] + err
        lib.edref_kernel_vertex.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p] + err
        _ref = lib
    return _ref


def orc():
    global _orc
    if _orc is None:
        lib = C.CDLL(ORACLE_SO)
        err = [C.c_char_p, C.c_size_t]
        lib.oracle_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_int32, C.POINTER(C.c_void_p), C.c_void_p,
                                       C.POINTER(C.c_int64)] + err
        lib.oracle_kernel_eval.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_int] + err
        lib.oracle_eval_expr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + err
        lib.oracle_chunk.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.oracle_assemble.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.oracle_max_rel_err.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        lib.oracle_max_rel_err.restype = C.c_double
        lib.oracle_generate_input.argtypes = [C.c_int64, C.c_int32, C.c_uint64, C.c_int32, C.c_void_p]
        _orc = lib
    return _orc


def _check(code, buf):
    if code != 0:
        raise RefError(code, buf.value.decode(errors="replace"))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ---- reference (compiled) --------------------------------------------------

def ref_plan_json(graph_text: str, p: int, n_machines: int, alpha: float = 0.01, pinned=None) -> dict:
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    pj = json.dumps(pinned).encode() if pinned else None
    _check(ref().edref_plan(graph_text.encode(), p, n_machines, alpha, pj, C.byref(out), err, 1024), err)
    s = C.cast(out, C.c_char_p).value.decode()
    ref().edref_free(out)
    d = json.loads(s)
    d["graph_text"] = graph_text
    if pinned:
        d["pinned"] = pinned
    return d


def ref_artifacts(graph_text: str, p: int, n_machines: int, alpha: float = 0.01, pinned=None):
    """(taskgraph/1, execgraph/1 with machines) as the reference's json_io writes them."""
    tg, eg = C.c_void_p(), C.c_void_p()
    err = C.create_string_buffer(1024)
    pj = json.dumps(pinned).encode() if pinned else None
    _check(ref().edref_artifacts(graph_text.encode(), p, n_machines, alpha, pj, C.byref(tg), C.byref(eg), err, 1024),
           err)
    out = (json.loads(C.cast(tg, C.c_char_p).value.decode()), json.loads(C.cast(eg, C.c_char_p).value.decode()))
    ref().edref_free(tg)
    ref().edref_free(eg)
    return out


def ref_generate_input(graph_text: str, seed: int, vid: int, shape) -> np.ndarray:
    out = np.empty(int(np.prod(shape)), dtype=np.float64)
    err = C.create_string_buffer(1024)
    _check(ref().edref_generate_input(graph_text.encode(), seed, vid, _ptr(out), out.size, err, 1024), err)
    return out.reshape(shape)


def ref_execute(plan_doc: dict, inputs: dict, threaded=True, f32=False, corrupt=False, machine_of=None):
    """Runs the reference run_end_to_end flow (planner re-run from the graph
    text, same p/L/alpha/pins, so the plan is identical). inputs: vid -> f64.
    machine_of (optional) replaces the planner's placement_t::machine_of.
    Returns (outputs dict vid->array, execute seconds, counters, total)."""
    g = plan_doc["graph_text"]
    verts = plan_doc["vertices"]
    arrs = [np.ascontiguousarray(inputs[i], dtype=np.float64) if verts[i]["expr"] is None else None
            for i in range(len(verts))]
    ins = (C.c_void_p * len(verts))(*[_ptr(a) for a in arrs])
    outs_np = [np.empty(verts[o]["bound"], dtype=np.float64) for o in plan_doc["outputs"]]
    outs = (C.c_void_p * max(1, len(outs_np)))(*[_ptr(a) for a in outs_np])
    secs = C.c_double()
    L = plan_doc["n_machines"]
    counters = (C.c_int64 * (3 * L))()
    total = C.c_int64()
    err = C.create_string_buffer(1024)
    pj = json.dumps(plan_doc["pinned"]).encode() if plan_doc.get("pinned") else None
    mo = (C.c_int32 * len(machine_of))(*machine_of) if machine_of is not None else None
    _check(ref().edref_execute_placed(g.encode(), plan_doc["p"], L, plan_doc["alpha"], pj, ins,
                                      int(threaded), int(f32), int(corrupt), mo,
                                      len(machine_of) if machine_of is not None else 0, outs, C.byref(secs),
                                      counters, C.byref(total), err, 1024), err)
    cnt = [(counters[3 * m], counters[3 * m + 1], counters[3 * m + 2]) for m in range(L)]
    return dict(zip(plan_doc["outputs"], outs_np)), secs.value, cnt, total.value


def ref_eval_reference(plan_doc: dict, inputs: dict) -> dict:
    g = plan_doc["graph_text"]
    verts = plan_doc["vertices"]
    arrs = [np.ascontiguousarray(inputs[i], dtype=np.float64) if verts[i]["expr"] is None else None
            for i in range(len(verts))]
    ins = (C.c_void_p * len(verts))(*[_ptr(a) for a in arrs])
    outs_np = [np.empty(v["bound"], dtype=np.float64) for v in verts]
    outs = (C.c_void_p * len(verts))(*[_ptr(a) for a in outs_np])
    err = C.create_string_buffer(1024)
    _check(ref().edref_eval_reference(g.encode(), ins, outs, err, 1024), err)
    return dict(enumerate(outs_np))


# ---- oracle (restatement) --------------------------------------------------

def oracle_generate_input(n: int, integer_valued: bool, seed: int, vid: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    orc().oracle_generate_input(n, int(integer_valued), seed, vid, _ptr(out))
    return out


def generate_inputs(plan, seed: int) -> dict:
    """generate_inputs (runtime.cc:552-571) via the oracle's restatement."""
    iv = plan.integer_valued()
    return {vid: oracle_generate_input(plan.numel(vid), iv, seed, vid).reshape(plan.vertices[vid].bound)
            for vid in plan.input_vertices()}


def oracle_execute(plan, inputs: dict, f32=False, want_chunks=False):
    """The restated executor over the same ed_plan_c the product consumes.
    Returns (outputs, chunks or None, counters, total)."""
    from paper_2410_02682_b200 import abi
    pc, keep = plan.to_c()
    arrs = {vid: np.ascontiguousarray(a, dtype=np.float64) for vid, a in inputs.items()}
    tin = (abi.ed_tensor_in_c * len(arrs))()
    for i, (vid, a) in enumerate(arrs.items()):
        tin[i] = abi.ed_tensor_in_c(vid, abi.DTYPE_F64, a.ctypes.data, a.size)
    outs_np = {o: np.empty(plan.vertices[o].bound, dtype=np.float64) for o in plan.outputs}
    outs = (abi.ed_output_c * max(1, len(outs_np)))()
    for i, (o, a) in enumerate(outs_np.items()):
        outs[i] = abi.ed_output_c(o, abi.DTYPE_F64, a.ctypes.data, a.size)
    chunks = None
    cptr = None
    if want_chunks:
        chunks = [np.empty(u.chunk_bound, dtype=np.float64) for u in plan.exec]
        cptr = (C.c_void_p * len(chunks))(*[_ptr(a) for a in chunks])
    counters = (abi.ed_machine_c * plan.n_machines)()
    total = C.c_int64()
    err = C.create_string_buffer(1024)
    code = orc().oracle_execute(C.byref(pc), tin, len(arrs), int(f32), outs, len(outs_np), cptr,
                                counters, C.byref(total), err, 1024)
    _check(code, err)
    cnt = [(c.fp, c.sent, c.received) for c in counters]
    return outs_np, chunks, cnt, total.value


def max_rel_err(got, expect) -> float:
    """max_rel_err (tensor.cc:9-19)."""
    g = np.asarray(got, dtype=np.float64).ravel()
    e = np.asarray(expect, dtype=np.float64).ravel()
    if g.size == 0:
        return 0.0
    return float(np.max(np.abs(g - e) / np.maximum(1.0, np.abs(e))))
