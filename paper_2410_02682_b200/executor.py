"""Python host over libed_gpu.so, mirroring the reference's executor API.

    report = execute(plan, inputs, precision="bf16")   # runtime.h:45-49

`plan` is a Plan (the reference planner's task graph + exec graph +
placement); `inputs` maps each input vertex id to its whole tensor (chunked
on the device, relation.cc:31-53) or to {exec_id: chunk}. The report mirrors
run_report_t (runtime.h:27-37). Errors mirror the reference's exception
classes: PlanError ~ plan_error_t, EvalError ~ eval_error_t.

There is no CPU fallback: if the CUDA library is missing or no B200 is
visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .plan import Plan

HERE = os.path.dirname(os.path.abspath(__file__))
# ED_LIB_PATH: a variant build of the same library (development experiments)
LIB_PATH = os.environ.get("ED_LIB_PATH") or os.path.join(HERE, "libed_gpu.so")
# Ranks sharing one GPU (Context.multi with a repeated device) run 2-4 streams
# each; with CUDA's default 8 hardware queues, streams of different ranks alias
# one queue, and a receive spinning on one rank's comm stream can block the
# kernel of another rank that would end its wait (8 ranks on one B200 timed
# out). Takes effect if the process has not created its CUDA context yet.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_lib = None


class EdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class PlanError(EdError):
    """plan_error_t (setup.h:40-42)."""


class EvalError(EdError):
    """eval_error_t (setup.h:45-47)."""


def library():
    """Loads the in-tree CUDA library. Raises if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2410_02682_b200.build`")
        _lib = abi.declare(C.CDLL(LIB_PATH))
        if _lib.ed_abi_version() != 1:
            raise ImportError("libed_gpu ABI version mismatch")
    return _lib


def _check(code, err):
    if code == abi.ED_OK:
        return
    msg = err.value.decode(errors="replace")
    if code == abi.ED_ERR_PLAN:
        raise PlanError(code, msg)
    if code == abi.ED_ERR_EVAL:
        raise EvalError(code, msg)
    raise EdError(code, msg)


def _err():
    return C.create_string_buffer(2048), 2048


@dataclass
class RunReport:
    """run_report_t (runtime.h:27-37) plus device timing."""
    machines: list = field(default_factory=list)     # (fp, sent, received) per machine
    total_transferred: int = 0
    wall_steps: int = 0
    max_site_cost: float = 0.0
    outputs: dict = field(default_factory=dict)      # output vertex -> assembled tensor
    device_ms: float = 0.0
    peer_bytes: int = 0
    contraction_flops: float = 0.0
    gpu_launches: int = 0


class Context:
    """One GPU (one process per GPU; rank/world for multi-GPU plans)."""

    def __init__(self, device=0, rank=0, world=1, nccl_id: bytes | None = None):
        lib = library()
        self.rank, self.world = rank, world
        h = C.c_void_p()
        err, n = _err()
        idbuf = C.create_string_buffer(nccl_id, len(nccl_id)) if nccl_id else None
        _check(lib.ed_ctx_create(device, rank, world, idbuf, len(nccl_id) if nccl_id else 0, C.byref(h), err, n), err)
        self.h = h

    @classmethod
    def multi(cls, device_ids) -> "Context":
        """One process driving len(device_ids) ranks (ed_ctx_create_multi):
        rank r on device_ids[r]; devices may repeat (ranks then share one)."""
        self = cls.__new__(cls)
        lib = library()
        self.rank, self.world = 0, len(device_ids)
        ids = (C.c_int32 * len(device_ids))(*device_ids)
        h = C.c_void_p()
        err, n = _err()
        _check(lib.ed_ctx_create_multi(len(device_ids), ids, C.byref(h), err, n), err)
        self.h = h
        return self

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        err, n = _err()
        _check(library().ed_nccl_unique_id(buf, 128, err, n), err)
        return buf.raw

    def close(self):
        if self.h:
            library().ed_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PreparedPlan:
    """A plan resident on the GPU: buffers allocated, kernels chosen, CUDA graph
    recorded (ed_prepare). Upload, run and download may be repeated."""

    def __init__(self, ctx: Context, plan: Plan, precision="bf16", corrupt=False, profile=False, graph=True,
                 transport="nccl"):
        self.ctx, self.plan = ctx, plan
        self._pc, self._keep = plan.to_c()
        opt = abi.ed_options_c()
        opt.precision = abi.PREC[precision]
        opt.corrupt = int(bool(corrupt))
        opt.profile = int(bool(profile))
        opt.no_graph = int(not graph)
        opt.transport = abi.TRANSPORT[transport]
        h = C.c_void_p()
        err, n = _err()
        _check(library().ed_prepare(ctx.h, C.byref(self._pc), C.byref(opt), C.byref(h), err, n), err)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            library().ed_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- inputs --------------------------------------------------------------
    def upload(self, inputs: dict):
        """inputs: vid -> whole tensor (f64 or f32 ndarray), or
        vid -> {exec_id: chunk ndarray} (a tensor relation)."""
        tensors, chunks, keep = [], [], []
        for vid, val in inputs.items():
            if isinstance(val, dict):
                for eid, ch in val.items():
                    a = _host(ch)
                    keep.append(a)
                    chunks.append(abi.ed_chunk_in_c(eid, _dt(a), a.ctypes.data, a.size))
            else:
                a = _host(val)
                keep.append(a)
                tensors.append(abi.ed_tensor_in_c(vid, _dt(a), a.ctypes.data, a.size))
        err, n = _err()
        if tensors:
            arr = (abi.ed_tensor_in_c * len(tensors))(*tensors)
            _check(library().ed_upload_tensors(self.h, arr, len(tensors), err, n), err)
        if chunks:
            arr = (abi.ed_chunk_in_c * len(chunks))(*chunks)
            _check(library().ed_upload(self.h, arr, len(chunks), err, n), err)

    def generate_inputs(self, seed: int):
        """generate_inputs(graph, seed) (runtime.cc:552-571) on the device, bit
        for bit, chunked into this rank's input chunks (ed_generate_inputs)."""
        err, n = _err()
        _check(library().ed_generate_inputs(self.h, C.c_uint64(seed), err, n), err)

    # ---- run -------------------------------------------------------------------
    def run(self) -> RunReport:
        L = self.plan.n_machines
        machines = (abi.ed_machine_c * L)()
        rep = abi.ed_report_c()
        rep.n_machines = L
        rep.machines = C.cast(machines, C.POINTER(abi.ed_machine_c))
        err, n = _err()
        _check(library().ed_run(self.h, C.byref(rep), err, n), err)
        return RunReport([(m.fp, m.sent, m.received) for m in machines], rep.total_transferred,
                         rep.wall_steps, rep.max_site_cost, {}, rep.device_ms, rep.peer_bytes,
                         rep.contraction_flops, rep.gpu_launches)

    # ---- outputs ---------------------------------------------------------------
    def download(self, dtype=np.float64, into: dict | None = None, vertices=None) -> dict:
        """Assembled graph outputs (or any input / output `vertices`)."""
        outs = {}
        descs = []
        for vid in (self.plan.outputs if vertices is None else vertices):
            a = into[vid] if into is not None else np.empty(self.plan.vertices[vid].bound, dtype=dtype)
            _out_ok(a, int(np.prod(self.plan.vertices[vid].bound)))
            outs[vid] = a
            descs.append(abi.ed_output_c(vid, _dt(a), a.ctypes.data, a.size))
        if descs:
            arr = (abi.ed_output_c * len(descs))(*descs)
            err, n = _err()
            _check(library().ed_download(self.h, arr, len(descs), err, n), err)
        return outs

    # ---- peer transport bootstrap (ED_TRANSPORT_PEER) -------------------------
    def peer_export(self) -> bytes:
        """This rank's blob (IPC handles + chunk offsets) for ed_peer_import."""
        n = C.c_size_t()
        err, en = _err()
        _check(library().ed_peer_export(self.h, None, 0, C.byref(n), err, en), err)
        buf = C.create_string_buffer(n.value)
        _check(library().ed_peer_export(self.h, buf, n.value, C.byref(n), err, en), err)
        return buf.raw[:n.value]

    def peer_import(self, blobs: list):
        """Every rank's blob, in rank order (e.g. from all_gather_object)."""
        if not blobs or any(len(b) != len(blobs[0]) for b in blobs):
            raise ValueError("one equally sized blob per rank")
        joined = b"".join(blobs)
        buf = C.create_string_buffer(joined, len(joined))
        err, en = _err()
        _check(library().ed_peer_import(self.h, buf, len(blobs[0]), len(blobs), err, en), err)

    def run_steps(self, inputs: list, outputs: list) -> RunReport:
        """ed_run_steps: len(inputs) end-to-end steps (upload inputs[s], run,
        download into outputs[s]) with step s+1's H2D overlapping step s's
        compute and D2H. inputs[s]: vid -> whole tensor; outputs[s]: vid ->
        preallocated array (pinned host memory for the copies to overlap)."""
        if len(inputs) != len(outputs):
            raise ValueError("one output dict per input dict")
        n_steps = len(inputs)
        n_in = len(inputs[0]) if n_steps else 0
        n_out = len(outputs[0]) if n_steps else 0
        tin = (abi.ed_tensor_in_c * max(1, n_steps * n_in))()
        tout = (abi.ed_output_c * max(1, n_steps * n_out))()
        keep = []
        for st in range(n_steps):
            if len(inputs[st]) != n_in or len(outputs[st]) != n_out:
                raise ValueError("every step needs the same inputs and outputs")
            for k, (vid, val) in enumerate(inputs[st].items()):
                a = _host(val)
                keep.append(a)
                tin[st * n_in + k] = abi.ed_tensor_in_c(vid, _dt(a), a.ctypes.data, a.size)
            for k, (vid, a) in enumerate(outputs[st].items()):
                _out_ok(a, int(np.prod(self.plan.vertices[vid].bound)))
                tout[st * n_out + k] = abi.ed_output_c(vid, _dt(a), a.ctypes.data, a.size)
        L = self.plan.n_machines
        machines = (abi.ed_machine_c * L)()
        rep = abi.ed_report_c()
        rep.n_machines = L
        rep.machines = C.cast(machines, C.POINTER(abi.ed_machine_c))
        err, n = _err()
        _check(library().ed_run_steps(self.h, n_steps, tin, n_in, tout, n_out, C.byref(rep), err, n), err)
        return RunReport([(m.fp, m.sent, m.received) for m in machines], rep.total_transferred,
                         rep.wall_steps, rep.max_site_cost, {}, rep.device_ms, rep.peer_bytes,
                         rep.contraction_flops, rep.gpu_launches)

    def download_chunk(self, exec_id: int, dtype=np.float64) -> np.ndarray:
        u = self.plan.exec[exec_id]
        a = np.empty(u.chunk_bound, dtype=dtype)
        _out_ok(a, int(np.prod(u.chunk_bound)))
        err, n = _err()
        _check(library().ed_download_chunk(self.h, exec_id, _dt(a), a.ctypes.data, a.size, err, n), err)
        return a

    def kernel_stats(self):
        cap = 256
        arr = (abi.ed_kernel_stat_c * cap)()
        k = C.c_int32()
        err, n = _err()
        _check(library().ed_kernel_stats(self.h, arr, cap, C.byref(k), err, n), err)
        return [dict(name=arr[i].name.decode(), launches=arr[i].launches, ms=arr[i].ms,
                     flops=arr[i].flops, bytes=arr[i].bytes) for i in range(min(k.value, cap))]


def _host(a):
    a = np.asarray(a)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    return np.ascontiguousarray(a)


def _dt(a):
    if a.dtype == np.float64:
        return abi.DTYPE_F64
    if a.dtype == np.float32:
        return abi.DTYPE_F32
    raise ValueError(f"unsupported dtype {a.dtype}: the library reads and writes float32 / float64 only")


def _out_ok(a, n):
    """An output buffer the library writes n elements into through a raw
    pointer: float32 / float64, C-contiguous, writeable, exactly n elements."""
    if not isinstance(a, np.ndarray):
        raise ValueError("output buffers must be numpy arrays")
    _dt(a)
    if not a.flags.c_contiguous or not a.flags.writeable:
        raise ValueError("output buffers must be C-contiguous and writeable")
    if a.size != n:
        raise ValueError(f"output buffer has {a.size} elements, the tensor {n}")


def plan_schedule(plan: Plan, rank: int, world: int):
    """Rank `rank`'s logical schedule (host-only; no GPU needed):
    [(kind, exec_id, peer, elems)] with kind in {"compute", "send", "recv"}."""
    pc, keep = plan.to_c()
    cap = 4 * len(plan.exec) + 16
    arr = (abi.ed_sched_op_c * cap)()
    n = C.c_int32()
    err, en = _err()
    _check(library().ed_plan_schedule(C.byref(pc), rank, world, arr, cap, C.byref(n), err, en), err)
    names = {abi.SCHED_COMPUTE: "compute", abi.SCHED_SEND: "send", abi.SCHED_RECV: "recv"}
    return [(names[arr[i].kind], arr[i].exec_id, arr[i].peer, arr[i].elems) for i in range(n.value)]


def gpu_placement(plan: Plan, tensor_tflops=1652.1, hbm_gbs=6548.8, link_gbs=900.0, elem_bytes=4, passes=0,
                  fuse_chains=True):
    """GPU-aware re-placement (ed_gpu_placement; host-only): returns
    (plan with the new machine_of, estimated busiest-GPU ms before, after).
    Defaults: MEASURED_PEAKS.json bf16 / HBM copy rates, NVLink 5 per
    direction. fuse_chains keeps each region of a fusable chain on one GPU."""
    pc, keep = plan.to_c()
    model = abi.ed_cost_model_c(tensor_tflops * 1e12, hbm_gbs * 1e9, link_gbs * 1e9, elem_bytes, passes,
                                int(fuse_chains), 0)
    m = (C.c_int32 * max(1, len(plan.exec)))()
    est = (C.c_double * 2)()
    err, en = _err()
    _check(library().ed_gpu_placement(C.byref(pc), C.byref(model), m, est, err, en), err)
    return plan.with_machines([m[i] for i in range(len(plan.exec))]), est[0], est[1]


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def execute(plan: Plan, inputs: dict, precision="bf16", corrupt=False, ctx: Context | None = None,
            out_dtype=np.float64) -> RunReport:
    """execute() (runtime.cc:382-451) on the GPU: seed, run, assemble outputs."""
    pp = PreparedPlan(ctx or default_context(), plan, precision=precision, corrupt=corrupt)
    try:
        pp.upload(inputs)
        rep = pp.run()
        rep.outputs = pp.download(dtype=out_dtype)
        return rep
    finally:
        pp.close()
