"""Host-side model of a placed ExecGraph (the reference planner's output).

Loads "edplan/1" JSON — the reference's task_graph_t (decomp.h:21-30),
exec_graph_t (execgraph.h:36-49) and placement_t::machine_of
(placement.h:9-15), as written by oracle/ref_shim.cc from the unmodified
reference planner — and flattens it into the C ABI's ed_plan_c
(include/ed_gpu.h). Mirrors the reference's data types by name so the
parity tests read like test_runtime.cc.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

from . import abi


@dataclass
class Expr:
    """einsum_expr_t (einsum.h:9-38); labels are strings."""
    out: list
    ins: list
    join: str | None
    map: str | None
    scale_c: float
    agg: str | None

    @property
    def is_binary(self):
        return len(self.ins) == 2

    def xy_labels(self):
        return [l for ls in self.ins for l in ls]

    def distinct_labels(self):
        r = list(self.ins[0])
        for l in (self.ins[1] if self.is_binary else []):
            if l not in r:
                r.append(l)
        return r

    def agg_labels(self):
        return [l for l in self.distinct_labels() if l not in self.out]


@dataclass
class Vertex:
    """ein_vertex_t (einsum.h:42-47) + its d (task_graph_t::d)."""
    vid: int
    name: str
    bound: list
    inputs: list
    expr: Expr | None
    d: list
    out_partition: list

    @property
    def is_input(self):
        return self.expr is None


@dataclass
class ExecVertex:
    """exec_vertex_t (execgraph.h:14-34) + machine_of."""
    id: int
    kind: int
    owner: int
    producer: int
    consumer: int
    slot: int
    key: list
    chunk_bound: list
    fp: int
    sz: int
    deps: list
    machine: int


@dataclass
class Plan:
    p: int
    n_machines: int
    alpha: float
    vertices: list
    outputs: list
    exec: list
    objective: int = 0
    source: dict = field(default_factory=dict)

    # ---- construction ----------------------------------------------------
    @staticmethod
    def from_json(obj) -> "Plan":
        if isinstance(obj, (str, bytes)):
            obj = json.loads(obj)
        if obj.get("schema") != "edplan/1":
            raise ValueError("not an edplan/1 document")
        verts = []
        for vid, jv in enumerate(obj["vertices"]):
            je = jv["expr"]
            expr = None
            if je is not None:
                expr = Expr(je["out"], je["in"], je["join"], je["map"], float(je["scale_c"]), je["agg"])
            verts.append(Vertex(vid, jv["name"], list(jv["bound"]), list(jv["inputs"]), expr,
                                list(jv["d"]), list(jv["out_partition"])))
        ex = [ExecVertex(j["id"], j["kind"], j["owner"], j["producer"], j["consumer"], j["slot"],
                         list(j["key"]), list(j["chunk_bound"]), j["fp"], j["sz"], list(j["deps"]),
                         j["machine"]) for j in obj["exec"]]
        return Plan(obj["p"], obj["n_machines"], obj["alpha"], verts, list(obj["outputs"]), ex,
                    obj.get("objective", 0), obj)

    @staticmethod
    def from_reference_artifacts(taskgraph, execgraph, alpha=0.01, n_machines=None) -> "Plan":
        """Plan ingestion from the reference's own artifacts: taskgraph/1
        (json_io.cc:63-103, `eindecomp optimize --out`) and execgraph/1 with
        machines (json_io.cc:131-155, `eindecomp place --out`). Fields the
        execgraph/1 schema omits are re-derived as explode() sets them
        (execgraph.cc:150-185): a refinement's consumer/slot from the join
        that reads it, its owner (the consumer for input-side layers), and
        every chunk_bound from the task graph's partitions."""
        if isinstance(taskgraph, (str, bytes)):
            taskgraph = json.loads(taskgraph)
        if isinstance(execgraph, (str, bytes)):
            execgraph = json.loads(execgraph)
        if taskgraph.get("schema") != "taskgraph/1" or execgraph.get("schema") != "execgraph/1":
            raise ValueError("expected taskgraph/1 and execgraph/1 documents")
        names = [jv["id"] for jv in taskgraph["vertices"]]
        index = {n: i for i, n in enumerate(names)}
        verts = []
        for vid, jv in enumerate(taskgraph["vertices"]):
            je = jv["einsum"]
            expr = None
            if je is not None:
                mp, c = je.get("map"), 0.0
                if mp is not None and mp.startswith("scale("):
                    mp, c = "scale", float(mp[6:-1])
                expr = Expr(je["out"], je["inns"], je.get("join"), mp, c, je.get("agg"))
            verts.append(Vertex(vid, jv["id"], list(jv["bound"]), [index[n] for n in jv["inputs"]], expr,
                                list(jv["d"]), list(jv["out_partition"])))
        kinds = {"input-chunk": 0, "join-kernel": 1, "refinement": 2}
        raw = execgraph["vertices"]
        readers = {}
        for jv in raw:
            if kinds[jv["kind"]] == 1:
                for slot, d in enumerate(jv["deps"]):
                    readers.setdefault(d, (index[jv["vertex"]], slot))

        def project(d, ls, lxy):
            return [d[lxy.index(l)] for l in ls]

        ex = []
        for jv in raw:
            kind = kinds[jv["kind"]]
            prod = index[jv["vertex"]]
            v = verts[prod]
            consumer, slot, owner = -1, -1, prod
            if kind == 0:
                cb = [b // d for b, d in zip(v.bound, v.d)]
            elif kind == 1:
                e = v.expr
                lxy = e.xy_labels()
                bxy = [b for i in v.inputs for b in verts[i].bound]
                local = [b // d for b, d in zip(bxy, v.d)]
                cb = project(local, e.out, lxy)
            else:
                if jv["id"] in readers:
                    consumer, slot = readers[jv["id"]]
                    ce = verts[consumer].expr
                    part = project(verts[consumer].d, ce.ins[slot], ce.xy_labels())
                    if v.expr is None:
                        owner = consumer
                else:
                    part = v.out_partition
                cb = [b // d for b, d in zip(v.bound, part)]
            ex.append(ExecVertex(jv["id"], kind, owner, prod, consumer, slot, list(jv["key"]), cb, jv["fp"],
                                 jv["sz"], list(jv["deps"]), jv.get("machine", 0)))
        if n_machines is None:
            n_machines = 1 + max((u.machine for u in ex), default=0)
        outputs = [index[n] for n in taskgraph["outputs"]]
        return Plan(None, n_machines, alpha, verts, outputs, ex, taskgraph.get("predicted_cost", 0),
                    {"taskgraph": taskgraph, "execgraph": execgraph})

    def with_machines(self, machine_of) -> "Plan":
        """The same plan under another placement (placement_t::machine_of):
        exec graph, keys and fold order unchanged."""
        import dataclasses
        if len(machine_of) != len(self.exec):
            raise ValueError("machine_of needs one entry per exec vertex")
        ex = [dataclasses.replace(u, deps=list(u.deps), machine=int(m)) for u, m in zip(self.exec, machine_of)]
        return dataclasses.replace(self, exec=ex)

    @staticmethod
    def load(path) -> "Plan":
        with open(path) as f:
            return Plan.from_json(json.load(f))

    # ---- exec_graph_t indices (execgraph.h:42-46) --------------------------
    def input_chunks_of(self, vid):
        return [u.id for u in self.exec if u.kind == abi.EXEC_INPUT_CHUNK and u.producer == vid]

    def joins_of(self, vid):
        return [u.id for u in self.exec if u.kind == abi.EXEC_JOIN and u.producer == vid]

    def output_refines_of(self, vid):
        return [u.id for u in self.exec
                if u.kind == abi.EXEC_REFINEMENT and u.producer == vid and u.consumer < 0]

    def input_vertices(self):
        return [v.vid for v in self.vertices if v.is_input]

    def find(self, name):
        for v in self.vertices:
            if v.name == name:
                return v.vid
        return -1

    def numel(self, vid):
        return math.prod(self.vertices[vid].bound)

    def contraction_flops(self):
        """2 * sum fp over mul/sum join kernels (SURVEY 8(d) unit of work)."""
        tot = 0
        for u in self.exec:
            if u.kind == abi.EXEC_JOIN:
                e = self.vertices[u.producer].expr
                if e.join == "mul" and e.agg == "sum":
                    tot += 2 * u.fp
        return tot

    def integer_valued(self):
        """uses_only_sum_mul (runtime.cc:358-378): generate_inputs' switch."""
        for v in self.vertices:
            e = v.expr
            if e is None:
                continue
            if e.join is not None and e.join not in ("mul", "add"):
                return False
            if e.map is not None and e.map not in ("identity", "relu", "neg"):
                return False
            if e.agg is not None and e.agg not in ("sum", "max"):
                return False
        return True

    # ---- C ABI flattening ------------------------------------------------
    def to_c(self):
        """Returns (ed_plan_c, keepalive). Keep the keepalive referenced for
        as long as the C struct is in use."""
        keep = []
        label_ids = {}

        def lab(ls):
            arr = (C.c_int32 * max(1, len(ls)))(*[label_ids.setdefault(l, len(label_ids)) for l in ls])
            keep.append(arr)
            return C.cast(arr, abi.i32p)

        def i64(xs):
            arr = (C.c_int64 * max(1, len(xs)))(*xs)
            keep.append(arr)
            return C.cast(arr, abi.i64p)

        V = (abi.ed_vertex_c * len(self.vertices))()
        for i, v in enumerate(self.vertices):
            c = V[i]
            name = v.name.encode()
            keep.append(name)
            c.name = name
            c.rank = len(v.bound)
            c.bound = i64(v.bound)
            c.rank_d = len(v.d)
            c.d = i64(v.d)
            c.inputs[0] = v.inputs[0] if len(v.inputs) > 0 else -1
            c.inputs[1] = v.inputs[1] if len(v.inputs) > 1 else -1
            e = v.expr
            if e is None:
                c.arity, c.join_op, c.map_op, c.agg_op = 0, -1, -1, -1
                c.rank_z = c.rank_x = c.rank_y = 0
                c.lz = c.lx = c.ly = lab([])
                continue
            c.arity = len(e.ins)
            c.join_op = abi.JOIN[e.join] if e.join else -1
            c.map_op = abi.MAP[e.map] if e.map else -1
            c.agg_op = abi.AGG[e.agg] if e.agg else -1
            c.scale_c = e.scale_c
            c.rank_z, c.lz = len(e.out), lab(e.out)
            c.rank_x, c.lx = len(e.ins[0]), lab(e.ins[0])
            if c.arity == 2:
                c.rank_y, c.ly = len(e.ins[1]), lab(e.ins[1])
            else:
                c.rank_y, c.ly = 0, lab([])
        X = (abi.ed_exec_vertex_c * len(self.exec))()
        for i, u in enumerate(self.exec):
            c = X[i]
            c.kind, c.owner, c.producer, c.consumer, c.slot = u.kind, u.owner, u.producer, u.consumer, u.slot
            c.key_rank, c.key = len(u.key), i64(u.key)
            c.chunk_rank, c.chunk_bound = len(u.chunk_bound), i64(u.chunk_bound)
            c.fp, c.sz = u.fp, u.sz
            deps = (C.c_int32 * max(1, len(u.deps)))(*u.deps)
            keep.append(deps)
            c.n_deps, c.deps = len(u.deps), C.cast(deps, abi.i32p)
            c.machine = u.machine
        outs = (C.c_int32 * max(1, len(self.outputs)))(*self.outputs)
        keep += [V, X, outs]
        plan = abi.ed_plan_c(len(self.vertices), C.cast(V, C.POINTER(abi.ed_vertex_c)),
                             len(self.exec), C.cast(X, C.POINTER(abi.ed_exec_vertex_c)),
                             len(self.outputs), C.cast(outs, abi.i32p), self.n_machines, self.alpha)
        return plan, keep
