"""ctypes mirror of include/ed_gpu.h (the C ABI of libed_gpu.so).

Kept field-for-field identical to the header; tests/test_abi.py checks the
struct sizes against the compiled library's own sizeof() exports.
"""
import ctypes as C

ED_OK, ED_ERR_USAGE, ED_ERR_PLAN, ED_ERR_EVAL = 0, 1, 2, 4
ED_ERR_CUDA, ED_ERR_NCCL, ED_ERR_OOM, ED_ERR_UNSUPPORTED = 5, 6, 7, 8

PREC = {"fp32": 0, "tf32": 1, "bf16": 2, "fp64": 3, "fp32x3": 4}
JOIN = {"mul": 0, "add": 1, "sub": 2, "div": 3, "sqdiff": 4, "absdiff": 5}
AGG = {"sum": 0, "max": 1}
MAP = {"relu": 0, "exp": 1, "neg": 2, "scale": 3, "identity": 4}
EXEC_INPUT_CHUNK, EXEC_JOIN, EXEC_REFINEMENT = 0, 1, 2
DTYPE_F64, DTYPE_F32 = 0, 1

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)


class ed_vertex_c(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("arity", C.c_int32),
        ("join_op", C.c_int32),
        ("map_op", C.c_int32),
        ("agg_op", C.c_int32),
        ("scale_c", C.c_double),
        ("rank", C.c_int32),
        ("bound", i64p),
        ("rank_z", C.c_int32),
        ("rank_x", C.c_int32),
        ("rank_y", C.c_int32),
        ("lz", i32p),
        ("lx", i32p),
        ("ly", i32p),
        ("rank_d", C.c_int32),
        ("d", i64p),
        ("inputs", C.c_int32 * 2),
    ]


class ed_exec_vertex_c(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("owner", C.c_int32),
        ("producer", C.c_int32),
        ("consumer", C.c_int32),
        ("slot", C.c_int32),
        ("key_rank", C.c_int32),
        ("key", i64p),
        ("chunk_rank", C.c_int32),
        ("chunk_bound", i64p),
        ("fp", C.c_int64),
        ("sz", C.c_int64),
        ("n_deps", C.c_int32),
        ("deps", i32p),
        ("machine", C.c_int32),
    ]


class ed_plan_c(C.Structure):
    _fields_ = [
        ("n_vertices", C.c_int32),
        ("vertices", C.POINTER(ed_vertex_c)),
        ("n_exec", C.c_int32),
        ("exec", C.POINTER(ed_exec_vertex_c)),
        ("n_outputs", C.c_int32),
        ("outputs", i32p),
        ("n_machines", C.c_int32),
        ("alpha", C.c_double),
    ]


class ed_options_c(C.Structure):
    _fields_ = [
        ("precision", C.c_int32),
        ("corrupt", C.c_int32),
        ("profile", C.c_int32),
        ("no_graph", C.c_int32),
        ("transport", C.c_int32),
        ("sched_mode", C.c_int32),
        ("reserved", C.c_int32 * 2),
    ]


class ed_chunk_in_c(C.Structure):
    _fields_ = [("exec_id", C.c_int32), ("dtype", C.c_int32), ("data", C.c_void_p), ("n", C.c_int64)]


class ed_tensor_in_c(C.Structure):
    _fields_ = [("vertex_id", C.c_int32), ("dtype", C.c_int32), ("data", C.c_void_p), ("n", C.c_int64)]


class ed_output_c(C.Structure):
    _fields_ = [("vertex_id", C.c_int32), ("dtype", C.c_int32), ("data", C.c_void_p), ("n", C.c_int64)]


class ed_machine_c(C.Structure):
    _fields_ = [("fp", C.c_int64), ("sent", C.c_int64), ("received", C.c_int64)]


class ed_report_c(C.Structure):
    _fields_ = [
        ("n_machines", C.c_int32),
        ("machines", C.POINTER(ed_machine_c)),
        ("total_transferred", C.c_int64),
        ("wall_steps", C.c_int64),
        ("max_site_cost", C.c_double),
        ("device_ms", C.c_double),
        ("peer_bytes", C.c_int64),
        ("contraction_flops", C.c_double),
        ("gpu_launches", C.c_int32),
    ]


class ed_kernel_stat_c(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64),
        ("launches", C.c_int32),
        ("ms", C.c_double),
        ("flops", C.c_double),
        ("bytes", C.c_double),
    ]


class ed_sched_op_c(C.Structure):
    _fields_ = [("kind", C.c_int32), ("exec_id", C.c_int32), ("peer", C.c_int32), ("elems", C.c_int64)]


SCHED_COMPUTE, SCHED_SEND, SCHED_RECV = 0, 1, 2
TRANSPORT = {"nccl": 0, "peer": 1}


class ed_cost_model_c(C.Structure):
    _fields_ = [("tensor_flops", C.c_double), ("hbm_bytes", C.c_double), ("link_bytes", C.c_double),
                ("elem_bytes", C.c_int32), ("max_passes", C.c_int32), ("fuse_chains", C.c_int32),
                ("reserved", C.c_int32)]


# Every symbol include/ed_gpu.h declares (tests/test_abi.py checks exports).
EXPORTED = [
    "ed_abi_version", "ed_nccl_unique_id", "ed_ctx_create", "ed_ctx_create_multi", "ed_ctx_destroy",
    "ed_prepare", "ed_plan_destroy", "ed_upload", "ed_upload_tensors", "ed_run",
    "ed_download", "ed_download_chunk", "ed_plan_schedule", "ed_kernel_stats", "ed_gpu_placement",
    "ed_run_steps", "ed_peer_export", "ed_peer_import", "ed_generate_inputs",
]


def declare(lib):
    """Attach argtypes/restypes to a loaded libed_gpu."""
    P = C.c_void_p
    err = [C.c_char_p, C.c_size_t]
    lib.ed_abi_version.restype = C.c_int32
    lib.ed_nccl_unique_id.argtypes = [C.c_void_p, C.c_size_t] + err
    lib.ed_ctx_create.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
                                  C.POINTER(P)] + err
    lib.ed_ctx_create_multi.argtypes = [C.c_int32, i32p, C.POINTER(P)] + err
    lib.ed_ctx_destroy.argtypes = [P]
    lib.ed_ctx_destroy.restype = None
    lib.ed_prepare.argtypes = [P, C.POINTER(ed_plan_c), C.POINTER(ed_options_c), C.POINTER(P)] + err
    lib.ed_plan_destroy.argtypes = [P]
    lib.ed_plan_destroy.restype = None
    lib.ed_upload.argtypes = [P, C.POINTER(ed_chunk_in_c), C.c_int32] + err
    lib.ed_upload_tensors.argtypes = [P, C.POINTER(ed_tensor_in_c), C.c_int32] + err
    lib.ed_run.argtypes = [P, C.POINTER(ed_report_c)] + err
    lib.ed_download.argtypes = [P, C.POINTER(ed_output_c), C.c_int32] + err
    lib.ed_download_chunk.argtypes = [P, C.c_int32, C.c_int32, C.c_void_p, C.c_int64] + err
    lib.ed_plan_schedule.argtypes = [C.POINTER(ed_plan_c), C.c_int32, C.c_int32, C.POINTER(ed_sched_op_c),
                                     C.c_int32, i32p] + err
    lib.ed_kernel_stats.argtypes = [P, C.POINTER(ed_kernel_stat_c), C.c_int32, i32p] + err
    lib.ed_run_steps.argtypes = [P, C.c_int32, C.POINTER(ed_tensor_in_c), C.c_int32, C.POINTER(ed_output_c),
                                 C.c_int32, C.POINTER(ed_report_c)] + err
    lib.ed_generate_inputs.argtypes = [P, C.c_uint64] + err
    lib.ed_peer_export.argtypes = [P, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)] + err
    lib.ed_peer_import.argtypes = [P, C.c_void_p, C.c_size_t, C.c_int32] + err
    lib.ed_gpu_placement.argtypes = [C.POINTER(ed_plan_c), C.POINTER(ed_cost_model_c), i32p,
                                     C.POINTER(C.c_double)] + err
    for name in EXPORTED[1:]:
        f = getattr(lib, name)
        if f.restype is C.c_int:  # default
            f.restype = C.c_int32
    return lib
