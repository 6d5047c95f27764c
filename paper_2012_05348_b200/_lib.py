"""ctypes declarations of the C-ABI in include/cbvh.h (argument marshalling only).

The shared library ``libcbvh.so`` is built in-tree by ``paper_2012_05348_b200.build``
(nvcc, sm_100a).  There is no fallback: if the library is missing, importing
this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CBVH_LIB") or os.path.join(HERE, "libcbvh.so")

CBVH_OK, CBVH_EINVAL, CBVH_EMESH, CBVH_EBLOB = 0, -1, -2, -3
CBVH_ECUDA, CBVH_ENOMEM, CBVH_EWORKSPACE, CBVH_EOVERFLOW, CBVH_EINTERNAL = -4, -5, -6, -7, -8
ERROR_NAMES = {0: "CBVH_OK", -1: "CBVH_EINVAL", -2: "CBVH_EMESH", -3: "CBVH_EBLOB", -4: "CBVH_ECUDA",
               -5: "CBVH_ENOMEM", -6: "CBVH_EWORKSPACE", -7: "CBVH_EOVERFLOW", -8: "CBVH_EINTERNAL"}


class cbvh_mesh(C.Structure):
    _fields_ = [("vertices", C.POINTER(C.c_float)), ("num_vertices", C.c_int64),
                ("triangles", C.POINTER(C.c_int32)), ("num_triangles", C.c_int64)]


class cbvh_build_opts(C.Structure):
    _fields_ = [("treelet_nodes", C.c_int), ("leaf_size", C.c_int), ("layout", C.c_int), ("kdop", C.c_int),
                ("align_treelets", C.c_int), ("zero_suppress", C.c_int)]


CBVH_LAYOUT_DELTA, CBVH_LAYOUT_FP16, CBVH_LAYOUT_FP32 = 0, 1, 2
CBVH_FLAG_ALIGNED_TREELETS, CBVH_FLAG_ZERO_SUPPRESSED = 1, 2
LAYOUTS = {"delta": CBVH_LAYOUT_DELTA, "fp16": CBVH_LAYOUT_FP16, "fp32": CBVH_LAYOUT_FP32}


class cbvh_header(C.Structure):
    _fields_ = [("branching", C.c_uint32), ("bits", C.c_uint32), ("treelet_nodes", C.c_uint32),
                ("leaf_size", C.c_uint32), ("code_width", C.c_uint32), ("num_nodes", C.c_uint32),
                ("num_tris", C.c_uint32), ("num_treelets", C.c_uint32), ("depth", C.c_uint32),
                ("num_leaves", C.c_uint32), ("lattice_exp", C.c_int32), ("origin", C.c_float * 3),
                ("root_box", C.c_int32 * 6), ("off_topo", C.c_uint64), ("off_codes", C.c_uint64),
                ("off_treelets", C.c_uint64), ("off_tris", C.c_uint64), ("off_tri_index", C.c_uint64),
                ("total_bytes", C.c_uint64), ("layout", C.c_uint32), ("kdop", C.c_uint32),
                ("off_axes", C.c_uint64), ("flags", C.c_uint32), ("real_nodes", C.c_uint32),
                ("off_blocks", C.c_uint64)]


class cbvh_info(C.Structure):
    _fields_ = [("h", cbvh_header), ("bvh_bytes", C.c_uint64), ("tri_bytes", C.c_uint64),
                ("bytes_per_node", C.c_double), ("code_bytes_per_node", C.c_double)]


class cbvh_bvh(C.Structure):
    _fields_ = [("d_blob", C.c_void_p), ("bytes", C.c_size_t), ("h", cbvh_header),
                ("root_topo", C.c_uint32), ("root_decoded", C.c_int32 * 6),
                ("max_abs_coord", C.c_float), ("axis_origin", C.c_float * 10),
                ("axis_exp", C.c_int32 * 10), ("axis_root", C.c_int32 * 20)]


class cbvh_stats(C.Structure):
    _fields_ = [("bv_tests", C.c_uint64), ("expansions", C.c_uint64), ("leaf_pairs", C.c_uint64),
                ("tri_tests", C.c_uint64), ("nodes_decoded", C.c_uint64), ("record_bytes", C.c_uint64),
                ("tri_bytes", C.c_uint64), ("spills", C.c_uint64), ("kernel_ns", C.c_uint64),
                ("tail_ns", C.c_uint64), ("dumped", C.c_uint64), ("timeline_ns", C.c_uint64 * 8),
                ("iterations", C.c_uint64), ("exact_tests", C.c_uint64), ("treelet_blocks", C.c_uint64),
                ("treelet_bytes", C.c_uint64), ("staged_reads", C.c_uint64)]


class cbvh_query_opts(C.Structure):
    _fields_ = [("descent", C.c_int), ("stats", C.c_int), ("early_exit", C.c_int), ("capped", C.c_int),
                ("treelet_staging", C.c_int)]


CBVH_DESCENT_SIMULTANEOUS, CBVH_DESCENT_LARGER = 0, 1
DESCENT = {"simultaneous": CBVH_DESCENT_SIMULTANEOUS, "alg1": CBVH_DESCENT_SIMULTANEOUS,
           "larger": CBVH_DESCENT_LARGER}

EXPORTS = ("build_compressed_bvh", "cbvh_free_blob", "cbvh_blob_info", "cbvh_bind",
           "cbvh_workspace_bytes", "collide_batch", "distance_batch", "collide_batch_stats",
           "distance_batch_stats", "cbvh_check", "cbvh_read_stats", "cbvh_last_launch_count",
           "cbvh_last_error", "cbvh_set_kernel_events", "collide_batch_ex", "distance_batch_ex")

_lib = None


def load():
    """Load libcbvh.so (raises if it was not built — no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA extension is required; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.build_compressed_bvh.argtypes = [P(cbvh_mesh), C.c_int, C.c_int, P(cbvh_build_opts),
                                       P(P(C.c_uint8)), P(C.c_size_t)]
    L.build_compressed_bvh.restype = C.c_int
    L.cbvh_free_blob.argtypes = [P(C.c_uint8)]
    L.cbvh_free_blob.restype = None
    L.cbvh_blob_info.argtypes = [P(C.c_uint8), C.c_size_t, P(cbvh_info)]
    L.cbvh_blob_info.restype = C.c_int
    L.cbvh_bind.argtypes = [P(C.c_uint8), C.c_size_t, C.c_void_p, P(cbvh_bvh)]
    L.cbvh_bind.restype = C.c_int
    L.cbvh_workspace_bytes.argtypes = [P(cbvh_bvh), P(cbvh_bvh), C.c_int64, C.c_int]
    L.cbvh_workspace_bytes.restype = C.c_size_t
    for name in ("collide_batch", "collide_batch_stats"):
        f = getattr(L, name)
        f.argtypes = [P(cbvh_bvh), P(cbvh_bvh), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_size_t, C.c_void_p]
        f.restype = C.c_int
    for name in ("distance_batch", "distance_batch_stats"):
        f = getattr(L, name)
        f.argtypes = [P(cbvh_bvh), P(cbvh_bvh), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                      C.c_size_t, C.c_void_p]
        f.restype = C.c_int
    L.collide_batch_ex.argtypes = [P(cbvh_bvh), P(cbvh_bvh), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_size_t, C.c_void_p, P(cbvh_query_opts)]
    L.collide_batch_ex.restype = C.c_int
    L.distance_batch_ex.argtypes = [P(cbvh_bvh), P(cbvh_bvh), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_size_t, C.c_void_p, P(cbvh_query_opts)]
    L.distance_batch_ex.restype = C.c_int
    L.cbvh_check.argtypes = [C.c_void_p, C.c_void_p]
    L.cbvh_check.restype = C.c_int
    L.cbvh_read_stats.argtypes = [C.c_void_p, P(cbvh_stats), C.c_void_p]
    L.cbvh_read_stats.restype = C.c_int
    L.cbvh_last_launch_count.argtypes = []
    L.cbvh_last_launch_count.restype = C.c_int
    L.cbvh_set_kernel_events.argtypes = [C.c_void_p, C.c_void_p]
    L.cbvh_set_kernel_events.restype = None
    L.cbvh_last_error.argtypes = []
    L.cbvh_last_error.restype = C.c_char_p
    _lib = L
    return L


class CbvhError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


def check(rc: int):
    if rc != CBVH_OK:
        raise CbvhError(rc, load().cbvh_last_error().decode(errors="replace"))
    return rc
