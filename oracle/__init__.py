"""ctypes front-end of the fp64 CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never by the product package
paper_2012_05348_b200/.  It shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp into oracle/liboracle.so with g++ (plain -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        dp, fp, ip, i64p, vp, u8p = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_void_p,
                                     C.POINTER(C.c_uint8))
        i64 = C.c_int64
        for name in ("oracle_tri_tri_distance", "oracle_tri_tri_pen", "oracle_signed_separation"):
            getattr(L, name).argtypes = [dp, dp]
            getattr(L, name).restype = C.c_double
        L.oracle_tri_tri_intersect.argtypes = [dp, dp]
        L.oracle_tri_tri_intersect.restype = C.c_int
        L.oracle_point_triangle_distance.argtypes = [dp, dp]
        L.oracle_point_triangle_distance.restype = C.c_double
        L.oracle_segment_segment_distance.argtypes = [dp, dp, dp, dp]
        L.oracle_segment_segment_distance.restype = C.c_double
        L.oracle_tree_from_mesh.argtypes = [fp, i64, ip, i64, C.c_int]
        L.oracle_tree_from_mesh.restype = vp
        L.oracle_tree_from_blob.argtypes = [u8p, C.c_uint64, fp, i64, ip, i64, C.c_int]
        L.oracle_tree_from_blob.restype = vp
        L.oracle_tree_free.argtypes = [vp]
        L.oracle_tree_free.restype = None
        L.oracle_tree_num_nodes.argtypes = [vp]
        L.oracle_tree_num_nodes.restype = i64
        L.oracle_collide.argtypes = [vp, vp, fp, i64, C.c_double, C.c_int, i64p, i64p, i64p, i64p]
        L.oracle_collide.restype = C.c_int
        L.oracle_collide_pairs.argtypes = [vp, vp, fp, C.c_double, i64p, i64]
        L.oracle_collide_pairs.restype = i64
        L.oracle_distance.argtypes = [vp, vp, fp, i64, C.c_int, dp, i64p]
        L.oracle_distance.restype = C.c_int
        L.oracle_bruteforce_collide.argtypes = [vp, vp, fp, i64, C.c_double, C.c_int, i64p, i64p, i64p]
        L.oracle_bruteforce_collide.restype = C.c_int
        L.oracle_bruteforce_pairs.argtypes = [vp, vp, fp, i64p, i64]
        L.oracle_bruteforce_pairs.restype = i64
        L.oracle_bruteforce_distance.argtypes = [vp, vp, fp, i64, C.c_int, dp]
        L.oracle_bruteforce_distance.restype = C.c_int
        L.oracle_check_blob.argtypes = [u8p, C.c_uint64, fp, i64, ip, i64, i64p]
        L.oracle_check_blob.restype = i64
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _tri(t) -> np.ndarray:
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float64).reshape(9))
    return t


# ---------------------------------------------------------------- primitives

def tri_tri_intersect(V, U) -> bool:
    V, U = _tri(V), _tri(U)
    return bool(lib().oracle_tri_tri_intersect(_p(V, C.c_double), _p(U, C.c_double)))


def tri_tri_distance(V, U) -> float:
    V, U = _tri(V), _tri(U)
    return lib().oracle_tri_tri_distance(_p(V, C.c_double), _p(U, C.c_double))


def tri_tri_pen(V, U) -> float:
    V, U = _tri(V), _tri(U)
    return lib().oracle_tri_tri_pen(_p(V, C.c_double), _p(U, C.c_double))


def signed_separation(V, U) -> float:
    V, U = _tri(V), _tri(U)
    return lib().oracle_signed_separation(_p(V, C.c_double), _p(U, C.c_double))


def point_triangle_distance(p, T) -> float:
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(3))
    T = _tri(T)
    return lib().oracle_point_triangle_distance(_p(p, C.c_double), _p(T, C.c_double))


def segment_segment_distance(p0, p1, q0, q1) -> float:
    a = [np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(3)) for x in (p0, p1, q0, q1)]
    return lib().oracle_segment_segment_distance(*[_p(x, C.c_double) for x in a])


# ---------------------------------------------------------------- trees

class Tree:
    """An oracle BVH: its own binary median split, or a blob's decoded topology."""

    def __init__(self, handle, verts, tris):
        self.h = handle
        self._keep = (verts, tris)

    @classmethod
    def from_mesh(cls, verts, tris, leaf_size: int = 4) -> "Tree":
        v = np.ascontiguousarray(verts, dtype=np.float32)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = lib().oracle_tree_from_mesh(_p(v, C.c_float), len(v), _p(t, C.c_int32), len(t), leaf_size)
        return cls(h, v, t)

    @classmethod
    def from_blob(cls, blob: bytes | np.ndarray, verts, tris, exact_boxes: bool = False) -> "Tree":
        b = np.frombuffer(bytes(blob), dtype=np.uint8) if not isinstance(blob, np.ndarray) else blob
        b = np.ascontiguousarray(b, dtype=np.uint8)
        v = np.ascontiguousarray(verts, dtype=np.float32)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = lib().oracle_tree_from_blob(_p(b, C.c_uint8), len(b), _p(v, C.c_float), len(v),
                                        _p(t, C.c_int32), len(t), int(exact_boxes))
        if not h:
            raise ValueError("malformed blob")
        return cls(h, v, t)

    @property
    def num_nodes(self) -> int:
        return int(lib().oracle_tree_num_nodes(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_tree_free(self.h)
            self.h = None


def model_extent(verts) -> float:
    """AABB diagonal of a mesh (reading R12: the moving model A's extent)."""
    v = np.asarray(verts, dtype=np.float64)
    return float(np.linalg.norm(v.max(axis=0) - v.min(axis=0)))


def band_delta(verts_A) -> float:
    """delta = 1e-6 x model extent of A (BASELINE.json north_star tolerance)."""
    return 1e-6 * model_extent(verts_A)


def collide(A: Tree, B: Tree, poses, delta: float, nthreads: int = 0):
    """Per pose: (count, H, Z, stats[bv_tests, leaf_pairs])."""
    P = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, 12)
    n = len(P)
    cnt, H, Z = (np.zeros(n, np.int64) for _ in range(3))
    st = np.zeros(2, np.int64)
    lib().oracle_collide(A.h, B.h, _p(P, C.c_float), n, float(delta), int(nthreads),
                         _p(cnt, C.c_int64), _p(H, C.c_int64), _p(Z, C.c_int64), _p(st, C.c_int64))
    return cnt, H, Z, st


def collide_pairs(A: Tree, B: Tree, pose, delta: float = 0.0) -> set:
    P = np.ascontiguousarray(pose, dtype=np.float32).reshape(12)
    cap = 1 << 16
    buf = np.zeros(2 * cap, np.int64)
    n = lib().oracle_collide_pairs(A.h, B.h, _p(P, C.c_float), float(delta), _p(buf, C.c_int64), cap)
    assert n <= cap
    return set(map(tuple, buf[: 2 * n].reshape(-1, 2).tolist()))


def distance(A: Tree, B: Tree, poses, nthreads: int = 0):
    P = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, 12)
    d = np.zeros(len(P), np.float64)
    st = np.zeros(1, np.int64)
    lib().oracle_distance(A.h, B.h, _p(P, C.c_float), len(P), int(nthreads), _p(d, C.c_double),
                          _p(st, C.c_int64))
    return d, st


def bruteforce_collide(A: Tree, B: Tree, poses, delta: float, nthreads: int = 0):
    P = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, 12)
    n = len(P)
    cnt, H, Z = (np.zeros(n, np.int64) for _ in range(3))
    lib().oracle_bruteforce_collide(A.h, B.h, _p(P, C.c_float), n, float(delta), int(nthreads),
                                    _p(cnt, C.c_int64), _p(H, C.c_int64), _p(Z, C.c_int64))
    return cnt, H, Z


def bruteforce_pairs(A: Tree, B: Tree, pose) -> set:
    P = np.ascontiguousarray(pose, dtype=np.float32).reshape(12)
    cap = 1 << 16
    buf = np.zeros(2 * cap, np.int64)
    n = lib().oracle_bruteforce_pairs(A.h, B.h, _p(P, C.c_float), _p(buf, C.c_int64), cap)
    assert n <= cap
    return set(map(tuple, buf[: 2 * n].reshape(-1, 2).tolist()))


def bruteforce_distance(A: Tree, B: Tree, poses, nthreads: int = 0):
    P = np.ascontiguousarray(poses, dtype=np.float32).reshape(-1, 12)
    d = np.zeros(len(P), np.float64)
    lib().oracle_bruteforce_distance(A.h, B.h, _p(P, C.c_float), len(P), int(nthreads),
                                     _p(d, C.c_double))
    return d


CHECK_FIELDS = ("malformed", "containment", "child_not_in_parent", "triangle_partition",
                "soup_mismatch", "treelet_partition", "treelet_oversize", "treelet_disconnected",
                "arity", "nodes_checked")


def check_blob(blob, verts, tris) -> dict:
    """Independent decode + invariant check of a blob; returns violation counts."""
    b = np.frombuffer(bytes(blob), dtype=np.uint8) if not isinstance(blob, np.ndarray) else blob
    b = np.ascontiguousarray(b, dtype=np.uint8)
    v = np.ascontiguousarray(verts, dtype=np.float32)
    t = np.ascontiguousarray(tris, dtype=np.int32)
    rep = np.zeros(10, np.int64)
    total = lib().oracle_check_blob(_p(b, C.c_uint8), len(b), _p(v, C.c_float), len(v),
                                    _p(t, C.c_int32), len(t), _p(rep, C.c_int64))
    out = dict(zip(CHECK_FIELDS, rep.tolist()))
    out["violations"] = int(total)
    return out
