"""Thin Python binding over the C-ABI (include/cbvh.h): argument marshalling only.

Every step of the hot path runs in libcbvh.so (host builder in C++, traversal
and leaf tests in sm_100a CUDA kernels).  PyTorch supplies device memory and
streams.  Names follow the C-ABI: build_compressed_bvh, collide_batch,
distance_batch.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L


def _torch():
    import torch
    return torch


@dataclass
class CompressedBVH:
    """A host blob (numpy uint8) plus, after ``to_device``, its bound device copy."""

    blob: np.ndarray
    info: dict
    device_blob: object = None  # torch.uint8 tensor on the GPU
    bound: L.cbvh_bvh = None

    @property
    def nbytes(self) -> int:
        return int(self.blob.nbytes)

    def to_device(self, device="cuda") -> "CompressedBVH":
        torch = _torch()
        d = torch.from_numpy(self.blob).to(device)
        if d.data_ptr() % 256:
            raise RuntimeError("device blob not 256-byte aligned")
        b = L.cbvh_bvh()
        L.check(L.load().cbvh_bind(self.blob.ctypes.data_as(C.POINTER(C.c_uint8)), self.blob.nbytes,
                                   C.c_void_p(d.data_ptr()), C.byref(b)))
        self.device_blob, self.bound = d, b
        return self


def blob_info(blob: np.ndarray) -> dict:
    info = L.cbvh_info()
    b = np.ascontiguousarray(blob, dtype=np.uint8)
    L.check(L.load().cbvh_blob_info(b.ctypes.data_as(C.POINTER(C.c_uint8)), b.nbytes, C.byref(info)))
    h = info.h
    return dict(branching=h.branching, bits=h.bits, treelet_nodes=h.treelet_nodes, leaf_size=h.leaf_size,
                code_width=h.code_width, num_nodes=h.num_nodes, num_tris=h.num_tris,
                num_treelets=h.num_treelets, depth=h.depth, num_leaves=h.num_leaves,
                lattice_exp=h.lattice_exp, origin=tuple(h.origin), root_box=tuple(h.root_box),
                off_topo=h.off_topo, off_codes=h.off_codes, off_treelets=h.off_treelets,
                off_tris=h.off_tris, off_tri_index=h.off_tri_index, total_bytes=h.total_bytes,
                layout={v: k for k, v in L.LAYOUTS.items()}[h.layout], kdop=h.kdop, off_axes=h.off_axes,
                aligned_treelets=bool(h.flags & L.CBVH_FLAG_ALIGNED_TREELETS), real_nodes=h.real_nodes,
                zero_suppressed=bool(h.flags & L.CBVH_FLAG_ZERO_SUPPRESSED), off_blocks=h.off_blocks,
                bvh_bytes=info.bvh_bytes, tri_bytes=info.tri_bytes, bytes_per_node=info.bytes_per_node,
                code_bytes_per_node=info.code_bytes_per_node)


def build_compressed_bvh(vertices, triangles, branching: int = 4, bits: int = 8,
                         treelet_nodes: int = 32, leaf_size: int = 4, layout: str = "delta",
                         kdop: int = 6, align_treelets: bool = False, zero_suppress: bool = False) -> CompressedBVH:
    """C-ABI build_compressed_bvh: host BVH build, lattice quantization,
    predictor–corrector codes and treelet packing.

    layout: "delta" (the compressed layout), or "fp16" / "fp32" absolute
    boxes for the paper's half-vs-float comparison (§III.A).
    kdop: 6 (AABB) or 14 / 18 / 26 — k-DOP bounding volumes (Table I), delta
    coded per slab direction; used for the static model B.
    align_treelets: whole treelets packed into T-slot blocks so the traversal
    can stage treelet blocks in shared memory.
    zero_suppress: integer-compressed corrections: per node a field
    presence mask and only the non-zero fields; implies align_treelets, and
    queries on such blobs decode from staged blocks."""
    if layout not in L.LAYOUTS:
        raise ValueError(f"layout must be one of {sorted(L.LAYOUTS)}")
    lib = L.load()
    v = np.ascontiguousarray(vertices, dtype=np.float32).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
    mesh = L.cbvh_mesh(v.ctypes.data_as(C.POINTER(C.c_float)), len(v),
                       t.ctypes.data_as(C.POINTER(C.c_int32)), len(t))
    opts = L.cbvh_build_opts(int(treelet_nodes), int(leaf_size), L.LAYOUTS[layout], int(kdop), int(bool(align_treelets)),
                             int(bool(zero_suppress)))
    out = C.POINTER(C.c_uint8)()
    n = C.c_size_t(0)
    L.check(lib.build_compressed_bvh(C.byref(mesh), int(branching), int(bits), C.byref(opts),
                                     C.byref(out), C.byref(n)))
    try:
        blob = np.ctypeslib.as_array(out, shape=(n.value,)).copy()
    finally:
        lib.cbvh_free_blob(out)
    return CompressedBVH(blob=blob, info=blob_info(blob))


class Workspace:
    """Device workspace (control words, stats, per-warp stack spill areas)."""

    def __init__(self, A: CompressedBVH, B: CompressedBVH, mode: int = 0, device="cuda"):
        torch = _torch()
        nb = L.load().cbvh_workspace_bytes(C.byref(A.bound), C.byref(B.bound), 0, int(mode))
        if nb == 0:
            raise L.CbvhError(L.CBVH_ECUDA, "cbvh_workspace_bytes failed: "
                              + L.load().cbvh_last_error().decode(errors="replace"))
        self.nbytes = int(nb)
        self.tensor = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        assert self.tensor.data_ptr() % 256 == 0

    @property
    def ptr(self) -> int:
        return self.tensor.data_ptr()


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _check_poses(poses):
    torch = _torch()
    if not (isinstance(poses, torch.Tensor) and poses.is_cuda and poses.dtype == torch.float32):
        raise TypeError("poses must be a CUDA float32 tensor [N, 12]")
    if poses.dim() != 2 or poses.shape[1] != 12 or not poses.is_contiguous():
        raise ValueError("poses must be contiguous [N, 12] row-major [R|t]")
    return int(poses.shape[0])


def _check_out(name, t, N, dtypes, device):
    """Caller-supplied output buffer: the kernels write N elements through its pointer."""
    torch = _torch()
    if not isinstance(t, torch.Tensor) or t.dtype not in dtypes:
        raise TypeError(f"{name} must be a tensor of dtype {' or '.join(map(str, dtypes))}")
    if t.device != device or not t.is_contiguous() or t.numel() < N:
        raise ValueError(f"{name} must be contiguous with >= {N} elements on {device}")


def _check_bvh(T: "CompressedBVH", device):
    if T.bound is None or T.device_blob is None:
        raise ValueError("CompressedBVH is not on a device: call .to_device() first")
    if T.device_blob.device != device:
        raise ValueError(f"blob is on {T.device_blob.device}, poses on {device}")


def _temp_workspace(A, B, mode, device, stream):
    """A call-local workspace, allocated on the call's stream so the caching
    allocator does not hand its memory out while the kernels still run."""
    torch = _torch()
    s = torch.cuda.current_stream(device) if stream is None else stream
    with torch.cuda.stream(s):
        return Workspace(A, B, mode, device)


def validate_poses(poses, tol: float = 1e-6) -> np.ndarray:
    """Host-side pose check (R orthonormal within 1e-6; finite values).

    Returns the indices of the poses that fail.  Optional and never done on
    the device; the kernels accept any finite [R|t] and apply R^T
    as the inverse rotation.  Accepts a numpy array or a tensor [N, 12]."""
    P = poses.detach().cpu().numpy() if hasattr(poses, "detach") else np.asarray(poses)
    P = np.asarray(P, dtype=np.float64).reshape(-1, 12)
    R = P[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]].reshape(-1, 3, 3)
    err = np.abs(np.einsum("nij,nkj->nik", R, R) - np.eye(3)).max(axis=(1, 2))
    bad = ~np.isfinite(P).all(axis=1) | ~(err <= tol) | (np.linalg.det(R) <= 0)
    return np.nonzero(bad)[0]


STAGING = {"auto": 0, "on": 1, "off": -1}


def _opts(descent: str, stats: bool, early_exit: bool = False, capped: bool = False,
          staging: str = "auto") -> L.cbvh_query_opts:
    if descent not in L.DESCENT:
        raise ValueError(f"descent must be one of {sorted(L.DESCENT)}")
    if staging not in STAGING:
        raise ValueError(f"staging must be one of {sorted(STAGING)}")
    return L.cbvh_query_opts(L.DESCENT[descent], 1 if stats else 0, 1 if early_exit else 0, 1 if capped else 0,
                             STAGING[staging])


def collide_batch(A: CompressedBVH, B: CompressedBVH, poses, hit=None, count=None,
                  workspace: Workspace | None = None, stream=None, stats: bool = False,
                  descent: str = "larger", early_exit: bool = False, staging: str = "auto"):
    """C-ABI collide_batch: per-pose hit flag (uint8) and colliding pair count (int32 view of uint32).

    descent: "larger" (default: descend the node with the larger box) or
    "simultaneous" (Alg. 1 verbatim).  Both give identical results.
    early_exit: stop each pose at its first hit (planning only needs the
    boolean); the hit flag is exact, the count a lower bound.
    staging: treelet blocks staged in shared memory — "auto" (when a blob
    was built with align_treelets), "on" (required) or "off".

    Device errors (a traversal-stack overflow) land in the workspace's error
    word: with a caller-supplied workspace, call ``check(workspace)`` after
    the call (it synchronises); without one, this call checks before it
    returns (and so synchronises the stream)."""
    torch = _torch()
    N = _check_poses(poses)
    dev = poses.device
    _check_bvh(A, dev)
    _check_bvh(B, dev)
    with torch.cuda.device(dev):
        if hit is None:
            hit = torch.empty(N, dtype=torch.uint8, device=dev)
        if count is None:
            count = torch.empty(N, dtype=torch.int32, device=dev)
        _check_out("hit", hit, N, (torch.uint8, torch.bool), dev)
        _check_out("count", count, N, (torch.int32, torch.uint32) if hasattr(torch, "uint32") else (torch.int32,), dev)
        temp = workspace is None
        if temp:
            workspace = _temp_workspace(A, B, 0, dev, stream)
        o = _opts(descent, stats, early_exit, staging=staging)
        L.check(L.load().collide_batch_ex(C.byref(A.bound), C.byref(B.bound), C.c_void_p(poses.data_ptr()), N,
                                          C.c_void_p(hit.data_ptr()), C.c_void_p(count.data_ptr()),
                                          C.c_void_p(workspace.ptr), workspace.nbytes,
                                          C.c_void_p(_stream_ptr(stream)), C.byref(o)))
        if temp:
            check(workspace, stream)
    return hit, count


def distance_batch(A: CompressedBVH, B: CompressedBVH, poses, dist=None,
                   workspace: Workspace | None = None, stream=None, stats: bool = False,
                   descent: str = "larger", caps=None, staging: str = "auto"):
    """C-ABI distance_batch: per-pose minimum triangle–triangle distance (fp32).
    caps (optional, fp32 [N] on the poses' device): per-pose caps — the result
    is min(distance, cap), exact below the cap (cbvh_query_opts.capped).
    Error checking as collide_batch."""
    torch = _torch()
    N = _check_poses(poses)
    dev = poses.device
    _check_bvh(A, dev)
    _check_bvh(B, dev)
    with torch.cuda.device(dev):
        if dist is None:
            dist = torch.empty(N, dtype=torch.float32, device=dev)
        _check_out("dist", dist, N, (torch.float32,), dev)
        if caps is not None:
            if caps.shape != (N,) or caps.dtype != torch.float32 or caps.device != dev:
                raise ValueError("caps must be fp32 [N] on the poses' device")
            with torch.cuda.stream(torch.cuda.current_stream(dev) if stream is None else stream):
                dist[:N].copy_(caps)
        temp = workspace is None
        if temp:
            workspace = _temp_workspace(A, B, 1, dev, stream)
        o = _opts(descent, stats, capped=caps is not None, staging=staging)
        L.check(L.load().distance_batch_ex(C.byref(A.bound), C.byref(B.bound), C.c_void_p(poses.data_ptr()), N,
                                           C.c_void_p(dist.data_ptr()), C.c_void_p(workspace.ptr), workspace.nbytes,
                                           C.c_void_p(_stream_ptr(stream)), C.byref(o)))
        if temp:
            check(workspace, stream)
    return dist


def check(workspace: Workspace, stream=None) -> None:
    """Sync the stream and raise on a device-side error (e.g. stack overflow)."""
    L.check(L.load().cbvh_check(C.c_void_p(workspace.ptr), C.c_void_p(_stream_ptr(stream))))


def read_stats(workspace: Workspace, stream=None) -> dict:
    s = L.cbvh_stats()
    L.check(L.load().cbvh_read_stats(C.c_void_p(workspace.ptr), C.byref(s), C.c_void_p(_stream_ptr(stream))))
    return {k: (list(getattr(s, k)) if k == "timeline_ns" else int(getattr(s, k))) for k, _ in L.cbvh_stats._fields_}


def last_launch_count() -> int:
    return int(L.load().cbvh_last_launch_count())
