"""Host builder + blob format (CPU; libcbvh.so loads without a GPU).

Checked by the oracle's INDEPENDENT decoder (oracle/oracle.cpp re-declares the
layout from DESIGN.md §3): containment of every decoded box, child ⊆
parent, leaves partition the triangles, treelets partition the
nodes and are connected, treelet size <= T; determinism; the
SPEC arithmetic example; fault injection; compression
invariance of the colliding pair sets and cost monotonicity.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2012_05348_b200 as M
from paper_2012_05348_b200 import _lib as L
from workloads import generators as G


@pytest.fixture(scope="module")
def cfg1():
    return G.make_config(1, num_poses=256)


@pytest.fixture(scope="module")
def mesh16k():
    return G.make_config(3, num_poses=1).A


def test_library_exports_every_header_symbol():
    text = open(L.HERE + "/../include/cbvh.h").read()
    names = set(re.findall(r"^\s*(?:int|void|size_t|const char\*)\s+(\w+)\(", text, re.M))
    assert {"build_compressed_bvh", "collide_batch", "distance_batch"} <= names
    lib = L.load()
    for n in names:
        assert hasattr(lib, n), n
    assert set(L.EXPORTS) == names


def test_ctypes_structs_match_header(tmp_path):
    # the binding's ctypes mirrors of the ABI structs must have the C layout:
    # compile a probe against include/cbvh.h that prints sizeof and every
    # field offset, and compare with ctypes
    import ctypes
    import subprocess
    structs = [L.cbvh_mesh, L.cbvh_build_opts, L.cbvh_header, L.cbvh_info, L.cbvh_bvh, L.cbvh_stats,
               L.cbvh_query_opts]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cbvh.h"', "int main(void) {"]
    for S in structs:
        lines.append(f'  printf("{S.__name__} %zu\\n", sizeof({S.__name__}));')
        for f, _ in S._fields_:
            lines.append(f'  printf("{S.__name__}.{f} %zu\\n", offsetof({S.__name__}, {f}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    inc = L.HERE + "/../include"
    subprocess.run(["gcc", "-std=c11", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], check=True, capture_output=True,
                                                 text=True).stdout.splitlines())
    for S in structs:
        assert int(got[S.__name__]) == ctypes.sizeof(S), S.__name__
        for f, _ in S._fields_:
            assert int(got[f"{S.__name__}.{f}"]) == getattr(S, f).offset, f"{S.__name__}.{f}"


@pytest.mark.parametrize("B", [2, 4, 8])
@pytest.mark.parametrize("bits", [2, 4, 5, 8, 11, 16])
def test_invariants_config1(cfg1, B, bits):
    A = cfg1.A
    bv = M.build_compressed_bvh(A.vertices, A.triangles, B, bits, 32, 4)
    r = O.check_blob(bv.blob, A.vertices, A.triangles)
    assert r["violations"] == 0, r
    assert r["nodes_checked"] == bv.info["num_nodes"]
    assert bv.info["code_width"] == (4 if bits <= 4 else 8 if bits <= 8 else 16)


@pytest.mark.parametrize("B,bits,T", [(2, 8, 32), (4, 8, 32), (8, 16, 32), (4, 4, 64), (4, 8, 4)])
def test_invariants_16k(mesh16k, B, bits, T):
    bv = M.build_compressed_bvh(mesh16k.vertices, mesh16k.triangles, B, bits, T, 4)
    r = O.check_blob(bv.blob, mesh16k.vertices, mesh16k.triangles)
    assert r["violations"] == 0, r


@pytest.mark.parametrize("B,bits,T", [(2, 8, 32), (4, 8, 32), (4, 8, 64), (8, 16, 64), (4, 4, 16)])
def test_aligned_treelets(cfg1, mesh16k, B, bits, T):
    # align_treelets: whole treelets packed next-fit into T-slot blocks; the padding
    # slots are unreachable and zero, the decoded boxes and the pair sets are
    # those of the packed numbering (independent checker + traversal)
    for m in (cfg1.A, mesh16k):
        al = M.build_compressed_bvh(m.vertices, m.triangles, B, bits, T, 4, align_treelets=True)
        pk = M.build_compressed_bvh(m.vertices, m.triangles, B, bits, T, 4)
        r = O.check_blob(al.blob, m.vertices, m.triangles)
        assert r["violations"] == 0, r
        i = al.info
        assert i["aligned_treelets"] and i["num_nodes"] % T == 0 and i["num_nodes"] >= i["real_nodes"]
        assert i["real_nodes"] == pk.info["num_nodes"] == r["nodes_checked"]
        assert i["num_treelets"] == pk.info["num_treelets"]
        topo_al = np.frombuffer(al.blob[i["off_topo"]:i["off_topo"] + 4 * i["num_nodes"]].tobytes(), np.uint32)
        assert np.count_nonzero(topo_al == 0x7FFFFFFF) == i["num_nodes"] - i["real_nodes"]
    A, Bm, P = cfg1.A, cfg1.B, cfg1.poses[:24]
    ta = O.Tree.from_blob(M.build_compressed_bvh(A.vertices, A.triangles, B, bits, T, 4, align_treelets=True).blob,
                          A.vertices, A.triangles)
    tb = O.Tree.from_blob(M.build_compressed_bvh(Bm.vertices, Bm.triangles, B, bits, T, 4, align_treelets=True).blob,
                          Bm.vertices, Bm.triangles)
    ra, rb = O.Tree.from_mesh(A.vertices, A.triangles), O.Tree.from_mesh(Bm.vertices, Bm.triangles)
    for p in P:
        assert O.collide_pairs(ta, tb, p) == O.collide_pairs(ra, rb, p)


@pytest.mark.parametrize("B,bits,T", [(2, 8, 32), (4, 8, 32), (4, 8, 64), (8, 16, 64), (4, 12, 16)])
def test_zero_suppressed_codes(cfg1, mesh16k, B, bits, T):
    # integer-compressed corrections: the oracle's own decoder of the
    # presence-mask format (oracle.cpp code_field) finds every box containing
    # its subtree, the pair sets equal the plain blob's, and the codes shrink
    for m in (cfg1.A, mesh16k):
        z = M.build_compressed_bvh(m.vertices, m.triangles, B, bits, T, 4, zero_suppress=True)
        al = M.build_compressed_bvh(m.vertices, m.triangles, B, bits, T, 4, align_treelets=True)
        r = O.check_blob(z.blob, m.vertices, m.triangles)
        assert r["violations"] == 0, r
        assert z.info["zero_suppressed"] and z.info["aligned_treelets"]
        assert z.info["num_nodes"] == al.info["num_nodes"] and z.info["real_nodes"] == al.info["real_nodes"]
        # at b = 8 zero corrections are common (a child sharing a parent
        # face) and each saves a byte: fewer hierarchy bytes than the same
        # aligned blob (at b = 16 the corrections rarely vanish)
        if bits == 8:
            assert z.info["bvh_bytes"] < al.info["bvh_bytes"]
    A, Bm, P = cfg1.A, cfg1.B, cfg1.poses[:24]
    ta = O.Tree.from_blob(M.build_compressed_bvh(A.vertices, A.triangles, B, bits, T, 4, zero_suppress=True).blob,
                          A.vertices, A.triangles)
    tb = O.Tree.from_blob(M.build_compressed_bvh(Bm.vertices, Bm.triangles, B, bits, T, 4, zero_suppress=True).blob,
                          Bm.vertices, Bm.triangles)
    ra, rb = O.Tree.from_mesh(A.vertices, A.triangles), O.Tree.from_mesh(Bm.vertices, Bm.triangles)
    for p in P:
        assert O.collide_pairs(ta, tb, p) == O.collide_pairs(ra, rb, p)


def test_zero_suppressed_errors_and_faults(cfg1):
    A = cfg1.A
    for kw in (dict(bits=4), dict(layout="fp16"), dict(kdop=14)):
        bits = kw.pop("bits", 8)
        with pytest.raises(L.CbvhError, match="EINVAL"):
            M.build_compressed_bvh(A.vertices, A.triangles, 4, bits, zero_suppress=True, **kw)
    z = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, 32, 4, zero_suppress=True)
    i = z.info
    region0 = i["off_codes"]
    lib = L.load()
    out = L.cbvh_bvh()

    def bind(blob):
        return lib.cbvh_bind(blob.ctypes.data_as(C.POINTER(C.c_uint8)), blob.nbytes, C.c_void_p(1 << 20), C.byref(out))

    assert bind(z.blob) == L.CBVH_OK
    # a presence mask with a 7th bit, and a mask that announces a field the
    # region does not hold, are rejected by bind and flagged by the checker
    bad = z.blob.copy()
    bad[region0 + 1] |= 64
    assert bind(bad) == L.CBVH_EBLOB
    assert O.check_blob(bad, A.vertices, A.triangles)["malformed"] > 0
    # flipping a mask bit shifts every later field: boxes decode wrong
    bad = z.blob.copy()
    j = next(k for k in range(1, 32) if bad[region0 + k] not in (0, 63))
    bad[region0 + j] ^= next(1 << f for f in range(6) if not (bad[region0 + j] >> f) & 1)
    assert O.check_blob(bad, A.vertices, A.triangles)["violations"] > 0


def test_aligned_treelets_errors_and_faults(cfg1):
    A = cfg1.A
    for kw in (dict(treelet_nodes=48), dict(treelet_nodes=128), dict(layout="fp32"), dict(kdop=14)):
        with pytest.raises(L.CbvhError, match="EINVAL"):
            M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, align_treelets=True, **kw)
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, 32, 4, align_treelets=True)
    i = bv.info
    topo = np.frombuffer(bv.blob[i["off_topo"]:i["off_topo"] + 4 * i["num_nodes"]].tobytes(), np.uint32)
    pad = int(np.nonzero(topo == 0x7FFFFFFF)[0][0])
    # a padding slot holding a code, or a parent pointing into padding, is caught
    bad = bv.blob.copy()
    bad[i["off_codes"] + 6 * pad] = 3
    assert O.check_blob(bad, A.vertices, A.triangles)["malformed"] > 0
    lib = L.load()
    out = L.cbvh_bvh()
    internal = int(np.nonzero((topo >> 31) == 0)[0][1])
    bad = bv.blob.copy()
    w = (int(topo[internal]) & ~0x0FFFFFFF) | (pad - 1)
    bad[i["off_topo"] + 4 * internal:i["off_topo"] + 4 * internal + 4] = np.frombuffer(np.uint32(w).tobytes(), np.uint8)
    rc = lib.cbvh_bind(bad.ctypes.data_as(C.POINTER(C.c_uint8)), bad.nbytes, C.c_void_p(1 << 20), C.byref(out))
    assert rc == L.CBVH_EBLOB


def test_node_counts_closed_form(cfg1):
    # equal-count median split, c = 4: a binary tree over 960 triangles has
    # 2 * 256 - 1 = 511 nodes (960 / 4 = 240 leaves -> padded split shape)
    A = cfg1.A
    n = {B: M.build_compressed_bvh(A.vertices, A.triangles, B, 8).info["num_nodes"] for B in (2, 4, 8)}
    assert n == {2: 511, 4: 341, 8: 329}


def test_determinism(cfg1):
    A = cfg1.A
    b1 = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8).blob
    b2 = M.build_compressed_bvh(A.vertices.copy(), A.triangles.copy(), 4, 8).blob
    assert b1.tobytes() == b2.tobytes()


def _tri_spanning(x0, x1):
    return np.array([[x0, 0, 0], [x1, 0, 0], [0.5 * (x0 + x1), 1, 0]], np.float32)


def test_spec_encode_example():
    # parent [0, 255], child [10.7, 200], b = 8 -> q_lo = 10, q_hi = 55.
    # On the lattice (cell 2^-14 for extent 255) the step is 2^14 cells = 1.0.
    V = np.concatenate([_tri_spanning(10.7, 200.0), _tri_spanning(0.0, 255.0)])
    T = np.arange(6, dtype=np.int32).reshape(2, 3)
    bv = M.build_compressed_bvh(V, T, 2, 8, 32, 1)
    info, blob = bv.info, bv.blob
    assert info["num_nodes"] == 3 and info["lattice_exp"] == -14
    topo = np.frombuffer(blob[info["off_topo"]:info["off_topo"] + 12].tobytes(), np.uint32)
    codes = blob[info["off_codes"]:info["off_codes"] + 18].reshape(3, 6)
    tri_index = np.frombuffer(blob[info["off_tri_index"]:info["off_tri_index"] + 8].tobytes(), np.uint32)
    assert topo[0] >> 31 == 0 and ((topo[0] >> 28) & 7) + 1 == 2
    assert np.all(codes[0] == 0)  # the root equals its anchor: zero corrections
    for node in (1, 2):
        first = topo[node] & 0x1FFFFFFF
        if tri_index[first] == 0:  # the [10.7, 200] triangle
            assert codes[node][0] == 10 and codes[node][3] == 55
        else:  # the [0, 255] triangle equals the parent on x: zero corrections
            assert codes[node][0] == 0 and codes[node][3] == 0
    assert O.check_blob(blob, V, T)["violations"] == 0


def test_treelet_closed_form_T_equals_B(cfg1):
    # T = B: every sibling group opens its own treelet -> 1 + #internal treelets
    A = cfg1.A
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 2, 8, 2, 4)
    i = bv.info
    assert i["num_treelets"] == 1 + (i["num_nodes"] - i["num_leaves"])
    big = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, 4096, 4).info
    assert big["num_treelets"] == 1  # tree smaller than the budget


def test_bytes_per_node_accounting(cfg1):
    A = cfg1.A
    for bits, cw in ((4, 3), (8, 6), (16, 12)):
        i = M.build_compressed_bvh(A.vertices, A.triangles, 4, bits, 32).info
        assert i["code_bytes_per_node"] == cw  # 6 corrections x field width
        # topology + codes; the treelet table is build metadata the device never reads
        assert i["bvh_bytes"] == (4 + cw) * i["num_nodes"]
        assert i["tri_bytes"] == 48 * A.num_triangles
        assert i["code_bytes_per_node"] <= 0.25 * 24 or bits == 16  # S:344 (b=8: 6 B vs 24 B fp32)


def test_fault_injection_detected(cfg1):
    A = cfg1.A
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, 32)
    info = bv.info
    assert O.check_blob(bv.blob, A.vertices, A.triangles)["violations"] == 0
    # (a) inflate one correction of a leaf: its decoded box no longer contains it
    topo = np.frombuffer(bv.blob[info["off_topo"]:info["off_topo"] + 4 * info["num_nodes"]].tobytes(), np.uint32)
    leaf = int(np.nonzero(topo >> 31)[0][5])
    bad = bv.blob.copy()
    bad[info["off_codes"] + 6 * leaf + 0] = 255
    bad[info["off_codes"] + 6 * leaf + 3] = 255
    r = O.check_blob(bad, A.vertices, A.triangles)
    assert r["containment"] > 0
    # (b) a triangle missing from the leaves
    bad = bv.blob.copy()
    ti = info["off_tri_index"]
    bad[ti:ti + 4] = bad[ti + 4:ti + 8]  # triangle index 0 slot now duplicates slot 1
    r = O.check_blob(bad, A.vertices, A.triangles)
    assert r["triangle_partition"] > 0
    # (c) corrupted topology word
    bad = bv.blob.copy()
    bad[info["off_topo"]:info["off_topo"] + 4] = np.frombuffer(np.uint32(0x0FFFFFF0).tobytes(), np.uint8)
    r = O.check_blob(bad, A.vertices, A.triangles)
    assert r["violations"] > 0


@pytest.mark.parametrize("B,bits", [(2, 8), (4, 4), (4, 8), (8, 16)])
def test_compression_invariance_and_cost(cfg1, B, bits):
    # BJ oracle self-check (3): the pair sets from traversing the DECODED
    # compressed boxes equal those over exact fp64 boxes; looser boxes cannot
    # prune more.
    A, Bm, P = cfg1.A, cfg1.B, cfg1.poses[:48]
    ba = M.build_compressed_bvh(A.vertices, A.triangles, B, bits)
    bb = M.build_compressed_bvh(Bm.vertices, Bm.triangles, B, bits)
    dA = O.Tree.from_blob(ba.blob, A.vertices, A.triangles)
    dB = O.Tree.from_blob(bb.blob, Bm.vertices, Bm.triangles)
    eA = O.Tree.from_blob(ba.blob, A.vertices, A.triangles, exact_boxes=True)
    eB = O.Tree.from_blob(bb.blob, Bm.vertices, Bm.triangles, exact_boxes=True)
    rA = O.Tree.from_mesh(A.vertices, A.triangles)
    rB = O.Tree.from_mesh(Bm.vertices, Bm.triangles)
    hits = 0
    for p in P:
        s = O.collide_pairs(dA, dB, p)
        assert s == O.collide_pairs(eA, eB, p) == O.collide_pairs(rA, rB, p)
        hits += bool(s)
    assert hits > 5
    _, _, _, st_dec = O.collide(dA, dB, P, 0.0)
    _, _, _, st_ex = O.collide(eA, eB, P, 0.0)
    assert st_dec[0] >= st_ex[0]


@pytest.mark.parametrize("kdop", [6, 14])
def test_degenerate_meshes_build(kdop):
    # zero-area triangles are kept: a point, a sliver, a tiny triangle
    # far from the origin and a flat mesh all build (the lattice search used to
    # loop forever on a zero-extent root) and pass the independent checker
    T1 = np.array([[0, 1, 2]], np.int32)
    cases = [np.array([[0.25, 0.25, 0]] * 3, np.float32),
             np.array([[2, 0, 0], [3, 0, 0], [4, 0, 0]], np.float32),
             np.array([[1000, 1000, 1000], [1000, 1000, 1000.0001], [1000, 1000.0001, 1000]], np.float32),
             np.zeros((3, 3), np.float32)]
    for V in cases:
        for B in (2, 4):
            bv = M.build_compressed_bvh(V, T1, B, 8, kdop=kdop if B == 4 else 6)
            assert O.check_blob(bv.blob, V, T1)["violations"] == 0
    rng = np.random.default_rng(5)
    V = rng.uniform(-1, 1, (60, 3)).astype(np.float32)
    V[:, 2] = 0  # flat: zero extent in z
    T = rng.integers(0, 60, (40, 3)).astype(np.int32)
    # duplicate-position (not duplicate-index) triangles: zero area
    T[:5, 1] = (T[:5, 0] + 1) % 60
    V[T[:5, 1]] = V[T[:5, 0]]
    bv = M.build_compressed_bvh(V, T, 4, 8, kdop=kdop)
    assert O.check_blob(bv.blob, V, T)["violations"] == 0


def test_error_paths():
    lib = L.load()
    V = np.zeros((3, 3), np.float32)
    V[1, 0] = V[2, 1] = 1
    T = np.array([[0, 1, 2]], np.int32)
    ok = M.build_compressed_bvh(V, T, 2, 8)
    assert ok.info["num_nodes"] == 1 and ok.info["num_leaves"] == 1
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.build_compressed_bvh(V, T, 3, 8)
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.build_compressed_bvh(V, T, 4, 1)
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.build_compressed_bvh(V, T, 4, 17)
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.build_compressed_bvh(V, T, 8, 8, treelet_nodes=4)
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.build_compressed_bvh(V, T, 4, 8, leaf_size=5)
    with pytest.raises(L.CbvhError, match="EMESH"):
        M.build_compressed_bvh(V, np.zeros((0, 3), np.int32), 4, 8)
    with pytest.raises(L.CbvhError, match="EMESH"):
        M.build_compressed_bvh(V, np.array([[0, 1, 3]], np.int32), 4, 8)
    Vn = V.copy()
    Vn[0, 0] = np.nan
    with pytest.raises(L.CbvhError, match="EMESH"):
        M.build_compressed_bvh(Vn, T, 4, 8)
    bad = ok.blob.copy()
    bad[0] = ord("X")
    with pytest.raises(L.CbvhError, match="EBLOB"):
        M.blob_info(bad)
    with pytest.raises(L.CbvhError, match="EBLOB"):
        M.blob_info(ok.blob[:-16])
    info = L.cbvh_info()
    assert lib.cbvh_blob_info(None, 0, C.byref(info)) == L.CBVH_EINVAL


# ------------------------------------------------------------------ node layouts (§III.A ablation)


@pytest.mark.parametrize("layout", ["fp16", "fp32"])
@pytest.mark.parametrize("B", [2, 4, 8])
def test_absolute_layouts_invariants(cfg1, mesh16k, layout, B):
    for m in (cfg1.A, mesh16k):
        bv = M.build_compressed_bvh(m.vertices, m.triangles, B, 8, 32, 4, layout=layout)
        r = O.check_blob(bv.blob, m.vertices, m.triangles)
        assert r["violations"] == 0, r
        assert bv.info["layout"] == layout
        assert bv.info["code_bytes_per_node"] == (12 if layout == "fp16" else 24)  # Table I: 6 floats / halves


def test_fp32_layout_is_exact(cfg1):
    A = cfg1.A
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, 32, 4, layout="fp32")
    dec = O.Tree.from_blob(bv.blob, A.vertices, A.triangles)
    ex = O.Tree.from_blob(bv.blob, A.vertices, A.triangles, exact_boxes=True)
    P = cfg1.poses[:16]
    # exact boxes: identical BV-test counts under the verbatim Alg. 1 oracle
    assert np.array_equal(O.collide(dec, dec, P, 0.0)[3], O.collide(ex, ex, P, 0.0)[3])


def test_fp16_directed_rounding_spec_examples():
    # 1.0 -> 0x3C00; 1.001 down -> 0x3C01 (1.0009765625), up -> 0x3C02
    V = np.array([[1.001, 1.0, 0.0], [3.0, 1.001, 0.0], [2.0, 2.0, 1.0]], np.float32)
    T = np.array([[0, 1, 2]], np.int32)
    bv = M.build_compressed_bvh(V, T, 2, 8, 32, 4, layout="fp16")
    off = bv.info["off_codes"]
    h = np.frombuffer(bv.blob[off:off + 12].tobytes(), np.uint16)
    lo, hi = h[:3], h[3:]
    assert lo[0] == 0x3C01 and hi[0] == 0x4200   # x in [1.001, 3]
    assert lo[1] == 0x3C00                         # y lo = 1.0 exactly
    assert hi[1] == 0x4000 and hi[2] == 0x3C00     # y hi = 2, z hi = 1
    Vu = np.array([[1.0, 1.001, 1.001], [0.5, 0.5, 0.5], [0.25, 0.25, 0.25]], np.float32)
    bu = M.build_compressed_bvh(Vu, T, 2, 8, 32, 4, layout="fp16")
    hu = np.frombuffer(bu.blob[bu.info["off_codes"] + 6:bu.info["off_codes"] + 12].tobytes(), np.uint16)
    assert hu[1] == 0x3C02                         # 1.001 rounded up
    assert O.check_blob(bu.blob, Vu, T)["violations"] == 0


def test_fp16_range_error():
    V = np.array([[0, 0, 0], [70000.0, 0, 0], [0, 1, 0]], np.float32)
    T = np.array([[0, 1, 2]], np.int32)
    with pytest.raises(L.CbvhError, match="EMESH"):
        M.build_compressed_bvh(V, T, 2, 8, layout="fp16")
    M.build_compressed_bvh(V, T, 2, 8, layout="fp32")


def test_layout_cost_monotone_under_alg1(cfg1):
    # S:419 / S:509: looser boxes cannot prune more (Alg. 1 verbatim oracle)
    A, Bm, P = cfg1.A, cfg1.B, cfg1.poses[:32]
    tests = {}
    for lay in ("fp32", "fp16", "delta"):
        ta = O.Tree.from_blob(M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, layout=lay).blob,
                              A.vertices, A.triangles)
        tb = O.Tree.from_blob(M.build_compressed_bvh(Bm.vertices, Bm.triangles, 4, 8, layout=lay).blob,
                              Bm.vertices, Bm.triangles)
        cnt, _, _, st = O.collide(ta, tb, P, 0.0)
        tests[lay] = (st[0], cnt)
    assert tests["fp16"][0] >= tests["fp32"][0] and tests["delta"][0] >= tests["fp32"][0]
    assert np.array_equal(tests["fp16"][1], tests["fp32"][1]) and np.array_equal(tests["delta"][1], tests["fp32"][1])


def test_bind_rejects_corrupt_topology(cfg1):
    # cbvh_bind validates the topology on the host (no device allocation needed:
    # bind only records the device pointer)
    A = cfg1.A
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 2, 8)
    lib = L.load()
    out = L.cbvh_bvh()
    fake_dev = C.c_void_p(1 << 20)  # 256-B aligned, never dereferenced by bind
    ok = lib.cbvh_bind(bv.blob.ctypes.data_as(C.POINTER(C.c_uint8)), bv.blob.nbytes, fake_dev, C.byref(out))
    assert ok == L.CBVH_OK
    off = bv.info["off_topo"]
    for bad_word in (0x0FFFFFF0, 0x00000000, 0x80000000 | 0x1FFFFFF0):  # far child / self-cycle / bad tris
        b = bv.blob.copy()
        b[off:off + 4] = np.frombuffer(np.uint32(bad_word).tobytes(), np.uint8)
        rc = lib.cbvh_bind(b.ctypes.data_as(C.POINTER(C.c_uint8)), b.nbytes, fake_dev, C.byref(out))
        assert rc == L.CBVH_EBLOB, hex(bad_word)


def test_leaf_slab_containment_and_fault(cfg1):
    # record pads carry each leaf's slab (unit n, [dmin, dmax] of n.v): the
    # independent checker verifies containment; a shrunk range is caught
    A = cfg1.A
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8)
    assert O.check_blob(bv.blob, A.vertices, A.triangles)["violations"] == 0
    info = bv.info
    topo = np.frombuffer(bv.blob[info["off_topo"]:info["off_topo"] + 4 * info["num_nodes"]].tobytes(), np.uint32)
    leaf = next(int(t) for t in topo if (t >> 31) and ((t >> 29) & 3) >= 1)  # a leaf with >= 2 triangles
    first = leaf & 0x1FFFFFFF
    rec1 = info["off_tris"] + 48 * (first + 1)
    bad = bv.blob.copy()
    dmin, dmax = np.frombuffer(bad[rec1 + 36:rec1 + 44].tobytes(), np.float32)
    bad[rec1 + 40:rec1 + 44] = np.frombuffer(np.float32(dmin + 0.25 * (dmax - dmin)).tobytes(), np.uint8)
    assert O.check_blob(bad, A.vertices, A.triangles)["containment"] > 0


# ------------------------------------------------------------------ k-DOP nodes for the static model (§8(f))

_KDOP_DIRS = {14: [(1, 1, 1), (1, 1, -1), (1, -1, 1), (-1, 1, 1)],
              18: [(1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1)]}
_KDOP_DIRS[26] = _KDOP_DIRS[14] + _KDOP_DIRS[18]


@pytest.mark.parametrize("kdop", [14, 18, 26])
@pytest.mark.parametrize("B,bits", [(2, 4), (4, 8), (8, 16)])
def test_kdop_invariants_and_aabb_part(cfg1, mesh16k, kdop, B, bits):
    # every extra slab axis nests child-in-parent and contains the exact
    # projections of its subtree (independent fp64 check); the x/y/z part of
    # the codes is the AABB blob's, field for field
    for m in (cfg1.B, mesh16k):
        kb = M.build_compressed_bvh(m.vertices, m.triangles, B, bits, 32, 4, kdop=kdop)
        r = O.check_blob(kb.blob, m.vertices, m.triangles)
        assert r["violations"] == 0, r
        ab = M.build_compressed_bvh(m.vertices, m.triangles, B, bits, 32, 4)
        w, n, nax = kb.info["code_width"], kb.info["num_nodes"], kdop // 2
        assert kb.info["kdop"] == kdop and kb.info["code_bytes_per_node"] == kdop * w // 8
        def fields(bv, k):
            c = bv.blob[bv.info["off_codes"]:bv.info["off_codes"] + n * k * w // 8]
            if w == 16:
                return np.frombuffer(c.tobytes(), np.uint16).reshape(n, k)
            if w == 8:
                return c.reshape(n, k)
            c = c.reshape(n, k // 2)
            return np.stack([c & 15, c >> 4], -1).reshape(n, k)
        fk, fa = fields(kb, kdop), fields(ab, 6)
        assert np.array_equal(fk[:, :3], fa[:, :3]) and np.array_equal(fk[:, nax:nax + 3], fa[:, 3:])


@pytest.mark.parametrize("kdop", [14, 18, 26])
def test_kdop_root_slabs_closed_form(kdop):
    # axis table: the root interval of direction d is [min d.v, max d.v] of the
    # mesh rounded outward by at most one cell 2^exp (exact fp64 projections)
    rng = np.random.default_rng(7)
    V = rng.normal(size=(30, 3)).astype(np.float32) * np.float32(3) + np.float32(10)
    T = np.arange(30, dtype=np.int32).reshape(10, 3)
    bv = M.build_compressed_bvh(V, T, 4, 8, 32, 4, kdop=kdop)
    off = bv.info["off_axes"]
    for a, d in enumerate(_KDOP_DIRS[kdop]):
        rec = bv.blob[off + 16 * a:off + 16 * a + 16].tobytes()
        org = float(np.frombuffer(rec[0:4], np.float32)[0])
        ex, lo, hi = (int(x) for x in np.frombuffer(rec[4:16], np.int32))
        pr = V.astype(np.float64) @ np.array(d, np.float64)
        cell = 2.0 ** ex
        assert org + lo * cell <= pr.min() < org + (lo + 1) * cell
        assert org + (hi - 1) * cell < pr.max() <= org + hi * cell
        assert hi - lo <= 2 ** 22
    assert O.check_blob(bv.blob, V, T)["violations"] == 0


def test_kdop_fault_and_errors(cfg1):
    A = cfg1.B
    bv = M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, 32, 4, kdop=14)
    info = bv.info
    topo = np.frombuffer(bv.blob[info["off_topo"]:info["off_topo"] + 4 * info["num_nodes"]].tobytes(), np.uint32)
    leaf = int(np.nonzero(topo >> 31)[0][3])
    bad = bv.blob.copy()
    # a diagonal-axis correction of one leaf inflated: its slab no longer holds it
    bad[info["off_codes"] + 14 * leaf + 3] = 255
    bad[info["off_codes"] + 14 * leaf + 7 + 3] = 255
    assert O.check_blob(bad, A.vertices, A.triangles)["containment"] > 0
    for k in (8, 12, 20):
        with pytest.raises(L.CbvhError, match="EINVAL"):
            M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, kdop=k)
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.build_compressed_bvh(A.vertices, A.triangles, 4, 8, layout="fp16", kdop=14)


def test_bind_kdop_axis_table(cfg1):
    # cbvh_bind reads the axis table and decodes node 0 of every extra axis
    # (no device access: bind only records the device pointer)
    B = cfg1.B
    lib = L.load()
    fake_dev = C.c_void_p(1 << 20)
    for k in (14, 18, 26):
        bv = M.build_compressed_bvh(B.vertices, B.triangles, 4, 8, 32, 4, kdop=k)
        out = L.cbvh_bvh()
        rc = lib.cbvh_bind(bv.blob.ctypes.data_as(C.POINTER(C.c_uint8)), bv.blob.nbytes, fake_dev, C.byref(out))
        assert rc == L.CBVH_OK
        off = bv.info["off_axes"]
        for a in range(k // 2 - 3):
            rec = np.frombuffer(bv.blob[off + 16 * a:off + 16 * a + 16].tobytes(), np.int32)
            assert out.axis_exp[a] == rec[1]
            assert out.axis_root[2 * a] == rec[2] and out.axis_root[2 * a + 1] == rec[3]  # node 0 == table root
        bad = bv.blob.copy()
        bad[off + 4:off + 8] = np.frombuffer(np.int32(500).tobytes(), np.uint8)  # absurd exponent
        rc = lib.cbvh_bind(bad.ctypes.data_as(C.POINTER(C.c_uint8)), bad.nbytes, fake_dev, C.byref(out))
        assert rc == L.CBVH_EBLOB


def test_production_kernels_do_not_spill(tmp_path):
    # both production traversal kernels (collide, distance; AABB blobs) stay
    # inside their register budgets with no local-memory spills: the ncu
    # captures showed spilled item boxes costing ~5 %
    import subprocess
    from paper_2012_05348_b200 import build as B
    out = subprocess.run(["nvcc", *[f for f in B.NVCC_FLAGS if f != "-shared"], "-c", "-Xptxas", "-v",
                          "-o", str(tmp_path / "k.o"), os.path.join(B.CSRC, "cbvh_device.cu")],
                         capture_output=True, text=True, check=True).stderr
    lines = out.splitlines()
    for mode in (0, 1):
        for fast in (0, 1, 2, 3, 4, 5):  # generic, and FAST: delta b = 8, fp16, fp32, delta in 4- / 16-bit fields
            tag = f"_ZN4cbvh15traverse_kernelILi{mode}ELb0ELi0ELb0ELi{fast}ELb0EEEvNS_6ParamsE"
            i = next(k for k, l in enumerate(lines) if "Function properties for " + tag in l)
            assert "0 bytes spill stores, 0 bytes spill loads" in lines[i + 1], lines[i + 1]
