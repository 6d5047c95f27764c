"""Golden fixtures (tests/golden/*.txt): values fixed by SPEC.md's worked
examples and by hand-derived closed forms, each row
citing its source.  The CPU tests pin the oracle's primitives and the host
builder's codes to them; the GPU test runs the same triangle pairs through the
C-ABI (single-triangle meshes at the identity pose).
"""
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rows(name):
    out = []
    with open(os.path.join(HERE, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                out.append([c.strip() for c in line.split("|")])
    return out


def _pairs():
    res = []
    for r in _rows("tri_pairs.txt"):
        V = np.array(r[2].split(), float).reshape(3, 3)
        U = np.array(r[3].split(), float).reshape(3, 3)
        res.append(pytest.param(V, U, int(r[4]), float(r[5]), int(r[6]), id=r[0]))
    return res


def test_golden_files_cite_their_source():
    for r in _rows("tri_pairs.txt") + _rows("encode.txt"):
        assert r[1].startswith("SPEC S:") or r[1].startswith("closed form"), r


@pytest.mark.parametrize("V,U,inter,dist,touch", _pairs())
def test_golden_pairs_oracle(V, U, inter, dist, touch):
    assert O.tri_tri_intersect(V, U) == bool(inter)
    assert O.tri_tri_intersect(U, V) == bool(inter)  # symmetry
    d = O.tri_tri_distance(V, U)
    assert abs(d - dist) <= 1e-12 * max(1.0, dist), (d, dist)
    assert abs(O.tri_tri_distance(U, V) - dist) <= 1e-12 * max(1.0, dist)


def _encode_rows():
    return [pytest.param(*[float(x) for x in r[2].split()], *[float(x) for x in r[3].split()], int(r[4]),
                         *[int(x) for x in r[5].split()], id=r[0]) for r in _rows("encode.txt")]


@pytest.mark.parametrize("plo,phi,clo,chi,bits,qlo,qhi", _encode_rows())
def test_golden_encode(plo, phi, clo, chi, bits, qlo, qhi):
    # the host builder's corrections on x for a two-leaf tree whose root is the
    # parent interval (reading R3: the step is 2^s lattice cells = 1.0 here)
    import paper_2012_05348_b200 as M

    def tri(x0, x1):
        return np.array([[x0, 0, 0], [x1, 0, 0], [0.5 * (x0 + x1), 1, 0]], np.float32)

    V = np.concatenate([tri(clo, chi), tri(plo, phi)])
    T = np.arange(6, dtype=np.int32).reshape(2, 3)
    bv = M.build_compressed_bvh(V, T, 2, bits, 32, 1)
    info, blob = bv.info, bv.blob
    topo = np.frombuffer(blob[info["off_topo"]:info["off_topo"] + 12].tobytes(), np.uint32)
    codes = blob[info["off_codes"]:info["off_codes"] + 18].reshape(3, 6)
    tri_index = np.frombuffer(blob[info["off_tri_index"]:info["off_tri_index"] + 8].tobytes(), np.uint32)
    found = False
    for node in (1, 2):
        if tri_index[topo[node] & 0x1FFFFFFF] == 0:  # the child triangle
            assert (int(codes[node][0]), int(codes[node][3])) == (qlo, qhi)
            found = True
    assert found


@pytest.mark.gpu
@pytest.mark.parametrize("V,U,inter,dist,touch", _pairs())
def test_golden_pairs_gpu(V, U, inter, dist, touch):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device")
    import paper_2012_05348_b200 as M
    from workloads import generators as G
    T = np.array([[0, 1, 2]], np.int32)
    A = M.build_compressed_bvh(V.astype(np.float32), T, 2, 8).to_device()
    B = M.build_compressed_bvh(U.astype(np.float32), T, 2, 8).to_device()
    P = torch.from_numpy(G.identity_poses(1)).cuda()
    hit, cnt = M.collide_batch(A, B, P)
    d = float(M.distance_batch(A, B, P).cpu().numpy()[0])
    c = int(cnt.cpu().numpy().view(np.uint32)[0])
    if touch:  # s = 0 exactly: inside the tolerance band, either answer is accepted
        assert c in (0, 1) and int(hit.cpu()[0]) == c
    else:
        assert c == inter and int(hit.cpu()[0]) == inter
    if dist == 0.0:
        assert d <= 1e-6
    else:
        assert abs(d - dist) <= 1e-5 * dist, (d, dist)
