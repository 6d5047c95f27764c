"""Pins of the oracle's traversal (Alg. 1) against brute force.

The oracle's hierarchical answer must equal the hierarchy-free all-pairs
answer: identical colliding pair SETS, identical counts and
band classifications, identical minimum distances.  Special cases: a mesh
against itself at identity (every triangle hits itself), far poses (only the
root test), config-4 geometry bracket.
"""
import numpy as np
import pytest

import oracle as O
from workloads import generators as G


@pytest.fixture(scope="module")
def tiny():
    out = {}
    for which in ("8x4", "16x8"):
        A, B, P = G.tiny_pair(which, seed=11, n_poses=400, half_width=2.0)
        out[which] = (A, B, P)
    return out


@pytest.mark.parametrize("which", ["8x4", "16x8"])
def test_pair_sets_equal_bruteforce(tiny, which):
    A, B, P = tiny[which]
    tA, tB = O.Tree.from_mesh(A.vertices, A.triangles), O.Tree.from_mesh(B.vertices, B.triangles)
    nonempty = 0
    for p in P[:150]:
        s_tree = O.collide_pairs(tA, tB, p)
        s_brute = O.bruteforce_pairs(tA, tB, p)
        assert s_tree == s_brute
        nonempty += bool(s_brute)
    assert nonempty > 10


@pytest.mark.parametrize("which", ["8x4", "16x8"])
def test_counts_and_band_equal_bruteforce(tiny, which):
    A, B, P = tiny[which]
    tA, tB = O.Tree.from_mesh(A.vertices, A.triangles), O.Tree.from_mesh(B.vertices, B.triangles)
    delta = O.band_delta(A.vertices)
    c1, h1, z1, st = O.collide(tA, tB, P, delta)
    c2, h2, z2 = O.bruteforce_collide(tA, tB, P, delta)
    assert np.array_equal(c1, c2) and np.array_equal(h1, h2) and np.array_equal(z1, z2)
    assert (c1 > 0).sum() > 20
    # H <= count <= H + Z (robust hits are hits; band pairs may go either way)
    assert np.all(h1 <= c1) and np.all(c1 <= h1 + z1)


def test_leaf_size_does_not_change_answer(tiny):
    A, B, P = tiny["16x8"]
    delta = O.band_delta(A.vertices)
    ref = None
    for c in (1, 2, 4, 7):
        tA, tB = O.Tree.from_mesh(A.vertices, A.triangles, c), O.Tree.from_mesh(B.vertices, B.triangles, c)
        out = O.collide(tA, tB, P[:100], delta)[:3]
        if ref is None:
            ref = out
        for a, b in zip(ref, out):
            assert np.array_equal(a, b)


def test_config1_meshes_against_bruteforce():
    w = G.make_config(1)
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
    delta = O.band_delta(w.A.vertices)
    P = w.poses[:24]
    c1, h1, z1, _ = O.collide(tA, tB, P, delta)
    c2, h2, z2 = O.bruteforce_collide(tA, tB, P, delta)
    assert np.array_equal(c1, c2) and np.array_equal(h1, h2) and np.array_equal(z1, z2)
    assert (c1 > 0).sum() >= 3


def test_self_at_identity_every_triangle_hits_itself():
    w = G.make_config(1)
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    I = G.identity_poses(1)
    pairs = O.collide_pairs(tA, tA, I[0])
    nt = w.A.num_triangles
    assert all((i, i) in pairs for i in range(nt))
    # neighbours sharing an edge or vertex also touch: count well above nt
    assert len(pairs) > 3 * nt


def test_far_pose_only_root_test():
    w = G.make_config(1)
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
    P = G.identity_poses(3)
    P[:, 3] = [6.0, -7.0, 0.0]
    P[:, 7] = [0.0, 0.0, 9.0]
    c, h, z, st = O.collide(tA, tB, P, 1e-6)
    assert c.sum() == 0 and h.sum() == 0 and z.sum() == 0
    assert st[0] == 3 and st[1] == 0  # one root BV test per pose, no leaf pair


@pytest.mark.parametrize("which", ["8x4", "16x8"])
def test_distance_equals_bruteforce(tiny, which):
    A, B, P = tiny[which]
    tA, tB = O.Tree.from_mesh(A.vertices, A.triangles), O.Tree.from_mesh(B.vertices, B.triangles)
    Q = P[:200].copy()
    Q[:, [3, 7, 11]] *= 2.0  # spread out so most poses are separated
    d1, _ = O.distance(tA, tB, Q)
    d2 = O.bruteforce_distance(tA, tB, Q)
    assert np.array_equal(d1, d2)
    assert (d1 > 0).sum() > 50 and (d1 == 0).sum() > 5
    # distance 0 exactly when the brute-force count is non-zero
    c, _, _ = O.bruteforce_collide(tA, tB, Q, 0.0)
    assert np.array_equal(d1 == 0, c > 0)


def test_distance_config4_bracket():
    w = G.make_config(4, num_poses=64)
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
    d, _ = O.distance(tA, tB, w.poses)
    t = w.poses[:, [3, 7, 11]].astype(np.float64)
    rho = np.sqrt((np.hypot(t[:, 0], t[:, 1]) - 3.0) ** 2 + t[:, 2] ** 2)
    assert np.all(rho >= 4.5 - 1e-5) and np.all(rho <= 6.0 + 1e-5)
    # surface of A within radius [0.95, 1.05]; torus tube within [0.97, 1.03]
    assert np.all(d >= rho - 1.05 - 1.03 - 1e-9)
    # chord sag of the polygonal surfaces is < 1e-3 at these resolutions
    assert np.all(d <= rho - 0.95 - 0.97 + 2e-3)
