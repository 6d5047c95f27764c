"""Generator pins (SURVEY §8(c) "what pins each part": mesh generators)."""
import numpy as np
import pytest

from workloads import generators as G


@pytest.mark.parametrize("u,v,nt,nv", [(32, 16, 960, 482), (64, 32, 3968, 1986), (128, 64, 16128, 8066),
                                       (318, 159, 100488, 50246)])
def test_uv_sphere_counts(u, v, nt, nv):
    dirs, tris = G.uv_sphere_topology(u, v)
    assert len(tris) == 2 * u * (v - 1) == nt and len(dirs) == 2 + u * (v - 1) == nv
    # closed 2-manifold: every edge is shared by exactly two triangles
    e = np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    assert np.all(cnt == 2)


def test_noise_ranges_and_torus():
    w = G.make_config(1, num_poses=4)
    r = np.linalg.norm(w.A.vertices.astype(np.float64), axis=1)
    assert r.min() >= 0.95 - 1e-6 and r.max() <= 1.05 + 1e-6
    v, t = G.noisy_torus(np.random.default_rng(0), 64, 32)
    assert len(t) == 2 * 64 * 32
    tube = np.sqrt((np.hypot(v[:, 0], v[:, 1]) - 3.0) ** 2 + v[:, 2] ** 2)
    assert tube.min() >= 0.97 - 1e-9 and tube.max() <= 1.03 + 1e-9


def test_poses_are_rigid():
    for P in (G.make_config(1, num_poses=256).poses, G.make_config(1, num_poses=64, preset="contact").poses):
        R = P[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]].reshape(-1, 3, 3).astype(np.float64)
        err = np.abs(np.einsum("nij,nkj->nik", R, R) - np.eye(3)).max()
        assert err < 1e-6
        assert np.allclose(np.linalg.det(R), 1.0, atol=1e-6)


def test_contact_preset_geometry():
    P = G.make_config(1, num_poses=512, preset="contact").poses
    d = np.linalg.norm(P[:, [3, 7, 11]].astype(np.float64), axis=1)
    assert np.allclose(d, 2.0, atol=1e-6)
    with pytest.raises(ValueError):
        G.make_config(5, num_poses=8, preset="contact")


def test_determinism_and_rank_offsets():
    a = G.make_config(2, num_poses=128)
    b = G.make_config(2, num_poses=128)
    c = G.make_config(2, num_poses=128, pose_seed_offset=1)
    assert np.array_equal(a.poses, b.poses) and np.array_equal(a.B.vertices, b.B.vertices)
    assert not np.array_equal(a.poses, c.poses) and np.array_equal(a.B.vertices, c.B.vertices)


def test_validate_poses():
    import paper_2012_05348_b200 as M
    P = G.make_config(1, num_poses=64).poses.copy()
    assert len(M.validate_poses(P)) == 0
    P[3, 0] *= 1.01          # not orthonormal
    P[7, 5] = np.nan          # not finite
    P[9, [0, 5, 10]] = [-1, -1, -1]   # reflection (det = -1)
    assert list(M.validate_poses(P)) == [3, 7, 9]


@pytest.mark.parametrize("k,n", [(1, 96), (3, 12)])
def test_zero_preset_table_is_the_oracles(k, n):
    # the zero-separation preset stores the
    # translation magnitudes tools/make_zero_preset.py bisected with the
    # oracle: re-evaluated here, the oracle distance of the generated fp32
    # poses equals the stored one and lies in (0, 1e-3)
    import os
    import oracle as O
    w = G.make_config(k, num_poses=n, preset="zero")
    tab = np.load(os.path.join(G.PRESET_DIR, f"zero_cfg{k}.npz"))
    assert len(tab["s"]) == (1024 if k == 1 else 32768)
    assert np.all((tab["distance"] > 0) & (tab["distance"] < 1e-3))
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
    d, _ = O.distance(tA, tB, w.poses)
    assert np.array_equal(d, tab["distance"][:n])
    # the rotation and direction are the seeded draws; |t| is the table's s
    assert np.allclose(np.linalg.norm(w.poses[:, [3, 7, 11]].astype(np.float64), axis=1), tab["s"][:n], rtol=1e-6)
