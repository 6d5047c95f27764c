"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Runs only on a B200 (-m gpu).  Every input comes from workloads.generators;
every expected value from oracle/ on the same arrays.  Sizes: config 1 in full
(1,024 poses, several thousand warp iterations, ragged tail), tiny meshes,
degenerate cases, and every BASELINE.json config at full size in the launch
configuration bench.py times, compared on seeded samples of poses the oracle
computes one by one, plus size-independent properties (hit == count > 0,
identical counts across all 9 config-3 layouts).
"""
import numpy as np
import pytest

import oracle as O
from tests.parity import check_collide, check_distance
from workloads import generators as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cuda_or_fail():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device")


@pytest.fixture(scope="module")
def M():
    _cuda_or_fail()
    import paper_2012_05348_b200 as M
    return M


def run_collide(M, A, B, poses, stats=False, descent="larger", early_exit=False):
    P = torch.from_numpy(np.ascontiguousarray(poses)).cuda()
    ws = M.Workspace(A, B, 0)
    hit, cnt = M.collide_batch(A, B, P, workspace=ws, stats=stats, descent=descent, early_exit=early_exit)
    M.check(ws)
    out = hit.cpu().numpy(), cnt.cpu().numpy().view(np.uint32).astype(np.int64)
    if stats:
        return out + (M.read_stats(ws),)
    return out


def run_distance(M, A, B, poses, stats=False, descent="larger"):
    P = torch.from_numpy(np.ascontiguousarray(poses)).cuda()
    ws = M.Workspace(A, B, 1)
    d = M.distance_batch(A, B, P, workspace=ws, stats=stats, descent=descent)
    M.check(ws)
    out = d.cpu().numpy()
    if stats:
        return out, M.read_stats(ws)
    return out


def build(M, mesh, B, bits, T=32, layout="delta", kdop=6, aligned=False, zs=False):
    return M.build_compressed_bvh(mesh.vertices, mesh.triangles, B, bits, T, 4, layout=layout,
                                  kdop=kdop, align_treelets=aligned, zero_suppress=zs).to_device()


def run_collide_staged(M, A, B, poses, staging):
    P = torch.from_numpy(np.ascontiguousarray(poses)).cuda()
    ws = M.Workspace(A, B, 0)
    hit, cnt = M.collide_batch(A, B, P, workspace=ws, stats=True, staging=staging)
    M.check(ws)
    return hit.cpu().numpy(), cnt.cpu().numpy().view(np.uint32).astype(np.int64), M.read_stats(ws)


def oracle_trees(w):
    return O.Tree.from_mesh(w.A.vertices, w.A.triangles), O.Tree.from_mesh(w.B.vertices, w.B.triangles)


# ------------------------------------------------------------------ config 1 in full


@pytest.fixture(scope="module")
def cfg1():
    w = G.make_config(1)
    tA, tB = oracle_trees(w)
    delta = O.band_delta(w.A.vertices)
    cnt, H, Z, _ = O.collide(tA, tB, w.poses, delta)
    return w, tA, tB, delta, cnt, H, Z


def test_config1_full_collide(M, cfg1):
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    hit, gc = run_collide(M, A, B, w.poses)
    rep = check_collide(hit, gc, H, Z, "cfg1")
    assert rep["hits"] > 200
    print("cfg1", rep)


@pytest.mark.parametrize("Bf,bits", [(2, 4), (4, 8), (8, 16), (4, 2)])
def test_config1_layouts(M, cfg1, Bf, bits):
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, Bf, bits), build(M, w.B, Bf, bits)
    hit, gc = run_collide(M, A, B, w.poses)
    check_collide(hit, gc, H, Z, f"cfg1 B={Bf} b={bits}")


@pytest.mark.parametrize("Bf", [2, 4, 8])
def test_config1_alg1_simultaneous_descent(M, cfg1, Bf):
    # Alg. 1 verbatim (descend both nodes) and the default larger-first rule
    # reach the same leaf pairs: identical counts on every pose, both in band
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, Bf, 8), build(M, w.B, Bf, 8)
    h1, c1, s1 = run_collide(M, A, B, w.poses, stats=True, descent="simultaneous")
    h2, c2, s2 = run_collide(M, A, B, w.poses, stats=True, descent="larger")
    check_collide(h1, c1, H, Z, f"alg1 B={Bf}")
    assert np.array_equal(c1, c2) and np.array_equal(h1, h2)
    assert s1["bv_tests"] > 0 and s2["bv_tests"] > 0
    d1 = run_distance(M, A, B, w.poses[:128], descent="simultaneous")
    d2 = run_distance(M, A, B, w.poses[:128], descent="larger")
    d64, _ = O.distance(tA, tB, w.poses[:128])
    check_distance(d1, d64, delta, "alg1 distance")
    check_distance(d2, d64, delta, "larger distance")


@pytest.mark.parametrize("layout", ["fp16", "fp32"])
def test_config1_absolute_layouts(M, cfg1, layout):
    # binary16 / fp32 node boxes (the paper's §III.A comparison) through the
    # same kernels: band rule vs the oracle, identical counts to the delta layout
    w, tA, tB, delta, cnt, H, Z = cfg1
    ref = run_collide(M, build(M, w.A, 4, 8), build(M, w.B, 4, 8), w.poses)
    A, B = build(M, w.A, 4, 8, layout=layout), build(M, w.B, 4, 8, layout=layout)
    hit, gc = run_collide(M, A, B, w.poses)
    check_collide(hit, gc, H, Z, f"cfg1 {layout}")
    assert np.array_equal(gc, ref[1])
    d = run_distance(M, A, B, w.poses[:128])
    d64, _ = O.distance(tA, tB, w.poses[:128])
    check_distance(d, d64, delta, f"cfg1 distance {layout}")


@pytest.mark.parametrize("kdop", [14, 18, 26])
@pytest.mark.parametrize("Bf,bits", [(2, 4), (4, 8), (8, 16)])
def test_config1_kdop(M, cfg1, kdop, Bf, bits):
    # k-DOP bounding volumes on the static model B (Table I): band rule
    # vs the oracle, the same counts as the AABB blob, and — the k-DOP is the
    # AABB cut by more slabs, the descent rule sees only the AABB part — no
    # more BV tests or leaf pairs than the AABB traversal
    w, tA, tB, delta, cnt, H, Z = cfg1
    A = build(M, w.A, Bf, bits)
    Bb = build(M, w.B, Bf, bits)
    Bk = build(M, w.B, Bf, bits, kdop=kdop)
    h0, c0, s0 = run_collide(M, A, Bb, w.poses, stats=True)
    hit, gc, sk = run_collide(M, A, Bk, w.poses, stats=True)
    check_collide(hit, gc, H, Z, f"cfg1 k={kdop}")
    assert np.array_equal(gc, c0)
    assert sk["bv_tests"] <= s0["bv_tests"] and sk["leaf_pairs"] <= s0["leaf_pairs"]
    d = run_distance(M, A, Bk, w.poses[:128])
    d64, _ = O.distance(tA, tB, w.poses[:128])
    check_distance(d, d64, delta, f"cfg1 distance k={kdop}")


def test_kdop_on_moving_model_rejected(M, cfg1):
    w = cfg1[0]
    A = build(M, w.A, 4, 8, kdop=14)
    B = build(M, w.B, 4, 8)
    with pytest.raises(Exception, match="EINVAL"):
        run_collide(M, A, B, w.poses[:4])


def test_config1_early_exit(M, cfg1):
    # early-exit hit flags equal the exhaustive ones; the count is a
    # lower bound that is >= 1 exactly for colliding poses
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    h1, c1 = run_collide(M, A, B, w.poses)
    h2, c2, st2 = run_collide(M, A, B, w.poses, stats=True, early_exit=True)
    _, _, st1 = run_collide(M, A, B, w.poses, stats=True)
    assert np.array_equal(h1, h2)
    assert np.array_equal(c2 > 0, h2 == 1) and np.all(c2 <= c1)
    assert st2["tri_tests"] < st1["tri_tests"]


def test_config1_stats_variant_same_answer(M, cfg1):
    w = cfg1[0]
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    h1, c1 = run_collide(M, A, B, w.poses)
    h2, c2, st = run_collide(M, A, B, w.poses, stats=True)
    assert np.array_equal(h1, h2) and np.array_equal(c1, c2)
    assert st["bv_tests"] > 0 and st["tri_tests"] >= int(c1.sum())
    assert st["expansions"] > 0 and st["leaf_pairs"] > 0


def test_config1_distance(M, cfg1):
    w, tA, tB, delta = cfg1[:4]
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    P = w.poses[:256]
    d64, _ = O.distance(tA, tB, P)
    g = run_distance(M, A, B, P)
    rep = check_distance(g, d64, delta, "cfg1 distance")
    assert rep["near_contact"] > 20


def test_config1_distance_caps(M, cfg1):
    # capped queries (cbvh_query_opts.capped): result = min(distance, cap),
    # exact below the cap; caps above the oracle's distance change nothing,
    # caps below it come back unchanged; NaN = no cap, negative = 0
    w, tA, tB, delta = cfg1[:4]
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    P = w.poses[:256]
    d64, _ = O.distance(tA, tB, P)
    Pt = torch.from_numpy(np.ascontiguousarray(P)).cuda()
    ws = M.Workspace(A, B, 1)
    far = d64 > 0.05
    above = np.where(far, d64 * 1.01 + 1e-3, np.inf).astype(np.float32)
    g = M.distance_batch(A, B, Pt, workspace=ws, caps=torch.from_numpy(above).cuda()).cpu().numpy()
    M.check(ws)
    check_distance(g, d64, delta, "cfg1 caps above")
    below = np.where(far, d64 * 0.5, np.float32(np.nan)).astype(np.float32)
    below[:4] = -1.0
    g = M.distance_batch(A, B, Pt, workspace=ws, caps=torch.from_numpy(below).cuda()).cpu().numpy()
    M.check(ws)
    cap_rows = far.copy()
    cap_rows[:4] = False
    assert np.array_equal(g[cap_rows], below[cap_rows])
    assert np.all(g[:4] == 0.0)
    nan_rows = ~far
    nan_rows[:4] = False
    check_distance(g[nan_rows], d64[nan_rows], delta, "cfg1 caps nan")


def test_contact_preset_collide_and_distance(M):
    # the paper's "distance of zero" preset: every pose at or near
    # contact — the band and the fp64 distance re-evaluation are exercised hardest
    w = G.make_config(1, num_poses=768, preset="contact")
    tA, tB = oracle_trees(w)
    delta = O.band_delta(w.A.vertices)
    _, H, Z, _ = O.collide(tA, tB, w.poses, delta)
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    hit, gc = run_collide(M, A, B, w.poses)
    rep = check_collide(hit, gc, H, Z, "contact")
    assert 0.5 < hit.mean() < 0.99
    d = run_distance(M, A, B, w.poses[:256])
    d64, _ = O.distance(tA, tB, w.poses[:256])
    drep = check_distance(d, d64, delta, "contact distance")
    assert np.median(d64[d64 > 0]) < 0.05
    print("contact", rep, drep)


@pytest.mark.parametrize("Bf,bits,T", [(2, 8, 32), (4, 8, 32), (4, 8, 64), (8, 16, 64), (4, 4, 16)])
def test_config1_treelet_staging(M, cfg1, Bf, bits, T):
    # treelet blocks staged in shared memory (align_treelets):
    # band rule vs the oracle, counts identical to the unstaged kernel on the
    # same blobs and on packed (unaligned) blobs, and blocks really staged
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, Bf, bits, T, aligned=True), build(M, w.B, Bf, bits, T, aligned=True)
    hit, gc, st = run_collide_staged(M, A, B, w.poses, "on")
    check_collide(hit, gc, H, Z, f"staged B={Bf} b={bits} T={T}")
    h0, c0, st0 = run_collide_staged(M, A, B, w.poses, "off")
    assert np.array_equal(gc, c0) and np.array_equal(hit, h0)
    hp, cp, _ = run_collide_staged(M, build(M, w.A, Bf, bits, T), build(M, w.B, Bf, bits, T), w.poses, "auto")
    assert np.array_equal(gc, cp)
    assert st["treelet_blocks"] > 0 and st["staged_reads"] > 0 and st0["treelet_blocks"] == 0
    assert st["bv_tests"] == st0["bv_tests"]
    # the staged reads plus the (all-slots-busy) global fallbacks are every decoded child
    assert st["staged_reads"] <= st["nodes_decoded"]
    # only one side aligned: that side is staged, the other read from global memory
    _, c1, s1 = run_collide_staged(M, A, build(M, w.B, Bf, bits, T), w.poses, "on")
    assert np.array_equal(c1, gc) and s1["treelet_blocks"] > 0
    P = torch.from_numpy(w.poses[:256]).cuda()
    d = M.distance_batch(A, B, P, staging="on").cpu().numpy()
    d64, _ = O.distance(tA, tB, w.poses[:256])
    check_distance(d, d64, delta, f"staged distance B={Bf}")
    with pytest.raises(M._lib.CbvhError, match="EINVAL"):
        M.collide_batch(build(M, w.A, Bf, bits, T), build(M, w.B, Bf, bits, T), P, staging="on")


@pytest.mark.parametrize("Bf,bits,T", [(2, 8, 32), (4, 8, 64), (8, 16, 64), (4, 12, 16)])
def test_config1_zero_suppressed_codes(M, cfg1, Bf, bits, T):
    # integer-compressed corrections: decoded from staged blocks and,
    # unstaged, straight from global memory (mask popcounts) — both in band
    # vs the oracle and identical to the plain aligned blob's counts
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, Bf, bits, T, zs=True), build(M, w.B, Bf, bits, T, zs=True)
    ref = run_collide(M, build(M, w.A, Bf, bits, T, aligned=True), build(M, w.B, Bf, bits, T, aligned=True), w.poses)
    for staging in ("on", "off"):
        hit, gc, st = run_collide_staged(M, A, B, w.poses, staging)
        check_collide(hit, gc, H, Z, f"zero-suppressed {staging} B={Bf} b={bits}")
        assert np.array_equal(gc, ref[1])
        assert (st["treelet_blocks"] > 0) == (staging == "on")
    P = torch.from_numpy(w.poses[:256]).cuda()
    d64, _ = O.distance(tA, tB, w.poses[:256])
    for staging in ("on", "off"):
        check_distance(M.distance_batch(A, B, P, staging=staging).cpu().numpy(), d64, delta, f"zs distance {staging}")


@pytest.mark.parametrize("k", [1, 3])
def test_zero_separation_preset(M, k):
    # the paper's "distance of zero" preset by bisection with the
    # oracle: every pose's oracle distance is in (0, 1e-3);
    # collide (band rule) and distance (1e-5 relative) through the C-ABI
    n = 1024 if k == 1 else 2048
    w = G.make_config(k, num_poses=n, preset="zero")
    tA, tB = oracle_trees(w)
    delta = O.band_delta(w.A.vertices)
    d64, _ = O.distance(tA, tB, w.poses)
    assert np.all((d64 > 0) & (d64 < 1e-3))
    _, H, Z, _ = O.collide(tA, tB, w.poses, delta)
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    hit, gc = run_collide(M, A, B, w.poses)
    rep = check_collide(hit, gc, H, Z, f"zero cfg{k}")
    drep = check_distance(run_distance(M, A, B, w.poses), d64, delta, f"zero cfg{k} distance")
    print("zero preset", k, rep, drep)


# ------------------------------------------------------------------ tiny + degenerate


@pytest.mark.parametrize("which", ["8x4", "16x8"])
def test_tiny_collide_and_distance(M, which):
    Am, Bm, P = G.tiny_pair(which, seed=5, n_poses=3000, half_width=1.5)
    tA, tB = O.Tree.from_mesh(Am.vertices, Am.triangles), O.Tree.from_mesh(Bm.vertices, Bm.triangles)
    delta = O.band_delta(Am.vertices)
    _, H, Z = O.bruteforce_collide(tA, tB, P, delta)
    for Bf in (2, 4, 8):
        A, B = build(M, Am, Bf, 8), build(M, Bm, Bf, 8)
        hit, gc = run_collide(M, A, B, P)
        check_collide(hit, gc, H, Z, f"tiny {which} B={Bf}")
        d = run_distance(M, A, B, P[:500])
        check_distance(d, O.bruteforce_distance(tA, tB, P[:500]), delta, f"tiny {which}")


def test_single_triangle_meshes(M):
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    T = np.array([[0, 1, 2]], np.int32)
    A = M.build_compressed_bvh(V, T, 2, 8).to_device()  # root is a leaf: leaf-leaf root pair
    P = G.identity_poses(4)
    P[1, 11] = 0.5   # lifted: no contact
    P[2, 11] = -1e-3  # below: no contact
    P[3, 3] = 0.2     # shifted in-plane: coplanar overlap
    hit, gc = run_collide(M, A, A, P)
    assert list(gc) == [1, 0, 0, 1] and list(hit) == [1, 0, 0, 1]
    d = run_distance(M, A, A, P)
    assert d[0] == 0 and d[3] == 0
    assert abs(d[1] - 0.5) < 1e-6 and abs(d[2] - 1e-3) < 1e-8


def test_self_identity_and_far(M, cfg1):
    w = cfg1[0]
    A = build(M, w.A, 4, 8)
    P = G.identity_poses(3)
    P[1, 3] = 10.0
    P[2, 7] = -3.0
    hit, gc = run_collide(M, A, A, P)
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    _, H, Z, _ = O.collide(tA, tA, P, O.band_delta(w.A.vertices))
    check_collide(hit, gc, H, Z, "self")
    # coincident geometry: every touching pair is a band pair (pen = 0); each
    # triangle meets itself exactly (identical fp32 coordinates, coplanar test)
    assert gc[0] >= w.A.num_triangles and hit[0] == 1
    assert gc[1] == 0 and gc[2] == 0


def test_empty_and_ragged_batches(M, cfg1):
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    hit, gc = run_collide(M, A, B, w.poses[:0])
    assert len(hit) == 0 and len(gc) == 0
    for n in (1, 7, 33, 257, 1023):
        hit, gc = run_collide(M, A, B, w.poses[:n])
        check_collide(hit, gc, H[:n], Z[:n], f"ragged {n}")


def test_error_paths_device(M, cfg1):
    from paper_2012_05348_b200 import _lib as L
    w = cfg1[0]
    A, B = build(M, w.A, 2, 8), build(M, w.B, 2, 8)
    P = torch.from_numpy(w.poses[:64]).cuda()
    ws = M.Workspace(A, B, 0)
    small = M.Workspace(A, B, 0)
    small.nbytes = 1024
    with pytest.raises(L.CbvhError, match="EWORKSPACE"):
        M.collide_batch(A, B, P, workspace=small)
    Pbig = torch.zeros(65 * 12 + 1, dtype=torch.float32, device="cuda")
    Pmis = Pbig[1:].view(65, 12)
    with pytest.raises(L.CbvhError, match="EINVAL"):
        M.collide_batch(A, B, Pmis, workspace=ws)
    M.collide_batch(A, B, P, workspace=ws)
    M.check(ws)
    assert M.last_launch_count() >= 2  # init + the load-balancing phases
    # the binding checks caller buffers before any kernel writes through them
    with pytest.raises(ValueError):
        M.collide_batch(A, B, P, hit=torch.empty(10, dtype=torch.uint8, device="cuda"), workspace=ws)
    with pytest.raises(TypeError):
        M.collide_batch(A, B, P, count=torch.empty(64, dtype=torch.float32, device="cuda"), workspace=ws)
    with pytest.raises(ValueError):
        M.distance_batch(A, B, P, dist=torch.empty(64, dtype=torch.float32), workspace=M.Workspace(A, B, 1))
    with pytest.raises(ValueError):
        M.collide_batch(A, M.build_compressed_bvh(w.B.vertices, w.B.triangles, 2, 8), P)  # not on the device
    # a call-local workspace on a side stream: the result is checked and synchronised before returning
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        hit, cnt = M.collide_batch(A, B, P, stream=side)
    ref_hit, ref_cnt = M.collide_batch(A, B, P, workspace=ws)
    M.check(ws)
    assert torch.equal(cnt, ref_cnt) and torch.equal(hit, ref_hit)


# ------------------------------------------------------------------ full-size configs, sampled


def _sample(n_total, k, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n_total, size=k, replace=False))


def test_config2_full_size_sampled(M):
    w = G.make_config(2)
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    hit, gc = run_collide(M, A, B, w.poses)
    assert 0.10 < hit.mean() < 0.25
    idx = _sample(len(w.poses), 1500, 2)
    # bias the sample towards colliding poses so the count check has teeth
    idx = np.unique(np.concatenate([idx, np.nonzero(hit)[0][:500]]))
    tA, tB = oracle_trees(w)
    delta = O.band_delta(w.A.vertices)
    _, H, Z, _ = O.collide(tA, tB, w.poses[idx], delta)
    rep = check_collide(hit[idx], gc[idx], H, Z, "cfg2")
    print("cfg2", rep)


def test_config3_all_layouts_agree(M):
    w = G.make_config(3)
    idx = _sample(len(w.poses), 1000, 3)
    tA, tB = oracle_trees(w)
    delta = O.band_delta(w.A.vertices)
    _, H, Z, _ = O.collide(tA, tB, w.poses[idx], delta)
    ref = None
    for Bf, bits in w.settings:
        A, B = build(M, w.A, Bf, bits), build(M, w.B, Bf, bits)
        hit, gc = run_collide(M, A, B, w.poses)
        check_collide(hit[idx], gc[idx], H, Z, f"cfg3 B={Bf} b={bits}")
        if ref is None:
            ref = gc
        # leaf tests are tree-independent and culling is conservative: every
        # layout must produce the same counts on all 262,144 poses
        assert np.array_equal(gc, ref), f"cfg3 B={Bf} b={bits} differs from B=2 b=4"


def test_config4_distance_full_size_sampled(M):
    w = G.make_config(4)
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    d = run_distance(M, A, B, w.poses)
    assert np.all(np.isfinite(d)) and d.min() >= 2.42 - 1e-4
    idx = _sample(len(w.poses), 512, 4)
    tA, tB = oracle_trees(w)
    d64, _ = O.distance(tA, tB, w.poses[idx])
    rep = check_distance(d[idx], d64, O.band_delta(w.A.vertices), "cfg4")
    print("cfg4", rep)


def test_config3_contact_distance_full_size_sampled(M):
    # the paper's zero-distance preset at config 3's full size (262,144
    # poses, the width-8 dive active): sampled poses against the fp64 oracle
    w = G.make_config(3, preset="contact")
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    d = run_distance(M, A, B, w.poses)
    assert np.all(np.isfinite(d)) and np.all(d >= 0)
    idx = _sample(len(w.poses), 48, 31)
    tA, tB = oracle_trees(w)
    d64, _ = O.distance(tA, tB, w.poses[idx])
    rep = check_distance(d[idx], d64, O.band_delta(w.A.vertices), "cfg3 contact")
    print("cfg3 contact distance", rep)


def test_config4_capped_full_size_sampled(M):
    # caps at config 4's full size: result = min(distance, cap) on every pose
    # (cap 3.5 falls inside the distance range [2.42, ~5]); sampled against
    # the oracle, and exactly the uncapped result wherever that is below 3.5
    w = G.make_config(4)
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    d = run_distance(M, A, B, w.poses)
    P = torch.from_numpy(w.poses).cuda()
    ws = M.Workspace(A, B, 1)
    cap = np.float32(3.5)
    dc = M.distance_batch(A, B, P, workspace=ws, caps=torch.full((len(P),), float(cap), device="cuda")).cpu().numpy()
    M.check(ws)
    below = d < cap
    assert 0 < below.sum() < len(d)
    assert np.array_equal(dc[below], d[below])
    assert np.all(dc[~below] == cap)
    idx = _sample(len(w.poses), 64, 41)
    tA, tB = oracle_trees(w)
    d64, _ = O.distance(tA, tB, w.poses[idx])
    ref = np.minimum(d64, float(cap))
    rel = np.abs(dc[idx] - ref) / ref
    assert rel.max() <= 1e-5


@pytest.mark.parametrize("layout,kdop", [("fp16", 6), ("fp32", 6), ("delta", 14)])
def test_config4_distance_layouts_sampled(M, layout, kdop):
    # the absolute layouts (the paper's half / float comparison) and a k-DOP
    # environment through the distance kernel at config 4's full size: the
    # same distances as the delta-AABB blobs wherever both are exact, and the
    # oracle's on a sample
    w = G.make_config(4)
    A = build(M, w.A, w.branching, w.bits, w.treelet, layout=layout)
    B = build(M, w.B, w.branching, w.bits, w.treelet, layout=layout, kdop=kdop)
    d = run_distance(M, A, B, w.poses)
    ref = run_distance(M, build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet),
                       w.poses)
    assert np.max(np.abs(d - ref) / ref) <= 2e-5
    idx = _sample(len(w.poses), 32, 51)
    tA, tB = oracle_trees(w)
    d64, _ = O.distance(tA, tB, w.poses[idx])
    check_distance(d[idx], d64, O.band_delta(w.A.vertices), f"cfg4 {layout} k={kdop}")


def test_config3_contact_early_exit_full_size(M):
    # zero-distance preset at full size: early-exit hit flags equal the
    # exhaustive ones on all 262,144 poses; counts are lower bounds >= 1 on hits
    w = G.make_config(3, preset="contact")
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    h1, c1 = run_collide(M, A, B, w.poses)
    h2, c2 = run_collide(M, A, B, w.poses, early_exit=True)
    assert np.array_equal(h1, h2)
    assert np.array_equal(c2 > 0, h2 == 1) and np.all(c2 <= c1)
    assert h1.sum() > len(h1) // 4


def test_config5_layouts_agree_full_size(M):
    # full config 5 batch: fp16 / fp32 layouts count exactly what delta counts
    w = G.make_config(5)
    ref = None
    for layout in ("delta", "fp16", "fp32"):
        A = build(M, w.A, w.branching, w.bits, w.treelet, layout)
        B = build(M, w.B, w.branching, w.bits, w.treelet, layout)
        hit, gc = run_collide(M, A, B, w.poses)
        if ref is None:
            ref = gc
        assert np.array_equal(gc, ref), layout


def test_config5_kdop_full_size(M):
    # full config 5 batch with 14- and 26-DOPs on B: the counts equal the
    # AABB blob's on every pose, and a sample matches the oracle (band rule)
    w = G.make_config(5)
    A = build(M, w.A, w.branching, w.bits, w.treelet)
    _, ref = run_collide(M, A, build(M, w.B, w.branching, w.bits, w.treelet), w.poses)
    idx = _sample(len(w.poses), 200, 7)
    tA, tB = oracle_trees(w)
    _, H, Z, _ = O.collide(tA, tB, w.poses[idx], O.band_delta(w.A.vertices))
    for k in (14, 26):
        hit, gc = run_collide(M, A, build(M, w.B, w.branching, w.bits, w.treelet, kdop=k), w.poses)
        assert np.array_equal(gc, ref), k
        check_collide(hit[idx], gc[idx], H, Z, f"cfg5 k={k}")


def test_config5_treelet_staging_full_size(M):
    # full config 5 batch on aligned blobs (T = 64): the staged kernel counts
    # exactly what the unstaged kernel counts on every pose
    w = G.make_config(5)
    A = build(M, w.A, w.branching, w.bits, w.treelet, aligned=True)
    B = build(M, w.B, w.branching, w.bits, w.treelet, aligned=True)
    h1, c1, s1 = run_collide_staged(M, A, B, w.poses, "on")
    h0, c0, s0 = run_collide_staged(M, A, B, w.poses, "off")
    assert np.array_equal(c1, c0) and np.array_equal(h1, h0)
    assert s1["treelet_blocks"] > 0 and s1["bv_tests"] == s0["bv_tests"]
    print("cfg5 staging", {k: s1[k] for k in ("treelet_blocks", "treelet_bytes", "staged_reads", "nodes_decoded")})


def test_config5_zero_suppressed_full_size(M):
    # full config 5 batch, zero-suppressed blobs: staged and unstaged decode
    # give the packed blob's counts on every pose
    w = G.make_config(5)
    _, ref = run_collide(M, build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet),
                         w.poses)
    A = build(M, w.A, w.branching, w.bits, w.treelet, zs=True)
    B = build(M, w.B, w.branching, w.bits, w.treelet, zs=True)
    for staging in ("on", "off"):
        _, gc, _ = run_collide_staged(M, A, B, w.poses, staging)
        assert np.array_equal(gc, ref), staging


def test_config5_early_exit_full_size(M):
    w = G.make_config(5)
    A = build(M, w.A, w.branching, w.bits, w.treelet)
    B = build(M, w.B, w.branching, w.bits, w.treelet)
    h1, c1 = run_collide(M, A, B, w.poses)
    h2, c2 = run_collide(M, A, B, w.poses, early_exit=True)
    assert np.array_equal(h1, h2)
    assert np.array_equal(c2 > 0, h2 == 1) and np.all(c2 <= c1)


def test_config5_full_size_sampled(M):
    w = G.make_config(5)
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    hit, gc = run_collide(M, A, B, w.poses)
    assert 0.02 < hit.mean() < 0.09
    # 6,000 random poses plus every 60th colliding pose (~1,000 more, so the
    # count check has teeth); bench.py checks a further ~45,000-pose prefix
    idx = _sample(len(w.poses), 6000, 5)
    idx = np.unique(np.concatenate([idx, np.nonzero(hit)[0][::60]]))
    tA, tB = oracle_trees(w)
    delta = O.band_delta(w.A.vertices)
    _, H, Z, _ = O.collide(tA, tB, w.poses[idx], delta)
    rep = check_collide(hit[idx], gc[idx], H, Z, "cfg5")
    print("cfg5", rep)


_PHASE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2012_05348_b200 as M
from workloads import generators as G
w = G.make_config(3, num_poses=65536)
A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet).to_device()
B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet).to_device()
P = torch.from_numpy(w.poses).cuda()
ws = M.Workspace(A, B, 0)
hit, cnt = M.collide_batch(A, B, P, workspace=ws, stats=True)
M.check(ws)
st = M.read_stats(ws)
wd = M.Workspace(A, B, 1)
d = M.distance_batch(A, B, P[:4096], workspace=wd)
M.check(wd)
np.savez({out!r}, cnt=cnt.cpu().numpy().view(np.uint32), d=d.cpu().numpy(), dumped=st["dumped"])
"""


@pytest.mark.parametrize("phases", ["0", "1,1,1,1,1,1", "4,0,2", "1000000"])
def test_load_balancing_phases_do_not_change_results(M, tmp_path, phases):
    # the continuation phases only move work between warps and
    # launches: any budget schedule (immediate dumps, many tiny phases, one
    # unbounded phase) gives the default schedule's counts and distances
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for tag, env in (("default", None), ("variant", phases)):
        out = str(tmp_path / f"{tag}.npz")
        e = dict(os.environ)
        e.pop("CBVH_PHASES", None)
        if env is not None:
            e["CBVH_PHASES"] = env
        subprocess.run([sys.executable, "-c", _PHASE_SCRIPT.format(root=root, out=out)], env=e, check=True,
                       timeout=600)
        res[tag] = np.load(out)
    assert np.array_equal(res["default"]["cnt"], res["variant"]["cnt"])
    assert np.array_equal(res["default"]["d"], res["variant"]["d"])
    if phases in ("0", "1,1,1,1,1,1"):
        assert int(res["variant"]["dumped"]) > 0  # the schedule really moved work between launches


_DIVE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2012_05348_b200 as M
from workloads import generators as G
out = {{}}
for cfg, n, preset in ((4, 8192, "random"), (3, 8192, "contact"), (2, 4096, "random")):
    w = G.make_config(cfg, num_poses=n, preset=preset)
    A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet).to_device()
    B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet).to_device()
    P = torch.from_numpy(w.poses).cuda()
    wd = M.Workspace(A, B, 1)
    d = M.distance_batch(A, B, P, workspace=wd)
    M.check(wd)
    out["d%d" % cfg] = d.cpu().numpy()
np.savez({out!r}, **out)
"""


def test_greedy_dive_does_not_change_distances(M, tmp_path):
    # the dive (reading R26) only seeds each pose's best with a real pair
    # distance computed as the leaf phase computes it: with and without it the
    # distances are bit-identical (configs 4, 3 contact, 2)
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for tag in ("0", "1"):
        out = str(tmp_path / f"dive{tag}.npz")
        e = dict(os.environ)
        e["CBVH_DIVE"] = tag
        subprocess.run([sys.executable, "-c", _DIVE_SCRIPT.format(root=root, out=out)], env=e, check=True,
                       timeout=600)
        res[tag] = np.load(out)
    for k in ("d4", "d3", "d2"):
        assert np.array_equal(res["0"][k], res["1"][k]), k


def test_config5_4x_poses_sampled(M):
    # 4,194,304 poses in one call (4x the headline batch): hit == (count > 0)
    # everywhere, the first 1M poses equal the 1M-pose call, and a sample of
    # the extra poses matches the oracle
    w = G.make_config(5)
    w4 = G.make_config(5, num_poses=4 * len(w.poses), pose_seed_offset=11)
    P = np.concatenate([w.poses, w4.poses[len(w.poses):]])
    A = build(M, w.A, w.branching, w.bits, w.treelet)
    B = build(M, w.B, w.branching, w.bits, w.treelet)
    hit, gc = run_collide(M, A, B, P)
    assert np.array_equal(hit == 1, gc > 0)
    _, ref = run_collide(M, A, B, w.poses)
    assert np.array_equal(gc[:len(w.poses)], ref)
    idx = len(w.poses) + _sample(len(P) - len(w.poses), 150, 9)
    tA, tB = oracle_trees(w)
    _, H, Z, _ = O.collide(tA, tB, P[idx], O.band_delta(w.A.vertices))
    check_collide(hit[idx], gc[idx], H, Z, "cfg5 x4")


def test_concurrent_streams_distinct_workspaces(M, cfg1):
    # include/cbvh.h: blobs are immutable; calls on different streams with
    # distinct workspaces may run concurrently
    w = cfg1[0]
    A, B = build(M, w.A, 4, 8), build(M, w.B, 4, 8)
    P1 = torch.from_numpy(np.ascontiguousarray(w.poses[:512])).cuda()
    P2 = torch.from_numpy(np.ascontiguousarray(w.poses[512:])).cuda()
    ref_hit, ref_cnt = run_collide(M, A, B, w.poses)
    ref_d = run_distance(M, A, B, w.poses[:256])
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ws1, ws2, ws3 = M.Workspace(A, B, 0), M.Workspace(A, B, 0), M.Workspace(A, B, 1)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            h1, c1 = M.collide_batch(A, B, P1, workspace=ws1, stream=s1)
        with torch.cuda.stream(s2):
            h2, c2 = M.collide_batch(A, B, P2, workspace=ws2, stream=s2)
        with torch.cuda.stream(s3):
            d3 = M.distance_batch(A, B, P1[:256], workspace=ws3, stream=s3)
        M.check(ws1, s1)
        M.check(ws2, s2)
        M.check(ws3, s3)
        torch.cuda.synchronize()
        cnt = np.concatenate([c1.cpu().numpy(), c2.cpu().numpy()]).view(np.uint32).astype(np.int64)
        hit = np.concatenate([h1.cpu().numpy(), h2.cpu().numpy()])
        assert np.array_equal(cnt, ref_cnt) and np.array_equal(hit, ref_hit)
        # (the visiting order may differ between runs; the minimum agrees to
        # fp32 rounding of near-tied candidates)
        assert np.allclose(d3.cpu().numpy(), ref_d, rtol=1e-6, atol=0)


@pytest.mark.parametrize("n", [1, 3, 64, 200, 257])
def test_small_batches_short_schedule(M, cfg1, n):
    # batches far below the grid size take the short phase schedule and the
    # early cursor polls: counts match the band rule and the
    # full batch's answers, distances the oracle's
    w, tA, tB, delta, cnt, H, Z = cfg1
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    # the heaviest poses first, so a tiny batch still has deep traversals to hand over
    order = np.argsort(-(H + Z), kind="stable")[:n]
    P = w.poses[order]
    hit, gc = run_collide(M, A, B, P)
    check_collide(hit, gc, H[order], Z[order], f"small batch {n}")
    full_hit, full_gc = run_collide(M, A, B, w.poses)
    assert np.array_equal(gc, full_gc[order]) and np.array_equal(hit, full_hit[order])
    d64, _ = O.distance(tA, tB, P[:64])
    g = run_distance(M, A, B, P[:64])
    check_distance(g, d64, delta, f"small batch {n} distance")


@pytest.mark.parametrize("Bf,kdop", [(8, 6), (2, 6), (8, 14), (4, 26)])
def test_warp_dive_arities(M, cfg1, Bf, kdop):
    # the warp dive gives a beam entry 4 or 8 lanes (the larger arity of the
    # two trees) and carries B's k-DOP slabs: distances against the oracle for
    # 8-ary and binary trees and k-DOP environments
    w, tA, tB, delta = cfg1[:4]
    A, B = build(M, w.A, Bf, 8), build(M, w.B, Bf, 8, kdop=kdop)
    P = w.poses[:192]
    d64, _ = O.distance(tA, tB, P)
    check_distance(run_distance(M, A, B, P), d64, delta, f"warp dive B={Bf} k={kdop}")


def test_fast_and_generic_kernels_agree_full_size(M):
    # default blobs run the FAST instantiations (format and options folded at
    # compile time, 7 CTAs / SM); the stats variant runs the generic kernel on
    # the same blobs: identical counts on the whole config-5 batch, identical
    # hit flags for the hit-only query, bit-identical distances on config 4
    w = G.make_config(5)
    A, B = build(M, w.A, w.branching, w.bits, w.treelet), build(M, w.B, w.branching, w.bits, w.treelet)
    hit_f, cnt_f = run_collide(M, A, B, w.poses)
    hit_g, cnt_g, st = run_collide(M, A, B, w.poses, stats=True)
    assert np.array_equal(cnt_f, cnt_g) and np.array_equal(hit_f, hit_g)
    assert st["bv_tests"] > 8e8
    hit_e, _ = run_collide(M, A, B, w.poses, early_exit=True)
    assert np.array_equal(hit_e, hit_f)
    w4 = G.make_config(4, num_poses=16384)
    A4, B4 = build(M, w4.A, w4.branching, w4.bits, w4.treelet), build(M, w4.B, w4.branching, w4.bits, w4.treelet)
    d_f = run_distance(M, A4, B4, w4.poses)
    d_g, _ = run_distance(M, A4, B4, w4.poses, stats=True)
    assert np.array_equal(d_f, d_g)
