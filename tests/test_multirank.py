"""N > 1 path of bench.py on CPU: two gloo ranks (world_size 2).

The path shards by pose batch (weak scaling): identical meshes
on every rank, an independent pose batch per rank, no data-path collective;
the only collective is the max-over-ranks reduction of the timed region.
Each rank also checks its shard against the oracle, as the GPU path would.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import bench
        import oracle as O

        w = bench.rank_workload(1, rank, num_poses=48)
        # same meshes everywhere, different poses per rank
        mesh_sig = torch.tensor([float(w.A.vertices.sum()), float(w.B.vertices.sum())], dtype=torch.float64)
        pose_sig = torch.tensor([float(w.poses.sum())], dtype=torch.float64)
        meshes = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        poses = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(meshes, mesh_sig)
        dist.all_gather(poses, pose_sig)
        # the timed region's reduction: max over ranks, identical on all ranks
        t = bench.max_over_ranks(1.0 + rank, dist)
        rate = bench.aggregate_rate(len(w.poses), 3, world, t)
        # each rank's shard is an independent problem: oracle per shard
        tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
        tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
        cnt, H, Z, _ = O.collide(tA, tB, w.poses, O.band_delta(w.A.vertices), nthreads=1)
        q.put((rank, [m.tolist() for m in meshes], [p.item() for p in poses], t, rate, int((cnt > 0).sum())))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_shard_and_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, p0, t0, v0, h0), (r1, m1, p1, t1, v1, h1) = res
    assert m0 == m1 and m0[0] == m0[1]          # identical meshes on both ranks
    assert p0 == p1 and p0[0] != p0[1]          # independent pose batches
    assert t0 == t1 == 2.0                      # max over ranks
    assert v0 == v1 == pytest.approx(48 * 3 * 2 / 2.0)
    assert h0 > 0 and h1 > 0


def test_single_rank_helpers():
    import bench
    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.aggregate_rate(100, 10, 4, 2.0) == 2000.0
    a = bench.rank_workload(1, 0, 16).poses
    b = bench.rank_workload(1, 1, 16).poses
    assert a.shape == b.shape and not np.array_equal(a, b)
