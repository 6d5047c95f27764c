#!/usr/bin/env python
"""Benchmark of the hot path: collide_batch over BASELINE.json's largest
config (config 5, "large planning batch": 1,048,576 poses, A = 100k-triangle
noisy sphere, B = 1,024 blobs / 4.06M triangles, 4-ary BVHs, 8-bit corrections,
64-node treelets) on N GPUs of one node.

One step = one collide_batch call over the rank's whole pose batch (all §8(a)
rows: pose setup, work acquisition, treelet fetch + decode, SAT child-pair
tests, compaction, leaf Möller tests, outputs).  Blobs and poses are resident
in HBM before the timed region; L2 is flushed (256 MiB write) between timed
steps, outside the CUDA events.  Multi-GPU: one process per GPU (torchrun),
each rank processes its own batch of the same size (weak scaling, no data-path
collective); the step time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from workloads import generators as G  # noqa: E402

METRIC = "collision queries (poses)/sec"
UNIT = "poses/s"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.3)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        # median under load: samples within the top half of observed clocks
        loaded = [x for x in sm if sm and x >= 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def rank_workload(config: int, rank: int, num_poses=None, preset: str = "random"):
    """Weak-scaling shard: every rank gets the same meshes and its own
    independent, equally sized pose batch (pose seed offset = rank)."""
    return G.make_config(config, num_poses=num_poses, pose_seed_offset=rank, preset=preset)


def max_over_ranks(seconds: float, dist=None, device=None) -> float:
    """The job's time is the slowest rank's (max all-reduce); no-op at N=1."""
    if dist is None:
        return seconds
    import torch
    t = torch.tensor([seconds], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank: int, steps: int, world: int, seconds: float) -> float:
    """Whole-job throughput: units all ranks processed / max-over-ranks time."""
    return units_per_rank * steps * world / seconds


def kernel_source_sha() -> str:
    """Hash of the kernel sources (tools/launch_totals.py stores the same hash
    with the ncu instruction counts it commits)."""
    import hashlib
    h = hashlib.sha256()
    for f in ("cbvh_device.cu", "leaf_geometry.cuh"):
        with open(os.path.join(ROOT, "paper_2012_05348_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_oracle_rate(w, n_sample: int, nthreads: int = 0, budget_s: float = 25.0, distance: bool = False):
    """The fp64 oracle (as it stands) on a bounded prefix of the workload's
    poses.  Returns the rate and the oracle's per-pose answers for that prefix
    (collide: count, H, Z; distance: d64) so the GPU's are checked against them."""
    import oracle as O
    t0 = time.time()
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
    build_s = time.time() - t0
    delta = O.band_delta(w.A.vertices)
    cores = nthreads or os.cpu_count()
    # grow the sample until ~budget_s of oracle time (bounded by n_sample)
    n, done, el = 64, 0, 0.0
    parts = []
    while True:
        P = w.poses[done:done + n]
        t = time.time()
        if distance:
            d64, _ = O.distance(tA, tB, P, nthreads)
            parts.append((d64,))
        else:
            cnt, H, Z, _ = O.collide(tA, tB, P, delta, nthreads)
            parts.append((cnt, H, Z))
        el += time.time() - t
        done += len(P)
        if el > budget_s or done >= n_sample:
            break
        n = min(n_sample - done, max(64, int(len(P) * max(1.0, (budget_s - el) / max(el, 1e-3)) * 0.5)))
    answers = tuple(np.concatenate([p[k] for p in parts]) for k in range(len(parts[0])))
    return {"value": done / el, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {done} of {len(w.poses)} poses of {w.name}, fp64 oracle with "
                      f"std::thread x {cores}; oracle BVH build {build_s:.1f} s not timed",
            "seconds": el, "poses": done, "answers": answers, "delta": delta}


def bench_parity(cpu, hit, cnt, dst, distance: bool) -> dict:
    """The GPU's answers of the timed run against the oracle's on the
    cpu_baseline sample (tests/parity.py rules: band rule for counts, 1e-5
    relative for distances)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity import check_collide, check_distance
    n = cpu["poses"]
    try:
        if distance:
            rep = check_distance(dst[:n].cpu().numpy(), cpu["answers"][0], cpu["delta"], "bench")
        else:
            _, H, Z = cpu["answers"]
            rep = check_collide(hit[:n].cpu().numpy(), cnt[:n].cpu().numpy().view(np.uint32), H, Z, "bench")
        rep["status"] = "ok"
    except AssertionError as e:
        rep = {"status": "FAIL", "error": str(e)[:300]}
    rep["poses_checked"] = n
    rep["rule"] = ("|gpu - d64| <= 1e-5 d64 (gpu <= 2 delta near contact)" if distance else
                   "H <= count <= H + Z per pose; hit exact outside the band (Z = pairs with |s| <= delta)")
    return rep


def l2_peak() -> dict | None:
    """Measured L2 read bandwidth (libcbvh_probe.so, csrc/probe_l2.cu)."""
    import ctypes as C
    path = os.path.join(ROOT, "paper_2012_05348_b200", "libcbvh_probe.so")
    if not os.path.exists(path):
        return None
    lib = C.CDLL(path)
    gbs, nb, l2 = C.c_double(0), C.c_size_t(0), C.c_size_t(0)
    msg = C.create_string_buffer(256)
    if lib.cbvh_probe_l2_read_gbs(C.byref(gbs), C.byref(nb), C.byref(l2), msg) != 0:
        return None
    return {"l2_read_gbs": gbs.value, "buffer_bytes": nb.value, "l2_bytes": l2.value,
            "source": "measured in this run: csrc/probe_l2.cu, 16-B ld.global.cg stream over an "
                      "L2-resident buffer (best of L2/8, L2/4, L2/2), CUDA events"}


CSV_COLUMNS = ("config", "workload", "mode", "poses", "branching", "bits", "treelet_nodes", "layout", "kdop_B", "seed",
               "steps", "ms_per_step", "poses_per_s", "e2e_poses_per_s", "bv_tests_per_s", "bytes_per_node_A",
               "bytes_per_node_B", "roofline_hbm_frac", "roofline_l2_frac", "roofline_issue_frac", "parity_status",
               "parity_poses", "band_pairs", "poses_with_band", "max_rel_err", "oracle_poses_per_s", "oracle_cores",
               "cpu_model", "sm_mhz")


def write_csv(path: str, line: dict, args) -> None:
    """One row per run (SURVEY §5 metrics: poses/s, BV tests/s, bytes/node,
    roofline fractions, band counts, oracle time, cores), appended to `path`."""
    import csv
    c, par, cpu = line["config"], line.get("parity") or {}, line.get("cpu_baseline") or {}
    row = {"config": args.config, "workload": c["workload"], "mode": "distance" if "proximity" in line["metric"] else "collide",
           "poses": c["poses_per_gpu"], "branching": c["branching"], "bits": c["bits"], "treelet_nodes": c["treelet_nodes"],
           "layout": c["layout"], "kdop_B": c["kdop_B"], "seed": args.seed, "steps": line["steps"],
           "ms_per_step": line["ms_per_step"], "poses_per_s": line["value"], "e2e_poses_per_s": line["e2e"]["value"],
           "bv_tests_per_s": line["bv_pair_tests_per_s"], "bytes_per_node_A": line["bytes_per_node"]["A"],
           "bytes_per_node_B": line["bytes_per_node"]["B"], "roofline_hbm_frac": line["roofline"]["frac"],
           "roofline_l2_frac": (line.get("roofline_l2") or {}).get("frac"),
           "roofline_issue_frac": (line.get("roofline_issue") or {}).get("frac"),
           "parity_status": par.get("status"), "parity_poses": par.get("poses_checked"),
           "band_pairs": par.get("band_pairs"), "poses_with_band": par.get("poses_with_band"),
           "max_rel_err": par.get("max_rel_err"), "oracle_poses_per_s": cpu.get("value"), "oracle_cores": cpu.get("cores"),
           "cpu_model": cpu.get("cpu_model"), "sm_mhz": (line.get("clocks") or {}).get("sm_mhz")}
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=CSV_COLUMNS)
        if new:
            wr.writeheader()
        wr.writerow(row)


def run_ncu(args, argv) -> int:
    """--ncu: after the plain run exited 0, the same command once more under
    ncu (a separate process; its printed numbers are not bench values) for the
    per-launch list: duration, warp / thread instructions, L2 and DRAM bytes."""
    out = args.ncu if args.ncu.endswith(".csv") else os.path.join(args.ncu, f"launches_cfg{args.config}.csv")
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    rest = [a for i, a in enumerate(argv) if a != "--ncu" and (i == 0 or argv[i - 1] != "--ncu")]
    cmd = ["ncu", "--metrics", "gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,"
           "lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "-c", "400",
           "--csv", "--log-file", out, sys.executable, os.path.abspath(__file__), *rest, "--no-cpu", "--quick"]
    return subprocess.call(cmd, stdout=subprocess.DEVNULL)


def run_reference(args):
    """--impl reference: the oracle on the host cores, same config/metric."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    w = G.make_config(args.config)
    import oracle as O
    tA = O.Tree.from_mesh(w.A.vertices, w.A.triangles)
    tB = O.Tree.from_mesh(w.B.vertices, w.B.triangles)
    delta = O.band_delta(w.A.vertices)
    per_step = args.ref_poses
    times = []
    for s in range(args.warmup + args.steps):
        lo = (s * per_step) % len(w.poses)
        P = w.poses[lo:lo + per_step]
        t = time.time()
        O.collide(tA, tB, P, delta, 0)
        dt = time.time() - t
        if s >= args.warmup:
            times.append(dt)
    T = sum(times)
    value = per_step * args.steps / T
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": w.name, "poses_per_step": per_step,
                                            "sample": "consecutive pose windows of the config-5 batch"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{per_step} poses per step x {args.steps} steps"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run(args):
    import torch
    import paper_2012_05348_b200 as M
    from paper_2012_05348_b200 import _lib as L

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    w = rank_workload(args.config, rank + args.seed, args.poses, args.preset)
    N = len(w.poses)
    if args.treelet:
        w.treelet = args.treelet
    t0 = time.time()
    if args.leaf:
        w.leaf = args.leaf
    if args.branching:
        w.branching = args.branching
    if args.bits:
        w.bits = args.bits
    A = M.build_compressed_bvh(w.A.vertices, w.A.triangles, w.branching, w.bits, w.treelet, args.leaf_a or w.leaf, args.layout,
                               align_treelets=args.align_treelets, zero_suppress=args.zero_suppress)
    B = M.build_compressed_bvh(w.B.vertices, w.B.triangles, w.branching, w.bits, w.treelet, args.leaf_b or w.leaf, args.layout,
                               kdop=args.kdop, align_treelets=args.align_treelets, zero_suppress=args.zero_suppress)
    distance = (w.mode if args.mode == "auto" else args.mode) == "distance"
    build_s = time.time() - t0
    A.to_device(dev)
    B.to_device(dev)
    poses_h = torch.from_numpy(w.poses).pin_memory()
    poses = poses_h.to(dev)
    hit = torch.empty(N, dtype=torch.uint8, device=dev)
    cnt = torch.empty(N, dtype=torch.int32, device=dev)
    dst = torch.empty(N, dtype=torch.float32, device=dev)
    ws = M.Workspace(A, B, 1 if distance else 0, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    lib = L.load()

    def step(stats=False):
        if distance:
            M.distance_batch(A, B, poses, dst, ws, stats=stats, descent=args.descent, staging=args.staging)
        else:
            M.collide_batch(A, B, poses, hit, cnt, ws, stats=stats, descent=args.descent,
                            early_exit=args.early_exit, staging=args.staging)

    # ---- first (cold) call, then warm-up (untimed by the contract; the cold
    # call's own time is reported as cold_first_call_ms)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    c0.record(stream)
    step()
    c1.record(stream)
    c1.synchronize()
    cold_ms = c0.elapsed_time(c1)
    for _ in range(max(3, args.warmup) - 1):
        step()
    M.check(ws)

    # ---- timed region: K steps, per-step CUDA events, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:  # torch creates the underlying cudaEvent_t lazily, on first record
        a.record(stream)
        b.record(stream)
    launches = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for k in range(args.steps):
            flush.fill_(k & 255)
            ev[k][0].record(stream)
            lib.cbvh_set_kernel_events(kev[k][0].cuda_event, kev[k][1].cuda_event)
            step()
            launches += M.last_launch_count()
            ev[k][1].record(stream)
        lib.cbvh_set_kernel_events(None, None)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    M.check(ws)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    T = max_over_ranks(sum(step_ms) / 1e3, dist, dev)
    value = aggregate_rate(N, args.steps, world, T)
    hits = 0 if distance else int(hit.sum().item())

    if args.quick:
        step(stats=True)
        st = M.read_stats(ws)
        if rank == 0:
            print(json.dumps({"quick": True, "value": value, "ms_per_step": 1e3 * T / args.steps,
                              "kernel_ms": statistics.mean(kern_ms), "hit_fraction": hits / N,
                              "lib": os.environ.get("CBVH_LIB", "default"),
                              "stats_kernel_ms": st["kernel_ns"] / 1e6, "stats_tail_ms": st["tail_ns"] / 1e6,
                              "dumped": st["dumped"], "launches": M.last_launch_count(),
                              "timeline_ms": [t / 1e6 for t in st["timeline_ns"]],
                              "lane_util": st["bv_tests"] / max(1, 32 * st["iterations"]),
                              "treelet_blocks": st["treelet_blocks"], "staged_reads": st["staged_reads"],
                              "nodes_decoded": st["nodes_decoded"],
                              "iterations": st["iterations"], "bv_tests": st["bv_tests"], "leaf_pairs": st["leaf_pairs"], "tri_tests": st["tri_tests"], "exact_tests": st["exact_tests"], "layout": args.layout, "kdop": args.kdop, "early_exit": args.early_exit,
                              "bytes_per_node": {"A": A.info["bytes_per_node"], "B": B.info["bytes_per_node"]},
                              "bvh_bytes": {"A": A.info["bvh_bytes"], "B": B.info["bvh_bytes"]}}), flush=True)
        return

    # ---- stats run (untimed): BV-pair tests and algorithmic bytes per launch
    step(stats=True)
    st = M.read_stats(ws)
    kern_s = statistics.mean(kern_ms) / 1e3
    alg_bytes = st["record_bytes"] + st["tri_bytes"] + N * (48 + 5)
    peaks = measured_peaks()
    achieved = alg_bytes / kern_s / 1e9
    traffic, nc = None, {}
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                nc = json.load(f).get(f"cfg{args.config}", {})
            # (the committed capture describes the kernel sources whose hash it
            # stores: after a kernel change it is not reported until re-captured)
            traffic = nc.get("dram_bytes_per_launch") if nc.get("kernel_source_sha256") == kernel_source_sha() else None
        except (OSError, ValueError):
            traffic, nc = None, {}
    # the issue ceiling the kernel actually runs into: warp
    # instructions of the committed ncu capture over the live kernel time,
    # against 148 SMs x 4 schedulers x the max SM clock
    issue = None
    winst = nc.get("warp_inst_per_launch") if not distance and args.layout == "delta" and args.kdop == 6 else None
    if winst and nc.get("kernel_source_sha256") != kernel_source_sha():
        winst = None  # the committed instruction count belongs to other kernel sources: not reported
    if winst:
        ipeak = 148 * 4 * peaks.get("sm_max_mhz", 1965.0) * 1e6
        issue = {"bound": "issue", "achieved": winst / kern_s, "peak": ipeak, "unit": "warp inst/s",
                 "frac": winst / kern_s / ipeak, "simt_efficiency": nc.get("thread_inst_per_warp_inst", 0) / 32,
                 "source": "warp instructions of all phases from profiles/ncu_traffic.json (ncu), live kernel time"}

    # ---- end-to-end through the public API with host buffers (pinned)
    hit_h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    cnt_h = torch.empty(N, dtype=torch.int32, pin_memory=True)
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        flush.fill_(k & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        poses.copy_(poses_h, non_blocking=True)
        step()
        if distance:
            cnt_h.view(torch.float32).copy_(dst, non_blocking=True)
        else:
            hit_h.copy_(hit, non_blocking=True)
            cnt_h.copy_(cnt, non_blocking=True)
        b.record(stream)
        b.synchronize()
        if k >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    E = max_over_ranks(sum(e2e_ms) / 1e3, dist, dev)

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_rate(w, n_sample=args.cpu_poses, nthreads=args.oracle_threads, budget_s=args.cpu_budget,
                              distance=distance)
        parity = bench_parity(cpu, hit, cnt, dst, distance)
    l2 = l2_peak() if rank == 0 else None

    if rank == 0:
        line = {
            "metric": ("proximity queries (poses)/sec" if distance else METRIC), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": w.name, "poses_per_gpu": N, "A_tris": w.A.num_triangles,
                       "B_tris": w.B.num_triangles, "branching": w.branching, "bits": w.bits,
                       "treelet_nodes": w.treelet, "leaf_size": w.leaf, "layout": args.layout, "kdop_B": args.kdop,
                       "descent": args.descent + (" (one side per internal pair, DESIGN R15)" if args.descent == "larger"
                                                  else " (Alg. 1 verbatim)"),
                       "early_exit": bool(args.early_exit), "preset": args.preset,
                       "align_treelets": bool(args.align_treelets), "zero_suppress": bool(args.zero_suppress),
                       "staging": args.staging,
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "parallelism": f"pose-sharded x{world} (independent batches)"},
            "bv_pair_tests_per_s": st["bv_tests"] / (statistics.median(step_ms) / 1e3),
            "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms)},
            "cold_first_call_ms": cold_ms,
            "rates_per_s": {k: st[k] / (statistics.median(step_ms) / 1e3)
                            for k in ("expansions", "leaf_pairs", "tri_tests", "exact_tests")},
            "bv_pair_tests_per_step": st["bv_tests"],
            "hit_fraction": hits / N,
            "bytes_per_node": {"A": A.info["bytes_per_node"], "B": B.info["bytes_per_node"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                         "traffic_source": (f"committed ncu capture {nc.get('source', 'profiles/ncu_traffic.json')}: "
                                            "dram__bytes_read.sum + dram__bytes_write.sum per launch"
                                            if traffic is not None else None),
                         "kernel": "traverse_kernel<%s> (all phases)" % ("distance" if distance else "collide"),
                         "kernel_ms": 1e3 * kern_s,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "peak_source": peaks["_source"] + " hbm_gbs (copy bandwidth)",
                         "limiter": ("warp-issue slots, not memory: the hierarchy and most triangle records are "
                                     "L1/L2-resident (DRAM traffic is a few % of the algorithmic bytes); see "
                                     "roofline_issue" + (" (frac %.2f)" % issue["frac"] if issue else "")
                                     + " and DESIGN.md §4.1")},
            "roofline_l2": ({"bound": "l2", "achieved": achieved, "peak": l2["l2_read_gbs"], "unit": "GB/s",
                            "frac": achieved / l2["l2_read_gbs"], "kernel": "traverse_kernel (all phases)",
                            "peak_source": l2["source"], "l2_bytes": l2["l2_bytes"],
                            "probe_buffer_bytes": l2["buffer_bytes"],
                            "note": "the same algorithmic bytes as roofline; the hierarchy and most "
                                    "triangle records are L1/L2-resident, so this is the level they are "
                                    "served from"} if l2 else None),
            "roofline_issue": issue,
            "parity": parity,
            "stats": st,
            "e2e": {"value": aggregate_rate(N, args.steps, world, E), "unit": UNIT,
                    "h2d_bytes_per_step": int(poses_h.numel() * 4),
                    "d2h_bytes_per_step": int(N * (4 if distance else 1 + 4))},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "build_s": build_s,
        }
        if cpu is not None:
            line["cpu_baseline"] = {k: v for k, v in cpu.items() if k in ("value", "unit", "cores", "kind", "sample",
                                                                          "cpu_model")}
        print(json.dumps(line), flush=True)
        if args.csv:
            write_csv(args.csv, line, args)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--poses", type=int, default=None, help="override the config's pose count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle leg")
    ap.add_argument("--quick", action="store_true", help="timed steps only (A/B comparisons)")
    ap.add_argument("--branching", type=int, default=0, help="override B (config-3 sweep)")
    ap.add_argument("--leaf", type=int, default=0, help="override the leaf size c (1..4)")
    ap.add_argument("--leaf-a", type=int, default=0, help="leaf size of the moving model A only (ablation)")
    ap.add_argument("--leaf-b", type=int, default=0, help="leaf size of the static model B only (ablation)")
    ap.add_argument("--bits", type=int, default=0, help="override b (config-3 sweep)")
    ap.add_argument("--descent", default="larger", choices=["larger", "simultaneous"])
    ap.add_argument("--preset", default="random", choices=["random", "contact", "zero"],
                    help="pose preset (configs 1, 3): 'zero' = the paper's zero-distance preset by bisection "
                         "(oracle distance in (0, 1e-3)), 'contact' = centres 2 apart")
    ap.add_argument("--early-exit", action="store_true",
                    help="hit-only collide (stop each pose at its first hit); not the headline metric")
    ap.add_argument("--mode", default="auto", choices=["auto", "collide", "distance"],
                    help="query of the timed step (auto: the config's own; others are ablations)")
    ap.add_argument("--kdop", type=int, default=6, choices=[6, 14, 18, 26],
                    help="bounding volumes of the static model B: 6 = AABB, 14/18/26-DOP (delta layout)")
    ap.add_argument("--layout", default="delta", choices=["delta", "fp16", "fp32"],
                    help="node box layout (fp16/fp32: the paper's half-vs-float ablation)")
    ap.add_argument("--align-treelets", action="store_true",
                    help="build aligned treelet blocks (staged in shared memory by default)")
    ap.add_argument("--zero-suppress", action="store_true",
                    help="integer-compressed corrections (presence masks; implies aligned treelet blocks)")
    ap.add_argument("--staging", default="auto", choices=["auto", "on", "off"],
                    help="treelet staging in shared memory (auto: when the blobs are aligned)")
    ap.add_argument("--treelet", type=int, default=0, help="override the treelet size T (nodes)")
    ap.add_argument("--seed", type=int, default=0, help="offset added to the config's pose seed (another pose batch)")
    ap.add_argument("--repeat", type=int, default=0, help="alias of --steps (timed repetitions)")
    ap.add_argument("--oracle-threads", type=int, default=0, help="host threads of the cpu_baseline oracle leg (0: all)")
    ap.add_argument("--csv", default="", help="append one CSV row of this run's metrics to this file")
    ap.add_argument("--ncu", default="", help="after the run, repeat it under ncu (separate process) and write the "
                                              "per-launch list to this .csv (or directory)")
    ap.add_argument("--cpu-poses", type=int, default=100000)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-poses", type=int, default=2048, help="poses per --impl reference step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.repeat:
        args.steps = args.repeat
    if args.impl == "reference":
        run_reference(args)
    else:
        run(args)
        if args.ncu and _env_int("WORLD_SIZE", 1) == 1:
            run_ncu(args, sys.argv[1:])


if __name__ == "__main__":
    main()
