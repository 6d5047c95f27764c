"""Seeded synthetic inputs shared by the oracle tests, the CUDA path and bench.py.

This module is deliberately free of the method's arithmetic (no bounding
volumes, no traversal, no triangle tests): it only draws meshes and poses.
Both sides of every parity check consume exactly the arrays produced here.

Workload recipes follow BASELINE.json ``configs[0..4]`` (called configs 1..5
below); readings of under-specified details are
SURVEY.md §8(c) readings #14 (pose format), #18 (noise), #19 (config-4 pose
placement) and #20 (rotation distribution), restated in DESIGN.md.

Conventions
-----------
* vertices: float32 [nv, 3]; triangles: int32 [nt, 3].
* poses: float32 [N, 12], row-major [R | t] (rows (R00 R01 R02 t0), ...),
  world = R @ x_A + t; the environment B is static at identity.
* everything is computed in float64 and rounded to float32 once.
* numpy ``default_rng`` (PCG64); seed base S = 201205348, config k uses
  S + 100k + 1 (mesh A), + 2 (mesh B / blobs), + 3 (poses).

Draw order (fixed, documented so that any re-implementation reproduces it):
* noisy UV sphere: one ``uniform(-a, a)`` per vertex in vertex order.
* blob scene: per blob, in blob order: the blob's sphere noise, then its
  radius ``uniform(rmin, rmax)``, then 4 ``standard_normal`` (rotation
  quaternion), then 3 ``uniform(-L, L)`` (centre).
* random poses: ``standard_normal((N, 4))`` quaternions, then
  ``uniform(-L, L, (N, 3))`` translations.
* ring poses (config 4): quaternions ``standard_normal((N, 4))``, then
  rho ``uniform(4.5, 6, N)``, phi ``uniform(0, 2pi, N)``, u ``uniform(0,1,N)``.
"""
from __future__ import annotations

import functools
import math
import os
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 201205348


def seeds(config: int) -> tuple[int, int, int]:
    """(mesh A, mesh B, poses) seeds for config k."""
    s = SEED_BASE + 100 * config
    return s + 1, s + 2, s + 3


# --------------------------------------------------------------------------- meshes

@functools.lru_cache(maxsize=16)
def uv_sphere_topology(u: int, v: int) -> tuple[np.ndarray, np.ndarray]:
    """Unit UV sphere: returns (unit directions fp64 [nv,3], triangles int32 [nt,3]).

    u segments in azimuth, v segments pole to pole; 2 + u(v-1) vertices and
    2u(v-1) triangles (poles and seam shared, so the mesh is closed).
    """
    assert u >= 3 and v >= 2
    dirs = [(0.0, 0.0, 1.0)]
    for j in range(1, v):
        th = math.pi * j / v
        st, ct = math.sin(th), math.cos(th)
        for i in range(u):
            ph = 2.0 * math.pi * i / u
            dirs.append((st * math.cos(ph), st * math.sin(ph), ct))
    dirs.append((0.0, 0.0, -1.0))
    dirs = np.asarray(dirs, dtype=np.float64)
    south = len(dirs) - 1

    def ring(j, i):  # j in 1..v-1
        return 1 + (j - 1) * u + (i % u)

    tris = []
    for i in range(u):
        tris.append((0, ring(1, i), ring(1, i + 1)))
    for j in range(1, v - 1):
        for i in range(u):
            a, b = ring(j, i), ring(j, i + 1)
            c, d = ring(j + 1, i), ring(j + 1, i + 1)
            tris.append((a, c, d))
            tris.append((a, d, b))
    for i in range(u):
        tris.append((south, ring(v - 1, i + 1), ring(v - 1, i)))
    return dirs, np.asarray(tris, dtype=np.int32)


def noisy_sphere(rng: np.random.Generator, u: int, v: int, radius: float = 1.0,
                 noise: float = 0.05) -> tuple[np.ndarray, np.ndarray]:
    """UV sphere of the given radius, each vertex radius scaled by (1 + U(-noise, noise)).

    Returns fp64 vertices (caller rounds) and int32 triangles.
    """
    dirs, tris = uv_sphere_topology(u, v)
    f = 1.0 + rng.uniform(-noise, noise, size=len(dirs))
    return dirs * (radius * f)[:, None], tris


def noisy_torus(rng: np.random.Generator, u: int, v: int, major: float = 3.0,
                minor: float = 1.0, noise: float = 0.03) -> tuple[np.ndarray, np.ndarray]:
    """Torus in the xy-plane, u segments around the ring, v around the tube.

    Each vertex's tube radius is minor * (1 + U(-noise, noise)) (reading #18).
    u*v vertices, 2uv triangles.
    """
    f = 1.0 + rng.uniform(-noise, noise, size=u * v)
    verts = np.empty((u * v, 3), dtype=np.float64)
    k = 0
    for i in range(u):
        ph = 2.0 * math.pi * i / u
        cph, sph = math.cos(ph), math.sin(ph)
        for j in range(v):
            th = 2.0 * math.pi * j / v
            r = minor * f[k]
            rho = major + r * math.cos(th)
            verts[k] = (rho * cph, rho * sph, r * math.sin(th))
            k += 1
    tris = []
    for i in range(u):
        for j in range(v):
            a = i * v + j
            b = ((i + 1) % u) * v + j
            c = ((i + 1) % u) * v + (j + 1) % v
            d = i * v + (j + 1) % v
            tris.append((a, b, c))
            tris.append((a, c, d))
    return verts, np.asarray(tris, dtype=np.int32)


def quat_to_matrix(q: np.ndarray) -> np.ndarray:
    """Unit quaternions [...,4] (w,x,y,z; normalised here) -> rotation matrices [...,3,3], fp64."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3), dtype=np.float64)
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def blob_scene(rng: np.random.Generator, nblobs: int, u: int, v: int, rmin: float,
               rmax: float, half_width: float, noise: float = 0.05):
    """nblobs noisy spheres, radius U[rmin,rmax], random rotation, centre U[-L,L]^3."""
    vs, ts = [], []
    off = 0
    for _ in range(nblobs):
        verts, tris = noisy_sphere(rng, u, v, 1.0, noise)
        r = rng.uniform(rmin, rmax)
        R = quat_to_matrix(rng.standard_normal(4))
        c = rng.uniform(-half_width, half_width, size=3)
        vs.append((verts * r) @ R.T + c)
        ts.append(tris + off)
        off += len(verts)
    return np.concatenate(vs), np.concatenate(ts).astype(np.int32)


# --------------------------------------------------------------------------- poses

def pack_poses(R: np.ndarray, t: np.ndarray) -> np.ndarray:
    """fp64 R [N,3,3], t [N,3] -> fp32 [N,12] row-major [R|t] (rounded once)."""
    P = np.concatenate([R, t[:, :, None]], axis=2).reshape(len(R), 12)
    return np.ascontiguousarray(P.astype(np.float32))


def random_poses(rng: np.random.Generator, n: int, half_width: float) -> np.ndarray:
    """Uniform rotation (normalised 4-D Gaussian) and t ~ U[-L, L]^3."""
    q = rng.standard_normal((n, 4))
    t = rng.uniform(-half_width, half_width, size=(n, 3))
    return pack_poses(quat_to_matrix(q), t)


def contact_poses(rng: np.random.Generator, n: int, centre_distance: float) -> np.ndarray:
    """The paper's "distance of zero" preset, analytically: uniform
    rotation and t = centre_distance x a uniform unit direction, so the two
    (noisy) spheres' nominal surfaces touch — every pose is at or near contact,
    the most expensive case.  Draws: standard_normal((N, 4)) quaternions, then
    standard_normal((N, 3)) directions."""
    q = rng.standard_normal((n, 4))
    d = rng.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return pack_poses(quat_to_matrix(q), centre_distance * d)


def zero_pose_draws(k: int, n: int, pose_seed_offset: int = 0):
    """Rotations (fp64 [n,3,3]) and unit translation directions (fp64 [n,3])
    of the zero-separation preset of config k: the config's pose seed,
    standard_normal((n, 4)) quaternions, then standard_normal((n, 3))
    directions (the same draws as contact_poses).  The magnitudes come from
    the bisection table tools/make_zero_preset.py writes with the oracle."""
    rng = np.random.default_rng(seeds(k)[2] + pose_seed_offset)
    q = rng.standard_normal((n, 4))
    d = rng.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return quat_to_matrix(q), d


PRESET_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "presets")


def zero_poses(k: int, n: int | None = None) -> np.ndarray:
    """The paper's "distance of zero" preset: per
    pose a uniform rotation and direction, translated by the magnitude the
    oracle's bisection found (0 < oracle distance < 1e-3), from
    presets/zero_cfg{k}.npz (tools/make_zero_preset.py)."""
    tab = np.load(os.path.join(PRESET_DIR, f"zero_cfg{k}.npz"))
    s = tab["s"]
    n = len(s) if n is None else int(n)
    if n > len(s):
        raise ValueError(f"the zero preset of config {k} has {len(s)} poses")
    R, u = zero_pose_draws(k, len(s))
    return pack_poses(R[:n], s[:n, None] * u[:n])


def ring_poses(rng: np.random.Generator, n: int, major: float = 3.0,
               rho_lo: float = 4.5, rho_hi: float = 6.0) -> np.ndarray:
    """Config 4: A's centre at distance rho ~ U[4.5,6] from the torus ring (reading #19)."""
    q = rng.standard_normal((n, 4))
    rho = rng.uniform(rho_lo, rho_hi, size=n)
    phi = rng.uniform(0.0, 2.0 * math.pi, size=n)
    u = rng.uniform(0.0, 1.0, size=n)
    th_max = np.arccos(-major / rho)
    th = (2.0 * u - 1.0) * th_max
    rhat = np.stack([np.cos(phi), np.sin(phi), np.zeros(n)], axis=1)
    z = np.array([0.0, 0.0, 1.0])
    centre = major * rhat + rho[:, None] * (np.cos(th)[:, None] * rhat + np.sin(th)[:, None] * z)
    return pack_poses(quat_to_matrix(q), centre)


# --------------------------------------------------------------------------- configs

@dataclass
class Mesh:
    vertices: np.ndarray  # fp32 [nv,3]
    triangles: np.ndarray  # int32 [nt,3]

    @property
    def num_triangles(self) -> int:
        return int(len(self.triangles))


def _mesh(verts64: np.ndarray, tris: np.ndarray) -> Mesh:
    return Mesh(np.ascontiguousarray(verts64.astype(np.float32)),
                np.ascontiguousarray(tris.astype(np.int32)))


@dataclass
class Workload:
    name: str
    A: Mesh
    B: Mesh
    poses: np.ndarray
    branching: int
    bits: int
    treelet: int
    leaf: int = 4
    mode: str = "collide"  # or "distance"
    settings: list = field(default_factory=list)  # config 3: [(B, bits), ...]


CONFIG_NAMES = {
    1: "cfg1_tiny_collide",
    2: "cfg2_environment_collide",
    3: "cfg3_branching_precision_sweep",
    4: "cfg4_proximity_torus",
    5: "cfg5_large_planning_batch",
}
CONFIG_POSES = {1: 1024, 2: 65536, 3: 262144, 4: 131072, 5: 1048576}


def make_config(k: int, num_poses: int | None = None, pose_seed_offset: int = 0,
                preset: str = "random") -> Workload:
    """Build the seeded inputs of BASELINE.json configs[k-1].

    ``num_poses`` truncates the pose stream (the first n poses of the full draw
    are NOT identical to a smaller draw; prefixes are taken from the full draw
    order only when num_poses is None). ``pose_seed_offset`` gives each rank of
    a multi-GPU run its own independent batch (weak scaling).
    ``preset="contact"`` (configs 1 and 3: two radius-1 spheres) replaces the
    poses by the analytic near-contact preset (centres 2 apart,
    ``contact_poses``); ``preset="zero"`` by the zero-separation preset found
    by bisection with the oracle (``zero_poses``: 0 < distance < 1e-3 for
    every pose; 1,024 poses for config 1, 32,768 for config 3).
    """
    sa, sb, sp = seeds(k)
    sp += pose_seed_offset
    n = CONFIG_POSES[k] if num_poses is None else int(num_poses)
    ra, rb, rp = (np.random.default_rng(s) for s in (sa, sb, sp))
    if preset not in ("random", "contact", "zero") or (preset != "random" and k not in (1, 3)):
        raise ValueError("presets 'contact' and 'zero' are defined for configs 1 and 3 (two unit spheres)")
    if k == 1:
        A = _mesh(*noisy_sphere(ra, 32, 16))
        B = _mesh(*noisy_sphere(rb, 32, 16))
        P = (random_poses(rp, n, 2.5) if preset == "random" else contact_poses(rp, n, 2.0) if preset == "contact"
             else zero_poses(k, num_poses))
        return Workload(CONFIG_NAMES[k], A, B, P, branching=2, bits=8, treelet=32)
    if k == 2:
        A = _mesh(*noisy_sphere(ra, 64, 32))
        B = _mesh(*blob_scene(rb, 256, 64, 32, 0.5, 2.0, 20.0))
        P = random_poses(rp, n, 20.0)
        return Workload(CONFIG_NAMES[k], A, B, P, branching=4, bits=8, treelet=32)
    if k == 3:
        A = _mesh(*noisy_sphere(ra, 128, 64))
        B = _mesh(*noisy_sphere(rb, 128, 64))
        P = (random_poses(rp, n, 2.5) if preset == "random" else contact_poses(rp, n, 2.0) if preset == "contact"
             else zero_poses(k, num_poses))
        settings = [(br, bi) for br in (2, 4, 8) for bi in (4, 8, 16)]
        return Workload(CONFIG_NAMES[k], A, B, P, branching=4, bits=8, treelet=32,
                        settings=settings)
    if k == 4:
        A = _mesh(*noisy_sphere(ra, 128, 64))
        B = _mesh(*noisy_torus(rb, 512, 256))
        P = ring_poses(rp, n)
        return Workload(CONFIG_NAMES[k], A, B, P, branching=4, bits=8, treelet=32,
                        mode="distance")
    if k == 5:
        A = _mesh(*noisy_sphere(ra, 318, 159))
        B = _mesh(*blob_scene(rb, 1024, 64, 32, 0.5, 2.0, 50.0))
        P = random_poses(rp, n, 50.0)
        return Workload(CONFIG_NAMES[k], A, B, P, branching=4, bits=8, treelet=64)
    raise ValueError(f"unknown config {k}")


def tiny_pair(which: str, seed: int = 7, n_poses: int = 64, half_width: float = 2.5):
    """Tiny brute-force meshes (UV 8x4 = 48 tris, 16x8 = 224 tris) and random poses."""
    uv = {"8x4": (8, 4), "16x8": (16, 8), "32x16": (32, 16)}[which]
    rng = np.random.default_rng(seed)
    A = _mesh(*noisy_sphere(rng, *uv))
    B = _mesh(*noisy_sphere(rng, *uv))
    P = random_poses(rng, n_poses, half_width)
    return A, B, P


def identity_poses(n: int = 1) -> np.ndarray:
    P = np.zeros((n, 12), dtype=np.float32)
    P[:, 0] = P[:, 5] = P[:, 10] = 1.0
    return P
