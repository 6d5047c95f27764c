"""Shared helpers for the GPU parity tests (tolerance rules of SURVEY.md §8(c)).

Collide (BASELINE.json north_star): per pose, with H = robust oracle hits
(signed separation < -delta) and Z = band pairs (|s| <= delta),
    H <= gpu_count <= H + Z,  gpu_hit = 1 if H > 0,  gpu_hit = 0 if H + Z = 0,
and gpu_hit == (gpu_count > 0).  Outside the band the count is bit-exact.

Distance: |gpu - d64| <= 1e-5 * d64, and gpu <= 2 delta when d64 <= delta.
"""
from __future__ import annotations

import numpy as np

REL_TOL_DIST = 1e-5


def check_collide(gpu_hit, gpu_count, H, Z, label=""):
    gpu_hit = np.asarray(gpu_hit).astype(np.int64)
    gpu_count = np.asarray(gpu_count).astype(np.int64)
    H, Z = np.asarray(H), np.asarray(Z)
    bad_lo = np.nonzero(gpu_count < H)[0]
    bad_hi = np.nonzero(gpu_count > H + Z)[0]
    assert len(bad_lo) == 0 and len(bad_hi) == 0, (
        f"{label}: count outside [H, H+Z] at poses {bad_lo[:5]} {bad_hi[:5]}: "
        f"gpu={gpu_count[np.r_[bad_lo[:5], bad_hi[:5]]]} H={H[np.r_[bad_lo[:5], bad_hi[:5]]]} "
        f"Z={Z[np.r_[bad_lo[:5], bad_hi[:5]]]}")
    assert np.array_equal(gpu_hit == 1, gpu_count > 0), f"{label}: hit flag != (count > 0)"
    assert np.all(gpu_hit[H > 0] == 1), f"{label}: robust hit missed"
    assert np.all(gpu_hit[(H + Z) == 0] == 0), f"{label}: spurious hit"
    return {"poses": len(H), "band_pairs": int(Z.sum()), "poses_with_band": int((Z > 0).sum()),
            "exact_poses": int((gpu_count == H).sum()), "hits": int((gpu_count > 0).sum())}


def check_distance(gpu, d64, delta, label=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    d64 = np.asarray(d64, dtype=np.float64)
    near = d64 <= delta
    far = ~near
    rel = np.abs(gpu[far] - d64[far]) / d64[far]
    worst = float(rel.max()) if far.any() else 0.0
    assert worst <= REL_TOL_DIST, f"{label}: max rel err {worst:.3e} at {np.argmax(rel)}"
    assert np.all(gpu[near] <= 2 * delta), f"{label}: near-contact distance above 2 delta"
    assert np.all(gpu >= 0)
    return {"poses": len(d64), "max_rel_err": worst, "near_contact": int(near.sum())}
