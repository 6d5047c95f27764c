#!/usr/bin/env python
"""Generate the rotated coplanar rows of tests/golden/tri_pairs.txt.

The coplanar branch of Möller's test projects both triangles onto
the coordinate plane that drops the dominant axis of the plane normal.  The
z=0 fixtures only exercise the z-dominant branch, so each z=0 closed form
below is carried into planes whose normal is x-dominant or y-dominant:

* by an axis permutation (normal exactly +x or +y), and
* by a rotation composed of two Pythagorean-triple rotations (cos 3/5,
  sin 4/5) after scaling by 25, so every vertex is an exact small integer
  combination and the rotated triangles stay exactly coplanar in fp32 and
  fp64.  Normals: (20, -12, 9)/25 (x-dominant), (12, 20, 9)/25 (y-dominant),
  (16, -12, 15)/25 (x-dominant by a small margin).

Rotations and permutations are isometries, so intersection results carry
over unchanged and distances scale by the factor (25 for the rotated rows,
1 for the permuted ones).  The expected values are the hand-derived z=0 closed
forms; this script computes only vertex coordinates (no method arithmetic)
and calls nothing from the product or the oracle.

    python tools/make_golden_coplanar.py >> tests/golden/tri_pairs.txt
"""
from fractions import Fraction as Fr
import math

T0 = [(0, 0), (1, 0), (0, 1)]


def shift(T, dx, dy):
    return [(x + dx, y + dy) for x, y in T]


# name, U (2-D in z=0), intersect, distance (z=0 closed form), touching, why
BASE = [
    ("coincident", T0, 1, "0", 1, "identical closed triangles"),
    ("gap1", shift(T0, 2, 0), 0, "1", 0, "T0 + (2,0): nearest points (1,0) and (2,0)"),
    ("shared_vertex", [(1, 0), (2, 0), (1, 1)], 1, "0", 1, "the triangles share the vertex (1,0)"),
    ("partial_overlap", shift(T0, Fr(1, 4), Fr(1, 4)), 1, "0", 1,
     "U's vertex (1/4,1/4) lies inside T0, the rest outside"),
    ("edges_cross", [(Fr(-1, 4), Fr(1, 2)), (Fr(1, 2), Fr(-1, 4)), (Fr(3, 4), Fr(3, 4))], 1, "0", 1,
     "no vertex of either lies in the other; edges cross"),
    ("box_overlap_gap", [(1, 1), (2, Fr(1, 2)), (Fr(1, 2), 2)], 0, "sqrt(1/2)", 0,
     "AABBs overlap; U lies in x+y>=2, nearest (1/2,1/2)-(1,1): sqrt(1/2)"),
]


def Rx(c, s):
    return [[1, 0, 0], [0, c, -s], [0, s, c]]


def Ry(c, s):
    return [[c, 0, s], [0, 1, 0], [-s, 0, c]]


def Rz(c, s):
    return [[c, -s, 0], [s, c, 0], [0, 0, 1]]


def mul(A, B):
    return [[sum(A[i][k] * B[k][j] for k in range(3)) for j in range(3)] for i in range(3)]


def app(R, p):
    return [sum(R[i][k] * p[k] for k in range(3)) for i in range(3)]


c, s = Fr(3, 5), Fr(4, 5)
FRAMES = [
    # name, map (x, y) of the z=0 plane -> 3-D point, scale, normal note
    ("perm_xdom", lambda p: [Fr(0), Fr(p[0]), Fr(p[1])], 1, "plane x=0 (normal +x)"),
    ("perm_ydom", lambda p: [Fr(p[1]), Fr(0), Fr(p[0])], 1, "plane y=0 (normal +y)"),
    ("rot_xdom", lambda p, R=mul(Rx(c, s), Ry(c, s)): app(R, [25 * Fr(p[0]), 25 * Fr(p[1]), 0]), 25,
     "x 25, rotated: normal (20,-12,9)/25"),
    ("rot_ydom", lambda p, R=mul(Ry(c, s), Rx(c, -s)): app(R, [25 * Fr(p[0]), 25 * Fr(p[1]), 0]), 25,
     "x 25, rotated: normal (12,20,9)/25"),
    ("rot_xdom_close", lambda p, R=mul(Rz(c, s), Rx(c, s)): app(R, [25 * Fr(p[0]), 25 * Fr(p[1]), 0]), 25,
     "x 25, rotated: normal (16,-12,15)/25"),
]


def fmt(pts):
    out = []
    for p in pts:
        for x in p:
            assert x.denominator & (x.denominator - 1) == 0, x  # dyadic: exact in binary
            out.append(repr(float(x)))
    return " ".join(out)


def normal(P):
    a = [P[1][k] - P[0][k] for k in range(3)]
    b = [P[2][k] - P[0][k] for k in range(3)]
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def main():
    print("# Rotated coplanar closed forms (tools/make_golden_coplanar.py): the z=0 rows carried into")
    print("# planes with an x- or y-dominant normal by exact isometries; distances scale with the frame.")
    for fname, f, scale, note in FRAMES:
        for name, U, inter, dist, touch, why in BASE:
            V3 = [f(p) for p in T0]
            U3 = [f(p) for p in U]
            n = [abs(x) for x in normal(V3)]
            dom = "xyz"[n.index(max(n))]
            assert dom == fname.split("_")[1][0], (fname, n)
            assert all(x == 0 for x in [sum(normal(V3)[k] * (q[k] - V3[0][k]) for k in range(3)) for q in U3])
            d = {"0": 0.0, "1": 1.0, "sqrt(1/2)": math.sqrt(0.5)}[dist] * scale
            print(f"coplanar_{name}_{fname} | closed form (S:95-103 coplanar branch) | {fmt(V3)} | {fmt(U3)} | "
                  f"{inter} | {d!r} | {touch} | z=0 case '{why}' in {note}; {dom}-dominant normal")


if __name__ == "__main__":
    main()
