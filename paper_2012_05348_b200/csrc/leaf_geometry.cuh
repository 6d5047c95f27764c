// leaf_geometry.cuh — checkPrimitives for the device: Möller's
// triangle–triangle interval test for closed triangles and the
// exact triangle–triangle distance, templated on the scalar type
// so the distance variant can re-evaluate near-contact candidates in fp64.
#pragma once

#include <cfloat>

namespace cbvh {

template <class F>
struct TriT {
  F v[3][3];
};

__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float div_(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return a / b; }
__device__ __forceinline__ float sqrt_(float a) { return sqrtf(a); }
__device__ __forceinline__ double sqrt_(double a) { return sqrt(a); }
__device__ __forceinline__ float clamp01(float a) { return __saturatef(a); }
__device__ __forceinline__ double clamp01(double a) { return fmin(1.0, fmax(0.0, a)); }

template <class F>
__device__ __forceinline__ void vsub(const F* a, const F* b, F* r) {
  r[0] = a[0] - b[0]; r[1] = a[1] - b[1]; r[2] = a[2] - b[2];
}
template <class F>
__device__ __forceinline__ F vdot(const F* a, const F* b) {
  return fma_(a[0], b[0], fma_(a[1], b[1], a[2] * b[2]));
}
template <class F>
__device__ __forceinline__ void vcross(const F* a, const F* b, F* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}

template <class F>
__device__ __forceinline__ F orient2(const F* a, const F* b, const F* c) {
  return (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
}

// closed 2-D segment intersection (touching counts)
template <class F>
__device__ bool seg2_intersect(const F* p1, const F* p2, const F* q1, const F* q2) {
  F d1 = orient2(q1, q2, p1), d2 = orient2(q1, q2, p2);
  F d3 = orient2(p1, p2, q1), d4 = orient2(p1, p2, q2);
  if (((d1 > 0 && d2 < 0) || (d1 < 0 && d2 > 0)) && ((d3 > 0 && d4 < 0) || (d3 < 0 && d4 > 0))) return true;
  auto on = [](const F* a, const F* b, const F* c) {
    return fmin(a[0], b[0]) <= c[0] && c[0] <= fmax(a[0], b[0]) && fmin(a[1], b[1]) <= c[1] &&
           c[1] <= fmax(a[1], b[1]);
  };
  return (d1 == 0 && on(q1, q2, p1)) || (d2 == 0 && on(q1, q2, p2)) || (d3 == 0 && on(p1, p2, q1)) ||
         (d4 == 0 && on(p1, p2, q2));
}

template <class F>
__device__ bool pt_in_tri2(const F* p, const F* a, const F* b, const F* c) {
  F o1 = orient2(a, b, p), o2 = orient2(b, c, p), o3 = orient2(c, a, p);
  bool neg = (o1 < 0) || (o2 < 0) || (o3 < 0);
  bool pos = (o1 > 0) || (o2 > 0) || (o3 > 0);
  return !(neg && pos);
}

// coplanar triangles: project on the plane dropping the normal's dominant axis
template <class F>
__device__ __noinline__ bool coplanar2(const F* N, const TriT<F>& V, const TriT<F>& U) {
  F a0 = fabs(N[0]), a1 = fabs(N[1]), a2 = fabs(N[2]);
  int i0, i1;
  if (a0 >= a1 && a0 >= a2) { i0 = 1; i1 = 2; }
  else if (a1 >= a2) { i0 = 0; i1 = 2; }
  else { i0 = 0; i1 = 1; }
  F v[3][2], u[3][2];
  for (int k = 0; k < 3; ++k) {
    v[k][0] = V.v[k][i0]; v[k][1] = V.v[k][i1];
    u[k][0] = U.v[k][i0]; u[k][1] = U.v[k][i1];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (seg2_intersect(v[i], v[(i + 1) % 3], u[j], u[(j + 1) % 3])) return true;
  return pt_in_tri2(v[0], u[0], u[1], u[2]) || pt_in_tri2(u[0], v[0], v[1], v[2]);
}

// (div_ is the fast fp32 division in the float instantiation: every
// parameter it produces is clamped / tested, so a candidate is always a real
// point pair and rounding can only over-estimate a distance.)

// Möller 1997: the interval a triangle cuts on the line of the two planes,
// from the projections p[] of its vertices and their plane distances d[]
// (k = the vertex alone on its side).
#ifndef CBVH_MOLLER_SELECT
#define CBVH_MOLLER_SELECT 1  // interval case analysis as selects (measured 0.5-1 % faster on configs 5 and 3)
#endif
template <class F>
__device__ __forceinline__ bool interval(const F p[3], const F d[3], F* t0, F* t1) {
#if CBVH_MOLLER_SELECT
  // the same case analysis as below, as selects (no divergent branches)
  // (bitwise operators on the flags: no short-circuit branches)
  const bool c1 = d[0] * d[1] > 0;
  const bool c2 = !c1 & (d[0] * d[2] > 0);
  const bool c3 = !c1 & !c2 & ((d[1] * d[2] > 0) | (d[0] != 0));
  const bool c4 = !c1 & !c2 & !c3 & (d[1] != 0);
  const bool c5 = !c1 & !c2 & !c3 & !c4 & (d[2] != 0);
  const bool k2 = c1 | c5, k1 = c2 | c4;  // else k = 0 (c3)
  const F pk = k2 ? p[2] : (k1 ? p[1] : p[0]), dk = k2 ? d[2] : (k1 ? d[1] : d[0]);
  const F pi = c3 ? p[1] : p[0], di = c3 ? d[1] : d[0];
  const F pj = k2 ? p[1] : p[2], dj = k2 ? d[1] : d[2];
  const F a = pk + (pi - pk) * div_(dk, dk - di);
  const F b = pk + (pj - pk) * div_(dk, dk - dj);
  *t0 = fmin(a, b);
  *t1 = fmax(a, b);
  return c1 | c2 | c3 | c4 | c5;
#else
  int k, i, j;
  if (d[0] * d[1] > 0) { k = 2; i = 0; j = 1; }
  else if (d[0] * d[2] > 0) { k = 1; i = 0; j = 2; }
  else if (d[1] * d[2] > 0 || d[0] != 0) { k = 0; i = 1; j = 2; }
  else if (d[1] != 0) { k = 1; i = 0; j = 2; }
  else if (d[2] != 0) { k = 2; i = 0; j = 1; }
  else return false;
  F a = p[k] + (p[i] - p[k]) * div_(d[k], d[k] - d[i]);
  F b = p[k] + (p[j] - p[k]) * div_(d[k], d[k] - d[j]);
  *t0 = fmin(a, b);
  *t1 = fmax(a, b);
  return true;
#endif
}

template <class F>
__device__ F seg_seg_d2(const F* p0, const F* p1, const F* q0, const F* q1);
template <class F>
__device__ __forceinline__ F pt_seg_d2(const F* p, const F* a, const F* b);

// ---- zero-area triangles.  SPEC allows duplicate-position triangles
// and asks for segment / point fallbacks: a closed triangle whose
// normal is the zero vector is the segment between its two farthest vertices
// (a point when all coincide).  Reached only from the rare branches of
// tri_tri_overlap where a normal has come out exactly zero.
template <class F>
__device__ __forceinline__ bool is_zero3(const F* n) { return n[0] == F(0) && n[1] == F(0) && n[2] == F(0); }

template <class F>
__device__ void far_pair(const TriT<F>& T, F a[3], F b[3]) {
  F d01[3], d12[3], d20[3];
  vsub(T.v[1], T.v[0], d01); vsub(T.v[2], T.v[1], d12); vsub(T.v[0], T.v[2], d20);
  const F l01 = vdot(d01, d01), l12 = vdot(d12, d12), l20 = vdot(d20, d20);
  const int i = (l01 >= l12 && l01 >= l20) ? 0 : (l12 >= l20 ? 1 : 2);
  for (int k = 0; k < 3; ++k) { a[k] = T.v[i][k]; b[k] = T.v[(i + 1) % 3][k]; }
}

// Closed segment ab against the closed non-degenerate triangle T with normal
// n.  Off the plane: the endpoints must not lie strictly on one side, and the
// line through a, b must pass through the closed triangle — the triple
// products (b - a) . ((t_i - a) x (t_i+1 - a)) share a sign (zeros allowed).
// In the plane: 2-D edge crossings or an endpoint inside, on the coordinate
// plane that drops n's dominant axis.
template <class F>
__device__ __noinline__ bool seg_tri_closed(const F* a, const F* b, const TriT<F>& T, const F* n) {
  F wa[3], wb[3];
  vsub(a, T.v[0], wa); vsub(b, T.v[0], wb);
  const F sa = vdot(n, wa), sb = vdot(n, wb);
  if ((sa > F(0) && sb > F(0)) || (sa < F(0) && sb < F(0))) return false;
  if (sa == F(0) && sb == F(0)) {
    const F ax = fabs(n[0]), ay = fabs(n[1]), az = fabs(n[2]);
    const int j0 = (ax >= ay && ax >= az) ? 1 : 0, j1 = (az > ax && az > ay) ? 1 : 2;
    const F p[2] = {a[j0], a[j1]}, q[2] = {b[j0], b[j1]};
    F t[3][2];
    for (int k = 0; k < 3; ++k) { t[k][0] = T.v[k][j0]; t[k][1] = T.v[k][j1]; }
    for (int k = 0; k < 3; ++k)
      if (seg2_intersect(p, q, t[k], t[(k + 1) % 3])) return true;
    return pt_in_tri2(p, t[0], t[1], t[2]);
  }
  F d[3];
  vsub(b, a, d);
  bool neg = false, pos = false;
  for (int k = 0; k < 3; ++k) {
    F p[3], q[3], c[3];
    vsub(T.v[k], a, p); vsub(T.v[(k + 1) % 3], a, q); vcross(p, q, c);
    const F s = vdot(d, c);
    neg = neg || s < F(0);
    pos = pos || s > F(0);
  }
  return !(neg && pos);
}

template <class F>
__device__ __noinline__ bool degenerate_overlap(const TriT<F>& V, const TriT<F>& U) {
  F e1[3], e2[3], N1[3], N2[3], a[3], b[3];
  vsub(V.v[1], V.v[0], e1); vsub(V.v[2], V.v[0], e2); vcross(e1, e2, N1);
  vsub(U.v[1], U.v[0], e1); vsub(U.v[2], U.v[0], e2); vcross(e1, e2, N2);
  if (is_zero3(N1) && is_zero3(N2)) {
    // two segments (or points): they meet iff their distance is zero —
    // the endpoint-to-segment terms and the interior stationary point
    F c[3], d[3];
    far_pair(V, a, b);
    far_pair(U, c, d);
    const F m = fmin(fmin(fmin(pt_seg_d2(a, c, d), pt_seg_d2(b, c, d)), fmin(pt_seg_d2(c, a, b), pt_seg_d2(d, a, b))),
                     seg_seg_d2(a, b, c, d));
    return m == F(0);
  }
  if (is_zero3(N1)) {
    far_pair(V, a, b);
    return seg_tri_closed(a, b, U, N2);
  }
  far_pair(U, a, b);
  return seg_tri_closed(a, b, V, N1);
}

// Möller's test in registers.  Returns 1 / 0 for the generic case, or -1
// when the planes are coplanar or parallel-touching, or a normal is zero —
// the rare cases tri_tri_overlap settles out of line.  The projections on the
// dominant axis of the intersection line are selects, not a run-time index,
// so neither triangle is ever written to local memory on this path.
template <class F>
__device__ __forceinline__ int moller_fast(const TriT<F>& V, const TriT<F>& U) {
  F e1[3], e2[3], N1[3], N2[3];
  vsub(V.v[1], V.v[0], e1); vsub(V.v[2], V.v[0], e2); vcross(e1, e2, N1);
  F d1 = -vdot(N1, V.v[0]);
  F du[3] = {vdot(N1, U.v[0]) + d1, vdot(N1, U.v[1]) + d1, vdot(N1, U.v[2]) + d1};
  if ((du[0] > 0 && du[1] > 0 && du[2] > 0) || (du[0] < 0 && du[1] < 0 && du[2] < 0)) return 0;
  vsub(U.v[1], U.v[0], e1); vsub(U.v[2], U.v[0], e2); vcross(e1, e2, N2);
  F d2 = -vdot(N2, U.v[0]);
  F dv[3] = {vdot(N2, V.v[0]) + d2, vdot(N2, V.v[1]) + d2, vdot(N2, V.v[2]) + d2};
  if ((dv[0] > 0 && dv[1] > 0 && dv[2] > 0) || (dv[0] < 0 && dv[1] < 0 && dv[2] < 0)) return 0;
  if (du[0] == 0 && du[1] == 0 && du[2] == 0) return -1;
  F D[3];
  vcross(N1, N2, D);
  const F m0 = fabs(D[0]), m1 = fabs(D[1]), m2 = fabs(D[2]);
  const bool x1 = m1 > m0, x2 = m2 > (x1 ? m1 : m0);  // dominant axis: 2 if x2, else 1 if x1, else 0
  if ((x2 ? m2 : (x1 ? m1 : m0)) == 0) return -1;
  F vp[3], up[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    vp[k] = x2 ? V.v[k][2] : (x1 ? V.v[k][1] : V.v[k][0]);
    up[k] = x2 ? U.v[k][2] : (x1 ? U.v[k][1] : U.v[k][0]);
  }
  F a0, a1, b0, b1;
  if (!interval(vp, dv, &a0, &a1) || !interval(up, du, &b0, &b1)) return -1;
  return !(a1 < b0 || b1 < a0) ? 1 : 0;
}

// The complete test (closed triangles), as one function: the
// distance variant's (fp32 and fp64) and the collide rare path's.  The
// generic case is the same arithmetic as moller_fast; the coplanar and
// zero-area cases branch off where the plane test and the line direction
// vanish.
template <class F>
__device__ bool tri_tri_overlap(const TriT<F>& V, const TriT<F>& U) {
  F e1[3], e2[3], N1[3], N2[3];
  vsub(V.v[1], V.v[0], e1); vsub(V.v[2], V.v[0], e2); vcross(e1, e2, N1);
  F d1 = -vdot(N1, V.v[0]);
  F du[3] = {vdot(N1, U.v[0]) + d1, vdot(N1, U.v[1]) + d1, vdot(N1, U.v[2]) + d1};
  if ((du[0] > 0 && du[1] > 0 && du[2] > 0) || (du[0] < 0 && du[1] < 0 && du[2] < 0)) return false;
  vsub(U.v[1], U.v[0], e1); vsub(U.v[2], U.v[0], e2); vcross(e1, e2, N2);
  F d2 = -vdot(N2, U.v[0]);
  F dv[3] = {vdot(N2, V.v[0]) + d2, vdot(N2, V.v[1]) + d2, vdot(N2, V.v[2]) + d2};
  if ((dv[0] > 0 && dv[1] > 0 && dv[2] > 0) || (dv[0] < 0 && dv[1] < 0 && dv[2] < 0)) return false;
  // (a zero normal — a zero-area triangle — makes du or the line direction D
  // vanish, so it can only arrive in these two branches)
  if (du[0] == 0 && du[1] == 0 && du[2] == 0)
    return (is_zero3(N1) || is_zero3(N2)) ? degenerate_overlap(V, U) : coplanar2(N1, V, U);
  F D[3];
  vcross(N1, N2, D);
  int ax = 0;
  F m = fabs(D[0]);
  if (fabs(D[1]) > m) { m = fabs(D[1]); ax = 1; }
  if (fabs(D[2]) > m) { m = fabs(D[2]); ax = 2; }
  if (m == 0) return (is_zero3(N1) || is_zero3(N2)) ? degenerate_overlap(V, U) : coplanar2(N1, V, U);
  F vp[3] = {V.v[0][ax], V.v[1][ax], V.v[2][ax]};
  F up[3] = {U.v[0][ax], U.v[1][ax], U.v[2][ax]};
  F a0, a1, b0, b1;
  if (!interval(vp, dv, &a0, &a1) || !interval(up, du, &b0, &b1)) return coplanar2(N1, V, U);
  return !(a1 < b0 || b1 < a0);
}

template <class F>
__device__ __forceinline__ F pt_seg_d2(const F* p, const F* a, const F* b) {
  F ab[3], ap[3];
  vsub(b, a, ab); vsub(p, a, ap);
  F L = vdot(ab, ab);
  F t = L > 0 ? clamp01(div_(vdot(ap, ab), L)) : F(0);
  F q[3] = {fma_(t, ab[0], a[0]) - p[0], fma_(t, ab[1], a[1]) - p[1], fma_(t, ab[2], a[2]) - p[2]};
  return vdot(q, q);
}

// Segment–segment candidate: the stationary point of |p(s) - q(t)|^2 when it
// lies inside [0,1]^2, else +inf.  A boundary minimum is an endpoint against
// the other segment — a vertex–edge distance, which pt_tri_d2 already covers
// (tri_tri_dist evaluates every vertex against every edge of the other
// triangle), so only the interior candidate is needed here.  Every candidate
// is a real pair of points, so rounding can only over-estimate the minimum.
template <class F>
__device__ F seg_seg_d2(const F* p0, const F* p1, const F* q0, const F* q1) {
  F d1[3], d2[3], r[3];
  vsub(p1, p0, d1); vsub(q1, q0, d2); vsub(p0, q0, r);
  F a = vdot(d1, d1), e = vdot(d2, d2), b = vdot(d1, d2), c = vdot(d1, r), f = vdot(d2, r);
  F den = a * e - b * b;
  F best = F(FLT_MAX);
  if (den > 0) {
    const F inv = div_(F(1), den);
    F s = (b * f - c * e) * inv, t = (a * f - b * c) * inv;
    if (s >= 0 && s <= 1 && t >= 0 && t <= 1) {
      F w[3] = {r[0] + s * d1[0] - t * d2[0], r[1] + s * d1[1] - t * d2[1], r[2] + s * d1[2] - t * d2[2]};
      best = vdot(w, w);
    }
  }
  return best;
}

// point–triangle: the plane distance when the projection lies inside the
// closed triangle, else the nearest edge.  (With tri_tri_dist's interior-only
// segment terms the minimum stays exact: a closest pair of two disjoint
// triangles has a vertex of one of them, or two edge-interior points.)
template <class F>
__device__ F pt_tri_d2(const F* p, const TriT<F>& T) {
  F e1[3], e2[3], n[3], w[3];
  vsub(T.v[1], T.v[0], e1); vsub(T.v[2], T.v[0], e2); vcross(e1, e2, n);
  F nn = vdot(n, n);
  if (nn > 0) {
    vsub(p, T.v[0], w);
    F h = div_(vdot(w, n), nn);
    F q[3] = {p[0] - h * n[0], p[1] - h * n[1], p[2] - h * n[2]};
    F a[3], b[3], c0[3];
    vsub(T.v[1], T.v[0], a); vsub(q, T.v[0], b); vcross(a, b, c0);
    bool in = vdot(c0, n) >= 0;
    vsub(T.v[2], T.v[1], a); vsub(q, T.v[1], b); vcross(a, b, c0);
    in = in && vdot(c0, n) >= 0;
    vsub(T.v[0], T.v[2], a); vsub(q, T.v[2], b); vcross(a, b, c0);
    in = in && vdot(c0, n) >= 0;
    if (in) {
      F d = p[0] - q[0], e = p[1] - q[1], f = p[2] - q[2];
      return d * d + e * e + f * f;
    }
  }
  return fmin(fmin(pt_seg_d2(p, T.v[0], T.v[1]), pt_seg_d2(p, T.v[1], T.v[2])), pt_seg_d2(p, T.v[2], T.v[0]));
}

// Distance of two triangles already known not to intersect: the minimum over
// the 6 vertex-triangle and 9 edge-edge terms.
template <class F>
__device__ F tri_tri_dist_disjoint(const TriT<F>& V, const TriT<F>& U) {
  F best = F(FLT_MAX);
  #pragma unroll 1
  for (int k = 0; k < 3; ++k) {
    best = fmin(best, pt_tri_d2(V.v[k], U));
    best = fmin(best, pt_tri_d2(U.v[k], V));
  }
  #pragma unroll 1
  for (int i = 0; i < 3; ++i)
    #pragma unroll 1
    for (int j = 0; j < 3; ++j)
      best = fmin(best, seg_seg_d2(V.v[i], V.v[(i + 1) % 3], U.v[j], U.v[(j + 1) % 3]));
  return sqrt_(best);
}

template <class F>
__device__ F tri_tri_dist(const TriT<F>& V, const TriT<F>& U) {
  if (tri_tri_overlap(V, U)) return F(0);
  return tri_tri_dist_disjoint(V, U);
}

}  // namespace cbvh
