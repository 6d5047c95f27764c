// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct fp64 CPU implementation of what the hot path
// computes.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or constant with the CUDA path under
// paper_2012_05348_b200/ (it even re-declares the blob layout from DESIGN.md §3
// on its own) and neither side includes the other.
//
// Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
//
//   * Algorithm 1 "BVHtraversal(BV a, BV b)" — the four cases, with
//     the last case read as the CROSS PRODUCT of children (reading R9).
//   * checkPrimitives — Möller's interval test for closed triangles
//     (S:95-103), fp64.
//   * separation distance variant — exact minimum
//     triangle–triangle distance with lower-bound pruning.
//   * signed separation / tolerance band (BASELINE.json north_star tolerance,
//     SURVEY.md §8(c)): s = d(T_A,T_B) if disjoint, -pen(T_A,T_B) if they
//     intersect, pen = min over the 11 Minkowski-facet axes.
//   * an independent decoder/checker of the compressed blob:
//     containment of every decoded box, child ⊆ parent, leaves partition the
//     triangles, treelets partition and are connected.
//
// Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC worked examples, brute
// force over all triangle pairs on tiny meshes, textbook edge–triangle
// reduction on random pairs, dense sampling for distances, closed forms for
// pen depth, and the blob checker's fault injection.
//
// Everything is scalar fp64 recursion; threads only split the pose batch.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace {

typedef double vec3[3];

inline void sub(const double* a, const double* b, double* r) { r[0] = a[0] - b[0]; r[1] = a[1] - b[1]; r[2] = a[2] - b[2]; }
inline double dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline void cross(const double* a, const double* b, double* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}

// ----------------------------------------------------------------------------
// Möller 1997 triangle–triangle interval test, closed triangles.
// ----------------------------------------------------------------------------

// 2-D orientation of (a, b, c): > 0 counter-clockwise.
inline double orient2(const double* a, const double* b, const double* c) {
  return (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
}

// Closed 2-D segment intersection test (touching counts).
bool segments_intersect_2d(const double* p1, const double* p2, const double* q1, const double* q2) {
  double d1 = orient2(q1, q2, p1), d2 = orient2(q1, q2, p2);
  double d3 = orient2(p1, p2, q1), d4 = orient2(p1, p2, q2);
  if (((d1 > 0 && d2 < 0) || (d1 < 0 && d2 > 0)) && ((d3 > 0 && d4 < 0) || (d3 < 0 && d4 > 0))) return true;
  auto on_seg = [](const double* a, const double* b, const double* c) {  // c on closed segment ab, given collinear
    return std::min(a[0], b[0]) <= c[0] && c[0] <= std::max(a[0], b[0]) &&
           std::min(a[1], b[1]) <= c[1] && c[1] <= std::max(a[1], b[1]);
  };
  if (d1 == 0 && on_seg(q1, q2, p1)) return true;
  if (d2 == 0 && on_seg(q1, q2, p2)) return true;
  if (d3 == 0 && on_seg(p1, p2, q1)) return true;
  if (d4 == 0 && on_seg(p1, p2, q2)) return true;
  return false;
}

// Closed point-in-triangle in 2-D.
bool point_in_tri_2d(const double* p, const double* a, const double* b, const double* c) {
  double o1 = orient2(a, b, p), o2 = orient2(b, c, p), o3 = orient2(c, a, p);
  bool has_neg = (o1 < 0) || (o2 < 0) || (o3 < 0);
  bool has_pos = (o1 > 0) || (o2 > 0) || (o3 > 0);
  return !(has_neg && has_pos);
}

// Coplanar case: project onto the coordinate plane that drops the dominant
// component of the normal N, then edge–edge and containment tests.
bool coplanar_tri_tri(const double* N, const double V[3][3], const double U[3][3]) {
  double a0 = std::fabs(N[0]), a1 = std::fabs(N[1]), a2 = std::fabs(N[2]);
  int i0, i1;
  if (a0 >= a1 && a0 >= a2) { i0 = 1; i1 = 2; }
  else if (a1 >= a2) { i0 = 0; i1 = 2; }
  else { i0 = 0; i1 = 1; }
  double v[3][2], u[3][2];
  for (int k = 0; k < 3; ++k) {
    v[k][0] = V[k][i0]; v[k][1] = V[k][i1];
    u[k][0] = U[k][i0]; u[k][1] = U[k][i1];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (segments_intersect_2d(v[i], v[(i + 1) % 3], u[j], u[(j + 1) % 3])) return true;
  if (point_in_tri_2d(v[0], u[0], u[1], u[2])) return true;
  if (point_in_tri_2d(u[0], v[0], v[1], v[2])) return true;
  return false;
}

// Interval of a triangle on the line of plane intersection, using the
// projections p[] of its vertices on the dominant axis of D and their signed
// plane distances d[].  Returns false for the fully coplanar case.
bool compute_interval(const double p[3], const double d[3], double* t0, double* t1) {
  int k, i, j;  // k = vertex alone on its side, i/j the other two
  if (d[0] * d[1] > 0) { k = 2; i = 0; j = 1; }
  else if (d[0] * d[2] > 0) { k = 1; i = 0; j = 2; }
  else if (d[1] * d[2] > 0 || d[0] != 0) { k = 0; i = 1; j = 2; }
  else if (d[1] != 0) { k = 1; i = 0; j = 2; }
  else if (d[2] != 0) { k = 2; i = 0; j = 1; }
  else return false;
  *t0 = p[k] + (p[i] - p[k]) * d[k] / (d[k] - d[i]);
  *t1 = p[k] + (p[j] - p[k]) * d[k] / (d[k] - d[j]);
  if (*t0 > *t1) std::swap(*t0, *t1);
  return true;
}

// ----------------------------------------------------------------------------
// Degenerate (zero-area) triangles.  SPEC allows duplicate-position triangles
// and requires the tests to fall back to segment / point logic.
// A closed triangle with a zero normal is the convex hull of three collinear
// points: the segment between its two farthest-apart vertices (a point when
// all three coincide).
// ----------------------------------------------------------------------------

bool is_zero(const double* v) { return v[0] == 0 && v[1] == 0 && v[2] == 0; }

void hull_segment(const double T[3][3], double a[3], double b[3]) {
  int bi = 0, bj = 1;
  double best = -1;
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j) {
      double d[3];
      sub(T[j], T[i], d);
      if (dot(d, d) > best) { best = dot(d, d); bi = i; bj = j; }
    }
  for (int k = 0; k < 3; ++k) { a[k] = T[bi][k]; b[k] = T[bj][k]; }
}

// Drop the dominant axis of the normal N: the two remaining coordinates.
void plane_axes(const double* N, int* i0, int* i1) {
  double a0 = std::fabs(N[0]), a1 = std::fabs(N[1]), a2 = std::fabs(N[2]);
  if (a0 >= a1 && a0 >= a2) { *i0 = 1; *i1 = 2; }
  else if (a1 >= a2) { *i0 = 0; *i1 = 2; }
  else { *i0 = 0; *i1 = 1; }
}

double point_segment_dist2(const double* p, const double* a, const double* b);
double segment_segment_dist2(const double* p0, const double* p1, const double* q0, const double* q1);

// Closed segment ab against a non-degenerate closed triangle U with normal N.
bool segment_triangle_intersect(const double* a, const double* b, const double U[3][3], const double* N) {
  double wa[3], wb[3];
  sub(a, U[0], wa); sub(b, U[0], wb);
  const double da = dot(N, wa), db = dot(N, wb);  // signed plane offsets (units of |N|)
  if ((da > 0 && db > 0) || (da < 0 && db < 0)) return false;
  int i0, i1;
  plane_axes(N, &i0, &i1);
  double u[3][2];
  for (int k = 0; k < 3; ++k) { u[k][0] = U[k][i0]; u[k][1] = U[k][i1]; }
  if (da == 0 && db == 0) {
    // the segment lies in U's plane: it meets U iff it crosses an edge or
    // an endpoint lies inside
    double pa[2] = {a[i0], a[i1]}, pb[2] = {b[i0], b[i1]};
    for (int j = 0; j < 3; ++j)
      if (segments_intersect_2d(pa, pb, u[j], u[(j + 1) % 3])) return true;
    return point_in_tri_2d(pa, u[0], u[1], u[2]);
  }
  // a single crossing point p = a + t (b - a), t = da / (da - db) in [0, 1]
  const double t = da / (da - db);
  double p2[2] = {a[i0] + t * (b[i0] - a[i0]), a[i1] + t * (b[i1] - a[i1])};
  return point_in_tri_2d(p2, u[0], u[1], u[2]);
}

bool tri_tri_intersect_degenerate(const double V[3][3], const double U[3][3], const double* N1, const double* N2) {
  double a[3], b[3], c[3], d[3];
  if (is_zero(N1) && is_zero(N2)) {
    // two segments (or points): closed sets meet iff their distance is zero
    hull_segment(V, a, b);
    hull_segment(U, c, d);
    return segment_segment_dist2(a, b, c, d) == 0.0;
  }
  if (is_zero(N1)) {
    hull_segment(V, a, b);
    return segment_triangle_intersect(a, b, U, N2);
  }
  hull_segment(U, a, b);
  return segment_triangle_intersect(a, b, V, N1);
}

bool tri_tri_intersect(const double V[3][3], const double U[3][3]) {
  double e1[3], e2[3], N1[3], N2[3];
  sub(V[1], V[0], e1); sub(V[2], V[0], e2); cross(e1, e2, N1);
  {
    double f1[3], f2[3];
    sub(U[1], U[0], f1); sub(U[2], U[0], f2); cross(f1, f2, N2);
    if (is_zero(N1) || is_zero(N2)) return tri_tri_intersect_degenerate(V, U, N1, N2);
  }
  double d1 = -dot(N1, V[0]);
  double du[3];
  for (int k = 0; k < 3; ++k) du[k] = dot(N1, U[k]) + d1;
  if ((du[0] > 0 && du[1] > 0 && du[2] > 0) || (du[0] < 0 && du[1] < 0 && du[2] < 0)) return false;

  sub(U[1], U[0], e1); sub(U[2], U[0], e2); cross(e1, e2, N2);
  double d2 = -dot(N2, U[0]);
  double dv[3];
  for (int k = 0; k < 3; ++k) dv[k] = dot(N2, V[k]) + d2;
  if ((dv[0] > 0 && dv[1] > 0 && dv[2] > 0) || (dv[0] < 0 && dv[1] < 0 && dv[2] < 0)) return false;

  if (du[0] == 0 && du[1] == 0 && du[2] == 0) return coplanar_tri_tri(N1, V, U);

  double D[3];
  cross(N1, N2, D);
  int ax = 0;
  double m = std::fabs(D[0]);
  if (std::fabs(D[1]) > m) { m = std::fabs(D[1]); ax = 1; }
  if (std::fabs(D[2]) > m) { m = std::fabs(D[2]); ax = 2; }
  if (m == 0) return coplanar_tri_tri(N1, V, U);  // parallel normals, planes touching
  double vp[3] = {V[0][ax], V[1][ax], V[2][ax]};
  double up[3] = {U[0][ax], U[1][ax], U[2][ax]};
  double a0, a1, b0, b1;
  if (!compute_interval(vp, dv, &a0, &a1)) return coplanar_tri_tri(N1, V, U);
  if (!compute_interval(up, du, &b0, &b1)) return coplanar_tri_tri(N1, V, U);
  return !(a1 < b0 || b1 < a0);
}

// ----------------------------------------------------------------------------
// Exact distances: point–segment, segment–segment, point–triangle.
// ----------------------------------------------------------------------------

double point_segment_dist2(const double* p, const double* a, const double* b) {
  double ab[3], ap[3];
  sub(b, a, ab); sub(p, a, ap);
  double L = dot(ab, ab);
  double t = L > 0 ? dot(ap, ab) / L : 0.0;
  t = std::min(1.0, std::max(0.0, t));
  double q[3] = {a[0] + t * ab[0] - p[0], a[1] + t * ab[1] - p[1], a[2] + t * ab[2] - p[2]};
  return dot(q, q);
}

// min over (s,t) in [0,1]^2 of |P0 + s d1 - (Q0 + t d2)|^2: the unconstrained
// stationary point if it lies inside the square, else the best of the four
// boundary edges (each a point–segment distance).
double segment_segment_dist2(const double* p0, const double* p1, const double* q0, const double* q1) {
  double best = std::min(std::min(point_segment_dist2(p0, q0, q1), point_segment_dist2(p1, q0, q1)),
                         std::min(point_segment_dist2(q0, p0, p1), point_segment_dist2(q1, p0, p1)));
  double d1[3], d2[3], r[3];
  sub(p1, p0, d1); sub(q1, q0, d2); sub(p0, q0, r);
  double a = dot(d1, d1), e = dot(d2, d2), b = dot(d1, d2), c = dot(d1, r), f = dot(d2, r);
  double den = a * e - b * b;
  if (den > 0) {
    double s = (b * f - c * e) / den;
    double t = (a * f - b * c) / den;
    if (s >= 0 && s <= 1 && t >= 0 && t <= 1) {
      double w[3] = {r[0] + s * d1[0] - t * d2[0], r[1] + s * d1[1] - t * d2[1], r[2] + s * d1[2] - t * d2[2]};
      best = std::min(best, dot(w, w));
    }
  }
  return best;
}

// Point–triangle: if the projection of p onto the plane lies inside the
// closed triangle, the plane distance; otherwise the nearest edge.
double point_triangle_dist2(const double* p, const double T[3][3]) {
  double e1[3], e2[3], n[3], w[3];
  sub(T[1], T[0], e1); sub(T[2], T[0], e2); cross(e1, e2, n);
  double nn = dot(n, n);
  double best = std::min(std::min(point_segment_dist2(p, T[0], T[1]), point_segment_dist2(p, T[1], T[2])),
                         point_segment_dist2(p, T[2], T[0]));
  if (nn > 0) {
    sub(p, T[0], w);
    double h = dot(w, n) / nn;  // signed plane offset in units of n
    double q[3] = {p[0] - h * n[0], p[1] - h * n[1], p[2] - h * n[2]};
    // barycentric sign test of q against the three edges (closed)
    double c0[3], c1[3], c2[3], a[3], b[3];
    sub(T[1], T[0], a); sub(q, T[0], b); cross(a, b, c0);
    sub(T[2], T[1], a); sub(q, T[1], b); cross(a, b, c1);
    sub(T[0], T[2], a); sub(q, T[2], b); cross(a, b, c2);
    if (dot(c0, n) >= 0 && dot(c1, n) >= 0 && dot(c2, n) >= 0) best = std::min(best, h * h * nn);
  }
  return best;
}

double tri_tri_distance(const double V[3][3], const double U[3][3]) {
  if (tri_tri_intersect(V, U)) return 0.0;
  double best = std::numeric_limits<double>::infinity();
  for (int k = 0; k < 3; ++k) {
    best = std::min(best, point_triangle_dist2(V[k], U));
    best = std::min(best, point_triangle_dist2(U[k], V));
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      best = std::min(best, segment_segment_dist2(V[i], V[(i + 1) % 3], U[j], U[(j + 1) % 3]));
  return std::sqrt(best);
}

// Penetration depth of two intersecting triangles: minimum over the facet
// normals of their Minkowski difference (n_V, n_U and the 9 edge crosses) of
// the overlap of the projections divided by the axis length.
double tri_tri_pen(const double V[3][3], const double U[3][3]) {
  double axes[11][3];
  int na = 0;
  double ev[3][3], eu[3][3];
  for (int k = 0; k < 3; ++k) { sub(V[(k + 1) % 3], V[k], ev[k]); sub(U[(k + 1) % 3], U[k], eu[k]); }
  cross(ev[0], ev[1], axes[na++]);
  cross(eu[0], eu[1], axes[na++]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) cross(ev[i], eu[j], axes[na++]);
  double best = std::numeric_limits<double>::infinity();
  for (int a = 0; a < na; ++a) {
    double L = std::sqrt(dot(axes[a], axes[a]));
    if (!(L > 0)) continue;
    double vmin = 1e300, vmax = -1e300, umin = 1e300, umax = -1e300;
    for (int k = 0; k < 3; ++k) {
      double pv = dot(axes[a], V[k]), pu = dot(axes[a], U[k]);
      vmin = std::min(vmin, pv); vmax = std::max(vmax, pv);
      umin = std::min(umin, pu); umax = std::max(umax, pu);
    }
    double ov = std::min(vmax - umin, umax - vmin) / L;
    best = std::min(best, ov);
  }
  return std::max(0.0, best);
}

double signed_separation(const double V[3][3], const double U[3][3]) {
  if (tri_tri_intersect(V, U)) return -tri_tri_pen(V, U);
  return tri_tri_distance(V, U);
}

// ----------------------------------------------------------------------------
// The oracle's own BVH: exact fp64 AABBs; either a binary
// equal-count median split built here, or the B-ary tree decoded from a blob.
// ----------------------------------------------------------------------------

struct Node {
  double lo[3], hi[3];
  std::vector<int> child;  // empty for leaves
  std::vector<int> tris;   // original triangle indices (leaves only)
};

struct Tree {
  std::vector<double> V;   // fp64 vertices [nv*3], exact lift of fp32
  std::vector<int> T;      // triangles [nt*3]
  std::vector<Node> nodes; // root = 0
};

void tri_verts(const Tree& t, int i, double out[3][3]) {
  for (int k = 0; k < 3; ++k)
    for (int a = 0; a < 3; ++a) out[k][a] = t.V[3 * t.T[3 * i + k] + a];
}

void fit_box(const Tree& t, const std::vector<int>& tris, double* lo, double* hi) {
  for (int a = 0; a < 3; ++a) { lo[a] = 1e300; hi[a] = -1e300; }
  for (int i : tris)
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) {
        double x = t.V[3 * t.T[3 * i + k] + a];
        lo[a] = std::min(lo[a], x); hi[a] = std::max(hi[a], x);
      }
}

int build_binary(Tree& t, std::vector<int> tris, int leaf_size) {
  int id = (int)t.nodes.size();
  t.nodes.emplace_back();
  fit_box(t, tris, t.nodes[id].lo, t.nodes[id].hi);
  if ((int)tris.size() <= leaf_size) { t.nodes[id].tris = tris; return id; }
  // longest axis of the centroid bounds, equal-count split, ties by index
  double clo[3] = {1e300, 1e300, 1e300}, chi[3] = {-1e300, -1e300, -1e300};
  auto centroid = [&](int i, int a) {
    return (t.V[3 * t.T[3 * i] + a] + t.V[3 * t.T[3 * i + 1] + a] + t.V[3 * t.T[3 * i + 2] + a]) / 3.0;
  };
  for (int i : tris)
    for (int a = 0; a < 3; ++a) { clo[a] = std::min(clo[a], centroid(i, a)); chi[a] = std::max(chi[a], centroid(i, a)); }
  int ax = 0;
  for (int a = 1; a < 3; ++a) if (chi[a] - clo[a] > chi[ax] - clo[ax]) ax = a;
  std::sort(tris.begin(), tris.end(), [&](int x, int y) {
    double cx = centroid(x, ax), cy = centroid(y, ax);
    return cx < cy || (cx == cy && x < y);
  });
  size_t h = tris.size() / 2;
  std::vector<int> left(tris.begin(), tris.begin() + h), right(tris.begin() + h, tris.end());
  int l = build_binary(t, left, leaf_size);
  int r = build_binary(t, right, leaf_size);
  t.nodes[id].child = {l, r};
  return id;
}

// ----------------------------------------------------------------------------
// Blob layout, re-declared here independently of the product.
// ----------------------------------------------------------------------------

struct BlobView {
  const uint8_t* p;
  size_t bytes;
  uint32_t B, bits, T, c, w, n_nodes, n_tris, n_treelets, depth, n_leaves;
  int32_t e;
  float origin[3];
  int32_t root[6];
  uint64_t off_topo, off_codes, off_treelets, off_tris, off_tri_index, total;
  uint32_t layout;  // 0 delta (lattice corrections), 1 absolute binary16, 2 absolute fp32
  uint32_t kdop;    // 6 (AABB) or 14 / 18 / 26: k/2 slab axes per node
  uint64_t off_axes;
  uint32_t flags;       // bit 0: aligned treelet blocks of T slots; bit 1: zero-suppressed codes
  uint32_t real_nodes;  // nodes of the tree; n_nodes counts slots (padding included)
  uint64_t off_blocks;  // zero-suppressed: per-block region offsets (u32, 16-byte units from off_codes)
  uint32_t nax() const { return kdop / 2; }
  bool aligned() const { return flags & 1u; }
  bool zero_suppressed() const { return flags & 2u; }
};

// Topology word of an unused (padding) slot of an aligned treelet.
constexpr uint32_t kPadSlot = 0x7FFFFFFFu;

template <class X> X rd(const uint8_t* p, size_t off) { X x; std::memcpy(&x, p + off, sizeof(X)); return x; }

bool parse_blob(const uint8_t* p, size_t bytes, BlobView* b) {
  if (bytes < 256 || std::memcmp(p, "CBVH", 4) != 0 || rd<uint32_t>(p, 4) != 5) return false;
  b->p = p; b->bytes = bytes;
  b->B = rd<uint32_t>(p, 8); b->bits = rd<uint32_t>(p, 12); b->T = rd<uint32_t>(p, 16);
  b->c = rd<uint32_t>(p, 20); b->w = rd<uint32_t>(p, 24); b->n_nodes = rd<uint32_t>(p, 28);
  b->n_tris = rd<uint32_t>(p, 32); b->n_treelets = rd<uint32_t>(p, 36); b->depth = rd<uint32_t>(p, 40);
  b->n_leaves = rd<uint32_t>(p, 44); b->e = rd<int32_t>(p, 48);
  for (int a = 0; a < 3; ++a) b->origin[a] = rd<float>(p, 52 + 4 * a);
  for (int a = 0; a < 6; ++a) b->root[a] = rd<int32_t>(p, 64 + 4 * a);
  b->off_topo = rd<uint64_t>(p, 88); b->off_codes = rd<uint64_t>(p, 96); b->off_treelets = rd<uint64_t>(p, 104);
  b->off_tris = rd<uint64_t>(p, 112); b->off_tri_index = rd<uint64_t>(p, 120); b->total = rd<uint64_t>(p, 128);
  b->layout = rd<uint32_t>(p, 136);
  b->kdop = rd<uint32_t>(p, 140);
  b->off_axes = rd<uint64_t>(p, 144);
  b->flags = rd<uint32_t>(p, 152);
  b->real_nodes = rd<uint32_t>(p, 156);
  b->off_blocks = rd<uint64_t>(p, 160);
  if (b->flags > 3u || b->real_nodes == 0 || b->real_nodes > b->n_nodes) return false;
  if (b->zero_suppressed() && (!b->aligned() || b->w < 8 || b->layout != 0 || b->kdop != 6)) return false;
  if (!b->aligned() && b->real_nodes != b->n_nodes) return false;
  if (b->aligned() && b->n_nodes % b->T != 0) return false;
  if (b->kdop != 6 && b->kdop != 14 && b->kdop != 18 && b->kdop != 26) return false;
  if (b->total != bytes) return false;
  if (b->layout == 0 && b->w != 4 && b->w != 8 && b->w != 16) return false;
  if (b->layout == 1 && b->w != 16) return false;
  if (b->layout == 2 && b->w != 32) return false;
  if (b->layout > 2) return false;
  return true;
}

// IEEE binary16 -> double, from the bit layout (1 sign, 5 exponent, 10 mantissa).
double half_to_double(uint16_t h) {
  const int e = (h >> 10) & 31, m = h & 1023;
  double v;
  if (e == 0) v = std::ldexp((double)m, -24);
  else if (e == 31) v = m ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
  else v = std::ldexp((double)(m + 1024), e - 25);
  return (h & 0x8000) ? -v : v;
}

// Absolute box of node n in the FP16 / FP32 layouts (lo xyz, hi xyz).
void abs_box(const BlobView& b, uint32_t n, double* lo, double* hi) {
  for (int a = 0; a < 3; ++a) {
    if (b.layout == 2) {
      lo[a] = (double)rd<float>(b.p, b.off_codes + 24ull * n + 4 * a);
      hi[a] = (double)rd<float>(b.p, b.off_codes + 24ull * n + 12 + 4 * a);
    } else {
      lo[a] = half_to_double(rd<uint16_t>(b.p, b.off_codes + 12ull * n + 2 * a));
      hi[a] = half_to_double(rd<uint16_t>(b.p, b.off_codes + 12ull * n + 6 + 2 * a));
    }
  }
}

uint32_t blob_topo(const BlobView& b, uint32_t n) { return rd<uint32_t>(b.p, b.off_topo + 4ull * n); }

// The six stored corrections of node n: order lo_x, lo_y, lo_z, hi_x, hi_y, hi_z.
// Stored field f of node n (fields: lo of the k/2 axes, then hi of the k/2
// axes; axes 0-2 are x, y, z): w-bit unsigned, little-endian, 4-bit fields
// packed two per byte (low nibble first).
uint32_t code_field(const BlobView& b, uint32_t n, uint32_t f) {
  if (b.zero_suppressed()) {
    // block n / T holds, from off_codes + 16 * table[block]: T presence masks
    // (bit f set = field f stored), then the stored fields of its nodes in
    // node order, w/8 bytes each, little-endian; absent fields are zero
    const uint32_t blk = n / b.T, j = n % b.T;
    const uint64_t region = b.off_codes + 16ull * rd<uint32_t>(b.p, b.off_blocks + 4ull * blk);
    const uint32_t m = b.p[region + j];
    if (!((m >> f) & 1u)) return 0;
    uint64_t k = 0;  // fields stored before this one
    for (uint32_t i = 0; i < j; ++i)
      for (int g = 0; g < 6; ++g) k += (b.p[region + i] >> g) & 1u;
    for (uint32_t g = 0; g < f; ++g) k += (m >> g) & 1u;
    const uint64_t at = region + b.T + k * (b.w / 8);
    return b.w == 16 ? (uint32_t)rd<uint16_t>(b.p, at) : (uint32_t)b.p[at];
  }
  const uint64_t base = b.off_codes + (uint64_t)n * (2ull * b.nax() * b.w / 8);
  if (b.w == 16) return rd<uint16_t>(b.p, base + 2 * f);
  if (b.w == 8) return b.p[base + f];
  return (b.p[base + f / 2] >> (4 * (f % 2))) & 15u;
}

// The box corrections of node n: lo_x, lo_y, lo_z, hi_x, hi_y, hi_z.
void blob_codes(const BlobView& b, uint32_t n, uint32_t q[6]) {
  for (int a = 0; a < 3; ++a) {
    q[a] = code_field(b, n, a);
    q[3 + a] = code_field(b, n, b.nax() + a);
  }
}

int bitlen(int64_t x) { int n = 0; while (x > 0) { ++n; x >>= 1; } return n; }

// Predictor-corrector decode ("delta to the parent nodes"):
// step 2^s with s = max(0, bitlen(E) - b), lo moves up, hi moves down.
void decode_child(const int64_t P[6], const uint32_t q[6], int bits, int64_t C[6]) {
  for (int a = 0; a < 3; ++a) {
    int64_t E = P[3 + a] - P[a];
    int s = std::max(0, bitlen(E) - bits);
    C[a] = P[a] + ((int64_t)q[a] << s);
    C[3 + a] = P[3 + a] - ((int64_t)q[3 + a] << s);
  }
}

// Lattice -> fp64: origin + k * 2^e, exact in fp64 for these magnitudes.
double lat(const BlobView& b, int a, int64_t k) { return (double)b.origin[a] + std::ldexp((double)k, b.e); }

// Build an oracle Tree from a blob; boxes are the DECODED boxes unless
// exact_boxes, in which case they are refit from the mesh (same topology) —
// used for the cost-monotonicity and compression-invariance pins.
bool tree_from_blob(const BlobView& b, Tree& t, bool exact_boxes) {
  t.nodes.assign(b.n_nodes, Node());
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(b.p + b.off_tri_index);
  std::vector<int64_t> box(6ull * b.n_nodes);
  std::vector<uint32_t> stack = {0}, order;
  std::vector<char> seen(b.n_nodes, 0);
  uint32_t q[6];
  blob_codes(b, 0, q);
  int64_t R[6];
  for (int a = 0; a < 6; ++a) R[a] = b.root[a];
  decode_child(R, q, b.bits, &box[0]);
  while (!stack.empty()) {
    uint32_t n = stack.back(); stack.pop_back();
    if (n >= b.n_nodes || seen[n]) return false;
    seen[n] = 1;
    order.push_back(n);
    Node& nd = t.nodes[n];
    if (b.layout == 0) {
      for (int a = 0; a < 3; ++a) { nd.lo[a] = lat(b, a, box[6ull * n + a]); nd.hi[a] = lat(b, a, box[6ull * n + 3 + a]); }
    } else {
      abs_box(b, n, nd.lo, nd.hi);
    }
    uint32_t tp = blob_topo(b, n);
    if (tp >> 31) {
      uint32_t first = tp & 0x1FFFFFFFu, cnt = ((tp >> 29) & 3u) + 1;
      for (uint32_t k = 0; k < cnt; ++k) {
        if (first + k >= b.n_tris) return false;
        nd.tris.push_back((int)idx[first + k]);
      }
    } else {
      uint32_t first = tp & 0x0FFFFFFFu, cnt = ((tp >> 28) & 7u) + 1;
      for (uint32_t k = 0; k < cnt; ++k) {
        uint32_t ch = first + k;
        if (ch >= b.n_nodes) return false;
        nd.child.push_back((int)ch);
        blob_codes(b, ch, q);
        decode_child(&box[6ull * n], q, b.bits, &box[6ull * ch]);
        stack.push_back(ch);
      }
    }
  }
  if (exact_boxes) {
    // refit bottom-up from the triangles (reverse DFS preorder: children first)
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      Node& nd = t.nodes[*it];
      if (nd.child.empty()) fit_box(t, nd.tris, nd.lo, nd.hi);
      else {
        for (int a = 0; a < 3; ++a) { nd.lo[a] = 1e300; nd.hi[a] = -1e300; }
        for (int ch : nd.child)
          for (int a = 0; a < 3; ++a) {
            nd.lo[a] = std::min(nd.lo[a], t.nodes[ch].lo[a]);
            nd.hi[a] = std::max(nd.hi[a], t.nodes[ch].hi[a]);
          }
      }
    }
  }
  return true;
}

// ----------------------------------------------------------------------------
// Traversal (Alg. 1) under a pose: world = R x_A + t, B at identity.
// ----------------------------------------------------------------------------

struct Pose { double R[3][3], t[3]; };

Pose load_pose(const float* p) {
  Pose P;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) P.R[r][c] = (double)p[4 * r + c];
    P.t[r] = (double)p[4 * r + 3];
  }
  return P;
}

void apply(const Pose& P, const double* x, double* w) {
  for (int r = 0; r < 3; ++r) w[r] = P.R[r][0] * x[0] + P.R[r][1] * x[1] + P.R[r][2] * x[2] + P.t[r];
}

// Conservative rebound of A's box into the world: the AABB of the
// 8 transformed corners.
void rebound(const Pose& P, const double* lo, const double* hi, double* wlo, double* whi) {
  for (int a = 0; a < 3; ++a) { wlo[a] = 1e300; whi[a] = -1e300; }
  for (int c = 0; c < 8; ++c) {
    double x[3] = {(c & 1) ? hi[0] : lo[0], (c & 2) ? hi[1] : lo[1], (c & 4) ? hi[2] : lo[2]}, w[3];
    apply(P, x, w);
    for (int a = 0; a < 3; ++a) { wlo[a] = std::min(wlo[a], w[a]); whi[a] = std::max(whi[a], w[a]); }
  }
}

struct CollideOut { int64_t count = 0, H = 0, Z = 0, bv_tests = 0, leaf_pairs = 0; };

struct Ctx {
  const Tree* A; const Tree* B; Pose P; double delta;
  CollideOut out;
  std::vector<int64_t>* pairs;  // optional: (i, j) of every fp64 Möller hit
};

bool boxes_overlap(const Ctx& c, int a, int b) {
  const Node& na = c.A->nodes[a];
  const Node& nb = c.B->nodes[b];
  double wlo[3], whi[3];
  rebound(c.P, na.lo, na.hi, wlo, whi);
  for (int k = 0; k < 3; ++k)
    if (whi[k] + c.delta < nb.lo[k] - c.delta || nb.hi[k] + c.delta < wlo[k] - c.delta) return false;
  return true;
}

// checkPrimitives plus the band classification of each pair.
void check_primitives(Ctx& c, int a, int b) {
  ++c.out.leaf_pairs;
  for (int i : c.A->nodes[a].tris) {
    double Vl[3][3], V[3][3];
    tri_verts(*c.A, i, Vl);
    for (int k = 0; k < 3; ++k) apply(c.P, Vl[k], V[k]);
    double vlo[3], vhi[3];
    for (int ax = 0; ax < 3; ++ax) {
      vlo[ax] = std::min(V[0][ax], std::min(V[1][ax], V[2][ax]));
      vhi[ax] = std::max(V[0][ax], std::max(V[1][ax], V[2][ax]));
    }
    for (int j : c.B->nodes[b].tris) {
      double U[3][3];
      tri_verts(*c.B, j, U);
      bool hit = tri_tri_intersect(V, U);
      double s;
      if (hit) {
        ++c.out.count;
        if (c.pairs) { c.pairs->push_back(i); c.pairs->push_back(j); }
        s = -tri_tri_pen(V, U);
      } else {
        double gap2 = 0;
        for (int ax = 0; ax < 3; ++ax) {
          double ulo = std::min(U[0][ax], std::min(U[1][ax], U[2][ax]));
          double uhi = std::max(U[0][ax], std::max(U[1][ax], U[2][ax]));
          double g = std::max(0.0, std::max(ulo - vhi[ax], vlo[ax] - uhi));
          gap2 += g * g;
        }
        s = (std::sqrt(gap2) <= c.delta) ? tri_tri_distance(V, U) : 2 * c.delta + 1;
      }
      if (s < -c.delta) ++c.out.H;
      else if (s <= c.delta) ++c.out.Z;
    }
  }
}

// Algorithm 1, verbatim structure; the last case takes all pairs (a_i, b_j).
void bvh_traversal(Ctx& c, int a, int b) {
  const Node& na = c.A->nodes[a];
  const Node& nb = c.B->nodes[b];
  bool la = na.child.empty(), lb = nb.child.empty();
  if (la && lb) {
    check_primitives(c, a, b);
  } else if (la) {
    for (int bi : nb.child) { ++c.out.bv_tests; if (boxes_overlap(c, a, bi)) bvh_traversal(c, a, bi); }
  } else if (lb) {
    for (int ai : na.child) { ++c.out.bv_tests; if (boxes_overlap(c, ai, b)) bvh_traversal(c, ai, b); }
  } else {
    for (int ai : na.child)
      for (int bj : nb.child) { ++c.out.bv_tests; if (boxes_overlap(c, ai, bj)) bvh_traversal(c, ai, bj); }
  }
}

CollideOut collide_one(const Tree& A, const Tree& B, const float* pose, double delta, std::vector<int64_t>* pairs) {
  Ctx c{&A, &B, load_pose(pose), delta, CollideOut(), pairs};
  ++c.out.bv_tests;
  if (boxes_overlap(c, 0, 0)) bvh_traversal(c, 0, 0);
  return c.out;
}

// Distance variant: same descent, prune a pair whose box–box distance (rebound
// A box vs B box) is >= the best distance found so far; nearest pairs first.
struct DCtx { const Tree* A; const Tree* B; Pose P; double best; int64_t bv_tests; };

double box_dist(const DCtx& c, int a, int b) {
  const Node& na = c.A->nodes[a];
  const Node& nb = c.B->nodes[b];
  double wlo[3], whi[3];
  rebound(c.P, na.lo, na.hi, wlo, whi);
  double g2 = 0;
  for (int k = 0; k < 3; ++k) {
    double g = std::max(0.0, std::max(nb.lo[k] - whi[k], wlo[k] - nb.hi[k]));
    g2 += g * g;
  }
  return std::sqrt(g2);
}

void dist_traversal(DCtx& c, int a, int b) {
  const Node& na = c.A->nodes[a];
  const Node& nb = c.B->nodes[b];
  bool la = na.child.empty(), lb = nb.child.empty();
  if (la && lb) {
    for (int i : na.tris) {
      double Vl[3][3], V[3][3];
      tri_verts(*c.A, i, Vl);
      for (int k = 0; k < 3; ++k) apply(c.P, Vl[k], V[k]);
      for (int j : nb.tris) {
        double U[3][3];
        tri_verts(*c.B, j, U);
        c.best = std::min(c.best, tri_tri_distance(V, U));
      }
    }
    return;
  }
  std::vector<std::pair<double, std::pair<int, int>>> cand;
  std::vector<int> as = la ? std::vector<int>{a} : na.child;
  std::vector<int> bs = lb ? std::vector<int>{b} : nb.child;
  for (int ai : as)
    for (int bj : bs) { ++c.bv_tests; cand.push_back({box_dist(c, ai, bj), {ai, bj}}); }
  std::sort(cand.begin(), cand.end());
  for (auto& x : cand) {
    if (x.first >= c.best) break;
    dist_traversal(c, x.second.first, x.second.second);
  }
}

double distance_one(const Tree& A, const Tree& B, const float* pose, int64_t* bv_tests) {
  DCtx c{&A, &B, load_pose(pose), std::numeric_limits<double>::infinity(), 0};
  dist_traversal(c, 0, 0);
  if (bv_tests) *bv_tests = c.bv_tests;
  return c.best;
}

template <class F> void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  // chunks of up to 64 poses, smaller for short batches so all threads get work
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(64, n / (8 * (int64_t)nthreads)));
  std::atomic<int64_t> next(0);
  auto work = [&]() {
    for (;;) {
      int64_t s = next.fetch_add(chunk);
      if (s >= n) return;
      for (int64_t i = s; i < std::min(n, s + chunk); ++i) f(i);
    }
  };
  if (nthreads == 1) { work(); return; }
  std::vector<std::thread> th;
  for (int k = 0; k < nthreads; ++k) th.emplace_back(work);
  for (auto& t : th) t.join();
}

Tree* make_tree_mesh(const float* verts, int64_t nv, const int32_t* tris, int64_t nt) {
  Tree* t = new Tree();
  t->V.assign(verts, verts + 3 * nv);
  t->T.assign(tris, tris + 3 * nt);
  return t;
}

}  // namespace

// ============================================================================
// C ABI used by tests/ and bench.py (ctypes).
// ============================================================================
extern "C" {

int oracle_tri_tri_intersect(const double* V, const double* U) {
  double a[3][3], b[3][3];
  std::memcpy(a, V, sizeof a); std::memcpy(b, U, sizeof b);
  return tri_tri_intersect(a, b) ? 1 : 0;
}
double oracle_tri_tri_distance(const double* V, const double* U) {
  double a[3][3], b[3][3];
  std::memcpy(a, V, sizeof a); std::memcpy(b, U, sizeof b);
  return tri_tri_distance(a, b);
}
double oracle_tri_tri_pen(const double* V, const double* U) {
  double a[3][3], b[3][3];
  std::memcpy(a, V, sizeof a); std::memcpy(b, U, sizeof b);
  return tri_tri_pen(a, b);
}
double oracle_signed_separation(const double* V, const double* U) {
  double a[3][3], b[3][3];
  std::memcpy(a, V, sizeof a); std::memcpy(b, U, sizeof b);
  return signed_separation(a, b);
}
double oracle_point_triangle_distance(const double* p, const double* T) {
  double t[3][3];
  std::memcpy(t, T, sizeof t);
  return std::sqrt(point_triangle_dist2(p, t));
}
double oracle_segment_segment_distance(const double* p0, const double* p1, const double* q0, const double* q1) {
  return std::sqrt(segment_segment_dist2(p0, p1, q0, q1));
}

// Oracle's own binary median-split BVH (leaf_size triangles per leaf).
void* oracle_tree_from_mesh(const float* verts, int64_t nv, const int32_t* tris, int64_t nt, int leaf_size) {
  Tree* t = make_tree_mesh(verts, nv, tris, nt);
  std::vector<int> all(nt);
  for (int64_t i = 0; i < nt; ++i) all[i] = (int)i;
  build_binary(*t, all, leaf_size);
  return t;
}

// Tree with the topology of a blob; decoded boxes (exact_boxes = 0) or boxes
// refit from the mesh (exact_boxes = 1).  Returns null on a malformed blob.
void* oracle_tree_from_blob(const uint8_t* blob, uint64_t bytes, const float* verts, int64_t nv,
                            const int32_t* tris, int64_t nt, int exact_boxes) {
  BlobView b;
  if (!parse_blob(blob, bytes, &b)) return nullptr;
  Tree* t = make_tree_mesh(verts, nv, tris, nt);
  if (!tree_from_blob(b, *t, exact_boxes != 0)) { delete t; return nullptr; }
  return t;
}

void oracle_tree_free(void* t) { delete static_cast<Tree*>(t); }
int64_t oracle_tree_num_nodes(void* t) { return (int64_t) static_cast<Tree*>(t)->nodes.size(); }

// Per-pose collide: fp64 Möller count, robust hits H (s < -delta) and band Z
// (|s| <= delta).  stats (nullable) receives [bv_tests, leaf_pairs] summed.
int oracle_collide(void* ta, void* tb, const float* poses, int64_t N, double delta, int nthreads,
                   int64_t* count, int64_t* H, int64_t* Z, int64_t* stats) {
  const Tree& A = *static_cast<Tree*>(ta);
  const Tree& B = *static_cast<Tree*>(tb);
  std::atomic<int64_t> bv(0), lp(0);
  parallel_for(N, nthreads, [&](int64_t i) {
    CollideOut o = collide_one(A, B, poses + 12 * i, delta, nullptr);
    count[i] = o.count; H[i] = o.H; Z[i] = o.Z;
    bv += o.bv_tests; lp += o.leaf_pairs;
  });
  if (stats) { stats[0] = bv.load(); stats[1] = lp.load(); }
  return 0;
}

// The (i, j) pairs (original triangle indices) of one pose; returns the
// number of pairs, writes at most cap of them.
int64_t oracle_collide_pairs(void* ta, void* tb, const float* pose, double delta, int64_t* pairs, int64_t cap) {
  std::vector<int64_t> v;
  collide_one(*static_cast<Tree*>(ta), *static_cast<Tree*>(tb), pose, delta, &v);
  int64_t n = (int64_t)v.size() / 2;
  for (int64_t k = 0; k < std::min(n, cap); ++k) { pairs[2 * k] = v[2 * k]; pairs[2 * k + 1] = v[2 * k + 1]; }
  return n;
}

int oracle_distance(void* ta, void* tb, const float* poses, int64_t N, int nthreads, double* dist, int64_t* stats) {
  const Tree& A = *static_cast<Tree*>(ta);
  const Tree& B = *static_cast<Tree*>(tb);
  std::atomic<int64_t> bv(0);
  parallel_for(N, nthreads, [&](int64_t i) {
    int64_t t = 0;
    dist[i] = distance_one(A, B, poses + 12 * i, &t);
    bv += t;
  });
  if (stats) stats[0] = bv.load();
  return 0;
}

// Brute force over all triangle pairs (no hierarchy at all).
int oracle_bruteforce_collide(void* ta, void* tb, const float* poses, int64_t N, double delta, int nthreads,
                              int64_t* count, int64_t* H, int64_t* Z) {
  const Tree& A = *static_cast<Tree*>(ta);
  const Tree& B = *static_cast<Tree*>(tb);
  int64_t na = (int64_t)A.T.size() / 3, nb = (int64_t)B.T.size() / 3;
  parallel_for(N, nthreads, [&](int64_t p) {
    Pose P = load_pose(poses + 12 * p);
    int64_t c = 0, h = 0, z = 0;
    for (int64_t i = 0; i < na; ++i) {
      double Vl[3][3], V[3][3];
      tri_verts(A, (int)i, Vl);
      for (int k = 0; k < 3; ++k) apply(P, Vl[k], V[k]);
      for (int64_t j = 0; j < nb; ++j) {
        double U[3][3];
        tri_verts(B, (int)j, U);
        double s = signed_separation(V, U);
        if (tri_tri_intersect(V, U)) ++c;
        if (s < -delta) ++h; else if (s <= delta) ++z;
      }
    }
    count[p] = c; H[p] = h; Z[p] = z;
  });
  return 0;
}

int64_t oracle_bruteforce_pairs(void* ta, void* tb, const float* pose, int64_t* pairs, int64_t cap) {
  const Tree& A = *static_cast<Tree*>(ta);
  const Tree& B = *static_cast<Tree*>(tb);
  Pose P = load_pose(pose);
  int64_t na = (int64_t)A.T.size() / 3, nb = (int64_t)B.T.size() / 3, n = 0;
  for (int64_t i = 0; i < na; ++i) {
    double Vl[3][3], V[3][3];
    tri_verts(A, (int)i, Vl);
    for (int k = 0; k < 3; ++k) apply(P, Vl[k], V[k]);
    for (int64_t j = 0; j < nb; ++j) {
      double U[3][3];
      tri_verts(B, (int)j, U);
      if (tri_tri_intersect(V, U)) {
        if (n < cap) { pairs[2 * n] = i; pairs[2 * n + 1] = j; }
        ++n;
      }
    }
  }
  return n;
}

int oracle_bruteforce_distance(void* ta, void* tb, const float* poses, int64_t N, int nthreads, double* dist) {
  const Tree& A = *static_cast<Tree*>(ta);
  const Tree& B = *static_cast<Tree*>(tb);
  int64_t na = (int64_t)A.T.size() / 3, nb = (int64_t)B.T.size() / 3;
  parallel_for(N, nthreads, [&](int64_t p) {
    Pose P = load_pose(poses + 12 * p);
    double best = std::numeric_limits<double>::infinity();
    for (int64_t i = 0; i < na; ++i) {
      double Vl[3][3], V[3][3];
      tri_verts(A, (int)i, Vl);
      for (int k = 0; k < 3; ++k) apply(P, Vl[k], V[k]);
      for (int64_t j = 0; j < nb; ++j) {
        double U[3][3];
        tri_verts(B, (int)j, U);
        best = std::min(best, tri_tri_distance(V, U));
      }
    }
    dist[p] = best;
  });
  return 0;
}

// Independent blob checker.  report[] receives counts of
// violations: [0] malformed/unreachable, [1] containment (a triangle vertex
// outside its decoded node box), [2] child ⊄ parent, [3] triangle partition
// (missing/duplicate), [4] triangle soup != mesh, [5] treelet partition,
// [6] treelet size > T, [7] treelet not connected / bad anchor, [8] arity,
// [9] number of nodes checked.  Returns the total number of violations.
int64_t oracle_check_blob(const uint8_t* blob, uint64_t bytes, const float* verts, int64_t nv,
                          const int32_t* tris, int64_t nt, int64_t* report) {
  for (int k = 0; k < 10; ++k) report[k] = 0;
  BlobView b;
  if (!parse_blob(blob, bytes, &b)) { report[0] = 1; return 1; }
  if ((int64_t)b.n_tris != nt) { report[3]++; }
  // decode every box by walking down from the root
  std::vector<int64_t> box(6ull * b.n_nodes, 0);
  std::vector<int> parent(b.n_nodes, -1);
  std::vector<char> seen(b.n_nodes, 0);
  std::vector<int> tri_seen(nt, 0);
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(b.p + b.off_tri_index);
  const float* soup = reinterpret_cast<const float*>(b.p + b.off_tris);
  uint32_t q[6];
  int64_t R[6];
  for (int a = 0; a < 6; ++a) R[a] = b.root[a];
  blob_codes(b, 0, q);
  decode_child(R, q, b.bits, &box[0]);
  // children are pushed after their parent was decoded, so a DFS works
  std::vector<uint32_t> stack = {0};
  std::vector<std::vector<uint32_t>> subtree_tris(b.n_nodes);
  std::vector<uint32_t> order;
  while (!stack.empty()) {
    uint32_t n = stack.back(); stack.pop_back();
    if (n >= b.n_nodes || seen[n]) { report[0]++; continue; }
    seen[n] = 1;
    order.push_back(n);
    report[9]++;
    uint32_t tp = blob_topo(b, n);
    const int64_t* Pn = &box[6ull * n];
    if (tp >> 31) {
      uint32_t first = tp & 0x1FFFFFFFu, cnt = ((tp >> 29) & 3u) + 1;
      if (cnt > b.c) report[8]++;
      for (uint32_t k = 0; k < cnt; ++k) {
        uint32_t s = first + k;
        if (s >= b.n_tris) { report[0]++; continue; }
        uint32_t ti = idx[s];
        if ((int64_t)ti >= nt) { report[3]++; continue; }
        tri_seen[ti]++;
        // soup must equal the mesh triangle, vertex by vertex
        for (int v = 0; v < 3; ++v)
          for (int a = 0; a < 3; ++a)
            if (soup[12ull * s + 3 * v + a] != verts[3 * tris[3 * ti + v] + a]) report[4]++;
        subtree_tris[n].push_back(ti);
      }
      // leaf slab: record 0's pad = normal n, record 1's pad =
      // (dmin, dmax); every vertex v of the leaf satisfies dmin <= n.v <= dmax
      // (exactly, in fp64); other pads are zero
      if (first < b.n_tris) {
        double nn[3] = {(double)soup[12ull * first + 9], (double)soup[12ull * first + 10], (double)soup[12ull * first + 11]};
        double lo = -INFINITY, hi = INFINITY;
        if (cnt > 1) { lo = (double)soup[12ull * (first + 1) + 9]; hi = (double)soup[12ull * (first + 1) + 10]; }
        if (std::fabs(std::sqrt(dot(nn, nn)) - 1.0) > 1e-6) report[4]++;
        for (uint32_t k = 0; k < cnt && first + k < b.n_tris; ++k) {
          for (int v = 0; v < 3; ++v) {
            double x[3] = {(double)soup[12ull * (first + k) + 3 * v], (double)soup[12ull * (first + k) + 3 * v + 1],
                           (double)soup[12ull * (first + k) + 3 * v + 2]};
            double d = dot(nn, x);
            if (cnt > 1 && (d < lo || d > hi)) report[1]++;
          }
          if (k >= 2 && (soup[12ull * (first + k) + 9] != 0.0f || soup[12ull * (first + k) + 10] != 0.0f ||
                         soup[12ull * (first + k) + 11] != 0.0f)) report[4]++;
          if (k == 1 && soup[12ull * (first + k) + 11] != 0.0f) report[4]++;
        }
      }
    } else {
      uint32_t first = tp & 0x0FFFFFFFu, cnt = ((tp >> 28) & 7u) + 1;
      if (cnt < 2 || cnt > b.B) report[8]++;
      for (uint32_t k = 0; k < cnt; ++k) {
        uint32_t ch = first + k;
        if (ch >= b.n_nodes) { report[0]++; continue; }
        if (parent[ch] != -1) { report[0]++; continue; }
        parent[ch] = (int)n;
        if (b.layout == 0) {
          blob_codes(b, ch, q);
          for (int f = 0; f < 6; ++f) if (q[f] >> b.bits) report[0]++;
          decode_child(Pn, q, b.bits, &box[6ull * ch]);
          const int64_t* C = &box[6ull * ch];
          for (int a = 0; a < 3; ++a)
            if (C[a] < Pn[a] || C[3 + a] > Pn[3 + a] || C[a] > C[3 + a]) report[2]++;
        } else {
          double plo[3], phi[3], clo[3], chi[3];
          abs_box(b, n, plo, phi);
          abs_box(b, ch, clo, chi);
          for (int a = 0; a < 3; ++a)
            if (clo[a] < plo[a] || chi[a] > phi[a] || clo[a] > chi[a]) report[2]++;
        }
        stack.push_back(ch);
      }
    }
  }
  // every slot is reached, except (aligned treelets) padding slots, which
  // must hold the padding word and zero codes
  uint64_t reached = 0;
  for (uint32_t n = 0; n < b.n_nodes; ++n) {
    if (seen[n]) { ++reached; continue; }
    if (!b.aligned() || blob_topo(b, n) != kPadSlot) { report[0]++; continue; }
    for (uint32_t f = 0; f < 2 * b.nax(); ++f) if (code_field(b, n, f) != 0) report[0]++;
    if (b.zero_suppressed() &&
        b.p[b.off_codes + 16ull * rd<uint32_t>(b.p, b.off_blocks + 4ull * (n / b.T)) + n % b.T] != 0)
      report[0]++;
  }
  if (reached != b.real_nodes) report[0]++;
  if (b.zero_suppressed()) {
    // regions in block order, inside [off_codes, off_blocks), each large
    // enough for its masks and the fields they announce; masks use 6 bits
    const uint64_t nblocks = b.n_nodes / b.T;
    for (uint64_t k = 0; k < nblocks; ++k) {
      const uint32_t o0 = rd<uint32_t>(b.p, b.off_blocks + 4 * k), o1 = rd<uint32_t>(b.p, b.off_blocks + 4 * (k + 1));
      if (o1 < o0 || b.off_codes + 16ull * o1 > b.off_blocks) { report[0]++; continue; }
      uint64_t need = b.T;
      for (uint32_t j = 0; j < b.T; ++j) {
        const uint32_t m = b.p[b.off_codes + 16ull * o0 + j];
        if (m > 63u) report[0]++;
        for (int g = 0; g < 6; ++g) need += ((m >> g) & 1u) * (b.w / 8);
      }
      if (need > 16ull * (o1 - o0)) report[0]++;
    }
  }
  // subtree triangle sets, bottom-up (reverse DFS preorder), then containment
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    uint32_t n = *it;
    if (parent[n] >= 0) {
      auto& dst = subtree_tris[parent[n]];
      dst.insert(dst.end(), subtree_tris[n].begin(), subtree_tris[n].end());
    }
    double nlo[3], nhi[3];
    if (b.layout == 0) {
      for (int a = 0; a < 3; ++a) { nlo[a] = lat(b, a, box[6ull * n + a]); nhi[a] = lat(b, a, box[6ull * n + 3 + a]); }
    } else {
      abs_box(b, n, nlo, nhi);
    }
    for (uint32_t ti : subtree_tris[n])
      for (int v = 0; v < 3; ++v)
        for (int a = 0; a < 3; ++a) {
          double x = (double)verts[3 * tris[3 * ti + v] + a];
          if (x < nlo[a] || x > nhi[a]) report[1]++;
        }
    if (parent[n] >= 0) subtree_tris[n].clear(), subtree_tris[n].shrink_to_fit();
  }
  for (int64_t i = 0; i < nt; ++i) if (tri_seen[i] != 1) report[3]++;
  // treelets: contiguous node ranges that partition [0, n_nodes); each <= T
  // nodes; every node's parent is in the same treelet except for the first
  // sibling group, whose parent's decoded box equals the treelet anchor.
  std::vector<int> treelet_of(b.n_nodes, -1);
  uint64_t expect_first = 0;
  for (uint32_t k = 0; k < b.n_treelets; ++k) {
    size_t o = b.off_treelets + 32ull * k;
    int32_t anchor[6];
    for (int a = 0; a < 6; ++a) anchor[a] = rd<int32_t>(b.p, o + 4 * a);
    uint32_t first = rd<uint32_t>(b.p, o + 24), cnt = rd<uint32_t>(b.p, o + 28);
    // contiguous ranges in order; aligned: a treelet that would straddle a
    // T-slot block boundary starts the next block instead (the slots skipped
    // are padding, checked above), and none straddles one
    const uint64_t next_block = (expect_first + b.T - 1) / b.T * b.T;
    const bool placed = first == expect_first ||
                        (b.aligned() && first == next_block && expect_first % b.T + cnt > b.T);
    if (!placed || cnt == 0) report[5]++;
    if (b.aligned() && cnt > 0 && first / b.T != (first + cnt - 1) / b.T) report[5]++;
    if (cnt > b.T) report[6]++;
    expect_first = (uint64_t)first + cnt;
    if ((uint64_t)first + cnt > b.n_nodes) { report[5]++; continue; }
    for (uint32_t n = first; n < first + cnt; ++n) treelet_of[n] = (int)k;
    // root group = the siblings of node `first`
    int pf = parent[first];
    for (uint32_t n = first; n < first + cnt; ++n) {
      int p = parent[n];
      bool in_root_group = (p == pf);
      if (!in_root_group && (p < 0 || treelet_of[p] != (int)k)) report[7]++;
    }
    // anchors re-anchor the delta layout; absolute layouts need none
    const int64_t* ab = (pf < 0) ? nullptr : &box[6ull * pf];
    for (int a = 0; a < 6 && b.layout == 0; ++a) {
      int64_t want = ab ? ab[a] : (int64_t)b.root[a];
      if (anchor[a] != want) report[7]++;
    }
  }
  if (b.aligned() ? (expect_first > b.n_nodes || b.n_nodes - expect_first >= b.T) : expect_first != b.n_nodes)
    report[5]++;
  // k-DOP slab axes (layout 0 only): decode every extra axis top-down (DFS
  // preorder has parents first), then check child-in-parent and containment of
  // the exact projections of each subtree's vertices (bottom-up).
  if (b.layout == 0 && b.kdop > 6) {
    static const int dirs[10][3] = {{1, 1, 1}, {1, 1, -1}, {1, -1, 1}, {-1, 1, 1}, {1, 1, 0},
                                    {1, -1, 0}, {1, 0, 1}, {1, 0, -1}, {0, 1, 1}, {0, 1, -1}};
    const int nx = (int)b.nax() - 3;
    const int d0 = (b.kdop == 18) ? 4 : 0;  // 18-DOP uses the 6 edge directions only
    for (int a = 0; a < nx; ++a) {
      const int* d = dirs[d0 + a];
      const size_t o = b.off_axes + 16ull * a;
      const float org = rd<float>(b.p, o);
      const int ex = rd<int32_t>(b.p, o + 4);
      const int64_t root_lo = rd<int32_t>(b.p, o + 8), root_hi = rd<int32_t>(b.p, o + 12);
      std::vector<int64_t> L(2ull * b.n_nodes, 0);
      std::vector<double> plo(b.n_nodes, 1e300), phi(b.n_nodes, -1e300);
      for (uint32_t n : order) {
        const int64_t P0 = parent[n] < 0 ? root_lo : L[2ull * parent[n]];
        const int64_t P1 = parent[n] < 0 ? root_hi : L[2ull * parent[n] + 1];
        const uint32_t ql = code_field(b, n, 3 + a), qh = code_field(b, n, b.nax() + 3 + a);
        if ((ql >> b.bits) || (qh >> b.bits)) report[0]++;
        const int s = std::max(0, bitlen(P1 - P0) - (int)b.bits);
        L[2ull * n] = P0 + ((int64_t)ql << s);
        L[2ull * n + 1] = P1 - ((int64_t)qh << s);
        if (L[2ull * n] < P0 || L[2ull * n + 1] > P1 || L[2ull * n] > L[2ull * n + 1]) report[2]++;
      }
      for (auto it = order.rbegin(); it != order.rend(); ++it) {
        const uint32_t n = *it;
        const uint32_t tp = blob_topo(b, n);
        if (tp >> 31) {
          const uint32_t first = tp & 0x1FFFFFFFu, cnt = ((tp >> 29) & 3u) + 1;
          for (uint32_t k = 0; k < cnt && first + k < b.n_tris; ++k) {
            const uint32_t ti = idx[first + k];
            if ((int64_t)ti >= nt) continue;
            for (int v = 0; v < 3; ++v) {
              const float* x = &verts[3 * tris[3 * ti + v]];
              const double pr = d[0] * (double)x[0] + d[1] * (double)x[1] + d[2] * (double)x[2];
              plo[n] = std::min(plo[n], pr);
              phi[n] = std::max(phi[n], pr);
            }
          }
        }
        if (parent[n] >= 0) {
          plo[parent[n]] = std::min(plo[parent[n]], plo[n]);
          phi[parent[n]] = std::max(phi[parent[n]], phi[n]);
        }
        const double lo = (double)org + std::ldexp((double)L[2ull * n], ex);
        const double hi = (double)org + std::ldexp((double)L[2ull * n + 1], ex);
        if (plo[n] < lo || phi[n] > hi) report[1]++;
      }
    }
  }
  int64_t total = 0;
  for (int k = 0; k < 9; ++k) total += report[k];
  return total;
}

}  // extern "C"
