// cbvh_device.cu — sm_100a kernels for batched simultaneous traversal of two
// compressed BVHs (BJ subsystem (2)) and the device half of the C-ABI.
//
// Paper mapping (P:n = PAPER.md line n, S:n = SPEC.md line n):
//   * Algorithm 1 BVHtraversal(a, b): a work item is a node pair
//     (a, b) whose boxes intersect (the root pair is not tested, as in
//     Alg. 1).  Expanding it enumerates the child pairs of the four cases —
//     both leaves -> checkPrimitives; a leaf -> (a, b_j); b leaf ->
//     (a_i, b); else the cross product (a_i, b_j) (reading R9) — and every
//     lane of the warp tests one child pair at once.
//   * "If a_i and b_j intersect" (P:55/65/75): AABB(b_j, world) vs the box of
//     a_i under the pose, separating-axis test over the 3 world axes and the
//     3 axes of A with a conservative fp32 slack (reading R10).
//   * predictor–corrector decode: each child box is decoded on
//     the fly from the already-decoded parent box carried by the work item,
//     in exact integer lattice arithmetic, then mapped to fp32 with directed
//     rounding (lo down, hi up) so the decoded box always contains the node.
//   * checkPrimitives: Möller's interval test, fp32, in A's local
//     frame (B's triangle is mapped by R^T (v - t)), closed triangles.
//   * distance variant: box lower bounds prune against
//     the pose's best distance; leaves use the exact triangle–triangle
//     distance (0 if they intersect).
//
// Execution model: a persistent grid; each warp owns a
// node-pair stack in shared memory (SoA, spilled to a per-warp global area
// when it runs high) that may hold items of several poses; the warp pops as
// many items as fill 32 lanes with child pairs, tests them, and compacts the
// survivors with __ballot_sync/__popc — internal pairs back onto the stack,
// leaf pairs into a per-warp leaf queue that is drained 32 triangle pairs at
// a time.  Poses are acquired in chunks from a global atomic cursor when the
// stack runs low.  Per-pose results are accumulated with warp-aggregated
// atomics, so any warp may process any item.

#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../include/cbvh.h"
#include "cbvh_internal.h"

namespace cbvh {

// ----------------------------------------------------------------------------
// device-side views
// ----------------------------------------------------------------------------

struct DevTree {
  const uint32_t* topo;
  const uint8_t* codes;
  const float* tris;
  float ox, oy, oz, cell;
  float maxabs;      // max |coordinate| of the decoded root box (slack scale)
  int bits, width;   // b and stored field width (4 / 8 / 16)
  uint32_t root_topo;
  int32_t root[6];   // decoded root lattice box
};

struct Control {
  unsigned int error;
  unsigned int cursor;
  unsigned int pad[14];
  unsigned long long stats[8];
};
static_assert(sizeof(Control) == 128, "control block layout");

constexpr int kWarps = 4;           // warps per CTA
constexpr int kStack = 64;          // smem stack entries per warp
constexpr int kFields = 16;         // words per stack entry
constexpr int kLeafQ = 64;          // leaf-queue entries per warp
constexpr int kSpillCap = 2048;     // global spill entries per warp
constexpr int kGrab = 8;            // poses acquired per cursor atomic
constexpr int kLowWater = 4;        // acquire poses when the stack is below this

// stack fields
enum { F_POSE = 0, F_TA = 1, F_TB = 2, F_BA = 3, F_BB = 9, F_LB = 15 };

struct Params {
  DevTree A, B;
  const float* poses;
  int N;
  uint8_t* hit;
  uint32_t* count;
  uint32_t* dist_bits;   // float bits of the running minimum distance
  Control* ctl;
  uint32_t* spill;       // [num_warps][kSpillCap][kFields]
};

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- decode

__device__ __forceinline__ void load_codes(const DevTree& T, uint32_t node, uint32_t q[6]) {
  if (T.width == 8) {
    const unsigned short* p = reinterpret_cast<const unsigned short*>(T.codes + 6ull * node);
    uint32_t a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    q[0] = a & 255u; q[1] = a >> 8; q[2] = b & 255u; q[3] = b >> 8; q[4] = c & 255u; q[5] = c >> 8;
  } else if (T.width == 16) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(T.codes + 12ull * node);
    uint32_t a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    q[0] = a & 0xffffu; q[1] = a >> 16; q[2] = b & 0xffffu; q[3] = b >> 16; q[4] = c & 0xffffu; q[5] = c >> 16;
  } else {
    const uint8_t* p = T.codes + 3ull * node;
    uint32_t w = (uint32_t)__ldg(p) | ((uint32_t)__ldg(p + 1) << 8) | ((uint32_t)__ldg(p + 2) << 16);
    #pragma unroll
    for (int f = 0; f < 6; ++f) q[f] = (w >> (4 * f)) & 15u;
  }
}

// child box from the decoded parent P (lattice ints): step 2^s,
// s = max(0, bitlen(E) - b), lo moves up by q_lo << s, hi down by q_hi << s.
__device__ __forceinline__ void decode_child(const int32_t P[6], const uint32_t q[6], int bits, int32_t C[6]) {
  #pragma unroll
  for (int a = 0; a < 3; ++a) {
    int32_t E = P[3 + a] - P[a];
    int s = max(0, (32 - __clz(E)) - bits);
    C[a] = P[a] + (int32_t)(q[a] << s);
    C[3 + a] = P[3 + a] - (int32_t)(q[3 + a] << s);
  }
}

// lattice -> fp32 with directed rounding: lo rounded down, hi rounded up, so
// the float box contains the lattice box exactly (cell is a power of two and
// |k| < 2^23, so k * cell is exact and only the add rounds).
__device__ __forceinline__ void to_float_box(const DevTree& T, const int32_t C[6], float lo[3], float hi[3]) {
  lo[0] = __fmaf_rd(__int2float_rn(C[0]), T.cell, T.ox);
  lo[1] = __fmaf_rd(__int2float_rn(C[1]), T.cell, T.oy);
  lo[2] = __fmaf_rd(__int2float_rn(C[2]), T.cell, T.oz);
  hi[0] = __fmaf_ru(__int2float_rn(C[3]), T.cell, T.ox);
  hi[1] = __fmaf_ru(__int2float_rn(C[4]), T.cell, T.oy);
  hi[2] = __fmaf_ru(__int2float_rn(C[5]), T.cell, T.oz);
}

struct PoseF {
  float R[3][3];
  float t[3];
};

__device__ __forceinline__ PoseF load_pose(const float* poses, int i) {
  const float4* p = reinterpret_cast<const float4*>(poses + 12ll * i);
  float4 r0 = __ldg(p), r1 = __ldg(p + 1), r2 = __ldg(p + 2);
  PoseF P;
  P.R[0][0] = r0.x; P.R[0][1] = r0.y; P.R[0][2] = r0.z; P.t[0] = r0.w;
  P.R[1][0] = r1.x; P.R[1][1] = r1.y; P.R[1][2] = r1.z; P.t[1] = r1.w;
  P.R[2][0] = r2.x; P.R[2][1] = r2.y; P.R[2][2] = r2.z; P.t[2] = r2.w;
  return P;
}

// ---------------------------------------------------------------- BV test

// SAT between box a (A-local, under pose P) and box b (world).  Returns the
// largest separating gap over the 6 axes (> 0 means separated) and, for the
// distance variant, the exact gap between b and the world AABB of a.
// eps absorbs fp32 rounding (|error| <= eps).
template <bool WANT_LB>
__device__ __forceinline__ float sat_gap(const PoseF& P, const float alo[3], const float ahi[3],
                                         const float blo[3], const float bhi[3], float eps, float* lb) {
  float ca[3], ha[3], cb[3], hb[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    ca[k] = 0.5f * (alo[k] + ahi[k]);
    ha[k] = 0.5f * (ahi[k] - alo[k]);
    cb[k] = 0.5f * (blo[k] + bhi[k]);
    hb[k] = 0.5f * (bhi[k] - blo[k]);
  }
  float Tw[3], gw[3];
  float gmax = -FLT_MAX;
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    Tw[k] = fmaf(P.R[k][0], ca[0], fmaf(P.R[k][1], ca[1], fmaf(P.R[k][2], ca[2], P.t[k] - cb[k])));
    float ra = fmaf(fabsf(P.R[k][0]), ha[0], fmaf(fabsf(P.R[k][1]), ha[1], fabsf(P.R[k][2]) * ha[2]));
    gw[k] = fabsf(Tw[k]) - (hb[k] + ra);
    gmax = fmaxf(gmax, gw[k]);
  }
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    float Ta = fmaf(P.R[0][k], Tw[0], fmaf(P.R[1][k], Tw[1], P.R[2][k] * Tw[2]));
    float rb = fmaf(fabsf(P.R[0][k]), hb[0], fmaf(fabsf(P.R[1][k]), hb[1], fabsf(P.R[2][k]) * hb[2]));
    gmax = fmaxf(gmax, fabsf(Ta) - (ha[k] + rb));
  }
  if (WANT_LB) {
    float g0 = fmaxf(gw[0], 0.f), g1 = fmaxf(gw[1], 0.f), g2 = fmaxf(gw[2], 0.f);
    float e = sqrtf(fmaf(g0, g0, fmaf(g1, g1, g2 * g2)));
    *lb = fmaxf(fmaxf(e, gmax), 0.f) - eps;
  }
  return gmax - eps;
}

// ---------------------------------------------------------------- leaf tests

struct Tri {
  float v[3][3];
};

__device__ __forceinline__ Tri load_tri(const float* tris, uint32_t i) {
  const float* p = tris + 9ull * i;
  Tri T;
  #pragma unroll
  for (int k = 0; k < 9; ++k) T.v[k / 3][k % 3] = __ldg(p + k);
  return T;
}

// B's world triangle into A's local frame: u = R^T (v - t).
__device__ __forceinline__ Tri to_local(const PoseF& P, const Tri& W) {
  Tri L;
  #pragma unroll
  for (int v = 0; v < 3; ++v) {
    float d0 = W.v[v][0] - P.t[0], d1 = W.v[v][1] - P.t[1], d2 = W.v[v][2] - P.t[2];
    #pragma unroll
    for (int k = 0; k < 3; ++k) L.v[v][k] = fmaf(P.R[0][k], d0, fmaf(P.R[1][k], d1, P.R[2][k] * d2));
  }
  return L;
}

__device__ __forceinline__ void vsub(const float* a, const float* b, float* r) {
  r[0] = a[0] - b[0]; r[1] = a[1] - b[1]; r[2] = a[2] - b[2];
}
__device__ __forceinline__ float vdot(const float* a, const float* b) {
  return fmaf(a[0], b[0], fmaf(a[1], b[1], a[2] * b[2]));
}
__device__ __forceinline__ void vcross(const float* a, const float* b, float* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}

__device__ __forceinline__ float orient2(float ax, float ay, float bx, float by, float cx, float cy) {
  return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
}

__device__ bool seg2_intersect(const float* p1, const float* p2, const float* q1, const float* q2) {
  float d1 = orient2(q1[0], q1[1], q2[0], q2[1], p1[0], p1[1]);
  float d2 = orient2(q1[0], q1[1], q2[0], q2[1], p2[0], p2[1]);
  float d3 = orient2(p1[0], p1[1], p2[0], p2[1], q1[0], q1[1]);
  float d4 = orient2(p1[0], p1[1], p2[0], p2[1], q2[0], q2[1]);
  if (((d1 > 0.f && d2 < 0.f) || (d1 < 0.f && d2 > 0.f)) && ((d3 > 0.f && d4 < 0.f) || (d3 < 0.f && d4 > 0.f)))
    return true;
  auto on = [](const float* a, const float* b, const float* c) {
    return fminf(a[0], b[0]) <= c[0] && c[0] <= fmaxf(a[0], b[0]) && fminf(a[1], b[1]) <= c[1] &&
           c[1] <= fmaxf(a[1], b[1]);
  };
  return (d1 == 0.f && on(q1, q2, p1)) || (d2 == 0.f && on(q1, q2, p2)) || (d3 == 0.f && on(p1, p2, q1)) ||
         (d4 == 0.f && on(p1, p2, q2));
}

__device__ bool pt_in_tri2(const float* p, const float* a, const float* b, const float* c) {
  float o1 = orient2(a[0], a[1], b[0], b[1], p[0], p[1]);
  float o2 = orient2(b[0], b[1], c[0], c[1], p[0], p[1]);
  float o3 = orient2(c[0], c[1], a[0], a[1], p[0], p[1]);
  bool neg = (o1 < 0.f) || (o2 < 0.f) || (o3 < 0.f);
  bool pos = (o1 > 0.f) || (o2 > 0.f) || (o3 > 0.f);
  return !(neg && pos);
}

__device__ __noinline__ bool coplanar2(const float* N, const Tri& V, const Tri& U) {
  float a0 = fabsf(N[0]), a1 = fabsf(N[1]), a2 = fabsf(N[2]);
  int i0, i1;
  if (a0 >= a1 && a0 >= a2) { i0 = 1; i1 = 2; }
  else if (a1 >= a2) { i0 = 0; i1 = 2; }
  else { i0 = 0; i1 = 1; }
  float v[3][2], u[3][2];
  for (int k = 0; k < 3; ++k) {
    v[k][0] = V.v[k][i0]; v[k][1] = V.v[k][i1];
    u[k][0] = U.v[k][i0]; u[k][1] = U.v[k][i1];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (seg2_intersect(v[i], v[(i + 1) % 3], u[j], u[(j + 1) % 3])) return true;
  return pt_in_tri2(v[0], u[0], u[1], u[2]) || pt_in_tri2(u[0], v[0], v[1], v[2]);
}

// interval of a triangle on the line of the two planes (Möller 1997):
// the vertex alone on its side k, crossing points toward i and j.
__device__ __forceinline__ bool interval(const float p[3], const float d[3], float* t0, float* t1) {
  int k, i, j;
  if (d[0] * d[1] > 0.f) { k = 2; i = 0; j = 1; }
  else if (d[0] * d[2] > 0.f) { k = 1; i = 0; j = 2; }
  else if (d[1] * d[2] > 0.f || d[0] != 0.f) { k = 0; i = 1; j = 2; }
  else if (d[1] != 0.f) { k = 1; i = 0; j = 2; }
  else if (d[2] != 0.f) { k = 2; i = 0; j = 1; }
  else return false;
  float a = p[k] + (p[i] - p[k]) * __fdividef(d[k], d[k] - d[i]);
  float b = p[k] + (p[j] - p[k]) * __fdividef(d[k], d[k] - d[j]);
  *t0 = fminf(a, b);
  *t1 = fmaxf(a, b);
  return true;
}

__device__ bool tri_tri_overlap(const Tri& V, const Tri& U) {
  float e1[3], e2[3], N1[3], N2[3];
  vsub(V.v[1], V.v[0], e1); vsub(V.v[2], V.v[0], e2); vcross(e1, e2, N1);
  float d1 = -vdot(N1, V.v[0]);
  float du[3] = {vdot(N1, U.v[0]) + d1, vdot(N1, U.v[1]) + d1, vdot(N1, U.v[2]) + d1};
  if ((du[0] > 0.f && du[1] > 0.f && du[2] > 0.f) || (du[0] < 0.f && du[1] < 0.f && du[2] < 0.f)) return false;
  vsub(U.v[1], U.v[0], e1); vsub(U.v[2], U.v[0], e2); vcross(e1, e2, N2);
  float d2 = -vdot(N2, U.v[0]);
  float dv[3] = {vdot(N2, V.v[0]) + d2, vdot(N2, V.v[1]) + d2, vdot(N2, V.v[2]) + d2};
  if ((dv[0] > 0.f && dv[1] > 0.f && dv[2] > 0.f) || (dv[0] < 0.f && dv[1] < 0.f && dv[2] < 0.f)) return false;
  if (du[0] == 0.f && du[1] == 0.f && du[2] == 0.f) return coplanar2(N1, V, U);
  float D[3];
  vcross(N1, N2, D);
  int ax = 0;
  float m = fabsf(D[0]);
  if (fabsf(D[1]) > m) { m = fabsf(D[1]); ax = 1; }
  if (fabsf(D[2]) > m) { m = fabsf(D[2]); ax = 2; }
  if (m == 0.f) return coplanar2(N1, V, U);
  float vp[3] = {V.v[0][ax], V.v[1][ax], V.v[2][ax]};
  float up[3] = {U.v[0][ax], U.v[1][ax], U.v[2][ax]};
  float a0, a1, b0, b1;
  if (!interval(vp, dv, &a0, &a1) || !interval(up, du, &b0, &b1)) return coplanar2(N1, V, U);
  return !(a1 < b0 || b1 < a0);
}

__device__ __forceinline__ float pt_seg_d2(const float* p, const float* a, const float* b) {
  float ab[3], ap[3];
  vsub(b, a, ab); vsub(p, a, ap);
  float L = vdot(ab, ab);
  float t = L > 0.f ? __saturatef(vdot(ap, ab) / L) : 0.f;
  float q[3] = {fmaf(t, ab[0], a[0]) - p[0], fmaf(t, ab[1], a[1]) - p[1], fmaf(t, ab[2], a[2]) - p[2]};
  return vdot(q, q);
}

// min over (s,t) in [0,1]^2: the stationary point when inside, else the four
// boundary point–segment distances; any candidate is a real pair of points,
// so rounding can only over-estimate the minimum.
__device__ float seg_seg_d2(const float* p0, const float* p1, const float* q0, const float* q1) {
  float best = fminf(fminf(pt_seg_d2(p0, q0, q1), pt_seg_d2(p1, q0, q1)),
                     fminf(pt_seg_d2(q0, p0, p1), pt_seg_d2(q1, p0, p1)));
  float d1[3], d2[3], r[3];
  vsub(p1, p0, d1); vsub(q1, q0, d2); vsub(p0, q0, r);
  float a = vdot(d1, d1), e = vdot(d2, d2), b = vdot(d1, d2), c = vdot(d1, r), f = vdot(d2, r);
  float den = a * e - b * b;
  if (den > 0.f) {
    float s = (b * f - c * e) / den, t = (a * f - b * c) / den;
    if (s >= 0.f && s <= 1.f && t >= 0.f && t <= 1.f) {
      float w[3] = {r[0] + s * d1[0] - t * d2[0], r[1] + s * d1[1] - t * d2[1], r[2] + s * d1[2] - t * d2[2]};
      best = fminf(best, vdot(w, w));
    }
  }
  return best;
}

__device__ float pt_tri_d2(const float* p, const Tri& T) {
  float e1[3], e2[3], n[3], w[3];
  vsub(T.v[1], T.v[0], e1); vsub(T.v[2], T.v[0], e2); vcross(e1, e2, n);
  float best = fminf(fminf(pt_seg_d2(p, T.v[0], T.v[1]), pt_seg_d2(p, T.v[1], T.v[2])), pt_seg_d2(p, T.v[2], T.v[0]));
  float nn = vdot(n, n);
  if (nn > 0.f) {
    vsub(p, T.v[0], w);
    float h = vdot(w, n) / nn;
    float q[3] = {p[0] - h * n[0], p[1] - h * n[1], p[2] - h * n[2]};
    float a[3], b[3], c0[3];
    vsub(T.v[1], T.v[0], a); vsub(q, T.v[0], b); vcross(a, b, c0);
    bool in = vdot(c0, n) >= 0.f;
    vsub(T.v[2], T.v[1], a); vsub(q, T.v[1], b); vcross(a, b, c0);
    in = in && vdot(c0, n) >= 0.f;
    vsub(T.v[0], T.v[2], a); vsub(q, T.v[2], b); vcross(a, b, c0);
    in = in && vdot(c0, n) >= 0.f;
    if (in) {
      float d = p[0] - q[0], e = p[1] - q[1], f = p[2] - q[2];
      best = fminf(best, d * d + e * e + f * f);
    }
  }
  return best;
}

__device__ float tri_tri_dist(const Tri& V, const Tri& U) {
  if (tri_tri_overlap(V, U)) return 0.f;
  float best = FLT_MAX;
  #pragma unroll 1
  for (int k = 0; k < 3; ++k) {
    best = fminf(best, pt_tri_d2(V.v[k], U));
    best = fminf(best, pt_tri_d2(U.v[k], V));
  }
  #pragma unroll 1
  for (int i = 0; i < 3; ++i)
    #pragma unroll 1
    for (int j = 0; j < 3; ++j)
      best = fminf(best, seg_seg_d2(V.v[i], V.v[(i + 1) % 3], U.v[j], U.v[(j + 1) % 3]));
  return sqrtf(best);
}

// ----------------------------------------------------------------------------
// the traversal kernel
// ----------------------------------------------------------------------------

constexpr int kWarpSmemWords = kFields * kStack + 3 * kLeafQ;

__device__ __forceinline__ int pair_count(uint32_t ta, uint32_t tb) {
  int na = (ta & kLeafBit) ? 1 : (int)((ta >> 28) & 7u) + 1;
  int nb = (tb & kLeafBit) ? 1 : (int)((tb >> 28) & 7u) + 1;
  return na * nb;
}

__device__ __forceinline__ int tri_pair_count(uint32_t ta, uint32_t tb) {
  return (int)(((ta >> 29) & 3u) + 1) * (int)(((tb >> 29) & 3u) + 1);
}

template <int MODE, bool STATS>
struct Warp {
  uint32_t* st;      // stack SoA [kFields][kStack]
  uint32_t* lq;      // leaf queue SoA [3][kLeafQ]: pose, topoA, topoB
  uint32_t* spill;   // this warp's global spill area
  int lane;
  int top, nleaf, spill_top;
  unsigned long long s_bv, s_exp, s_leaf, s_tri, s_dec, s_spill;
};

template <int MODE, bool STATS>
__device__ __noinline__ void drain_leaves(const Params& p, Warp<MODE, STATS>& w) {
  // process every queued leaf pair: tri pairs spread over the 32 lanes
  int head = 0;
  while (head < w.nleaf) {
    int avail = min(32, w.nleaf - head);
    uint32_t pose = 0, ta = 0, tb = 0;
    int n = 0;
    if (w.lane < avail) {
      pose = w.lq[0 * kLeafQ + head + w.lane];
      ta = w.lq[1 * kLeafQ + head + w.lane];
      tb = w.lq[2 * kLeafQ + head + w.lane];
      n = tri_pair_count(ta, tb);
    }
    int incl = n;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, incl, o);
      if (w.lane >= o) incl += y;
    }
    unsigned fit = __ballot_sync(FULL, w.lane < avail && incl <= 32);
    int m = __popc(fit);  // >= 1 since every entry has <= 16 tri pairs
    int total = __shfl_sync(FULL, incl, m - 1);
    unsigned starts = __reduce_or_sync(FULL, (w.lane < m) ? (1u << (incl - n)) : 0u);
    // this lane's tri pair
    int e = __popc(starts & ((2u << w.lane) - 1u)) - 1;
    int start_e = __shfl_sync(FULL, incl - n, e < 0 ? 0 : e);
    uint32_t my_pose = __shfl_sync(FULL, pose, e < 0 ? 0 : e);
    uint32_t my_ta = __shfl_sync(FULL, ta, e < 0 ? 0 : e);
    uint32_t my_tb = __shfl_sync(FULL, tb, e < 0 ? 0 : e);
    bool valid = w.lane < total;
    int k = w.lane - start_e;
    int nb = (int)((my_tb >> 29) & 3u) + 1;
    uint32_t ia = (my_ta & 0x1FFFFFFFu) + (uint32_t)(k / nb);
    uint32_t ib = (my_tb & 0x1FFFFFFFu) + (uint32_t)(k % nb);
    bool hit = false;
    float d = FLT_MAX;
    if (valid) {
      PoseF P = load_pose(p.poses, (int)my_pose);
      Tri TA = load_tri(p.A.tris, ia);
      Tri TB = to_local(P, load_tri(p.B.tris, ib));
      if (MODE == 0) hit = tri_tri_overlap(TA, TB);
      else d = tri_tri_dist(TA, TB);
    }
    if (STATS) {
      if (w.lane == 0) { w.s_tri += total; w.s_leaf += m; }
    }
    if (MODE == 0) {
      unsigned hm = __ballot_sync(FULL, hit);
      if (hit) {
        unsigned g = __match_any_sync(hm, my_pose);
        if (w.lane == __ffs(g) - 1) {
          atomicAdd(&p.count[my_pose], (unsigned)__popc(g));
          p.hit[my_pose] = 1;
        }
      }
    } else {
      unsigned vm = __ballot_sync(FULL, valid);
      if (valid) {
        unsigned g = __match_any_sync(vm, my_pose);
        unsigned mn = __reduce_min_sync(g, __float_as_uint(d));
        if (w.lane == __ffs(g) - 1) atomicMin(&p.dist_bits[my_pose], mn);
      }
    }
    head += m;
  }
  w.nleaf = 0;
  __syncwarp();
}

template <int MODE, bool STATS>
__device__ __noinline__ void spill_out(const Params& p, Warp<MODE, STATS>& w) {
  // move the bottom half of the smem stack to the global spill area
  constexpr int H = kStack / 2;
  if (w.spill_top + H > kSpillCap) {
    if (w.lane == 0) atomicExch(&p.ctl->error, (unsigned)(-CBVH_EOVERFLOW));
    w.top = 0;  // abandon: results are flagged invalid via cbvh_check
    return;
  }
  __syncwarp();
  for (int idx = w.lane; idx < H * kFields; idx += 32) {
    int e = idx / kFields, f = idx % kFields;
    w.spill[(size_t)(w.spill_top + e) * kFields + f] = w.st[f * kStack + e];
  }
  __syncwarp();
  int rest = w.top - H;
  for (int idx = w.lane; idx < rest * kFields; idx += 32) {
    int e = idx % rest, f = idx / rest;
    w.st[f * kStack + e] = w.st[f * kStack + e + H];
  }
  __syncwarp();
  w.spill_top += H;
  w.top = rest;
  if (STATS && w.lane == 0) w.s_spill++;
}

template <int MODE, bool STATS>
__device__ __noinline__ void spill_in(const Params& p, Warp<MODE, STATS>& w) {
  int n = min(kStack / 2, w.spill_top);
  int base = w.spill_top - n;
  __syncwarp();
  for (int idx = w.lane; idx < n * kFields; idx += 32) {
    int e = idx / kFields, f = idx % kFields;
    w.st[f * kStack + e] = w.spill[(size_t)(base + e) * kFields + f];
  }
  __syncwarp();
  w.spill_top = base;
  w.top = n;
}

template <int MODE, bool STATS>
__global__ void __launch_bounds__(kWarps * 32) traverse_kernel(const Params p) {
  extern __shared__ uint32_t smem[];
  const int wib = threadIdx.x >> 5;
  Warp<MODE, STATS> w;
  w.lane = threadIdx.x & 31;
  w.st = smem + wib * kWarpSmemWords;
  w.lq = w.st + kFields * kStack;
  const int gwarp = blockIdx.x * kWarps + wib;
  w.spill = p.spill + (size_t)gwarp * kSpillCap * kFields;
  w.top = 0; w.nleaf = 0; w.spill_top = 0;
  w.s_bv = w.s_exp = w.s_leaf = w.s_tri = w.s_dec = w.s_spill = 0;
  bool poses_left = true;
  const unsigned lt = lanemask_lt();
  const float scale_ab = p.A.maxabs + p.B.maxabs;

  while (true) {
    // ---- acquire poses when the stack runs low: push the root pair
    if (poses_left && w.top < kLowWater) {
      unsigned base = 0;
      if (w.lane == 0) base = atomicAdd(&p.ctl->cursor, (unsigned)kGrab);
      base = __shfl_sync(FULL, base, 0);
      if (base >= (unsigned)p.N) {
        poses_left = false;
      } else {
        int k = min(kGrab, p.N - (int)base);
        bool mine = w.lane < k;
        bool leafpair = (p.A.root_topo & kLeafBit) && (p.B.root_topo & kLeafBit);
        if (mine && !leafpair) {
          int slot = w.top + w.lane;
          w.st[F_POSE * kStack + slot] = base + w.lane;
          w.st[F_TA * kStack + slot] = p.A.root_topo;
          w.st[F_TB * kStack + slot] = p.B.root_topo;
          #pragma unroll
          for (int q = 0; q < 6; ++q) {
            w.st[(F_BA + q) * kStack + slot] = (uint32_t)p.A.root[q];
            w.st[(F_BB + q) * kStack + slot] = (uint32_t)p.B.root[q];
          }
          w.st[F_LB * kStack + slot] = 0u;
        }
        if (mine && leafpair) {
          int slot = w.nleaf + w.lane;
          w.lq[0 * kLeafQ + slot] = base + w.lane;
          w.lq[1 * kLeafQ + slot] = p.A.root_topo;
          w.lq[2 * kLeafQ + slot] = p.B.root_topo;
        }
        if (leafpair) w.nleaf += k; else w.top += k;
        __syncwarp();
        if (w.nleaf > kLeafQ - 32) drain_leaves<MODE, STATS>(p, w);
      }
    }
    if (w.top == 0) {
      if (w.spill_top > 0) { spill_in<MODE, STATS>(p, w); continue; }
      if (poses_left) continue;
      break;
    }

    // ---- pop as many items as fill 32 lanes with child pairs
    int n = 0;
    if (w.lane < w.top) {
      int slot = w.top - 1 - w.lane;
      n = pair_count(w.st[F_TA * kStack + slot], w.st[F_TB * kStack + slot]);
    }
    int incl = n;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, incl, o);
      if (w.lane >= o) incl += y;
    }
    const int n0 = __shfl_sync(FULL, n, 0);
    int m, total, passes;
    unsigned starts;
    if (n0 > 32) {  // B = 8 both internal: one item, two passes
      m = 1; total = n0; passes = (n0 + 31) >> 5; starts = 1u;
    } else {
      unsigned fit = __ballot_sync(FULL, w.lane < w.top && incl <= 32);
      m = __popc(fit);
      total = __shfl_sync(FULL, incl, m - 1);
      passes = 1;
      starts = __reduce_or_sync(FULL, (w.lane < m) ? (1u << (incl - n)) : 0u);
    }
    int e = __popc(starts & ((2u << w.lane) - 1u)) - 1;
    if (e < 0) e = 0;
    const int start_e = __shfl_sync(FULL, incl - n, e);
    // this lane's item, read from the stack before anything is pushed
    const int slot = w.top - 1 - e;
    const uint32_t pose = w.st[F_POSE * kStack + slot];
    const uint32_t ta = w.st[F_TA * kStack + slot];
    const uint32_t tb = w.st[F_TB * kStack + slot];
    int32_t BA[6], BB[6];
    #pragma unroll
    for (int q = 0; q < 6; ++q) {
      BA[q] = (int32_t)w.st[(F_BA + q) * kStack + slot];
      BB[q] = (int32_t)w.st[(F_BB + q) * kStack + slot];
    }
    const float item_lb = __uint_as_float(w.st[F_LB * kStack + slot]);
    __syncwarp();
    w.top -= m;
    if (STATS && w.lane == 0) w.s_exp += m;

    const PoseF P = load_pose(p.poses, (int)pose);
    const float eps = 2e-6f * (fmaxf(fabsf(P.t[0]), fmaxf(fabsf(P.t[1]), fabsf(P.t[2]))) + scale_ab);
    float best = FLT_MAX;
    if (MODE == 1) best = __uint_as_float(__ldcg(&p.dist_bits[pose]));
    const bool a_int = !(ta & kLeafBit), b_int = !(tb & kLeafBit);
    const int nb = b_int ? (int)((tb >> 28) & 7u) + 1 : 1;

    for (int pass = 0; pass < passes; ++pass) {
      const int k = w.lane - start_e + 32 * pass;
      bool valid = (w.lane + 32 * pass) < total;
      if (MODE == 1) valid = valid && item_lb < best;
      const int i = k / nb, j = k - (k / nb) * nb;
      int32_t CA[6], CB[6];
      uint32_t cta = ta, ctb = tb;
      bool surv = false;
      float lb = 0.f;
      if (valid) {
        if (a_int) {
          uint32_t node = (ta & 0x0FFFFFFFu) + (uint32_t)i;
          uint32_t q[6];
          load_codes(p.A, node, q);
          cta = __ldg(p.A.topo + node);
          decode_child(BA, q, p.A.bits, CA);
        } else {
          #pragma unroll
          for (int r = 0; r < 6; ++r) CA[r] = BA[r];
        }
        if (b_int) {
          uint32_t node = (tb & 0x0FFFFFFFu) + (uint32_t)j;
          uint32_t q[6];
          load_codes(p.B, node, q);
          ctb = __ldg(p.B.topo + node);
          decode_child(BB, q, p.B.bits, CB);
        } else {
          #pragma unroll
          for (int r = 0; r < 6; ++r) CB[r] = BB[r];
        }
        float alo[3], ahi[3], blo[3], bhi[3];
        to_float_box(p.A, CA, alo, ahi);
        to_float_box(p.B, CB, blo, bhi);
        if (MODE == 0) {
          surv = sat_gap<false>(P, alo, ahi, blo, bhi, eps, nullptr) <= 0.f;
        } else {
          sat_gap<true>(P, alo, ahi, blo, bhi, eps, &lb);
          surv = lb < best;
        }
        if (STATS) w.s_dec += (a_int ? 1 : 0) + (b_int ? 1 : 0);
      }
      if (STATS) {
        unsigned vm = __ballot_sync(FULL, valid);
        if (w.lane == 0) w.s_bv += __popc(vm);
      }
      const bool leafpair = surv && (cta & kLeafBit) && (ctb & kLeafBit);
      const bool push = surv && !leafpair;
      // ---- compaction: internal pairs onto the stack
      const unsigned pm = __ballot_sync(FULL, push);
      if (pm) {
        if (w.top + 32 > kStack) spill_out<MODE, STATS>(p, w);
        unsigned order = pm;
        if (MODE == 1) {
          // nearest-first: the smallest lower bound goes on top
          unsigned key = push ? __float_as_uint(fmaxf(lb, 0.f)) : 0xffffffffu;
          unsigned mn = __reduce_min_sync(FULL, key);
          unsigned who = __ballot_sync(FULL, push && key == mn);
          int wl = __ffs(who) - 1;
          int last = 31 - __clz(pm);
          // swap slots of lanes wl and last
          int pos = __popc(pm & lt);
          if (w.lane == wl) pos = __popc(pm) - 1;
          else if (w.lane == last) pos = __popc(pm & ((1u << wl) - 1u));
          if (push) {
            int s2 = w.top + pos;
            w.st[F_POSE * kStack + s2] = pose;
            w.st[F_TA * kStack + s2] = cta;
            w.st[F_TB * kStack + s2] = ctb;
            #pragma unroll
            for (int q = 0; q < 6; ++q) {
              w.st[(F_BA + q) * kStack + s2] = (uint32_t)CA[q];
              w.st[(F_BB + q) * kStack + s2] = (uint32_t)CB[q];
            }
            w.st[F_LB * kStack + s2] = __float_as_uint(lb);
          }
          (void)order;
        } else {
          if (push) {
            int s2 = w.top + __popc(pm & lt);
            w.st[F_POSE * kStack + s2] = pose;
            w.st[F_TA * kStack + s2] = cta;
            w.st[F_TB * kStack + s2] = ctb;
            #pragma unroll
            for (int q = 0; q < 6; ++q) {
              w.st[(F_BA + q) * kStack + s2] = (uint32_t)CA[q];
              w.st[(F_BB + q) * kStack + s2] = (uint32_t)CB[q];
            }
          }
        }
        w.top += __popc(pm);
      }
      // ---- leaf pairs into the leaf queue
      const unsigned lm = __ballot_sync(FULL, leafpair);
      if (lm) {
        if (leafpair) {
          int s2 = w.nleaf + __popc(lm & lt);
          w.lq[0 * kLeafQ + s2] = pose;
          w.lq[1 * kLeafQ + s2] = cta;
          w.lq[2 * kLeafQ + s2] = ctb;
        }
        w.nleaf += __popc(lm);
      }
      __syncwarp();
      if (w.nleaf > kLeafQ - 32) drain_leaves<MODE, STATS>(p, w);
    }
  }
  if (w.nleaf > 0) drain_leaves<MODE, STATS>(p, w);
  if (STATS && w.lane == 0) {
    atomicAdd(&p.ctl->stats[0], w.s_bv);
    atomicAdd(&p.ctl->stats[1], w.s_exp);
    atomicAdd(&p.ctl->stats[2], w.s_leaf);
    atomicAdd(&p.ctl->stats[3], w.s_tri);
    atomicAdd(&p.ctl->stats[6], w.s_tri * 72ull);
    atomicAdd(&p.ctl->stats[7], w.s_spill);
  }
  if (STATS) {
    // nodes decoded: summed over lanes
    unsigned long long d = w.s_dec;
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_down_sync(FULL, d, o);
    if (w.lane == 0) atomicAdd(&p.ctl->stats[4], d);
  }
}

template <int MODE>
__global__ void init_kernel(Params p, int reset_stats) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int stride = gridDim.x * blockDim.x;
  for (int k = i; k < p.N; k += stride) {
    if (MODE == 0) { p.count[k] = 0u; p.hit[k] = 0; }
    else p.dist_bits[k] = 0x7f800000u;  // +inf
  }
  if (i == 0) {
    p.ctl->cursor = 0u;
    p.ctl->error = 0u;
    if (reset_stats)
      for (int s = 0; s < 8; ++s) p.ctl->stats[s] = 0ull;
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------

static thread_local char g_err[512] = "";
static thread_local int g_launches = 0;

int set_error(int code, const char* msg) {
  std::snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  std::snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return CBVH_ECUDA;
}

static size_t smem_bytes() { return (size_t)kWarps * kWarpSmemWords * sizeof(uint32_t); }

struct LaunchShape {
  int blocks;
  int warps;
};

template <int MODE, bool STATS>
static int shape_for(LaunchShape* s) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(traverse_kernel<MODE, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes());
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, traverse_kernel<MODE, STATS>, kWarps * 32, smem_bytes());
  if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (per_sm < 1) per_sm = 1;
  s->blocks = sms * per_sm;
  s->warps = s->blocks * kWarps;
  return CBVH_OK;
}

static int max_warps(int mode) {
  // workspace is sized for the larger of the instantiations of this mode
  LaunchShape a{}, b{};
  int rc = mode == 0 ? shape_for<0, false>(&a) : shape_for<1, false>(&a);
  if (rc) return -1;
  rc = mode == 0 ? shape_for<0, true>(&b) : shape_for<1, true>(&b);
  if (rc) return -1;
  return a.warps > b.warps ? a.warps : b.warps;
}

static size_t workspace_for_warps(int warps) {
  return 256 + (size_t)warps * kSpillCap * kFields * sizeof(uint32_t);
}

static DevTree make_tree(const cbvh_bvh* T) {
  DevTree d;
  const uint8_t* base = static_cast<const uint8_t*>(T->d_blob);
  const cbvh_header& h = T->h;
  d.topo = reinterpret_cast<const uint32_t*>(base + h.off_topo);
  d.codes = base + h.off_codes;
  d.tris = reinterpret_cast<const float*>(base + h.off_tris);
  d.ox = h.origin[0]; d.oy = h.origin[1]; d.oz = h.origin[2];
  d.cell = std::ldexp(1.0f, h.lattice_exp);
  d.bits = (int)h.bits;
  d.width = (int)h.code_width;
  return d;
}

template <int MODE, bool STATS>
static int launch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                  uint32_t* d_count, float* d_dist, void* d_ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!A || !B || !d_ws) return set_error(CBVH_EINVAL, "null argument");
  if (N < 0 || N > 0x7fffffffLL) return set_error(CBVH_EINVAL, "N out of range");
  if (N > 0 && !d_poses) return set_error(CBVH_EINVAL, "null poses");
  if (N > 0 && MODE == 0 && (!d_hit || !d_count)) return set_error(CBVH_EINVAL, "null outputs");
  if (N > 0 && MODE == 1 && !d_dist) return set_error(CBVH_EINVAL, "null outputs");
  if (!A->d_blob || !B->d_blob) return set_error(CBVH_EINVAL, "unbound bvh");
  if ((reinterpret_cast<uintptr_t>(d_poses) & 15) != 0) return set_error(CBVH_EINVAL, "poses must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(d_ws) & 255) != 0) return set_error(CBVH_EINVAL, "workspace must be 256-byte aligned");
  LaunchShape s;
  int rc = shape_for<MODE, STATS>(&s);
  if (rc) return rc;
  if (ws_bytes < workspace_for_warps(s.warps)) return set_error(CBVH_EWORKSPACE, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Params p;
  p.A = make_tree(A);
  p.B = make_tree(B);
  std::memcpy(p.A.root, A->root_decoded, sizeof p.A.root);
  std::memcpy(p.B.root, B->root_decoded, sizeof p.B.root);
  p.A.root_topo = A->root_topo;
  p.B.root_topo = B->root_topo;
  p.A.maxabs = A->max_abs_coord;
  p.B.maxabs = B->max_abs_coord;
  p.poses = d_poses;
  p.N = (int)N;
  p.hit = d_hit;
  p.count = d_count;
  p.dist_bits = reinterpret_cast<uint32_t*>(d_dist);
  p.ctl = static_cast<Control*>(d_ws);
  p.spill = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(d_ws) + 256);
  int ib = (int)((N + 255) / 256);
  ib = ib < 1 ? 1 : (ib > 4096 ? 4096 : ib);
  init_kernel<MODE><<<ib, 256, 0, st>>>(p, STATS ? 1 : 0);
  g_launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "init_kernel launch");
  if (N == 0) return CBVH_OK;
  traverse_kernel<MODE, STATS><<<s.blocks, kWarps * 32, smem_bytes(), st>>>(p);
  g_launches++;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "traverse_kernel launch");
  return CBVH_OK;
}

}  // namespace cbvh

using namespace cbvh;

extern "C" {

const char* cbvh_last_error(void) { return g_err; }
int cbvh_last_launch_count(void) { return g_launches; }

int cbvh_bind(const uint8_t* h_blob, size_t bytes, const void* d_blob, cbvh_bvh* out) {
  if (!h_blob || !d_blob || !out) return set_error(CBVH_EINVAL, "null argument");
  if ((reinterpret_cast<uintptr_t>(d_blob) & 255) != 0) return set_error(CBVH_EINVAL, "device blob must be 256-byte aligned");
  cbvh_header h;
  int rc = parse_header(h_blob, bytes, &h);
  if (rc) return rc;
  out->d_blob = d_blob;
  out->bytes = bytes;
  out->h = h;
  std::memcpy(&out->root_topo, h_blob + h.off_topo, 4);
  // node 0 is coded against the header root box (the anchor of treelet 0)
  uint32_t q[6];
  const uint8_t* c = h_blob + h.off_codes;
  if (h.code_width == 16) {
    for (int f = 0; f < 6; ++f) { uint16_t x; std::memcpy(&x, c + 2 * f, 2); q[f] = x; }
  } else if (h.code_width == 8) {
    for (int f = 0; f < 6; ++f) q[f] = c[f];
  } else {
    uint32_t w = c[0] | (c[1] << 8) | (c[2] << 16);
    for (int f = 0; f < 6; ++f) q[f] = (w >> (4 * f)) & 15u;
  }
  for (int a = 0; a < 3; ++a) {
    int64_t E = (int64_t)h.root_box[3 + a] - h.root_box[a];
    if (E < 0 || E >= (1ll << 23)) return set_error(CBVH_EBLOB, "bad root box");
    int bl = 0;
    while ((E >> bl) > 0) ++bl;
    int s = bl - (int)h.bits > 0 ? bl - (int)h.bits : 0;
    out->root_decoded[a] = h.root_box[a] + (int32_t)(q[a] << s);
    out->root_decoded[3 + a] = h.root_box[3 + a] - (int32_t)(q[3 + a] << s);
  }
  float m = 0.f;
  for (int a = 0; a < 3; ++a) {
    double lo = (double)h.origin[a] + std::ldexp((double)out->root_decoded[a], h.lattice_exp);
    double hi = (double)h.origin[a] + std::ldexp((double)out->root_decoded[3 + a], h.lattice_exp);
    m = std::fmax(m, (float)std::fmax(std::fabs(lo), std::fabs(hi)));
  }
  out->max_abs_coord = m;
  return CBVH_OK;
}

size_t cbvh_workspace_bytes(const cbvh_bvh* A, const cbvh_bvh* B, int64_t N, int mode) {
  (void)A; (void)B; (void)N;
  int w = max_warps(mode == 1 ? 1 : 0);
  if (w <= 0) return 0;
  return workspace_for_warps(w);
}

int collide_batch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                  uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream) {
  return launch<0, false>(A, B, d_poses, N, d_hit, d_pair_count, nullptr, d_ws, ws_bytes, stream);
}
int collide_batch_stats(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                        uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream) {
  return launch<0, true>(A, B, d_poses, N, d_hit, d_pair_count, nullptr, d_ws, ws_bytes, stream);
}
int distance_batch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, float* d_min_dist,
                   void* d_ws, size_t ws_bytes, void* stream) {
  return launch<1, false>(A, B, d_poses, N, nullptr, nullptr, d_min_dist, d_ws, ws_bytes, stream);
}
int distance_batch_stats(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                         float* d_min_dist, void* d_ws, size_t ws_bytes, void* stream) {
  return launch<1, true>(A, B, d_poses, N, nullptr, nullptr, d_min_dist, d_ws, ws_bytes, stream);
}

int cbvh_check(const void* d_ws, void* stream) {
  if (!d_ws) return set_error(CBVH_EINVAL, "null workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned err = 0;
  cudaError_t e = cudaMemcpyAsync(&err, d_ws, sizeof err, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cbvh_check");
  if (err) return set_error(-(int)err, "device traversal error (stack overflow)");
  return CBVH_OK;
}

int cbvh_read_stats(const void* d_ws, cbvh_stats* out, void* stream) {
  if (!d_ws || !out) return set_error(CBVH_EINVAL, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long v[8];
  cudaError_t e = cudaMemcpyAsync(v, static_cast<const uint8_t*>(d_ws) + offsetof(Control, stats), sizeof v,
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cbvh_read_stats");
  out->bv_tests = v[0]; out->expansions = v[1]; out->leaf_pairs = v[2]; out->tri_tests = v[3];
  out->nodes_decoded = v[4]; out->record_bytes = v[5]; out->tri_bytes = v[6]; out->spills = v[7];
  return CBVH_OK;
}

}  // extern "C"
