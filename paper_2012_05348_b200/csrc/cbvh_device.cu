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
//   * distance variant: separating-axis lower bounds
//     (box gaps and the axis through the centres, reading R24) prune against
//     the pose's best distance, which a beam-search dive seeds with a real
//     leaf-pair distance before the traversal (R26); leaves use the exact
//     triangle–triangle distance (0 if they intersect).
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

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <atomic>

#include <cfloat>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/cbvh.h"
#include "cbvh_internal.h"
#include "leaf_geometry.cuh"

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
  int bits, width;   // b and stored field width (4 / 8 / 16; 16 / 32 for the absolute layouts)
  int layout;        // CBVH_LAYOUT_DELTA / _FP16 / _FP32
  uint32_t n_nodes, n_tris;  // bounds for the checked build
  uint32_t root_topo;
  int32_t root[6];   // decoded root lattice box
  int tlog;          // aligned treelet blocks: log2 T (node id = block << tlog | offset); -1: not staged
  int cb;            // code bytes per node (6 w / 8)
  const uint32_t* zoff;  // zero-suppressed codes: per-block region offsets (16-byte units from codes); else null
  int stage_ok;          // blocks can be staged (aligned, 16-byte multiples)
};

// k-DOP slab axes of the static model B beyond x, y, z (kdop/2 - 3 <= 10):
// per axis the lattice origin and cell
struct KDopB {
  float org[10], cell[10];
  int32_t root[20];  // node 0 decoded (lo, hi per axis)
};

constexpr int kMaxPhases = 8;

struct Control {
  unsigned int error;
  unsigned int pad0;
  unsigned int cursor[kMaxPhases];  // per phase: next pose (phase 0) / continuation item to acquire
  unsigned int count[kMaxPhases];   // per phase: items dumped for the next phase
  unsigned long long t_start, t_exhausted, t_end, dumped;  // globaltimer (stats variant), items dumped
  unsigned long long stats[8];
  unsigned long long t_frac[8];  // stats variant: when the pose cursor passed k/8 of N
  unsigned long long iterations; // stats variant: expansion passes (warp iterations)
  unsigned long long exact;      // stats variant: triangle pairs past the culls (exact Möller / distance)
  unsigned long long stage_blocks, stage_bytes, stage_reads;  // stats variant: treelet blocks staged in smem,
                                                              // their bytes, child records read from smem
};
constexpr size_t kCtlBytes = 512;  // workspace header holding the control block
static_assert(sizeof(Control) <= kCtlBytes, "control block must fit the workspace header");

#ifndef CBVH_MIN_BLOCKS_DIST
#define CBVH_MIN_BLOCKS_DIST 3
#endif
#ifndef CBVH_MIN_BLOCKS
#define CBVH_MIN_BLOCKS 5
#endif
#ifndef CBVH_WARPS
#define CBVH_WARPS 4
#endif
constexpr int kWarps = CBVH_WARPS;  // warps per CTA
#ifndef CBVH_STACK
#define CBVH_STACK 96
#endif
constexpr int kStack = CBVH_STACK;  // smem stack entries per warp
// entries moved to the global spill area when a pass's pushes would not fit:
// at least the 32 a pass can push (the stack may be full), at most what leaves
// the stack non-empty.  32 measured 0.5 % (config 5) to 1.3 % (config 4)
// faster than half the stack.
#ifndef CBVH_SPILL_H
#define CBVH_SPILL_H 32
#endif
static_assert(CBVH_SPILL_H >= 32 && CBVH_SPILL_H <= CBVH_STACK - 32, "a spill must make room for 32 pushes");
constexpr int kFields = 16;         // words per stack entry (AABB pairs)
// words per stack entry with KX extra k-DOP axes on B (their decoded lo, hi)
__host__ __device__ constexpr int nfields(int kx) { return kFields + 2 * kx; }
constexpr int kLeafQ = 64;          // leaf-queue entries per warp
constexpr int kSpillCap = 2048;     // global spill entries per warp
constexpr int kContCap = 1 << 19;   // continuation-buffer items (per buffer, two buffers)
constexpr int kGrabItems = 1;       // continuation items acquired per cursor atomic
#ifndef CBVH_GRAB
#define CBVH_GRAB 8
#endif
#ifndef CBVH_LOW_WATER
#define CBVH_LOW_WATER 4
#endif
#ifndef CBVH_POLL
#define CBVH_POLL 1
#endif
#ifndef CBVH_POLL_EVERY
#define CBVH_POLL_EVERY 128
#endif
constexpr unsigned kPoll = CBVH_POLL_EVERY;  // iterations between polls of the input cursor (power of two)
constexpr int kGrab = CBVH_GRAB;          // poses acquired per cursor atomic
constexpr int kLowWater = CBVH_LOW_WATER; // acquire poses when the stack is below this

// stack fields
enum { F_POSE = 0, F_TA = 1, F_TB = 2, F_BA = 3, F_BB = 9, F_LB = 15, F_XB = 16 };

struct Params {
  DevTree A, B;
  KDopB X;               // B's extra k-DOP axes (kernel instantiations with KX > 0)
  const float* poses;
  int N;
  uint8_t* hit;
  uint32_t* count;
  uint32_t* dist_bits;   // float bits of the running minimum distance
  Control* ctl;
  uint32_t* spill;       // [num_warps][kSpillCap][kFields]
  uint32_t* cont_in;     // continuation items of the previous phase [kContCap][kFields]
  uint32_t* cont_out;    // continuation items for the next phase
  int phase;             // 0: poses; >= 1: the previous phase's continuation items
  int nwarps;            // warps in the grid
  int budget;            // iterations a warp may run after its input is exhausted (< 0: unbounded)
  int descent;           // CBVH_DESCENT_SIMULTANEOUS (Alg. 1 verbatim) or CBVH_DESCENT_LARGER
  int early_exit;        // collide: stop a pose's traversal at its first hit
  int capped;            // distance: dist holds per-pose caps on entry (cbvh_query_opts.capped)
  int stage_slot_words;  // staging: words per smem slot (one treelet block: T topology words + T x cb code bytes)
  int stage_sides;       // staging: bit 0 tree A, bit 1 tree B (CBVH_STAGE_SIDES, tuning; default both)
  int bmax;              // the larger branching factor of the two trees (warp dive: lanes per beam entry)
};

// item pose word: bits 0..29 pose id, bit 30 = descend a, bit 31 = descend b
constexpr uint32_t kPoseMask = 0x3FFFFFFFu;

// Checked build (-DCBVH_CHECKED): device-side bounds checks of every node,
// triangle, pose and queue index; a violation sets CBVH_EINTERNAL in the error
// word (cbvh_check reports it).  compute-sanitizer is unavailable on the GPU
// pool, so this is the memory-safety evidence (tests/test_gpu_checked.py).
#ifdef CBVH_CHECKED
#define CBVH_GUARD(p, cond, fix) \
  do { if (!(cond)) { atomicExch(&(p).ctl->error, (unsigned)(-CBVH_EINTERNAL)); fix; } } while (0)
#else
#define CBVH_GUARD(p, cond, fix) do { } while (0)
#endif
#define CBVH_CHECK(p, cond) CBVH_GUARD(p, cond, (void)0)
constexpr uint32_t kDescA = 0x40000000u;
constexpr uint32_t kDescB = 0x80000000u;

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch (sm_90+): wait until the previous kernel of
// the stream has completed and its writes are visible; let the next kernel's
// CTAs become resident as soon as there is room for them.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Inclusive warp prefix sum: shfl.up's in-range predicate guards the add, so a
// step is two instructions (the intrinsic form compiles to a shuffle, a lane
// compare, a select and an add).
#ifndef CBVH_ASM_SCAN
#define CBVH_ASM_SCAN 1
#endif
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#if CBVH_ASM_SCAN
  (void)lane;
  #pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    asm volatile("{ .reg .s32 r; .reg .pred q; shfl.sync.up.b32 r|q, %0, %1, 0, 0xffffffff; @q add.s32 %0, %0, r; }"
                 : "+r"(v) : "r"(o));
#else
  #pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
#endif
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- decode

// FAST (template parameter of the decode helpers and of traverse_kernel): a
// blob format as compile-time constants, so the per-child format branches (and
// their constant loads) disappear from the kernel — 1: the default format
// (delta layout, b = 8 in 8-bit fields, codes not zero-suppressed), 2 / 3: the
// absolute binary16 / fp32 layouts of the paper's half-vs-float comparison
// (§III.A); 0: any format, decided at run time (the generic instantiation).
// 4 / 5: the delta layout in 4- / 16-bit fields (any b up to the field width;
// BJ config 3 sweeps b = 4, 8, 16), not zero-suppressed.
template <int FAST>
__device__ __forceinline__ int fast_layout(const DevTree& T) {
  return FAST == 0 ? T.layout : FAST == 2 ? CBVH_LAYOUT_FP16 : FAST == 3 ? CBVH_LAYOUT_FP32 : CBVH_LAYOUT_DELTA;
}
template <int FAST>
__device__ __forceinline__ int fast_width(const DevTree& T) {
  return FAST == 1 ? 8 : FAST == 4 ? 4 : FAST == 5 ? 16 : T.width;
}
template <int FAST = 0>
__device__ __forceinline__ void load_codes(const DevTree& T, uint32_t node, uint32_t q[6]) {
  const int width = fast_width<FAST>(T);
  if (width == 8) {
    const unsigned short* p = reinterpret_cast<const unsigned short*>(T.codes + 6ull * node);
    uint32_t a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    q[0] = a & 255u; q[1] = a >> 8; q[2] = b & 255u; q[3] = b >> 8; q[4] = c & 255u; q[5] = c >> 8;
  } else if (width == 16) {
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

#ifndef CBVH_ZS
#define CBVH_ZS 1
#endif
// Zero-suppressed codes (integer compression): node j
// of block b has presence mask m = region[j] (region = codes + 16 zoff[b]),
// and its non-zero fields follow, in field order, at byte
// T + (w/8) x (set bits of the masks of nodes 0..j-1).  From global memory
// the prefix is a popcount over the preceding mask bytes (<= 16 words).
__device__ __forceinline__ void load_codes_zs(const uint8_t* region, const uint8_t* fields0, uint32_t m, uint32_t before,
                                              int width, uint32_t q[6]) {
  const int wb = width >> 3;
  const uint8_t* x = fields0 + wb * before;
  #pragma unroll
  for (int f = 0; f < 6; ++f) {
    const bool on = (m >> f) & 1u;
    const uint32_t v = on ? (wb == 2 ? (uint32_t)x[0] | ((uint32_t)x[1] << 8) : (uint32_t)x[0]) : 0u;
    q[f] = v;
    x += on ? wb : 0;
  }
  (void)region;
}

// (returns the six fields packed in pairs, q0 | q1 << 16 ..., in registers)
__device__ __noinline__ uint3 load_codes_zs_global(const uint8_t* codes, const uint32_t* zoff, int tlog, int width,
                                                   uint32_t node) {
  uint32_t q[6];
  const uint32_t blk = node >> tlog, loc = node & ((1u << tlog) - 1u);
  const uint8_t* region = codes + 16ull * __ldg(zoff + blk);
  const uint32_t* mw = reinterpret_cast<const uint32_t*>(region);
  uint32_t before = 0;
  for (uint32_t k = 0; 4 * k < loc; ++k) {
    uint32_t wv = __ldg(mw + k);
    const uint32_t nb = loc - 4 * k;  // mask bytes of this word that precede node loc
    if (nb < 4) wv &= (1u << (8 * nb)) - 1u;
    before += __popc(wv);
  }
  const uint32_t m = __ldg(region + loc);
  load_codes_zs(region, region + (1u << tlog), m, before, width, q);
  return make_uint3(q[0] | (q[1] << 16), q[2] | (q[3] << 16), q[4] | (q[5] << 16));
}

// ---------------------------------------------------------------- node boxes
// A node's box travels as 6 words: lattice ints (DELTA) or fp32 bits
// (FP16 / FP32, absolute).  The child box comes from the parent's words
// (DELTA: predictor-corrector decode) or straight from the record.
template <int FAST = 0>
__device__ __forceinline__ void fetch_child_box(const DevTree& T, uint32_t node, const int32_t P[6], int32_t C[6]) {
  const int layout = fast_layout<FAST>(T);
  if (layout == CBVH_LAYOUT_DELTA) {
    uint32_t q[6];
    // (zero-suppressed blobs: an out-of-line call, so the common path keeps
    // its registers and code layout; CBVH_ZS=0 builds without the branch)
    if (FAST == 0 && CBVH_ZS && T.zoff) {
      const uint3 z = load_codes_zs_global(T.codes, T.zoff, T.tlog, T.width, node);
      q[0] = z.x & 0xffffu; q[1] = z.x >> 16; q[2] = z.y & 0xffffu; q[3] = z.y >> 16; q[4] = z.z & 0xffffu; q[5] = z.z >> 16;
    } else {
      load_codes<FAST>(T, node, q);
    }
    decode_child(P, q, FAST == 1 ? 8 : T.bits, C);  // (FAST 4 / 5: b at run time, one constant load)
  } else if (layout == CBVH_LAYOUT_FP16) {
    // binary16 descriptors (§III.A): widened exactly to fp32
    const uint32_t* w = reinterpret_cast<const uint32_t*>(T.codes + 12ull * node);
    const uint32_t a = __ldg(w), b = __ldg(w + 1), c = __ldg(w + 2);
    const uint32_t h[6] = {a & 0xffffu, a >> 16, b & 0xffffu, b >> 16, c & 0xffffu, c >> 16};
    #pragma unroll
    for (int k = 0; k < 6; ++k) C[k] = __float_as_int(__half2float(__ushort_as_half((unsigned short)h[k])));
  } else {
    const float2* w = reinterpret_cast<const float2*>(T.codes + 24ull * node);
    const float2 a = __ldg(w), b = __ldg(w + 1), c = __ldg(w + 2);
    C[0] = __float_as_int(a.x); C[1] = __float_as_int(a.y); C[2] = __float_as_int(b.x);
    C[3] = __float_as_int(b.y); C[4] = __float_as_int(c.x); C[5] = __float_as_int(c.y);
  }
}

template <int FAST = 0>
__device__ __forceinline__ void words_to_float(const DevTree& T, const int32_t C[6], float lo[3], float hi[3]) {
  if (fast_layout<FAST>(T) == CBVH_LAYOUT_DELTA) {
    to_float_box(T, C, lo, hi);
  } else {
    #pragma unroll
    for (int k = 0; k < 3; ++k) { lo[k] = __int_as_float(C[k]); hi[k] = __int_as_float(C[3 + k]); }
  }
}

// sum of the box's extents (the larger-first descent rule's size measure)
template <int FAST = 0>
__device__ __forceinline__ float words_extent(const DevTree& T, const int32_t C[6]) {
  if (fast_layout<FAST>(T) == CBVH_LAYOUT_DELTA)
    return (float)((C[3] - C[0]) + (C[4] - C[1]) + (C[5] - C[2])) * T.cell;
  return (__int_as_float(C[3]) - __int_as_float(C[0])) + (__int_as_float(C[4]) - __int_as_float(C[1])) +
         (__int_as_float(C[5]) - __int_as_float(C[2]));
}

struct PoseF {
  float R[3][3];
  float t[3];
};

// ---------------------------------------------------------------- k-DOP (B)
// Extra slab directions of a k-DOP (Table I; reading R22), in the
// builder's order — 14: the 4 body diagonals; 18: the 6 edge directions;
// 26: the diagonals, then the edges.  Integer components in {-1, 0, 1}.
__host__ __device__ constexpr int diag_dir(int a, int k) {
  // (1,1,1) (1,1,-1) (1,-1,1) (-1,1,1)
  return a == 0 ? 1 : a == 1 ? (k == 2 ? -1 : 1) : a == 2 ? (k == 1 ? -1 : 1) : (k == 0 ? -1 : 1);
}
__host__ __device__ constexpr int edge_dir(int a, int k) {
  // (1,1,0) (1,-1,0) (1,0,1) (1,0,-1) (0,1,1) (0,1,-1)
  return k == (a < 4 ? 0 : 1) ? 1 : k == (a < 2 ? 1 : 2) ? ((a & 1) ? -1 : 1) : 0;
}
__host__ __device__ constexpr int kdop_dir(int kx, int a, int k) {
  return (kx == 6 || (kx == 10 && a >= 4)) ? edge_dir(kx == 10 ? a - 4 : a, k) : diag_dir(a, k);
}

// the 2 * NAX stored fields of a k-DOP record: lo of the NAX axes, then hi
template <int NAX>
__device__ __forceinline__ void load_codes_k(const DevTree& T, uint32_t node, uint32_t q[2 * NAX]) {
  if (T.width == 8) {
    const unsigned short* p = reinterpret_cast<const unsigned short*>(T.codes + 2ull * NAX * node);
    #pragma unroll
    for (int i = 0; i < NAX; ++i) { const uint32_t a = __ldg(p + i); q[2 * i] = a & 255u; q[2 * i + 1] = a >> 8; }
  } else if (T.width == 16) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(T.codes + 4ull * NAX * node);
    #pragma unroll
    for (int i = 0; i < NAX; ++i) { const uint32_t a = __ldg(p + i); q[2 * i] = a & 0xffffu; q[2 * i + 1] = a >> 16; }
  } else {
    const uint8_t* p = T.codes + (uint64_t)NAX * node;
    #pragma unroll
    for (int i = 0; i < NAX; ++i) { const uint32_t a = __ldg(p + i); q[2 * i] = a & 15u; q[2 * i + 1] = a >> 4; }
  }
}

// child k-DOP from the decoded parent (box P, extra axes PX): the same
// predictor-corrector step per axis as decode_child
template <int KX>
__device__ __forceinline__ void fetch_child_kdop(const DevTree& T, uint32_t node, const int32_t P[6],
                                                 const int32_t* PX, int32_t C[6], int32_t* CX) {
  constexpr int NAX = 3 + KX;
  uint32_t q[2 * NAX];
  load_codes_k<NAX>(T, node, q);
  #pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int s = max(0, (32 - __clz(P[3 + a] - P[a])) - T.bits);
    C[a] = P[a] + (int32_t)(q[a] << s);
    C[3 + a] = P[3 + a] - (int32_t)(q[NAX + a] << s);
  }
  #pragma unroll
  for (int a = 0; a < KX; ++a) {
    const int s = max(0, (32 - __clz(PX[2 * a + 1] - PX[2 * a])) - T.bits);
    CX[2 * a] = PX[2 * a] + (int32_t)(q[3 + a] << s);
    CX[2 * a + 1] = PX[2 * a + 1] - (int32_t)(q[NAX + 3 + a] << s);
  }
}

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

#ifndef CBVH_DIST_BOXB
#define CBVH_DIST_BOXB 5  // world-AABB gap + centre axis: 4 alone is 2-4 % faster at config 4 but 17 % slower on config 2 distance; 7 no tighter
#endif
#ifndef CBVH_DIST_LEAFB
#define CBVH_DIST_LEAFB 4  // centroid axis only: 1 | 2 | 4 prune the same, measured 12 % slower (config 4)
#endif
#ifndef CBVH_SAT_EDGES
#define CBVH_SAT_EDGES 0
#endif
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
  float ga[3], Ta[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    Ta[k] = fmaf(P.R[0][k], Tw[0], fmaf(P.R[1][k], Tw[1], P.R[2][k] * Tw[2]));
    float rb = fmaf(fabsf(P.R[0][k]), hb[0], fmaf(fabsf(P.R[1][k]), hb[1], fabsf(P.R[2][k]) * hb[2]));
    ga[k] = fabsf(Ta[k]) - (ha[k] + rb);
    gmax = fmaxf(gmax, ga[k]);
  }
#if CBVH_SAT_EDGES
  if (!WANT_LB && gmax <= eps) {
    // the 9 edge axes L = A_i x e_j (Gottschalk's OBB test): A's
    // columns are orthonormal up to ~1e-7, so A's radius on L uses
    // A_k x A_i = +-A_m; the unnormalised gap (|L| <= 1) is compared with eps
    #pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
      #pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        // L = A_i x e_j: L[j] = 0, L[j1] = A_i[j2], L[j2] = -A_i[j1]
        const float l1 = P.R[j2][i], l2 = -P.R[j1][i];
        const float tl = fmaf(Tw[j1], l1, Tw[j2] * l2);
        const float ra = fmaf(ha[i1], fabsf(P.R[j][i2]), ha[i2] * fabsf(P.R[j][i1]));
        const float rb = fmaf(hb[j1], fabsf(l1), hb[j2] * fabsf(l2));
        gmax = fmaxf(gmax, fabsf(tl) - (ra + rb));
      }
    }
  }
#endif
  if (WANT_LB) {
    // lower bounds on the box distance, CBVH_DIST_BOXB bits: 1 the Euclidean
    // gap of b against the world AABB of a, 2 of a against the A-frame AABB
    // of b (both contain the posed boxes), 4 the axis through the two box
    // centres, u = Tw / |Tw|: |Tw| less the radii of both boxes on u (A's
    // from Ta = R^T Tw) — nearly the true distance for boxes far apart
    // relative to their size
    float l = 0.f;
    if (CBVH_DIST_BOXB & 1) {
      const float g0 = fmaxf(gw[0], 0.f), g1 = fmaxf(gw[1], 0.f), g2 = fmaxf(gw[2], 0.f);
      l = sqrtf(fmaf(g0, g0, fmaf(g1, g1, g2 * g2)));
    }
    if (CBVH_DIST_BOXB & 2) {
      const float g0 = fmaxf(ga[0], 0.f), g1 = fmaxf(ga[1], 0.f), g2 = fmaxf(ga[2], 0.f);
      l = fmaxf(l, sqrtf(fmaf(g0, g0, fmaf(g1, g1, g2 * g2))));
    }
    if (CBVH_DIST_BOXB & 4) {
      const float T2 = fmaf(Tw[0], Tw[0], fmaf(Tw[1], Tw[1], Tw[2] * Tw[2]));
      const float rs = fmaf(ha[0], fabsf(Ta[0]), fmaf(ha[1], fabsf(Ta[1]), fmaf(ha[2], fabsf(Ta[2]),
                       fmaf(hb[0], fabsf(Tw[0]), fmaf(hb[1], fabsf(Tw[1]), hb[2] * fabsf(Tw[2]))))));
      l = fmaxf(l, T2 > 0.f ? (T2 - rs) * rsqrtf(T2) : 0.f);
    }
    *lb = fmaxf(l, 0.f) - eps;
  }
  return gmax - eps;
}

// A's box (A-local, under pose P) against B's extra k-DOP slabs: the gap
// along each direction d (unnormalised, |d|_1 <= 3) between the projection
// interval of the posed box and B's slab, less |d|_1 eps for the rounding of
// the projections, divided by |d|_2 (reciprocal rounded down) — a lower bound
// on the separation along the unit direction; > 0 means separated.
template <int KX>
__device__ __forceinline__ float kdop_gap(const PoseF& P, const float alo[3], const float ahi[3],
                                          const KDopB& X, const int32_t* CX, float eps) {
  float ca[3], ha[3], wc[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    ca[k] = 0.5f * (alo[k] + ahi[k]);
    ha[k] = 0.5f * (ahi[k] - alo[k]);
  }
  #pragma unroll
  for (int k = 0; k < 3; ++k) wc[k] = fmaf(P.R[k][0], ca[0], fmaf(P.R[k][1], ca[1], fmaf(P.R[k][2], ca[2], P.t[k])));
  float g = -FLT_MAX;
  #pragma unroll
  for (int a = 0; a < KX; ++a) {
    const float d0 = (float)kdop_dir(KX, a, 0), d1 = (float)kdop_dir(KX, a, 1), d2 = (float)kdop_dir(KX, a, 2);
    const float c = d0 * wc[0] + d1 * wc[1] + d2 * wc[2];
    float r = 0.f;
    #pragma unroll
    for (int i = 0; i < 3; ++i) r = fmaf(fabsf(d0 * P.R[0][i] + d1 * P.R[1][i] + d2 * P.R[2][i]), ha[i], r);
    const float xlo = __fmaf_rd(__int2float_rn(CX[2 * a]), X.cell[a], X.org[a]);
    const float xhi = __fmaf_ru(__int2float_rn(CX[2 * a + 1]), X.cell[a], X.org[a]);
    const float gap = fmaxf(xlo - (c + r), (c - r) - xhi);
    const bool diag = kdop_dir(KX, a, 0) != 0 && kdop_dir(KX, a, 1) != 0 && kdop_dir(KX, a, 2) != 0;
    g = fmaxf(g, (gap - (diag ? 3.f : 2.f) * eps) * (diag ? 0.57735020f : 0.70710670f));
  }
  return g;
}

// ---------------------------------------------------------------- leaf tests

using Tri = TriT<float>;
using Tri64 = TriT<double>;

// 48-byte triangle records: three 16-byte vector loads
__device__ __forceinline__ Tri load_tri(const float* tris, uint32_t i) {
  const float4* p = reinterpret_cast<const float4*>(tris + 12ull * i);
  const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  Tri T;
  T.v[0][0] = a.x; T.v[0][1] = a.y; T.v[0][2] = a.z;
  T.v[1][0] = a.w; T.v[1][1] = b.x; T.v[1][2] = b.y;
  T.v[2][0] = b.z; T.v[2][1] = b.w; T.v[2][2] = c.x;
  return T;
}

// B's world triangle into A's local frame: u = R^T (v - t).  Near contact
// |v - t| is small, so the subtraction is (almost) exact and the local-frame
// error stays ~1e-7 even at |t| = 50 (SURVEY §8(c) reading R12).
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

__device__ __forceinline__ bool tri_boxes_overlap(const Tri& V, const Tri& U) {
  bool ok = true;
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float vlo = fminf(V.v[0][k], fminf(V.v[1][k], V.v[2][k]));
    const float vhi = fmaxf(V.v[0][k], fmaxf(V.v[1][k], V.v[2][k]));
    const float ulo = fminf(U.v[0][k], fminf(U.v[1][k], U.v[2][k]));
    const float uhi = fmaxf(U.v[0][k], fmaxf(U.v[1][k], U.v[2][k]));
    ok = ok && !(vhi < ulo || uhi < vlo);
  }
  return ok;
}

// Conservative box–triangle overlap (separating-axis test, Akenine-Möller's
// triangle–box formulation): the 3 box axes, the triangle normal and, with
// CBVH_TRIBOX_EDGES, the 9 edge x box-axis crosses.  Testing fewer axes
// only makes the filter looser, never wrong; eps covers fp32 rounding.
#ifndef CBVH_TRIBOX_EDGES
#define CBVH_TRIBOX_EDGES 0
#endif
// the leaf filter maps triangles straight to box-centred coordinates (the
// pose offset and the box centre folded into one FMA chain per coordinate)
#ifndef CBVH_FOLD_CENTRE
#define CBVH_FOLD_CENTRE 1
#endif
// axes of the box-triangle filter: 1 the box axes, 2 the triangle normal —
// for A's boxes against B's triangles (DIR 0) and B's boxes against A's (DIR 1)
#ifndef CBVH_COL_LEAFB0
#define CBVH_COL_LEAFB0 3
#endif
#ifndef CBVH_COL_LEAFB1
#define CBVH_COL_LEAFB1 1  // box axes only: B's boxes against A's small triangles (measured 2-5 % faster than 3 on configs 5, 3, 2)
#endif
#ifndef CBVH_PAIR_AFILTER
#define CBVH_PAIR_AFILTER 2
#endif
#ifndef CBVH_PAIR_RATIO
#define CBVH_PAIR_RATIO 1.5f  // measured: config 5 -4.5 %, configs 3 / 2 +1 / +2 % (always: config 3 -3.5 %; never: config 5 +6 %)
#endif
// (The early return after the box axes stays: straight-line code without it
// measured 1 % slower on config 5 and 3 % on config 3 — whole warps do leave
// here.  The same for Möller's plane rejections: neutral.)
template <int AXES>
__device__ __forceinline__ bool box_tri_overlap(const float c[3], const float h[3], const Tri& T, float eps) {
  float v[3][3];
  #pragma unroll
  for (int q = 0; q < 3; ++q)
    #pragma unroll
    for (int k = 0; k < 3; ++k) v[q][k] = CBVH_FOLD_CENTRE ? T.v[q][k] : T.v[q][k] - c[k];  // box-centred
  bool sep = false;
  if (AXES & 1) {
    #pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float tlo = fminf(v[0][k], fminf(v[1][k], v[2][k]));
      const float thi = fmaxf(v[0][k], fmaxf(v[1][k], v[2][k]));
      sep = sep || tlo > h[k] + eps || thi < -h[k] - eps;
    }
    if (sep) return false;
  }
  float e[3][3];
  vsub(v[1], v[0], e[0]);
  vsub(v[2], v[1], e[1]);
  vsub(v[0], v[2], e[2]);
  if (AXES & 2) {
    float n[3];
    vcross(e[0], e[1], n);
    const float nrm = fabsf(n[0]) + fabsf(n[1]) + fabsf(n[2]);
    const float rad_n = fmaf(fabsf(n[0]), h[0], fmaf(fabsf(n[1]), h[1], fabsf(n[2]) * h[2]));
    sep = sep || fabsf(vdot(n, v[0])) > fmaf(eps, nrm, rad_n);
  }
  if (sep) return false;
#if CBVH_TRIBOX_EDGES
  #pragma unroll
  for (int i = 0; i < 3; ++i) {
    // axis a = e_i x unit_k: only two components are non-zero
    #pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int k1 = (k + 1) % 3, k2 = (k + 2) % 3;
      // a = e_i x u_k  ->  a[k1] = e[i][k2], a[k2] = -e[i][k1]
      const float a1 = e[i][k2], a2 = -e[i][k1];
      const float p0 = a1 * v[0][k1] + a2 * v[0][k2];
      const float p1 = a1 * v[1][k1] + a2 * v[1][k2];
      const float p2 = a1 * v[2][k1] + a2 * v[2][k2];
      const float r = fabsf(a1) * h[k1] + fabsf(a2) * h[k2];
      const float sl = eps * (fabsf(a1) + fabsf(a2));
      if (fminf(p0, fminf(p1, p2)) > r + sl || fmaxf(p0, fmaxf(p1, p2)) < -r - sl) return false;
    }
  }
#endif
  return true;
}

// Triangle q of a leaf as three 16-byte vectors.
struct TriRec {
  float4 a, b, c;
};
__device__ __forceinline__ TriRec load_rec(const float* tris, uint32_t i) {
  const float4* p = reinterpret_cast<const float4*>(tris + 12ull * i);
  return TriRec{__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}
__device__ __forceinline__ Tri rec_tri(const TriRec& r) {
  Tri T;
  T.v[0][0] = r.a.x; T.v[0][1] = r.a.y; T.v[0][2] = r.a.z;
  T.v[1][0] = r.a.w; T.v[1][1] = r.b.x; T.v[1][2] = r.b.y;
  T.v[2][0] = r.b.z; T.v[2][1] = r.b.w; T.v[2][2] = r.c.x;
  return T;
}


// The box (centre c, half extents h) against the triangles of a leaf, each
// mapped into the box's frame (DIR 0: B's world triangles into A's frame by
// R^T (v - t); DIR 1: A's local triangles into the world by R v + t).  Bit q
// of the result: triangle q of the leaf may touch the box.  The next
// triangle's record is fetched while the current one is tested.
#ifndef CBVH_FILTER_INLINE
#define CBVH_FILTER_INLINE 1
#endif
#if CBVH_FILTER_INLINE
#define CBVH_FILTER_ATTR __forceinline__
#else
#define CBVH_FILTER_ATTR __noinline__
#endif
// Only the triangles in `todo` are tested: a triangle the parent box missed
// cannot touch the child box (child ⊆ parent, same eps), so the mask an item
// inherits from its parent's refinement is a valid starting set.
// PF: the next triangle's record is fetched while the current one is tested —
// worth 6 % at 5 CTAs / SM (round 1: 95 -> 89 ms), but at the FAST kernels' 7
// CTAs the other warps hide the latency and the 12 registers of the
// prefetched record cost more: without it config 5 37.2 -> 36.3 ms, config 3
// 41.9 -> 41.1, config 2 3.56 -> 3.43 and no spills at 72 registers
// (profiles/round2_ab_prefetch.txt).
template <int DIR, bool PF = true>
__device__ CBVH_FILTER_ATTR uint32_t box_hits_leaf(const PoseF& P, const float lo[3], const float hi[3],
                                               const float* tris, uint32_t leaf, float eps, uint32_t todo) {
  const uint32_t first = leaf & 0x1FFFFFFFu;
  todo &= (2u << ((leaf >> 29) & 3u)) - 1u;
  float c[3], h[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) { c[k] = 0.5f * (lo[k] + hi[k]); h[k] = 0.5f * (hi[k] - lo[k]); }
#if CBVH_FOLD_CENTRE
  float off[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k)
    off[k] = DIR == 0 ? -fmaf(P.R[0][k], P.t[0], fmaf(P.R[1][k], P.t[1], fmaf(P.R[2][k], P.t[2], c[k]))) : P.t[k] - c[k];
#endif
  uint32_t m = 0;
  if (todo == 0u) return 0u;
  uint32_t qn = (uint32_t)__ffs(todo) - 1u;
  todo &= todo - 1u;
  TriRec next;
  if (PF) next = load_rec(tris, first + qn);
  #pragma unroll 1
  while (true) {
    const uint32_t q = qn;
    TriRec cur;
    if (PF) cur = next; else cur = load_rec(tris, first + q);
    const bool more = todo != 0u;
    if (more) {
      qn = (uint32_t)__ffs(todo) - 1u;
      todo &= todo - 1u;
      if (PF) next = load_rec(tris, first + qn);
    }
    const Tri L = rec_tri(cur);
    Tri W;
#if CBVH_FOLD_CENTRE
    // DIR 0: w = R^T v - (R^T t + c); DIR 1: w = R v + (t - c) — the filter
    // is conservative by eps, which covers the rounding of the folded offset
    #pragma unroll
    for (int v = 0; v < 3; ++v)
      #pragma unroll
      for (int k = 0; k < 3; ++k)
        W.v[v][k] = DIR == 0 ? fmaf(P.R[0][k], L.v[v][0], fmaf(P.R[1][k], L.v[v][1], fmaf(P.R[2][k], L.v[v][2], off[k])))
                             : fmaf(P.R[k][0], L.v[v][0], fmaf(P.R[k][1], L.v[v][1], fmaf(P.R[k][2], L.v[v][2], off[k])));
#else
    if (DIR == 0) {
      W = to_local(P, L);
    } else {
      #pragma unroll
      for (int v = 0; v < 3; ++v)
        #pragma unroll
        for (int k = 0; k < 3; ++k)
          W.v[v][k] = fmaf(P.R[k][0], L.v[v][0], fmaf(P.R[k][1], L.v[v][1], fmaf(P.R[k][2], L.v[v][2], P.t[k])));
    }
#endif
    if (box_tri_overlap<DIR == 0 ? CBVH_COL_LEAFB0 : CBVH_COL_LEAFB1>(c, h, W, eps)) m |= 1u << q;
    if (!more) break;
  }
  return m;
}

// Distance variant of the leaf refinement: per triangle of the leaf (mapped
// into the box's frame as above) a lower bound on its distance to the box —
// the larger of the gap between the box and the triangle's AABB and the gap
// along the triangle's normal (separating axes: a lower bound on the distance
// between the convex sets), less 2 eps.  Bit q: triangle q's bound is below
// `best`; *lbmin = the smallest bound over the leaf's triangles.
// collide: an item carries the leaf-triangle masks of its refinement, so a
// child box is tested only against the triangles its parent box touched
#ifndef CBVH_MASK_PROP
#define CBVH_MASK_PROP 1
#endif
#ifndef CBVH_DIST_FILTER
#define CBVH_DIST_FILTER 1
#endif
#ifndef CBVH_NEAR_NATIVE
#define CBVH_NEAR_NATIVE 1  // the leaf bound in the triangle's frame (no vertex transform)
#endif
template <int DIR>
__device__ CBVH_FILTER_ATTR uint32_t box_near_leaf(const PoseF& P, const float lo[3], const float hi[3],
                                               const float* tris, uint32_t leaf, float eps, float best,
                                               float* lbmin, uint32_t todo) {
  // only the triangles in `todo`: one the parent box's bound already put at
  // or beyond the pose's best stays there for the child box (child ⊆ parent,
  // best only decreases)
  const uint32_t first = leaf & 0x1FFFFFFFu;
  todo &= (2u << ((leaf >> 29) & 3u)) - 1u;
  float c[3], h[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) { c[k] = 0.5f * (lo[k] + hi[k]); h[k] = 0.5f * (hi[k] - lo[k]); }
  uint32_t m = 0;
  float lbm = FLT_MAX;
  *lbmin = lbm;
  if (todo == 0u) return 0u;
#if CBVH_DIST_LEAFB == 4 && CBVH_NEAR_NATIVE
  // the box centre in the triangles' frame: DIR 0 world, R c + t; DIR 1 A-local, R^T (c - t)
  float cf[3];
  {
    const float e0 = c[0] - P.t[0], e1 = c[1] - P.t[1], e2 = c[2] - P.t[2];
    #pragma unroll
    for (int k = 0; k < 3; ++k)
      cf[k] = DIR == 0 ? fmaf(P.R[k][0], c[0], fmaf(P.R[k][1], c[1], fmaf(P.R[k][2], c[2], P.t[k])))
                       : fmaf(P.R[0][k], e0, fmaf(P.R[1][k], e1, P.R[2][k] * e2));
  }
#endif
  uint32_t qn = (uint32_t)__ffs(todo) - 1u;
  todo &= todo - 1u;
  TriRec next = load_rec(tris, first + qn);
  #pragma unroll 1
  while (true) {
    const TriRec cur = next;
    const uint32_t q = qn;
    const bool more = todo != 0u;
    if (more) {
      qn = (uint32_t)__ffs(todo) - 1u;
      todo &= todo - 1u;
      next = load_rec(tris, first + qn);
    }
    const Tri L = rec_tri(cur);
#if CBVH_DIST_LEAFB == 4 && CBVH_NEAR_NATIVE
    // the centroid-axis bound in the triangle's own frame: only the box
    // centre is mapped (once per lane, cf above), and the box's radius along
    // the axis s = 3 x (centroid - centre) uses the box axes as they appear in
    // this frame — the columns (DIR 0) / rows (DIR 1) of R.  No vertex is
    // transformed: 44 instead of ~75 operations per triangle.
    {
      float d[3][3], sv[3], a[3];
      #pragma unroll
      for (int u = 0; u < 3; ++u)
        #pragma unroll
        for (int k = 0; k < 3; ++k) d[u][k] = L.v[u][k] - cf[k];
      #pragma unroll
      for (int k = 0; k < 3; ++k) sv[k] = d[0][k] + d[1][k] + d[2][k];
      const float c2 = fmaf(sv[0], sv[0], fmaf(sv[1], sv[1], sv[2] * sv[2]));
      const float pmin = fminf(vdot(sv, d[0]), fminf(vdot(sv, d[1]), vdot(sv, d[2])));
      #pragma unroll
      for (int k = 0; k < 3; ++k)
        a[k] = DIR == 0 ? fmaf(P.R[0][k], sv[0], fmaf(P.R[1][k], sv[1], P.R[2][k] * sv[2]))
                        : fmaf(P.R[k][0], sv[0], fmaf(P.R[k][1], sv[1], P.R[k][2] * sv[2]));
      const float rb = fmaf(fabsf(a[0]), h[0], fmaf(fabsf(a[1]), h[1], fabsf(a[2]) * h[2]));
      const float lb = (c2 > 0.f ? (pmin - rb) * rsqrtf(c2) : 0.f) - 2.f * eps;
      if (lb < best) m |= 1u << q;
      lbm = fminf(lbm, lb);
      if (!more) break;
    }
#else
    float v[3][3];
    #pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (DIR == 0) {
        const float d0 = L.v[u][0] - P.t[0], d1 = L.v[u][1] - P.t[1], d2 = L.v[u][2] - P.t[2];
        #pragma unroll
        for (int k = 0; k < 3; ++k) v[u][k] = fmaf(P.R[0][k], d0, fmaf(P.R[1][k], d1, P.R[2][k] * d2)) - c[k];
      } else {
        #pragma unroll
        for (int k = 0; k < 3; ++k)
          v[u][k] = fmaf(P.R[k][0], L.v[u][0], fmaf(P.R[k][1], L.v[u][1], fmaf(P.R[k][2], L.v[u][2], P.t[k]))) - c[k];
      }
    }
    // separating-axis gaps (each a lower bound on the box-triangle
    // distance), CBVH_DIST_LEAFB bits: 1 the box axes (triangle AABB gap),
    // 2 the triangle normal, 4 the box-centre-to-centroid axis
    float lb = 0.f;
    if (CBVH_DIST_LEAFB & 1) {
      float g2 = 0.f;
      #pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float tlo = fminf(v[0][k], fminf(v[1][k], v[2][k]));
        const float thi = fmaxf(v[0][k], fmaxf(v[1][k], v[2][k]));
        const float g = fmaxf(0.f, fmaxf(tlo - h[k], -h[k] - thi));
        g2 = fmaf(g, g, g2);
      }
      lb = sqrtf(g2);
    }
    if (CBVH_DIST_LEAFB & 2) {
      float e1[3], e2[3], n[3];
      vsub(v[1], v[0], e1);
      vsub(v[2], v[0], e2);
      vcross(e1, e2, n);
      const float nn = vdot(n, n);
      const float rad_n = fmaf(fabsf(n[0]), h[0], fmaf(fabsf(n[1]), h[1], fabsf(n[2]) * h[2]));
      lb = fmaxf(lb, nn > 0.f ? (fabsf(vdot(n, v[0])) - rad_n) * rsqrtf(nn) : 0.f);
    }
    if (CBVH_DIST_LEAFB & 4) {
      // the axis from the box centre (the origin here) to the triangle's
      // centroid: the triangle's nearest projection less the box radius
      float ct[3];
      #pragma unroll
      for (int k = 0; k < 3; ++k) ct[k] = (v[0][k] + v[1][k] + v[2][k]) * (1.f / 3.f);
      const float c2 = fmaf(ct[0], ct[0], fmaf(ct[1], ct[1], ct[2] * ct[2]));
      const float pmin = fminf(vdot(ct, v[0]), fminf(vdot(ct, v[1]), vdot(ct, v[2])));
      const float rb = fmaf(fabsf(ct[0]), h[0], fmaf(fabsf(ct[1]), h[1], fabsf(ct[2]) * h[2]));
      lb = fmaxf(lb, c2 > 0.f ? (pmin - rb) * rsqrtf(c2) : 0.f);
    }
    lb -= 2.f * eps;
    if (lb < best) m |= 1u << q;
    lbm = fminf(lbm, lb);
    if (!more) break;
#endif
  }
  *lbmin = lbm;
  return m;
}

#ifndef CBVH_DRAIN_INLINE
#define CBVH_DRAIN_INLINE 1
#endif
#if CBVH_DRAIN_INLINE
#define CBVH_DRAIN_ATTR __forceinline__
#else
#define CBVH_DRAIN_ATTR __noinline__
#endif
#ifndef CBVH_EE_ORDER
#define CBVH_EE_ORDER 1  // early-exit collide: deepest overlap on top (config 5 -8 %, config 3 -2 %, config 2 +3 %)
#endif
#ifndef CBVH_EE_DRAIN
#define CBVH_EE_DRAIN 4  // early-exit collide: drain the leaf queue at this many pairs (64 / 16 / 4 / 1 measured: 4 best, config 3 -22 %)
#endif
#ifndef CBVH_DRAIN_AABB
#define CBVH_DRAIN_AABB 0  // collide: triangle-AABB cull before Möller in the leaf drain (measured 2-3 % slower: Möller's plane tests reject as early)
#endif
#ifndef CBVH_DIST_DRAIN
#define CBVH_DIST_DRAIN 32  // distance: drain the leaf queue once it holds this many pairs (2 / 8 / 16 / 32 measured: 32 best, -8..-20 %)
#endif
#ifndef CBVH_LEAF_SLAB
#define CBVH_LEAF_SLAB 0
#endif

// A box against the slab of a leaf (the range [dmin, dmax] of n.v over the
// leaf's vertices, stored in the triangle records' pads — DESIGN.md §3): the
// box, as an oriented box in the leaf's frame, is projected on n.
// DIR 0: A's box (A-local) vs a B leaf (world): centre R c + t, radius sum_m |n.R_m| h_m
// DIR 1: B's box (world) vs an A leaf (A-local): centre R^T (c - t), radius sum_k |(R n)_k| h_k
template <int DIR>
__device__ __forceinline__ bool box_vs_slab(const PoseF& P, const float lo[3], const float hi[3],
                                            const float* tris, uint32_t leaf, float eps) {
  const uint32_t first = leaf & 0x1FFFFFFFu, cnt = ((leaf >> 29) & 3u) + 1;
  const float4* r0 = reinterpret_cast<const float4*>(tris + 12ull * first);
  const float4 c0 = __ldg(r0 + 2);
  const float n[3] = {c0.y, c0.z, c0.w};
  float dlo, dhi;
  if (cnt > 1) {
    const float4 c1 = __ldg(reinterpret_cast<const float4*>(tris + 12ull * (first + 1)) + 2);
    dlo = c1.y;
    dhi = c1.z;
  } else {
    const float4 a0 = __ldg(r0), b0 = __ldg(r0 + 1);
    const float d0 = fmaf(n[0], a0.x, fmaf(n[1], a0.y, n[2] * a0.z));
    const float d1 = fmaf(n[0], a0.w, fmaf(n[1], b0.x, n[2] * b0.y));
    const float d2 = fmaf(n[0], b0.z, fmaf(n[1], b0.w, n[2] * c0.x));
    dlo = fminf(d0, fminf(d1, d2));
    dhi = fmaxf(d0, fmaxf(d1, d2));
  }
  float cw[3], rad = 0.f;
  #pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float cr = 0.5f * (lo[r] + hi[r]), hr = 0.5f * (hi[r] - lo[r]);
    // projection of the box's axis r on n
    const float nr = DIR == 0 ? fmaf(n[0], P.R[0][r], fmaf(n[1], P.R[1][r], n[2] * P.R[2][r]))
                              : fmaf(n[0], P.R[r][0], fmaf(n[1], P.R[r][1], n[2] * P.R[r][2]));
    rad = fmaf(fabsf(nr), hr, rad);
    cw[r] = cr;
  }
  float s;
  if (DIR == 0) {
    float x[3];
    #pragma unroll
    for (int k = 0; k < 3; ++k) x[k] = fmaf(P.R[k][0], cw[0], fmaf(P.R[k][1], cw[1], fmaf(P.R[k][2], cw[2], P.t[k])));
    s = fmaf(n[0], x[0], fmaf(n[1], x[1], n[2] * x[2]));
  } else {
    const float d0 = cw[0] - P.t[0], d1 = cw[1] - P.t[1], d2 = cw[2] - P.t[2];
    float x[3];
    #pragma unroll
    for (int k = 0; k < 3; ++k) x[k] = fmaf(P.R[0][k], d0, fmaf(P.R[1][k], d1, P.R[2][k] * d2));
    s = fmaf(n[0], x[0], fmaf(n[1], x[1], n[2] * x[2]));
  }
  return s + rad + 2.f * eps >= dlo && s - rad - 2.f * eps <= dhi;
}

// packed list of the set bits of a <= 4-bit mask: 2-bit indices, count
__device__ __forceinline__ uint32_t pack_list(uint32_t m) {
  uint32_t list = 0, n = 0;
  #pragma unroll
  for (int q = 0; q < 4; ++q)
    if (m & (1u << q)) { list |= (uint32_t)q << (2 * n); ++n; }
  return list | (n << 8);
}

// Euclidean gap between the AABBs of two triangles (a lower bound on their
// distance)
__device__ __forceinline__ float tri_box_gap(const Tri& V, const Tri& U) {
  float g2 = 0.f;
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float vlo = fminf(V.v[0][k], fminf(V.v[1][k], V.v[2][k]));
    const float vhi = fmaxf(V.v[0][k], fmaxf(V.v[1][k], V.v[2][k]));
    const float ulo = fminf(U.v[0][k], fminf(U.v[1][k], U.v[2][k]));
    const float uhi = fmaxf(U.v[0][k], fmaxf(U.v[1][k], U.v[2][k]));
    const float g = fmaxf(0.f, fmaxf(ulo - vhi, vlo - uhi));
    g2 = fmaf(g, g, g2);
  }
  return sqrtf(g2);
}

// Gap between two triangles along the line through their centroids (a
// separating-axis lower bound on their distance; for small triangles far
// apart it is within ~size^2 / distance of the true distance, where the AABB
// gap is off by ~size x tilt).  Projections are taken relative to V's
// centroid so the magnitudes stay small.
#ifndef CBVH_DIST_TRIB
#define CBVH_DIST_TRIB 3
#endif
__device__ __forceinline__ float tri_axis_gap(const Tri& V, const Tri& U) {
  float cv[3], u[3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    cv[k] = (V.v[0][k] + V.v[1][k] + V.v[2][k]) * (1.f / 3.f);
    u[k] = (U.v[0][k] + U.v[1][k] + U.v[2][k]) * (1.f / 3.f) - cv[k];
  }
  const float L2 = fmaf(u[0], u[0], fmaf(u[1], u[1], u[2] * u[2]));
  if (!(L2 > 0.f)) return 0.f;
  float vmax = -FLT_MAX, umin = FLT_MAX;
  #pragma unroll
  for (int q = 0; q < 3; ++q) {
    vmax = fmaxf(vmax, fmaf(u[0], V.v[q][0] - cv[0], fmaf(u[1], V.v[q][1] - cv[1], u[2] * (V.v[q][2] - cv[2]))));
    umin = fminf(umin, fmaf(u[0], U.v[q][0] - cv[0], fmaf(u[1], U.v[q][1] - cv[1], u[2] * (U.v[q][2] - cv[2]))));
  }
  return (umin - vmax) * rsqrtf(L2);
}

// The rare cases of Möller's test (coplanar or touching planes, zero-area
// triangles) for triangle pair (ia, ib) under pose `pose`: the triangles are
// re-read and re-mapped (bit-identical to the caller's copies) rather than
// passed by reference, so the common register path never writes them to
// local memory.
__device__ __noinline__ bool overlap_rare(const Params& p, uint32_t pose, uint32_t ia, uint32_t ib) {
  const PoseF P = load_pose(p.poses, (int)pose);
  const Tri TA = load_tri(p.A.tris, ia);
  const Tri TB = to_local(P, load_tri(p.B.tris, ib));
  return tri_tri_overlap(TA, TB);
}

// fp64 re-evaluation of a near-contact distance candidate,
// in the world frame as the distance is defined: A's fp32
// triangle mapped by the fp32 pose lifted exactly to fp64, B's fp32 triangle
// as is.  (The fp32 path works in A's frame with R^T, whose ~1e-7
// non-orthonormality is an absolute error that a 1e-5 relative bound cannot
// absorb at small distances.)
__device__ __noinline__ float tri_dist_fp64(const PoseF& P, const float* trisA, uint32_t ia,
                                            const float* trisB, uint32_t ib) {
  Tri64 a, b;
  const Tri TA = load_tri(trisA, ia), TB = load_tri(trisB, ib);
  #pragma unroll
  for (int v = 0; v < 3; ++v) {
    #pragma unroll
    for (int k = 0; k < 3; ++k) {
      a.v[v][k] = fma((double)P.R[k][0], (double)TA.v[v][0],
                      fma((double)P.R[k][1], (double)TA.v[v][1], fma((double)P.R[k][2], (double)TA.v[v][2], (double)P.t[k])));
      b.v[v][k] = (double)TB.v[v][k];
    }
  }
  return (float)tri_tri_dist(a, b);
}

// ----------------------------------------------------------------------------
// the traversal kernel
// ----------------------------------------------------------------------------

#ifndef CBVH_LATE_LOADS
#define CBVH_LATE_LOADS 1
#endif
#ifndef CBVH_SMEM_BOXES
#define CBVH_SMEM_BOXES 2  // bit 0: collide, bit 1: distance (measured: distance config 4 -6 %, collide +1.5..2 %)
#endif
__host__ __device__ constexpr bool smem_boxes(int mode) { return (CBVH_SMEM_BOXES >> mode) & 1; }
constexpr int kSurv = 64;  // exact-test queue entries per warp (pose, tri A, tri B)
// per-warp shared memory: stack + leaf queue (+ the exact-test queue, distance only)
#ifndef CBVH_PACK_LUT
#define CBVH_PACK_LUT 1  // pack_list of a 4-bit mask from a 16-word per-warp table (one LDS instead of ~17 ALU operations)
#endif
__host__ __device__ constexpr int warp_smem_words(int mode, int kx) {
  return nfields(kx) * kStack + 5 * kLeafQ + (mode == 1 ? 3 * kSurv : 0) + (smem_boxes(mode) ? 12 * 32 : 0) +
         (CBVH_PACK_LUT ? 16 : 0);
}

// child pairs of an item: Alg. 1 enumerates children of every side it
// descends (flags chosen at push time, see descent_flags)
__device__ __forceinline__ int pair_count(uint32_t pw, uint32_t ta, uint32_t tb) {
  int na = (pw & kDescA) ? (int)((ta >> 28) & 7u) + 1 : 1;
  int nb = (pw & kDescB) ? (int)((tb >> 28) & 7u) + 1 : 1;
  return na * nb;
}

// Which side(s) an internal pair (a, b) descends.  Alg. 1 descends
// both when both are internal; the LARGER rule descends only the node with the
// larger box (sum of extents, A-local vs world — rotation-invariant up to
// sqrt 3), which visits the same leaf pairs (reading R15).
template <int FAST = 0>
__device__ __forceinline__ uint32_t descent_flags(int rule, uint32_t ta, uint32_t tb, const int32_t CA[6],
                                                  const int32_t CB[6], const DevTree& TA, const DevTree& TB) {
  const bool ai = !(ta & kLeafBit), bi = !(tb & kLeafBit);
  if (!(ai && bi) || rule == 0) return (ai ? kDescA : 0u) | (bi ? kDescB : 0u);
  const float ea = words_extent<FAST>(TA, CA), eb = words_extent<FAST>(TB, CB);
  return ea >= eb ? kDescA : kDescB;
}

// floor(k / d) for 0 <= k < 2^12, 1 <= d <= 8 without an integer divide:
// (k + 1/2) / d is at least 1/(2d) away from the next integer, far above the
// ~1e-6 relative error of the fp32 reciprocal.
__device__ __forceinline__ int small_div(int k, int d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)d));  // one MUFU, ~1 ulp
  return __float2int_rz(((float)k + 0.5f) * r);
}

// all triangles of a leaf: low (ntri) bits set
__device__ __forceinline__ uint32_t full_mask(uint32_t t) { return (2u << ((t >> 29) & 3u)) - 1u; }

// The distance of triangle pair (ia, ib) under pose P as the leaf phase
// reports it: fp32 in A's frame; fp32 error here is ~1e-7 x (|t| + model
// extents), so candidates too small for a 1e-5 relative bound are
// re-evaluated in fp64.
__device__ __forceinline__ float pair_distance(const Params& p, const PoseF& P, const Tri& TA, const Tri& TB,
                                               uint32_t ia, uint32_t ib) {
  float d = tri_tri_dist(TA, TB);
  const float tmax = fmaxf(fabsf(P.t[0]), fmaxf(fabsf(P.t[1]), fabsf(P.t[2])));
  if (d < 0.05f * (tmax + p.A.maxabs + p.B.maxabs)) d = tri_dist_fp64(P, p.A.tris, ia, p.B.tris, ib);
  return d;
}

// Greedy dive (distance): a beam search from the root pair — each step
// expands every beam entry (the larger-first side, or the non-leaf side),
// scores the children by the box lower bound and keeps the W best; a kept leaf
// pair is evaluated (its triangle pairs' distances, computed exactly as the
// leaf phase computes them) and leaves the beam.  The smallest distance found
// becomes the pose's starting best.  These are distances of real triangle
// pairs, so the traversal's result is unchanged (min over a superset of the
// same values); it only prunes from the start instead of from +inf (R26).
// One warp per pose: the beam lives in shared memory and the lanes expand all
// of its entries' children at once (lane = entry x child; W = 8 entries of
// <= 4 children, or 4 of <= 8), the kept candidates are the W smallest bounds
// (W rounds of a warp min-reduction), and a kept leaf pair's triangle pairs
// are evaluated one per lane.  A pose's dive is ~20 dependent steps of one
// decode + one bound; the first version ran the whole beam serially in one
// thread per pose, which is what a batch too small to fill the GPU waited for
// (158 us for 64 poses; config 4 at 64 poses 2.17 -> 1.96 ms, config 1 at
// 1,024 poses 0.97 -> 0.72 ms, full config 4 within 1 %).
__device__ __forceinline__ float dive_leaf_pair_warp(const Params& p, const PoseF& P, uint32_t ta, uint32_t tb, int lane) {
  const uint32_t fa = ta & 0x1FFFFFFFu, na = ((ta >> 29) & 3u) + 1;
  const uint32_t fb = tb & 0x1FFFFFFFu, nb = ((tb >> 29) & 3u) + 1;
  float d = FLT_MAX;
  if ((uint32_t)lane < na * nb) {
    const uint32_t v = (uint32_t)lane / nb, u = (uint32_t)lane - v * nb;
    d = pair_distance(p, P, load_tri(p.A.tris, fa + v), to_local(P, load_tri(p.B.tris, fb + u)), fa + v, fb + u);
  }
  return __uint_as_float(__reduce_min_sync(FULL, __float_as_uint(fmaxf(d, 0.f))));
}

template <int KX>
__global__ void __launch_bounds__(128) dive_warp_kernel(const __grid_constant__ Params p) {
  constexpr int NW = 14 + 2 * KX;  // words per beam entry: topo A, topo B, box A, box B, B's extra slabs
  __shared__ uint32_t sm[4][2][8][NW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int i = blockIdx.x * 4 + wib;
  grid_dependency_wait();  // init_kernel's distances / caps
  grid_launch_dependents();
  if (i >= p.N) return;
  const PoseF P = load_pose(p.poses, i);
  const float tmax = fmaxf(fabsf(P.t[0]), fmaxf(fabsf(P.t[1]), fabsf(P.t[2])));
  const float eps = 2e-6f * (tmax + p.A.maxabs + p.B.maxabs);
  const unsigned lt = lanemask_lt();
  // lanes per beam entry (the larger arity, 4 or 8) and the beam width that fills the warp
  const int sh = p.bmax <= 4 ? 2 : 3, W = 32 >> sh;
  uint32_t(*cur)[NW] = sm[wib][0];
  uint32_t(*nxt)[NW] = sm[wib][1];
  if (lane == 0) {
    cur[0][0] = p.A.root_topo;
    cur[0][1] = p.B.root_topo;
    #pragma unroll
    for (int q = 0; q < 6; ++q) { cur[0][2 + q] = (uint32_t)p.A.root[q]; cur[0][8 + q] = (uint32_t)p.B.root[q]; }
    #pragma unroll
    for (int q = 0; q < 2 * KX; ++q) cur[0][14 + q] = (uint32_t)p.X.root[q];
  }
  __syncwarp();
  int nb = 1;
  float dmin = __uint_as_float(__ldcg(&p.dist_bits[i]));  // +inf, or the caller's cap
  if ((p.A.root_topo & kLeafBit) && (p.B.root_topo & kLeafBit)) {
    dmin = fminf(dmin, dive_leaf_pair_warp(p, P, p.A.root_topo, p.B.root_topo, lane));
    nb = 0;
  }
  #pragma unroll 1
  for (int step = 0; step < 128 && nb > 0; ++step) {
    const int e = lane >> sh, k = lane & ((1 << sh) - 1);
    bool valid = e < nb;
    uint32_t cta = 0, ctb = 0;
    int32_t CA[6], CB[6], CX[2 * KX + 1];
    float lb = FLT_MAX;
    if (valid) {
      const uint32_t ta = cur[e][0], tb = cur[e][1];
      int32_t BA[6], BB[6], BX[2 * KX + 1];
      #pragma unroll
      for (int q = 0; q < 6; ++q) { BA[q] = (int32_t)cur[e][2 + q]; BB[q] = (int32_t)cur[e][8 + q]; }
      #pragma unroll
      for (int q = 0; q < 2 * KX; ++q) BX[q] = (int32_t)cur[e][14 + q];
      const bool la = (ta & kLeafBit) != 0, lbf = (tb & kLeafBit) != 0;
      const bool descA = !la && (lbf || (descent_flags(CBVH_DESCENT_LARGER, ta, tb, BA, BB, p.A, p.B) & kDescA));
      const uint32_t t = descA ? ta : tb;
      const uint32_t first = t & 0x0FFFFFFFu, n = ((t >> 28) & 7u) + 1;
      valid = (uint32_t)k < n;
      if (valid) {
        cta = ta; ctb = tb;
        #pragma unroll
        for (int q = 0; q < 6; ++q) { CA[q] = BA[q]; CB[q] = BB[q]; }
        #pragma unroll
        for (int q = 0; q < 2 * KX; ++q) CX[q] = BX[q];
        if (descA) {
          cta = __ldg(p.A.topo + first + k);
          fetch_child_box(p.A, first + k, BA, CA);
        } else {
          ctb = __ldg(p.B.topo + first + k);
          if constexpr (KX > 0) fetch_child_kdop<KX>(p.B, first + k, BB, BX, CB, CX);
          else fetch_child_box(p.B, first + k, BB, CB);
        }
        float alo[3], ahi[3], blo[3], bhi[3];
        words_to_float(p.A, CA, alo, ahi);
        words_to_float(p.B, CB, blo, bhi);
        sat_gap<true>(P, alo, ahi, blo, bhi, eps, &lb);
        valid = lb < dmin;
      }
    }
    // keep the W smallest bounds: W rounds of a warp minimum over (bound, lane) keys
    unsigned key = valid ? ((__float_as_uint(fmaxf(lb, 0.f)) & ~31u) | (unsigned)lane) : 0xffffffffu;
    bool sel = false;
    #pragma unroll 1
    for (int r = 0; r < W; ++r) {
      const unsigned mn = __reduce_min_sync(FULL, key);
      if (mn == 0xffffffffu) break;
      if (key == mn) { sel = true; key = 0xffffffffu; }
    }
    // kept leaf pairs are evaluated (one triangle pair per lane) and leave the beam
    const bool leafpair = sel && (cta & kLeafBit) && (ctb & kLeafBit);
    unsigned lpm = __ballot_sync(FULL, leafpair);
    while (lpm) {
      const int src = __ffs(lpm) - 1;
      lpm &= lpm - 1;
      const uint32_t a = __shfl_sync(FULL, cta, src), b = __shfl_sync(FULL, ctb, src);
      const float l = __shfl_sync(FULL, lb, src);
      if (l < dmin) dmin = fminf(dmin, dive_leaf_pair_warp(p, P, a, b, lane));
    }
    const bool keep = sel && !leafpair && lb < dmin;
    const unsigned km = __ballot_sync(FULL, keep);
    if (keep) {
      const int pos = __popc(km & lt);
      nxt[pos][0] = cta;
      nxt[pos][1] = ctb;
      #pragma unroll
      for (int q = 0; q < 6; ++q) { nxt[pos][2 + q] = (uint32_t)CA[q]; nxt[pos][8 + q] = (uint32_t)CB[q]; }
      #pragma unroll
      for (int q = 0; q < 2 * KX; ++q) nxt[pos][14 + q] = (uint32_t)CX[q];
    }
    nb = __popc(km);
    uint32_t(*t2)[NW] = cur; cur = nxt; nxt = t2;
    __syncwarp();
  }
  if (lane == 0) atomicMin(&p.dist_bits[i], __float_as_uint(dmin));
}

// per-warp constant context (registers); mutable counters live in the kernel
struct WarpCtx {
  uint32_t* st;     // stack SoA [nfields(KX)][kStack]
  uint32_t* lq;     // leaf queue SoA [5][kLeafQ]: pose, topoA, topoB, triangle lists, lower bound (distance)
  uint32_t* sq;     // exact-test queue SoA [3][kSurv]: pose, triangle of A, triangle of B
  uint32_t* scr;    // per-lane parking of the child boxes [12][32] (CBVH_SMEM_BOXES)
  uint32_t* lut;    // pack_list of every 4-bit mask [16] (CBVH_PACK_LUT)
  uint32_t* spill;  // this warp's global spill area [kSpillCap][nfields(KX)]
  uint32_t* stag;   // staging: slot tags [kStageSlots] (tree bit | block id; kNoBlock = empty)
  uint32_t* stg;    // staging: slots [kStageSlots][stage_slot_words]
  int lane;
};

// ---------------------------------------------------------------- treelet staging
// Treelet blocks in shared memory ("clustering BVHs into smaller
// parts"; BJ north_star (2): "treelet blocks fetched with coalesced 16-byte
// vector loads into shared memory").  With an aligned blob (align_treelets)
// a T-slot block holds whole treelets and is one fixed-size span of the
// topology and code arrays.  Each warp keeps kStageSlots blocks; every pass
// the lanes that descend a side look their child's block up (one leader per
// distinct block, __match_any_sync); a missing block is copied in by the
// whole warp with 16-byte loads into the round-robin slot no lane of this
// pass uses, and when every slot is taken the lane reads global memory as the
// unstaged kernel does.  Children are then decoded from shared memory.
#ifndef CBVH_STAGE_SLOTS
#define CBVH_STAGE_SLOTS 4
#endif
static_assert(CBVH_STAGE_SLOTS >= 1 && CBVH_STAGE_SLOTS <= 8, "1..8 staging slots");
constexpr int kStageSlots = CBVH_STAGE_SLOTS;
constexpr int kStageTagWords = (kStageSlots + 3) & ~3;  // tags padded so the slots stay 16-byte aligned
constexpr uint32_t kNoBlock = 0xFFFFFFFFu;
constexpr uint32_t kTreeB = 0x40000000u;  // tag bit of tree B's blocks

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}

// Look up (and, on a miss, copy in) the block of each lane's `node` of tree
// T; returns the lane's slot or -1 (no node, or no free slot: read global).
// All misses of the pass are copied together with asynchronous 16-byte
// global->shared copies (cp.async, LDGSTS), so their latencies overlap.
// Slot layout (words): T topology words; the codes (T x cb bytes, or a
// zero-suppressed region of at most T + 6 T w/8 bytes); zero-suppressed only:
// T u16 byte offsets of each node's first field within the region.
__host__ __device__ __forceinline__ int region_words(const DevTree& T) {
  const int n = 1 << T.tlog;
  return T.zoff ? ((n + 6 * n * (T.width >> 3) + 15) / 16) * 4 : (n * T.cb) / 4;
}
__host__ __device__ __forceinline__ int slot_words(const DevTree& T) {
  const int n = 1 << T.tlog;
  return n + region_words(T) + (T.zoff ? n / 2 : 0);
}

template <bool STATS>
__device__ __forceinline__ int stage_block(const Params& p, const WarpCtx& c, const DevTree& T, uint32_t tree_bit,
                                           uint32_t node, unsigned* used, unsigned* rr,
                                           unsigned long long* s_blocks, unsigned long long* s_bytes) {
  const uint32_t key = (node == kNoBlock || !T.stage_ok) ? kNoBlock : ((node >> T.tlog) | tree_bit);
  if (!__any_sync(FULL, key != kNoBlock)) return -1;
  const unsigned grp = __match_any_sync(FULL, key);
  const int leader = __ffs(grp) - 1;
  const bool lead = key != kNoBlock && c.lane == leader;
  int s = -1;
  if (lead) {
    #pragma unroll
    for (int q = 0; q < kStageSlots; ++q) s = c.stag[q] == key ? q : s;
  }
  *used |= __reduce_or_sync(FULL, (lead && s >= 0) ? (1u << s) : 0u);
  unsigned miss = __ballot_sync(FULL, lead && s < 0);
  if (miss) {
    __syncwarp();  // every lane's reads of the previous pass are done before a slot is overwritten
    // assign slots (round robin over the slots no lane of this pass uses)
    unsigned long long fill = 0;  // bits 8k..8k+7: the slot of the k-th copied block
    int nfill = 0;
    unsigned m = miss;
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      int v = -1;
      #pragma unroll
      for (int t = kStageSlots - 1; t >= 0; --t) {
        const int q = (int)((*rr + (unsigned)t) % kStageSlots);
        v = ((*used >> q) & 1u) ? v : q;
      }
      if (v < 0) break;  // every slot serves this pass: the rest read global memory
      *rr = (unsigned)(v + 1) % kStageSlots;
      *used |= 1u << v;
      const uint32_t k = __shfl_sync(FULL, key, l);
      if (c.lane == l) s = v;
      if (c.lane == 0) c.stag[v] = k;
      fill |= (unsigned long long)v << (8 * nfill);
      ++nfill;
    }
    __syncwarp();  // the new tags are visible to every lane
    // copy: per block nt topology chunks + its code chunks (16 bytes each),
    // all blocks' copies in flight together
    const int nt = (1 << T.tlog) >> 2;
    unsigned long long bytes = 0;
    for (int b = 0; b < nfill; ++b) {
      const int v = (int)((fill >> (8 * b)) & 255u);
      const uint32_t blk = c.stag[v] & ~kTreeB;
      const size_t first = (size_t)blk << T.tlog;
      const uint8_t* csrc = T.zoff ? T.codes + 16ull * __ldg(T.zoff + blk) : T.codes + first * T.cb;
      const int nc = T.zoff ? (int)(__ldg(T.zoff + blk + 1) - __ldg(T.zoff + blk)) : ((1 << T.tlog) * T.cb) >> 4;
      uint32_t* dst = c.stg + v * p.stage_slot_words;
      for (int q = c.lane; q < nt + nc; q += 32)
        cp_async16(dst + 4 * q, q < nt ? static_cast<const void*>(T.topo + first + 4 * q)
                                       : static_cast<const void*>(csrc + 16 * (q - nt)));
      bytes += 16ull * (nt + nc);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (T.zoff) {
      // zero-suppressed: each node's field offset = T + (w/8) x (set mask
      // bits of the nodes before it), a warp prefix sum over the masks
      __syncwarp();
      const int n = 1 << T.tlog, wb = T.width >> 3;
      for (int b = 0; b < nfill; ++b) {
        uint32_t* slotp = c.stg + ((fill >> (8 * b)) & 255u) * p.stage_slot_words;
        const uint8_t* reg = reinterpret_cast<const uint8_t*>(slotp + n);
        unsigned short* offs = reinterpret_cast<unsigned short*>(slotp + n + region_words(T));
        uint32_t carry = 0;
        for (int h = 0; h < n; h += 32) {
          const int j = h + c.lane;
          const uint32_t x = j < n ? (uint32_t)__popc(reg[j]) : 0u;
          uint32_t inc = x;
          #pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (c.lane >= o) inc += y;
          }
          if (j < n) offs[j] = (unsigned short)(n + wb * (carry + inc - x));
          carry += __shfl_sync(FULL, inc, 31);
        }
      }
    }
    if (STATS && c.lane == 0) { *s_blocks += nfill; *s_bytes += bytes; }
  }
  __syncwarp();
  s = __shfl_sync(FULL, s, leader);
  return key == kNoBlock ? -1 : s;
}

// The codes of a node record at `rec` (global or shared memory), fields as load_codes
__device__ __forceinline__ void load_codes_at(const uint8_t* rec, int width, uint32_t q[6]) {
  if (width == 8) {
    const unsigned short* r = reinterpret_cast<const unsigned short*>(rec);
    const uint32_t a = r[0], b = r[1], c = r[2];
    q[0] = a & 255u; q[1] = a >> 8; q[2] = b & 255u; q[3] = b >> 8; q[4] = c & 255u; q[5] = c >> 8;
  } else if (width == 16) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(rec);
    const uint32_t a = r[0], b = r[1], c = r[2];
    q[0] = a & 0xffffu; q[1] = a >> 16; q[2] = b & 0xffffu; q[3] = b >> 16; q[4] = c & 0xffffu; q[5] = c >> 16;
  } else {
    const uint32_t w = (uint32_t)rec[0] | ((uint32_t)rec[1] << 8) | ((uint32_t)rec[2] << 16);
    #pragma unroll
    for (int f = 0; f < 6; ++f) q[f] = (w >> (4 * f)) & 15u;
  }
}

// A child's topology word and decoded box: from its staged block (slot >= 0)
// or from global memory.
__device__ __forceinline__ uint32_t fetch_child(const WarpCtx& c, const Params& p, const DevTree& T, int slot,
                                                uint32_t node, const int32_t P[6], int32_t C[6]) {
  if (slot >= 0) {
    const uint32_t* blk = c.stg + slot * p.stage_slot_words;
    const uint32_t loc = node & ((1u << T.tlog) - 1u);
    const uint8_t* reg = reinterpret_cast<const uint8_t*>(blk + (1 << T.tlog));
    uint32_t q[6];
    if (T.zoff) {
      const unsigned short* offs = reinterpret_cast<const unsigned short*>(blk + (1 << T.tlog) + region_words(T));
      load_codes_zs(reg, reg + offs[loc], reg[loc], 0u, T.width, q);
    } else {
      load_codes_at(reg + loc * T.cb, T.width, q);
    }
    decode_child(P, q, T.bits, C);
    return blk[loc];
  }
  fetch_child_box(T, node, P, C);
  return __ldg(T.topo + node);
}

// Drain the leaf queue: checkPrimitives over every queued leaf pair,
// the c_A x c_B triangle pairs spread over the 32 lanes.  Returns the number
// of triangle-pair tests (for stats).
// The expensive exact tests of up to 32 queued triangle pairs (the cheap
// culls ran before they were queued), one pair per lane, full SIMT:
// collide — Möller, hits summed per pose (__match_any_sync + one atomicAdd);
// distance — triangle distance (fp64 re-evaluation when small), per-pose
// minimum (__reduce_min_sync on float bits + atomicMin).
template <int MODE>
__device__ __forceinline__ void exact_batch(const Params& p, const WarpCtx c, int k) {
  const bool valid = c.lane < k;
  uint32_t pose = 0, ia = 0, ib = 0;
  if (valid) {
    pose = c.sq[0 * kSurv + c.lane];
    ia = c.sq[1 * kSurv + c.lane];
    ib = c.sq[2 * kSurv + c.lane];
  }
  bool hit = false;
  float d = FLT_MAX;
  if (valid) {
    const PoseF P = load_pose(p.poses, (int)pose);
    const Tri TA = load_tri(p.A.tris, ia);
    const Tri TB = to_local(P, load_tri(p.B.tris, ib));
    if (MODE == 0) {
      const int r = moller_fast(TA, TB);
      hit = r > 0 || (r < 0 && overlap_rare(p, pose, ia, ib));
    } else {
      d = pair_distance(p, P, TA, TB, ia, ib);
    }
  }
  if (MODE == 0) {
    const unsigned hm = __ballot_sync(FULL, hit);
    if (hit) {
      const unsigned g = __match_any_sync(hm, pose);
      if (c.lane == __ffs(g) - 1) {
        atomicAdd(&p.count[pose], (unsigned)__popc(g));
        p.hit[pose] = 1;
      }
    }
  } else {
    const unsigned vm = __ballot_sync(FULL, valid);
    if (valid) {
      const unsigned g = __match_any_sync(vm, pose);
      const unsigned mn = __reduce_min_sync(g, __float_as_uint(d));
      if (c.lane == __ffs(g) - 1) atomicMin(&p.dist_bits[pose], mn);
    }
  }
  __syncwarp();
}

// Drain the leaf queue: checkPrimitives over every queued leaf pair.
// Stage 1 spreads the c_A x c_B triangle pairs (only the triangles the box
// filters kept) over the lanes and applies the cheap exact culls (collide:
// disjoint triangle AABBs; distance: AABB gap >= the pose's best); survivors
// are compacted into a per-warp queue and stage 2 (exact_batch) runs the
// expensive tests 32 at a time, so Möller / the distance code run with full
// lanes instead of the ~20-30 % the culls leave.  Returns the number of
// triangle-pair tests (stats).
template <int MODE, bool STATS, int FAST = 0, bool EE = false>
__device__ CBVH_DRAIN_ATTR unsigned drain_leaves(const Params& p, const WarpCtx c, int nleaf,
                                                 unsigned long long* exact) {
  unsigned tests = 0;
  int head = 0, nsq = 0;
  const unsigned lt = lanemask_lt();
  while (head < nleaf) {
    int avail = min(32, nleaf - head);
    uint32_t pose = 0, ta = 0, tb = 0, mk = 0;
    int n = 0;
    if (c.lane < avail) {
      pose = c.lq[0 * kLeafQ + head + c.lane];
      ta = c.lq[1 * kLeafQ + head + c.lane];
      tb = c.lq[2 * kLeafQ + head + c.lane];
      mk = c.lq[3 * kLeafQ + head + c.lane];
      n = (int)((mk >> 8) & 7u) * (int)((mk >> 19) & 7u);  // only triangles the box filters kept
      // early exit: a pose that already has a hit needs no more tests
      if (MODE == 0 && (FAST ? EE : p.early_exit != 0) && __ldcg(&p.hit[pose])) n = 0;
      // distance: a leaf pair whose box bound no longer beats the pose's best
      // distance (tightened since it was queued) is skipped
      if (MODE == 1 && __uint_as_float(c.lq[4 * kLeafQ + head + c.lane]) >= __uint_as_float(__ldcg(&p.dist_bits[pose])))
        n = 0;
    }
    const int incl = warp_incl_scan(n, c.lane);
    const unsigned fit = __ballot_sync(FULL, c.lane < avail && incl <= 32);
    const int m = __popc(fit);  // >= 2: an entry has at most 16 triangle pairs
    const int total = __shfl_sync(FULL, incl, m - 1);
    // lane -> entry: rank among the non-empty entries.  Empty entries (pruned
    // distance pairs, early-exit poses) share a start position with their
    // successor, so the non-empty ones are first compacted (in registers of
    // the lanes: entry of rank r moves to lane r) — a shuffle, not __fns.
    const bool nonempty = c.lane < m && n > 0;
    const unsigned nz = __ballot_sync(FULL, nonempty);
    const unsigned starts = __reduce_or_sync(FULL, nonempty ? (1u << (incl - n)) : 0u);
    const int r = max(__popc(starts & ((2u << c.lane) - 1u)) - 1, 0);
    int e = r;
    if ((nz & (nz + 1u)) != 0u) {  // the non-empty entries are not a prefix
      // lane r needs the index of the r-th non-empty entry: scatter it
      // through the entries' lower-bound slots (already read this round)
      if (nonempty) c.lq[4 * kLeafQ + head + __popc(nz & lt)] = (uint32_t)c.lane;
      __syncwarp();
      e = (int)c.lq[4 * kLeafQ + head + min(r, __popc(nz) - 1)];
      __syncwarp();
    }
    const int start_e = __shfl_sync(FULL, incl - n, e);
    const uint32_t my_pose = __shfl_sync(FULL, pose, e);
    const uint32_t my_ta = __shfl_sync(FULL, ta, e);
    const uint32_t my_tb = __shfl_sync(FULL, tb, e);
    const uint32_t my_mk = __shfl_sync(FULL, mk, e);
    const bool valid = c.lane < total;
    const int k = c.lane - start_e;
    // my_mk: bits 0-7 / 11-18 packed 2-bit triangle lists of A / B, counts at 8 / 19
    const int nb = max(1, (int)((my_mk >> 19) & 7u));
    const int ka = small_div(k, nb), kb = k - ka * nb;
    const uint32_t ia = (my_ta & 0x1FFFFFFFu) + ((my_mk >> (2 * ka)) & 3u);
    const uint32_t ib = (my_tb & 0x1FFFFFFFu) + ((my_mk >> (11 + 2 * kb)) & 3u);
    CBVH_CHECK(p, !valid || (ia < p.A.n_tris && ib < p.B.n_tris && my_pose < (uint32_t)p.N));
    bool keep = false, hit = false;
    if (valid) {
      const PoseF P = load_pose(p.poses, (int)my_pose);
      const Tri TA = load_tri(p.A.tris, ia);
      const Tri TB = to_local(P, load_tri(p.B.tris, ib));
      if (MODE == 0) {
        // exact cull on the same fp32 coordinates Möller uses: closed
        // triangles whose AABBs are disjoint cannot intersect.  Collide runs
        // Möller in place (measured: the compaction costs more than the
        // ~30 % SIMT it recovers for this cheaper test).
        const bool cand = !CBVH_DRAIN_AABB || tri_boxes_overlap(TA, TB);
        if (STATS && cand) ++*exact;
        if (cand) {
          const int r = moller_fast(TA, TB);
          hit = r > 0 || (r < 0 && overlap_rare(p, my_pose, ia, ib));
        }
      } else {
        // triangle AABB gap: a lower bound; skip pairs that cannot beat the best
        const float tmax0 = fmaxf(fabsf(P.t[0]), fmaxf(fabsf(P.t[1]), fabsf(P.t[2])));
        const float best = __uint_as_float(__ldcg(&p.dist_bits[my_pose]));
        const float slack = 2e-6f * (tmax0 + p.A.maxabs + p.B.maxabs);
        // CBVH_DIST_TRIB bits: 1 the triangle AABB gap, 2 the centroid axis
        keep = true;
        if (CBVH_DIST_TRIB & 1) keep = tri_box_gap(TA, TB) - slack < best;
        if ((CBVH_DIST_TRIB & 2) && keep) keep = tri_axis_gap(TA, TB) - slack < best;
        if (STATS && keep) ++*exact;
      }
    }
    tests += (unsigned)total;
    if (MODE == 0) {
      const unsigned hm = __ballot_sync(FULL, hit);
      if (hit) {
        const unsigned g = __match_any_sync(hm, my_pose);
        if (c.lane == __ffs(g) - 1) {
          atomicAdd(&p.count[my_pose], (unsigned)__popc(g));
          p.hit[my_pose] = 1;
        }
      }
      head += m;
      continue;
    }
    // distance: compact the survivors into the exact-test queue
    const unsigned km = __ballot_sync(FULL, keep);
    if (keep) {
      const int s2 = nsq + __popc(km & lt);
      c.sq[0 * kSurv + s2] = my_pose;
      c.sq[1 * kSurv + s2] = ia;
      c.sq[2 * kSurv + s2] = ib;
    }
    nsq += __popc(km);
    __syncwarp();
    if (nsq >= 32) {
      exact_batch<MODE>(p, c, 32);
      // move the rest (< 32) to the front
      uint32_t v0 = 0, v1 = 0, v2 = 0;
      const bool mv = c.lane < nsq - 32;
      if (mv) {
        v0 = c.sq[0 * kSurv + 32 + c.lane];
        v1 = c.sq[1 * kSurv + 32 + c.lane];
        v2 = c.sq[2 * kSurv + 32 + c.lane];
      }
      __syncwarp();
      if (mv) {
        c.sq[0 * kSurv + c.lane] = v0;
        c.sq[1 * kSurv + c.lane] = v1;
        c.sq[2 * kSurv + c.lane] = v2;
      }
      nsq -= 32;
      __syncwarp();
    }
    head += m;
  }
  if (nsq > 0) exact_batch<MODE>(p, c, nsq);
  __syncwarp();
  return tests;
}

// Move the bottom H entries (default half the stack, at most `top`) of the
// smem stack to the warp's global spill area.  Returns the new (top,
// spill_top).  On overflow the warp abandons its smem stack: it flags
// CBVH_EOVERFLOW and marks every pose with an abandoned item conservatively —
// collide: hit = 1 (the count stays a lower bound); distance: 0 — so a caller
// that skips cbvh_check never sees a missed contact as a clear pose.
template <int MODE, int NF>
__device__ __noinline__ int2 spill_out(const Params& p, const WarpCtx c, int top, int spill_top, int H = kStack / 2) {
  if (spill_top + H > kSpillCap) {
    if (c.lane == 0) atomicExch(&p.ctl->error, (unsigned)(-CBVH_EOVERFLOW));
    for (int e = c.lane; e < top; e += 32) {
      const uint32_t pose = c.st[F_POSE * kStack + e] & kPoseMask;
      if (MODE == 0) p.hit[pose] = 1;
      else atomicMin(&p.dist_bits[pose], 0u);
    }
    __syncwarp();
    return make_int2(0, spill_top);  // abandon; cbvh_check reports the error
  }
  __syncwarp();
  for (int idx = c.lane; idx < H * NF; idx += 32) {
    int e = idx / NF, f = idx % NF;
    c.spill[(size_t)(spill_top + e) * NF + f] = c.st[f * kStack + e];
  }
  __syncwarp();
  const int rest = top - H;
  for (int idx = c.lane; idx < rest * NF; idx += 32) {
    int e = idx % rest, f = idx / rest;
    c.st[f * kStack + e] = c.st[f * kStack + e + H];
  }
  __syncwarp();
  return make_int2(rest, spill_top + H);
}

// Refill an empty smem stack from the top of the spill area.
template <int NF>
__device__ __noinline__ int2 spill_in(const WarpCtx c, int spill_top) {
  const int n = min(kStack / 2, spill_top);
  const int base = spill_top - n;
  __syncwarp();
  for (int idx = c.lane; idx < n * NF; idx += 32) {
    int e = idx / NF, f = idx % NF;
    c.st[f * kStack + e] = c.spill[(size_t)(base + e) * NF + f];
  }
  __syncwarp();
  return make_int2(n, base);
}

// ---------------------------------------------------------------- load balancing
// Persistent warps acquire input from a global cursor.  Once a warp's input
// is exhausted it may run `budget` more iterations; then it dumps its whole
// remaining stack (smem + spill) into the continuation buffer and exits.  The
// next launch (phase) spreads those items over every warp, so a few heavy
// sub-traversals no longer leave the GPU idle behind them; the last phase
// runs unbounded.  Items carry their pose id and results are accumulated with
// atomics, so any warp may finish any item.

// Reserve n slots of the continuation buffer (compare-and-swap so a failed
// reservation never leaves a hole); returns the first slot or -1 when full.
__device__ __forceinline__ int reserve_cont(unsigned* count, int n, int lane) {
  int base = -1;
  if (lane == 0) {
    unsigned cur = __ldcg(count);
    while (cur + (unsigned)n <= (unsigned)kContCap) {
      const unsigned prev = atomicCAS(count, cur, cur + (unsigned)n);
      if (prev == cur) { base = (int)cur; break; }
      cur = prev;
    }
  }
  return __shfl_sync(FULL, base, 0);
}

// Dump the smem stack and the spill area; false if the buffer is full.
template <int NF>
__device__ __noinline__ bool dump_items(const Params& p, const WarpCtx c, int top, int spill_top) {
  const int n = top + spill_top;
  const int base = reserve_cont(&p.ctl->count[p.phase], n, c.lane);
  if (base < 0) return false;
  uint32_t* out = p.cont_out + (size_t)base * NF;
  for (int idx = c.lane; idx < spill_top * NF; idx += 32) out[idx] = c.spill[idx];
  out += (size_t)spill_top * NF;
  for (int idx = c.lane; idx < top * NF; idx += 32) {
    const int e = idx / NF, f = idx % NF;
    out[idx] = c.st[f * kStack + e];
  }
  return true;
}

// resident CTAs per SM the register allocation targets (k-DOP stacks take
// more shared memory and registers)
// The FAST collide instantiation needs fewer registers (80 at 6 CTAs / SM
// without a spill, 72 at 7 with 16 bytes of them), so more warps hide the
// latencies of this issue-bound kernel: measured 5 / 6 / 7 / 8 CTAs per SM
// (8 with a 80-entry stack to fit shared memory): config 5 40.1 / 38.1 /
// 37.3 / 38.0 ms, config 3 45.4 / 42.8 / 42.0 / 42.7, config 2 3.44 / 3.46 /
// 3.55 / 3.94 (profiles/round2_ab_occupancy.txt).
#ifndef CBVH_MIN_BLOCKS_FAST
#define CBVH_MIN_BLOCKS_FAST 7
#endif
__host__ __device__ constexpr int min_blocks(int mode, int kx, int fast = 0) {
  return kx == 0 ? (mode == 0 ? (fast ? CBVH_MIN_BLOCKS_FAST : CBVH_MIN_BLOCKS) : CBVH_MIN_BLOCKS_DIST)
                 : (mode == 0 ? (kx >= 10 ? 3 : 4) : 3);
}

template <int MODE, bool STATS, int KX, bool STAGE, int FAST, bool EE = false>
__global__ void __launch_bounds__(kWarps * 32, min_blocks(MODE, KX, FAST)) traverse_kernel(const __grid_constant__ Params p) {
  constexpr int NF = nfields(KX);
  extern __shared__ uint32_t smem[];
  const int wib = threadIdx.x >> 5;
  grid_dependency_wait();  // the previous phase's continuation items, init_kernel's outputs and control block
  grid_launch_dependents();
  static_assert(!FAST || (!STATS && KX == 0 && !STAGE), "FAST is the default-format production kernel");
  static_assert(!EE || (FAST == 1 && MODE == 0), "EE: the hit-only FAST collide kernel");
  const int early_exit = FAST ? (EE ? 1 : 0) : p.early_exit;  // (FAST: the option is the template parameter EE)
  const int descent = FAST ? CBVH_DESCENT_LARGER : p.descent;
  WarpCtx c;
  c.lane = threadIdx.x & 31;
  c.st = smem + wib * warp_smem_words(MODE, KX);
  c.lq = c.st + NF * kStack;
  c.sq = c.lq + 5 * kLeafQ;
  c.scr = c.sq + (MODE == 1 ? 3 * kSurv : 0);
  c.lut = c.scr + (smem_boxes(MODE) ? 12 * 32 : 0);
  if (CBVH_PACK_LUT) {
    if (c.lane < 16) c.lut[c.lane] = pack_list((uint32_t)c.lane);
    __syncwarp();
  }
  c.spill = p.spill + (size_t)(blockIdx.x * kWarps + wib) * kSpillCap * NF;
  // staging area after all warps' stacks and queues
  c.stag = smem + kWarps * warp_smem_words(MODE, KX) + wib * (kStageTagWords + kStageSlots * p.stage_slot_words);
  c.stg = c.stag + kStageTagWords;
  unsigned st_used = 0, st_rr = 0;
  unsigned long long s_sblk = 0, s_sbytes = 0, s_sreads = 0;
  if (STAGE) {
    if (c.lane < kStageSlots) c.stag[c.lane] = kNoBlock;
    __syncwarp();
  }
  int top = 0, nleaf = 0, spill_top = 0;
  int after = 0;  // iterations since the input ran out (before that: the poll counter)
  unsigned long long s_dump = 0, s_iter = 0, s_exact = 0;
  unsigned long long s_bv = 0, s_exp = 0, s_leaf = 0, s_tri = 0, s_dec = 0, s_rec = 0, s_lbytes = 0, s_spill = 0;
  bool poses_left = true;
  const unsigned lt = lanemask_lt();
  const float scale_ab = p.A.maxabs + p.B.maxabs;
  const bool root_leafpair = (p.A.root_topo & kLeafBit) && (p.B.root_topo & kLeafBit);
  if (STATS && c.lane == 0) atomicMin(&p.ctl->t_start, globaltimer_ns());

  while (true) {
    // ---- acquire poses when the stack runs low: push their root pairs
    // (only when nothing is spilled: spilled items are finished first, which
    // bounds the stack by the deepest single traversal, not the batch size)
    if (poses_left && top < kLowWater && spill_top == 0) {
      if (p.phase == 0) {
        // chunks of kGrab poses while plenty remain, single poses near the end
        // (a chunk of several heavy poses in one warp is the tail otherwise)
        unsigned base = 0, g = 1;
        if (c.lane == 0) {
          const unsigned hint = __ldcg(&p.ctl->cursor[0]);
          g = (hint + (unsigned)kGrab * (unsigned)p.nwarps * 8u < (unsigned)p.N) ? (unsigned)kGrab : 1u;
          base = atomicAdd(&p.ctl->cursor[0], g);
        }
        base = __shfl_sync(FULL, base, 0);
        g = __shfl_sync(FULL, g, 0);
        if (STATS && c.lane == 0 && base < (unsigned)p.N) {
          const unsigned long long f = (8ull * base) / (unsigned)p.N;
          if (f != (8ull * (base + g)) / (unsigned)p.N || base == 0) atomicMin(&p.ctl->t_frac[f], globaltimer_ns());
        }
        if (base >= (unsigned)p.N) {
          poses_left = false;
          after = 0;
          if (STATS && c.lane == 0) atomicMin(&p.ctl->t_exhausted, globaltimer_ns());
        } else {
          const int k = min((int)g, p.N - (int)base);
          if (c.lane < k) {
            if (root_leafpair) {
              const int slot = nleaf + c.lane;
              c.lq[0 * kLeafQ + slot] = base + c.lane;
              c.lq[1 * kLeafQ + slot] = p.A.root_topo;
              c.lq[2 * kLeafQ + slot] = p.B.root_topo;
              c.lq[3 * kLeafQ + slot] = pack_list(full_mask(p.A.root_topo)) | (pack_list(full_mask(p.B.root_topo)) << 11);
              c.lq[4 * kLeafQ + slot] = 0u;
            } else {
              const int slot = top + c.lane;
              c.st[F_POSE * kStack + slot] =
                  (base + c.lane) | descent_flags<FAST>(descent, p.A.root_topo, p.B.root_topo, p.A.root, p.B.root,
                                                  p.A, p.B);
              c.st[F_TA * kStack + slot] = p.A.root_topo;
              c.st[F_TB * kStack + slot] = p.B.root_topo;
              #pragma unroll
              for (int q = 0; q < 6; ++q) {
                c.st[(F_BA + q) * kStack + slot] = (uint32_t)p.A.root[q];
                c.st[(F_BB + q) * kStack + slot] = (uint32_t)p.B.root[q];
              }
              #pragma unroll
              for (int q = 0; q < 2 * KX; ++q) c.st[(F_XB + q) * kStack + slot] = (uint32_t)p.X.root[q];
              c.st[F_LB * kStack + slot] = 0xFFu;  // inherited leaf masks: all (distance: lower bound 0)
            }
          }
          if (root_leafpair) nleaf += k; else top += k;
          __syncwarp();
          if (nleaf > kLeafQ - 32) {
            s_tri += drain_leaves<MODE, STATS, FAST, EE>(p, c, nleaf, &s_exact);
            nleaf = 0;
          }
        }
      } else {
        // continuation items dumped by the previous phase
        const unsigned avail = p.ctl->count[p.phase - 1];
        unsigned base = 0;
        if (c.lane == 0) base = atomicAdd(&p.ctl->cursor[p.phase], (unsigned)kGrabItems);
        base = __shfl_sync(FULL, base, 0);
        if (base >= avail) {
          poses_left = false;
          after = 0;
        } else {
          const int k = min(kGrabItems, (int)(avail - base));
          for (int idx = c.lane; idx < k * NF; idx += 32) {
            const int e = idx / NF, f = idx % NF;
            c.st[f * kStack + top + e] = p.cont_in[(size_t)(base + e) * NF + f];
          }
          top += k;
          __syncwarp();
        }
      }
    }
    if (top == 0) {
      if (spill_top > 0) {
        int2 r = spill_in<NF>(c, spill_top);
        top = r.x; spill_top = r.y;
        continue;
      }
      if (poses_left) continue;
      break;
    }
    // ---- every warp learns when the input runs out, not only the warps that
    // try to acquire: a warp deep in a heavy traversal polls the cursor every
    // kPoll iterations (one L2 load by lane 0), so its budget starts and its
    // backlog moves to the next phase with everybody else's
    // (and at iterations 8, 16, 32, 64 of the warp's life, so a batch smaller
    // than the grid — every pose taken at once — is handed on after a few
    // iterations, not after kPoll of them)
    if (CBVH_POLL && poses_left && p.budget >= 0 &&
        ((++after & (kPoll - 1)) == 0 || (after < (int)kPoll && after >= 8 && (after & (after - 1)) == 0))) {
      unsigned cur = 0, lim = 0;
      if (c.lane == 0) {
        cur = __ldcg(&p.ctl->cursor[p.phase]);
        lim = p.phase == 0 ? (unsigned)p.N : __ldcg(&p.ctl->count[p.phase - 1]);
      }
      if (__shfl_sync(FULL, cur >= lim ? 1 : 0, 0)) {
        poses_left = false;
        after = 0;
        if (STATS && c.lane == 0 && p.phase == 0) atomicMin(&p.ctl->t_exhausted, globaltimer_ns());
      }
    }
    // ---- bounded work after the input ran out: hand the rest to the next phase
    if (!poses_left && p.budget >= 0 && ++after > p.budget) {
      if (nleaf > 0) {
        s_tri += drain_leaves<MODE, STATS, FAST, EE>(p, c, nleaf, &s_exact);
        nleaf = 0;
      }
      if (dump_items<NF>(p, c, top, spill_top)) {
        if (STATS) s_dump += top + spill_top;
        top = 0;
        spill_top = 0;
        break;
      }
      after = INT_MIN;  // buffer full: finish here
    }

    // ---- pop as many items as fill 32 lanes with child pairs
    int n = 0;
    if (c.lane < top) {
      const int slot = top - 1 - c.lane;
      n = pair_count(c.st[F_POSE * kStack + slot], c.st[F_TA * kStack + slot], c.st[F_TB * kStack + slot]);
    }
    const int incl = warp_incl_scan(n, c.lane);
    const int n0 = __shfl_sync(FULL, n, 0);
    int m, total, passes;
    unsigned starts;
    // (FAST descends one side per item — the larger-first rule — so an item
    // has at most 8 child pairs and never needs a second pass)
    if (!FAST && n0 > 32) {  // B = 8, both internal: one item in two passes
      m = 1; total = n0; passes = (n0 + 31) >> 5; starts = 1u;
#if CBVH_LATE_LOADS
      // the item stays on the stack during its passes (its boxes are read
      // where they are decoded), so make room for both passes' pushes first
      if (top + 32 * passes > kStack) {
        int2 r = spill_out<MODE, NF>(p, c, top, spill_top, top + 32 * passes - kStack);
        top = r.x; spill_top = r.y;
        if (top == 0) continue;  // spill area full: the error is flagged, the item abandoned
      }
#endif
    } else {
      const unsigned fit = __ballot_sync(FULL, c.lane < top && incl <= 32);
      m = __popc(fit);
      total = __shfl_sync(FULL, incl, m - 1);
      passes = 1;
      starts = __reduce_or_sync(FULL, (c.lane < m) ? (1u << (incl - n)) : 0u);
    }
    const int e = __popc(starts & ((2u << c.lane) - 1u)) - 1;
    const int start_e = __shfl_sync(FULL, incl - n, e);
    // this lane's item, read before anything is pushed over it
    const int slot = top - 1 - e;
    const uint32_t pword = c.st[F_POSE * kStack + slot];
    const uint32_t pose = pword & kPoseMask;
    const uint32_t ta = c.st[F_TA * kStack + slot];
    const uint32_t tb = c.st[F_TB * kStack + slot];
#if !CBVH_LATE_LOADS
    int32_t BA[6], BB[6], BX[2 * KX + 1];
    #pragma unroll
    for (int q = 0; q < 6; ++q) {
      BA[q] = (int32_t)c.st[(F_BA + q) * kStack + slot];
      BB[q] = (int32_t)c.st[(F_BB + q) * kStack + slot];
    }
    #pragma unroll
    for (int q = 0; q < 2 * KX; ++q) BX[q] = (int32_t)c.st[(F_XB + q) * kStack + slot];
#endif
    // leaf masks in bits 0-7; distance: the lower bound's float bits above
    // (rounded down to a multiple of 256 ulp)
    const uint32_t item_w = c.st[F_LB * kStack + slot];
    const float item_lb = __uint_as_float(item_w & ~0xFFu);
    __syncwarp();
    const bool hold = CBVH_LATE_LOADS && passes > 1;
    if (!hold) top -= m;
    if (STATS) { s_exp += m; s_iter += passes; }

    CBVH_CHECK(p, pose < (uint32_t)p.N && slot >= 0 && slot < kStack);
#if !CBVH_LATE_LOADS
    const PoseF P = load_pose(p.poses, (int)pose);
    const float tmax = fmaxf(fabsf(P.t[0]), fmaxf(fabsf(P.t[1]), fabsf(P.t[2])));
    const float eps = 2e-6f * (tmax + scale_ab);
#endif
    const bool early_done = MODE == 0 && early_exit && __ldcg(&p.hit[pose]) != 0;
    float best = FLT_MAX;
    if (MODE == 1) best = __uint_as_float(__ldcg(&p.dist_bits[pose]));
    const bool a_int = (pword & kDescA) != 0, b_int = (pword & kDescB) != 0;  // sides descended
    const int nb = b_int ? (int)((tb >> 28) & 7u) + 1 : 1;

    for (int pass = 0; pass < passes; ++pass) {
      const int k = c.lane - start_e + 32 * pass;
      bool valid = (c.lane + 32 * pass) < total;
      if (MODE == 1) valid = valid && item_lb < best;
      if (MODE == 0 && early_exit) valid = valid && !early_done;
      // child indices on the two sides; with one side descended (FAST) the
      // pair index is the child index of that side
      const int i = FAST ? (b_int ? 0 : k) : small_div(k, nb), j = FAST ? (b_int ? k : 0) : k - i * nb;
      int32_t CA[6], CB[6], CX[2 * KX + 1];
      uint32_t cta = ta, ctb = tb;
      float sg = 0.f;  // collide: the SAT gap (early-exit push order)
      bool surv = false;
      float lb = 0.f;
      // triangles of a leaf side the parent's refinement kept (collide; a
      // descended side is a new node: all)
      uint32_t mskA = 15u, mskB = 15u;
      // (collide only: for distance the inherited masks rarely exclude a
      // triangle and measured 4 % slower on config 4)
      if (MODE == 0 && CBVH_MASK_PROP) {
        if (!a_int) mskA = item_w & 15u;
        if (!b_int) mskB = (item_w >> 4) & 15u;
      }
      bool bad = false;  // checked build: an out-of-range child drops the lane
#if CBVH_LATE_LOADS
      // the pose and the item's parent boxes are loaded where they are used
      // (short live ranges: at the register cap they were spilled to local
      // memory across the pop bookkeeping); the item's slot is intact — the
      // pushes of this pass come after the __syncwarp below, and a held
      // multi-pass item is not popped until its last pass
      const PoseF P = load_pose(p.poses, (int)pose);
      const float tmax = fmaxf(fabsf(P.t[0]), fmaxf(fabsf(P.t[1]), fabsf(P.t[2])));
      const float eps = 2e-6f * (tmax + scale_ab);
      int32_t BA[6], BB[6], BX[2 * KX + 1];
#endif
      // treelet staging: the blocks of this pass's children, warp-wide
      int slotA = -1, slotB = -1;
      if (STAGE) {
        st_used = 0;
        uint32_t na = kNoBlock, nbn = kNoBlock;
        if (valid && a_int) na = (ta & 0x0FFFFFFFu) + (uint32_t)i;
        if (valid && b_int) nbn = (tb & 0x0FFFFFFFu) + (uint32_t)j;
        if (na != kNoBlock && na >= p.A.n_nodes) na = kNoBlock;
        if (nbn != kNoBlock && nbn >= p.B.n_nodes) nbn = kNoBlock;
        if (p.stage_sides & 1) slotA = stage_block<STATS>(p, c, p.A, 0u, na, &st_used, &st_rr, &s_sblk, &s_sbytes);
        if (p.stage_sides & 2) slotB = stage_block<STATS>(p, c, p.B, kTreeB, nbn, &st_used, &st_rr, &s_sblk, &s_sbytes);
        if (STATS) s_sreads += (slotA >= 0 ? 1 : 0) + (slotB >= 0 ? 1 : 0);
      }
      if (valid) {
#if CBVH_LATE_LOADS
        #pragma unroll
        for (int q = 0; q < 6; ++q) {
          BA[q] = (int32_t)c.st[(F_BA + q) * kStack + slot];
          BB[q] = (int32_t)c.st[(F_BB + q) * kStack + slot];
        }
        #pragma unroll
        for (int q = 0; q < 2 * KX; ++q) BX[q] = (int32_t)c.st[(F_XB + q) * kStack + slot];
#endif
        if (a_int) {
          uint32_t node = (ta & 0x0FFFFFFFu) + (uint32_t)i;
          CBVH_GUARD(p, node < p.A.n_nodes, (node = 0, bad = true));
          if (STAGE) cta = fetch_child(c, p, p.A, slotA, node, BA, CA);
          else {
            cta = __ldg(p.A.topo + node);
            fetch_child_box<FAST>(p.A, node, BA, CA);
          }
        } else {
          #pragma unroll
          for (int r = 0; r < 6; ++r) CA[r] = BA[r];
        }
        if (b_int) {
          uint32_t node = (tb & 0x0FFFFFFFu) + (uint32_t)j;
          CBVH_GUARD(p, node < p.B.n_nodes, (node = 0, bad = true));
          if constexpr (KX > 0) {
            ctb = __ldg(p.B.topo + node);
            fetch_child_kdop<KX>(p.B, node, BB, BX, CB, CX);
          } else if (STAGE) {
            ctb = fetch_child(c, p, p.B, slotB, node, BB, CB);
          } else {
            ctb = __ldg(p.B.topo + node);
            fetch_child_box<FAST>(p.B, node, BB, CB);
          }
        } else {
          #pragma unroll
          for (int r = 0; r < 6; ++r) CB[r] = BB[r];
          #pragma unroll
          for (int r = 0; r < 2 * KX; ++r) CX[r] = BX[r];
        }
        float alo[3], ahi[3], blo[3], bhi[3];
        words_to_float<FAST>(p.A, CA, alo, ahi);
        words_to_float<FAST>(p.B, CB, blo, bhi);
        if (smem_boxes(MODE) && !FAST) {
          // park the child boxes in shared memory across the tests: under
          // register pressure the compiler spills them to local memory (the
          // FAST distance kernel has the registers: 165, no spills, -1 %)
          #pragma unroll
          for (int q = 0; q < 6; ++q) {
            c.scr[q * 32 + c.lane] = (uint32_t)CA[q];
            c.scr[(6 + q) * 32 + c.lane] = (uint32_t)CB[q];
          }
        }
        if (MODE == 0) {
          sg = sat_gap<false>(P, alo, ahi, blo, bhi, eps, nullptr);
          surv = sg <= 0.f;
          if constexpr (KX > 0) {
            if (surv) surv = kdop_gap<KX>(P, alo, ahi, p.X, CX, eps) <= 0.f;
          }
          // Against a leaf, "intersect" is refined to the leaf's triangles
          // themselves (still conservative): the partner's box must touch at
          // least one of them.  B's leaves are ~10x A's in config 5, so the
          // box alone lets every A leaf crossing a B leaf box through.  For a
          // leaf pair both sides are filtered and the surviving triangles are
          // recorded as masks for the leaf phase.
          const bool la = (cta & kLeafBit) != 0, lbf = (ctb & kLeafBit) != 0;
#if CBVH_LEAF_SLAB
          // an internal box against a leaf: the leaf's slab (one plane pair,
          // DESIGN.md §4.2) — a leaf pair still refines per triangle (masks)
          if (surv && lbf && !la) surv = box_vs_slab<0>(P, alo, ahi, p.B.tris, ctb, eps);
          if (surv && la && !lbf) surv = box_vs_slab<1>(P, blo, bhi, p.A.tris, cta, eps);
#if CBVH_LEAF_SLAB == 2
          const bool doB = lbf, doA = la;
#else
          const bool doB = lbf && la, doA = la && lbf;
#endif
#else
          // A leaf pair filters A's triangles against B's leaf box only when
          // that box is not much larger than A's leaf box (sum of extents):
          // a large B box rarely excludes one of A's small triangles
          // (CBVH_PAIR_AFILTER: 0 never, 1 always, 2 by the size ratio)
          bool doA = la;
          if (la && lbf) {
            if (CBVH_PAIR_AFILTER == 0) doA = false;
            else if (CBVH_PAIR_AFILTER == 2)
              doA = words_extent<FAST>(p.B, CB) < CBVH_PAIR_RATIO * words_extent<FAST>(p.A, CA);
          }
          const bool doB = lbf;
#endif
          if (surv && doB) {
            mskB = box_hits_leaf<0, FAST == 0>(P, alo, ahi, p.B.tris, ctb, eps, mskB);
            surv = mskB != 0u;
          }
          if (surv && doA) {
            mskA = box_hits_leaf<1, FAST == 0>(P, blo, bhi, p.A.tris, cta, eps, mskA);
            surv = mskA != 0u;
          }
        } else {
          sat_gap<true>(P, alo, ahi, blo, bhi, eps, &lb);
          if constexpr (KX > 0) {
            if (lb < best) lb = fmaxf(lb, kdop_gap<KX>(P, alo, ahi, p.X, CX, eps));
          }
          surv = lb < best;
#if CBVH_DIST_FILTER
          // against a leaf: per-triangle bounds (masks for the leaf phase, and
          // a tighter pair bound)
          const bool refine = CBVH_DIST_FILTER == 1 || ((cta & kLeafBit) && (ctb & kLeafBit));
          if (surv && refine && (ctb & kLeafBit)) {
            float l2;
            mskB = box_near_leaf<0>(P, alo, ahi, p.B.tris, ctb, eps, best, &l2, mskB);
            lb = fmaxf(lb, l2);
            surv = mskB != 0u;
          }
          if (surv && refine && (cta & kLeafBit)) {
            float l2;
            mskA = box_near_leaf<1>(P, blo, bhi, p.A.tris, cta, eps, best, &l2, mskA);
            lb = fmaxf(lb, l2);
            surv = mskA != 0u;
          }
#endif
        }
        if (STATS) {
          s_dec += (a_int ? 1 : 0) + (b_int ? 1 : 0);
          s_rec += (a_int ? 4 + 3 * p.A.width / 4 : 0) + (b_int ? 4 + (3 + KX) * p.B.width / 4 : 0);
        }
      }
      if (bad) surv = false;
      if (STATS) s_bv += __popc(__ballot_sync(FULL, valid)) * (c.lane == 0 ? 1 : 0);
      const bool leafpair = surv && (cta & kLeafBit) && (ctb & kLeafBit);
      const bool push = surv && !leafpair;
      // ---- ballot/popc compaction: internal pairs back onto the stack
#if CBVH_LATE_LOADS
      __syncwarp();  // every lane has read its item before any push lands on it
#endif
      const unsigned pm = __ballot_sync(FULL, push);
      if (pm) {
        if (top + 32 > kStack) {
          int2 r = spill_out<MODE, NF>(p, c, top, spill_top, CBVH_SPILL_H);
          top = r.x; spill_top = r.y;
          if (STATS) s_spill++;
        }
        int pos = __popc(pm & lt);
        if (MODE == 1) {
          // nearest-first: the smallest lower bound goes on top of the stack
          const unsigned key = push ? __float_as_uint(fmaxf(lb, 0.f)) : 0xffffffffu;
          const unsigned mn = __reduce_min_sync(FULL, key);
          const int wl = __ffs(__ballot_sync(FULL, push && key == mn)) - 1;
          const int last = 31 - __clz(pm);
          if (c.lane == wl) pos = __popc(pm) - 1;
          else if (c.lane == last) pos = __popc(pm & ((1u << wl) - 1u));
        }
#if CBVH_EE_ORDER
        if (MODE == 0 && early_exit) {
          // early exit: the deepest-overlapping pair (most negative SAT gap)
          // goes on top, to reach a first hit sooner
          const unsigned b = __float_as_uint(sg);
          const unsigned key = push ? ((b & 0x80000000u) ? ~b : (b | 0x80000000u)) : 0xffffffffu;
          const unsigned mn = __reduce_min_sync(FULL, key);
          const int wl = __ffs(__ballot_sync(FULL, push && key == mn)) - 1;
          const int last = 31 - __clz(pm);
          if (c.lane == wl) pos = __popc(pm) - 1;
          else if (c.lane == last) pos = __popc(pm & ((1u << wl) - 1u));
        }
#endif
        if (push) {
          const int s2 = top + pos;
          CBVH_CHECK(p, s2 < kStack);
          if (smem_boxes(MODE) && !FAST) {
            #pragma unroll
            for (int q = 0; q < 6; ++q) {
              CA[q] = (int32_t)c.scr[q * 32 + c.lane];
              CB[q] = (int32_t)c.scr[(6 + q) * 32 + c.lane];
            }
          }
          c.st[F_POSE * kStack + s2] = pose | descent_flags<FAST>(descent, cta, ctb, CA, CB, p.A, p.B);
          c.st[F_TA * kStack + s2] = cta;
          c.st[F_TB * kStack + s2] = ctb;
          #pragma unroll
          for (int q = 0; q < 6; ++q) {
            c.st[(F_BA + q) * kStack + s2] = (uint32_t)CA[q];
            c.st[(F_BB + q) * kStack + s2] = (uint32_t)CB[q];
          }
          #pragma unroll
          for (int q = 0; q < 2 * KX; ++q) c.st[(F_XB + q) * kStack + s2] = (uint32_t)CX[q];
          c.st[F_LB * kStack + s2] = (MODE == 1 ? (__float_as_uint(fmaxf(lb, 0.f)) & ~0xFFu) : 0u) |
                                     (mskA & 15u) | ((mskB & 15u) << 4);
        }
        top += __popc(pm);
      }
      // ---- leaf pairs into the leaf queue
      const unsigned lm = __ballot_sync(FULL, leafpair);
      if (lm) {
        if (leafpair) {
          const int s2 = nleaf + __popc(lm & lt);
          CBVH_CHECK(p, s2 < kLeafQ);
          c.lq[0 * kLeafQ + s2] = pose;
          c.lq[1 * kLeafQ + s2] = cta;
          c.lq[2 * kLeafQ + s2] = ctb;
          c.lq[3 * kLeafQ + s2] = CBVH_PACK_LUT ? (c.lut[mskA & full_mask(cta)] | (c.lut[mskB & full_mask(ctb)] << 11))
                                                : (pack_list(mskA & full_mask(cta)) | (pack_list(mskB & full_mask(ctb)) << 11));
          if (MODE == 1) c.lq[4 * kLeafQ + s2] = __float_as_uint(lb);
        }
        nleaf += __popc(lm);
        if (STATS) {
          s_leaf += __popc(lm) * (c.lane == 0 ? 1 : 0);
          if (leafpair) s_lbytes += 36u * (((cta >> 29) & 3u) + ((ctb >> 29) & 3u) + 2u);
        }
      }
      __syncwarp();
      // drain in full rounds (collide above 32 entries, distance at
      // CBVH_DIST_DRAIN: a sooner drain tightens a pose's best earlier, but
      // the half-empty rounds cost more than the pruning gains)
      if (nleaf > kLeafQ - 32 || (MODE == 1 && nleaf >= CBVH_DIST_DRAIN) ||
          (MODE == 0 && early_exit && nleaf >= CBVH_EE_DRAIN)) {
        s_tri += drain_leaves<MODE, STATS, FAST, EE>(p, c, nleaf, &s_exact);
        nleaf = 0;
      }
    }
    if (hold) {
      // pop the held multi-pass item: the top entry moves into its slot
      if (top - 1 != slot)
        for (int f = c.lane; f < NF; f += 32) c.st[f * kStack + slot] = c.st[f * kStack + top - 1];
      __syncwarp();
      top -= 1;
    }
    if (MODE == 1 && nleaf > 0 && top == 0) {
      s_tri += drain_leaves<MODE, STATS, FAST, EE>(p, c, nleaf, &s_exact);
      nleaf = 0;
    }
  }
  if (nleaf > 0) s_tri += drain_leaves<MODE, STATS, FAST, EE>(p, c, nleaf, &s_exact);
  if (STATS && c.lane == 0) atomicMax(&p.ctl->t_end, globaltimer_ns());
  if (STATS) {
    unsigned long long d = s_dec, r = s_rec, lb = s_lbytes, ex = s_exact;
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ex += __shfl_down_sync(FULL, ex, o);
      d += __shfl_down_sync(FULL, d, o);
      r += __shfl_down_sync(FULL, r, o);
      lb += __shfl_down_sync(FULL, lb, o);
    }
    if (c.lane == 0) {
      atomicAdd(&p.ctl->stats[0], s_bv);
      atomicAdd(&p.ctl->stats[1], s_exp);
      atomicAdd(&p.ctl->stats[2], s_leaf);
      atomicAdd(&p.ctl->stats[3], s_tri);
      atomicAdd(&p.ctl->stats[4], d);
      atomicAdd(&p.ctl->stats[5], r);
      atomicAdd(&p.ctl->stats[6], lb);
      atomicAdd(&p.ctl->stats[7], s_spill);
      atomicAdd(&p.ctl->dumped, s_dump);
      atomicAdd(&p.ctl->iterations, s_iter);
      atomicAdd(&p.ctl->exact, ex);
    }
    if (STAGE) {
      unsigned long long sr = s_sreads;
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) sr += __shfl_down_sync(FULL, sr, o);
      if (c.lane == 0) {
        atomicAdd(&p.ctl->stage_blocks, s_sblk);
        atomicAdd(&p.ctl->stage_bytes, s_sbytes);
        atomicAdd(&p.ctl->stage_reads, sr);
      }
    }
  }
}

template <int MODE>
__global__ void init_kernel(Params p, int reset_stats) {
  grid_launch_dependents();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int stride = gridDim.x * blockDim.x;
  for (int k = i; k < p.N; k += stride) {
    if (MODE == 0) { p.count[k] = 0u; p.hit[k] = 0; }
    else if (!p.capped) p.dist_bits[k] = 0x7f800000u;  // +inf
    else {
      // caller-supplied caps: NaN -> +inf (no cap), negative -> 0; the float
      // bits of non-negative values order like uint32 (atomicMin)
      const uint32_t b = p.dist_bits[k];
      if (b & 0x80000000u) p.dist_bits[k] = 0u;
      else if (b > 0x7f800000u) p.dist_bits[k] = 0x7f800000u;
    }
  }
  if (i == 0) {
    p.ctl->error = 0u;
    for (int k = 0; k < kMaxPhases; ++k) {
      p.ctl->cursor[k] = 0u;
      p.ctl->count[k] = 0u;
    }
    if (reset_stats) {
      for (int s = 0; s < 8; ++s) p.ctl->stats[s] = 0ull;
      p.ctl->t_start = ~0ull;
      p.ctl->t_exhausted = ~0ull;
      p.ctl->t_end = 0ull;
      p.ctl->dumped = 0ull;
      p.ctl->iterations = 0ull;
      p.ctl->exact = 0ull;
      p.ctl->stage_blocks = p.ctl->stage_bytes = p.ctl->stage_reads = 0ull;
      for (int s = 0; s < 8; ++s) p.ctl->t_frac[s] = ~0ull;
    }
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------

static thread_local char g_err[512] = "";
static thread_local int g_launches = 0;
static thread_local cudaEvent_t g_ev_start = nullptr, g_ev_stop = nullptr;

int set_error(int code, const char* msg) {
  std::snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  std::snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return CBVH_ECUDA;
}

static size_t smem_bytes(int mode, int kx) { return (size_t)kWarps * warp_smem_words(mode, kx) * sizeof(uint32_t); }

struct LaunchShape {
  int blocks;
  int warps;
};

constexpr int kMaxDevices = 64;

// Grid of the persistent traversal kernel: SMs x resident CTAs at `smem`
// bytes of dynamic shared memory per CTA.
template <int MODE, bool STATS, int KX, bool STAGE, int FAST = 0, bool EE = false>
static int shape_for(LaunchShape* s, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  // the dynamic shared-memory opt-in and the occupancy are per device: cached
  // per device (a race only repeats the idempotent calls); the staged kernel's
  // shared memory depends on the blobs, so its occupancy is queried per call
  static std::atomic<int> cached[kMaxDevices];
  const int slot = dev < kMaxDevices ? dev : -1;
  per_sm = (slot >= 0 && !STAGE) ? cached[slot].load(std::memory_order_acquire) : 0;
  if (per_sm == 0) {
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    if (smem > (size_t)optin) return set_error(CBVH_EINVAL, "shared memory of the staged kernel exceeds the device limit");
    e = cudaFuncSetAttribute(traverse_kernel<MODE, STATS, KX, STAGE, FAST, EE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             STAGE ? optin : (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, traverse_kernel<MODE, STATS, KX, STAGE, FAST, EE>, kWarps * 32,
                                                      smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (per_sm < 1) per_sm = 1;
    if (slot >= 0 && !STAGE) cached[slot].store(per_sm, std::memory_order_release);
  }
  s->blocks = sms * per_sm;
  s->warps = s->blocks * kWarps;
  return CBVH_OK;
}

template <int KX>
static int max_warps_kx(int mode) {
  // workspace is sized for the larger of the instantiations of this mode
  LaunchShape a{}, b{};
  // (the staged kernel uses more shared memory, so never more warps)
  int rc = mode == 0 ? shape_for<0, false, KX, false>(&a, smem_bytes(0, KX))
                     : shape_for<1, false, KX, false>(&a, smem_bytes(1, KX));
  if (rc) return -1;
  rc = mode == 0 ? shape_for<0, true, KX, false>(&b, smem_bytes(0, KX)) : shape_for<1, true, KX, false>(&b, smem_bytes(1, KX));
  if (rc) return -1;
  int w = a.warps > b.warps ? a.warps : b.warps;
  if constexpr (KX == 0) {
    LaunchShape f[6] = {};
    rc = mode == 0 ? shape_for<0, false, 0, false, 4>(&f[4], smem_bytes(0, 0)) : shape_for<1, false, 0, false, 4>(&f[4], smem_bytes(1, 0));
    if (!rc) rc = mode == 0 ? shape_for<0, false, 0, false, 5>(&f[5], smem_bytes(0, 0)) : shape_for<1, false, 0, false, 5>(&f[5], smem_bytes(1, 0));
    if (rc) return -1;
    if (mode == 0 && shape_for<0, false, 0, false, 1, true>(&f[3], smem_bytes(0, 0))) return -1;
    rc = mode == 0 ? shape_for<0, false, 0, false, 1>(&f[0], smem_bytes(0, 0)) : shape_for<1, false, 0, false, 1>(&f[0], smem_bytes(1, 0));
    if (!rc) rc = mode == 0 ? shape_for<0, false, 0, false, 2>(&f[1], smem_bytes(0, 0)) : shape_for<1, false, 0, false, 2>(&f[1], smem_bytes(1, 0));
    if (!rc) rc = mode == 0 ? shape_for<0, false, 0, false, 3>(&f[2], smem_bytes(0, 0)) : shape_for<1, false, 0, false, 3>(&f[2], smem_bytes(1, 0));
    if (rc) return -1;
    for (const LaunchShape& x : f) w = x.warps > w ? x.warps : w;
  }
  return w;
}

static int max_warps(int mode, int kx) {
  switch (kx) {
    case 0: return max_warps_kx<0>(mode);
    case 4: return max_warps_kx<4>(mode);
    case 6: return max_warps_kx<6>(mode);
    case 10: return max_warps_kx<10>(mode);
  }
  return -1;
}

static size_t workspace_for_warps(int warps, int kx) {
  return kCtlBytes + (size_t)warps * kSpillCap * nfields(kx) * sizeof(uint32_t) +
         2 * (size_t)kContCap * nfields(kx) * sizeof(uint32_t);
}

// extra k-DOP axes of B (0 for an AABB blob)
static int extra_axes(const cbvh_bvh* B) { return B ? (int)B->h.kdop / 2 - 3 : 0; }

// Greedy dive before a distance traversal (reading R26); CBVH_DIVE=0 turns it
// off (A/B only).
static bool dive_enabled() {
  static const bool on = [] {  // thread-safe one-time initialisation
    const char* env = std::getenv("CBVH_DIVE");
    return (env && *env) ? (std::atoi(env) != 0) : true;
  }();
  return on;
}

// CBVH_FAST=0 sends the default format through the generic kernel too (A/B only)
static bool fast_enabled() {
  static const bool on = [] {
    const char* env = std::getenv("CBVH_FAST");
    return (env && *env) ? (std::atoi(env) != 0) : true;
  }();
  return on;
}

// Phase schedule: budgets of the bounded phases, then one
// unbounded phase.  CBVH_PHASES="b0,b1,..." overrides (tuning only).
constexpr int64_t kSmallBatch = 256;
struct PhaseSchedule {
  int n = 0;
  int b[kMaxPhases];
};
static int phase_budgets(int* out, int64_t N) {
  static const PhaseSchedule sched = [] {  // thread-safe one-time initialisation
    PhaseSchedule r;
    const char* env = std::getenv("CBVH_PHASES");
    if (env && *env) {
      const char* q = env;
      while (*q && r.n < kMaxPhases - 1) {
        r.b[r.n++] = std::atoi(q);
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    } else {
      // seven bounded phases of 32 iterations, then the unbounded one: the
      // last phase has no hand-over, so its longest chain is the call's tail
      // (16k poses of config 5: 0.5 ms at 10 % SM activity behind 32, 32, 64);
      // more, equally short phases leave it almost nothing, and a phase with
      // nothing to do costs ~7 us (tools/ab_phases_full.sh, small_batch.py:
      // config 5 at 16k / 131k / 1M poses -12 / -3 / -0.5 %, config 4 distance
      // at 1,024 poses -16 %)
      for (int k = 0; k < kMaxPhases - 1; ++k) r.b[r.n++] = 32;
    }
    return r;
  }();
  static const bool overridden = [] { const char* env = std::getenv("CBVH_PHASES"); return env && *env; }();
  if (!overridden && N <= kSmallBatch) {
    // a batch far smaller than the grid: what the caller waits for is the
    // longest chain of dependent iterations, so the first hand-overs come
    // sooner (measured, tools/ab_phases_small.sh: 64 poses of config 3
    // 513 -> 345 us, config 4 distance 1058 -> 853 us; at 1,024 poses the
    // longer budgets are better again)
    static const int small[4] = {8, 16, 32, 64};
    for (int k = 0; k < 4; ++k) out[k] = small[k];
    return 4;
  }
  for (int k = 0; k < sched.n; ++k) out[k] = sched.b[k];
  return sched.n;
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
  d.layout = (int)h.layout;
  d.n_nodes = h.num_nodes;
  d.n_tris = h.num_tris;
  d.cb = (int)(h.kdop * h.code_width / 8);
  d.tlog = -1;
  d.stage_ok = 0;
  d.zoff = nullptr;
  const uint32_t Tn = h.treelet_nodes;
  if ((h.flags & CBVH_FLAG_ALIGNED_TREELETS) && h.kdop == 6 && Tn >= 4 && (Tn & (Tn - 1)) == 0) {
    for (d.tlog = 0; (1u << d.tlog) < Tn; ++d.tlog) {}
    if (h.flags & CBVH_FLAG_ZERO_SUPPRESSED) d.zoff = reinterpret_cast<const uint32_t*>(base + h.off_blocks);
    d.stage_ok = (d.zoff || (Tn * (uint32_t)d.cb) % 16 == 0) ? 1 : 0;
  }
  return d;
}

// Launch a kernel of the call's chain (dive, traversal phases) with
// programmatic dependent launch: its CTAs may become resident while the
// previous kernel of the stream drains, and every thread waits in
// grid_dependency_wait() until that kernel has completed and its memory is
// visible — the launch latency of the 4-7 kernels of a call overlaps the
// previous kernel's tail instead of adding to it (CBVH_PDL=0: plain launches).
template <class... KArgs, class... Args>
static cudaError_t launch_after(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args&&... args) {
  static const bool pdl = [] {
    const char* env = std::getenv("CBVH_PDL");
    return (env && *env) ? (std::atoi(env) != 0) : true;
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int MODE, bool STATS, int KX>
static int launch_kx(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                     uint32_t* d_count, float* d_dist, void* d_ws, size_t ws_bytes, void* stream, int descent,
                     int early_exit, int capped, int stage) {
  g_launches = 0;
  if (!A || !B || !d_ws) return set_error(CBVH_EINVAL, "null argument");
  if (N < 0 || N > 0x3fffffffLL) return set_error(CBVH_EINVAL, "N out of range [0, 2^30)");
  if (descent != CBVH_DESCENT_LARGER && descent != CBVH_DESCENT_SIMULTANEOUS)
    return set_error(CBVH_EINVAL, "bad descent rule");
  if (N > 0 && !d_poses) return set_error(CBVH_EINVAL, "null poses");
  if (N > 0 && MODE == 0 && (!d_hit || !d_count)) return set_error(CBVH_EINVAL, "null outputs");
  if (N > 0 && MODE == 1 && !d_dist) return set_error(CBVH_EINVAL, "null outputs");
  if (!A->d_blob || !B->d_blob) return set_error(CBVH_EINVAL, "unbound bvh");
  if ((reinterpret_cast<uintptr_t>(d_poses) & 15) != 0) return set_error(CBVH_EINVAL, "poses must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(d_ws) & 255) != 0) return set_error(CBVH_EINVAL, "workspace must be 256-byte aligned");
  Params p;
  p.A = make_tree(A);
  p.B = make_tree(B);
  // treelet staging (KX = 0 only): the slot holds the larger of the two
  // trees' blocks; a tree whose blob is not aligned is read from global memory
  if (KX != 0 || (!p.A.stage_ok && !p.B.stage_ok)) stage = 0;
  p.stage_slot_words = 0;
  static const int sides = [] {
    const char* env = std::getenv("CBVH_STAGE_SIDES");
    return (env && *env) ? std::atoi(env) : 3;
  }();
  p.stage_sides = sides;
  for (const DevTree* T : {&p.A, &p.B})
    if (stage && T->stage_ok) p.stage_slot_words = std::max(p.stage_slot_words, slot_words(*T));
  const size_t smem = smem_bytes(MODE, KX) +
                      (stage ? (size_t)kWarps * (kStageTagWords + kStageSlots * p.stage_slot_words) * sizeof(uint32_t) : 0);
  // the default blob format and query options run the FAST instantiation
  // (format constants folded at compile time); everything else the generic one
  auto plain = [](const DevTree& T, int w) { return T.layout == CBVH_LAYOUT_DELTA && T.width == w && !T.zoff; };
  int fast = 0;
  const bool ee = MODE == 0 && early_exit;
  if (!STATS && KX == 0 && !stage && descent == CBVH_DESCENT_LARGER && fast_enabled()) {
    if (plain(p.A, 8) && plain(p.B, 8) && p.A.bits == 8 && p.B.bits == 8) fast = 1;  // (also hit-only collide: the EE instantiation)
    else if (ee) fast = 0;
    else if (plain(p.A, 4) && plain(p.B, 4)) fast = 4;
    else if (plain(p.A, 16) && plain(p.B, 16)) fast = 5;
    else if (p.A.layout == CBVH_LAYOUT_FP16 && p.B.layout == CBVH_LAYOUT_FP16) fast = 2;
    else if (p.A.layout == CBVH_LAYOUT_FP32 && p.B.layout == CBVH_LAYOUT_FP32) fast = 3;
  }
  LaunchShape s;
  int rc;
  if constexpr (KX == 0 && !STATS) {
    rc = stage ? shape_for<MODE, STATS, KX, true>(&s, smem)
         : (fast == 1 && ee) ? shape_for<0, STATS, KX, false, 1, true>(&s, smem)
         : fast == 1 ? shape_for<MODE, STATS, KX, false, 1>(&s, smem)
         : fast == 2 ? shape_for<MODE, STATS, KX, false, 2>(&s, smem)
         : fast == 3 ? shape_for<MODE, STATS, KX, false, 3>(&s, smem)
         : fast == 4 ? shape_for<MODE, STATS, KX, false, 4>(&s, smem)
         : fast == 5 ? shape_for<MODE, STATS, KX, false, 5>(&s, smem)
                     : shape_for<MODE, STATS, KX, false>(&s, smem);
  } else if constexpr (KX == 0) {
    rc = stage ? shape_for<MODE, STATS, KX, true>(&s, smem) : shape_for<MODE, STATS, KX, false>(&s, smem);
  } else {
    rc = shape_for<MODE, STATS, KX, false>(&s, smem);
  }
  if (rc) return rc;
  if (ws_bytes < workspace_for_warps(s.warps, KX)) return set_error(CBVH_EWORKSPACE, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::memcpy(p.A.root, A->root_decoded, sizeof p.A.root);
  std::memcpy(p.B.root, B->root_decoded, sizeof p.B.root);
  p.A.root_topo = A->root_topo;
  p.B.root_topo = B->root_topo;
  p.A.maxabs = A->max_abs_coord;
  p.B.maxabs = B->max_abs_coord;
  std::memset(&p.X, 0, sizeof p.X);
  for (int a = 0; a < KX; ++a) {
    p.X.org[a] = B->axis_origin[a];
    p.X.cell[a] = std::ldexp(1.0f, B->axis_exp[a]);
    p.X.root[2 * a] = B->axis_root[2 * a];
    p.X.root[2 * a + 1] = B->axis_root[2 * a + 1];
  }
  p.poses = d_poses;
  p.N = (int)N;
  p.hit = d_hit;
  p.count = d_count;
  p.dist_bits = reinterpret_cast<uint32_t*>(d_dist);
  p.ctl = static_cast<Control*>(d_ws);
  p.spill = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(d_ws) + kCtlBytes);
  uint32_t* cont0 = p.spill + (size_t)s.warps * kSpillCap * nfields(KX);
  uint32_t* cont1 = cont0 + (size_t)kContCap * nfields(KX);
  p.descent = descent;
  p.early_exit = (MODE == 0 && early_exit) ? 1 : 0;
  p.capped = (MODE == 1 && capped) ? 1 : 0;
  p.nwarps = s.warps;
  p.bmax = (int)std::max(A->h.branching, B->h.branching);
  int ib = (int)((N + 255) / 256);
  ib = ib < 1 ? 1 : (ib > 4096 ? 4096 : ib);
  init_kernel<MODE><<<ib, 256, 0, st>>>(p, STATS ? 1 : 0);
  g_launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "init_kernel launch");
  if (N == 0) return CBVH_OK;
  if (MODE == 1 && dive_enabled()) {
    e = launch_after(dive_warp_kernel<KX>, (int)((N + 3) / 4), 128, 0, st, p);
    g_launches++;
    if (e != cudaSuccess) return cuda_fail(e, "dive_kernel launch");
  }
  int budgets[kMaxPhases];
  const int nb = phase_budgets(budgets, N);
  if (g_ev_start) cudaEventRecord(g_ev_start, st);
  for (int ph = 0; ph <= nb; ++ph) {
    p.phase = ph;
    p.budget = ph < nb ? budgets[ph] : -1;
    p.cont_in = (ph & 1) ? cont0 : cont1;   // phase ph reads what ph - 1 wrote
    p.cont_out = (ph & 1) ? cont1 : cont0;
    if constexpr (KX == 0 && !STATS) {
      if (stage) e = launch_after(traverse_kernel<MODE, STATS, KX, true, 0>, s.blocks, kWarps * 32, smem, st, p);
      else if (fast == 1 && ee) e = launch_after(traverse_kernel<0, STATS, KX, false, 1, true>, s.blocks, kWarps * 32, smem, st, p);
      else if (fast == 1) e = launch_after(traverse_kernel<MODE, STATS, KX, false, 1>, s.blocks, kWarps * 32, smem, st, p);
      else if (fast == 2) e = launch_after(traverse_kernel<MODE, STATS, KX, false, 2>, s.blocks, kWarps * 32, smem, st, p);
      else if (fast == 3) e = launch_after(traverse_kernel<MODE, STATS, KX, false, 3>, s.blocks, kWarps * 32, smem, st, p);
      else if (fast == 4) e = launch_after(traverse_kernel<MODE, STATS, KX, false, 4>, s.blocks, kWarps * 32, smem, st, p);
      else if (fast == 5) e = launch_after(traverse_kernel<MODE, STATS, KX, false, 5>, s.blocks, kWarps * 32, smem, st, p);
      else e = launch_after(traverse_kernel<MODE, STATS, KX, false, 0>, s.blocks, kWarps * 32, smem, st, p);
    } else if constexpr (KX == 0) {
      if (stage) e = launch_after(traverse_kernel<MODE, STATS, KX, true, 0>, s.blocks, kWarps * 32, smem, st, p);
      else e = launch_after(traverse_kernel<MODE, STATS, KX, false, 0>, s.blocks, kWarps * 32, smem, st, p);
    } else {
      e = launch_after(traverse_kernel<MODE, STATS, KX, false, 0>, s.blocks, kWarps * 32, smem, st, p);
    }
    g_launches++;
    if (e != cudaSuccess) return cuda_fail(e, "traverse_kernel launch");
  }
  if (g_ev_stop) cudaEventRecord(g_ev_stop, st);
  return CBVH_OK;
}

// k-DOPs bound the static model B only (reading R22): the kernel is
// instantiated per number of B's extra slab axes
template <int MODE, bool STATS>
static int launch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                  uint32_t* d_count, float* d_dist, void* d_ws, size_t ws_bytes, void* stream, int descent,
                  int early_exit, int capped, int stage) {
  g_launches = 0;
  if (!A || !B) return set_error(CBVH_EINVAL, "null argument");
  if (A->h.kdop != 6) return set_error(CBVH_EINVAL, "k-DOP blobs bound the static model B only; A must be an AABB blob");
  // treelet staging: auto (0) = on when a blob has aligned treelet blocks
  const bool aligned = ((A->h.flags | B->h.flags) & CBVH_FLAG_ALIGNED_TREELETS) != 0;
  if (stage > 0 && (!aligned || extra_axes(B) != 0))
    return set_error(CBVH_EINVAL, "treelet staging needs an aligned-treelet blob (align_treelets) and AABBs");
  const int st = stage < 0 ? 0 : (aligned ? 1 : 0);
  switch (extra_axes(B)) {
    case 0: return launch_kx<MODE, STATS, 0>(A, B, d_poses, N, d_hit, d_count, d_dist, d_ws, ws_bytes, stream, descent, early_exit, capped, st);
    case 4: return launch_kx<MODE, STATS, 4>(A, B, d_poses, N, d_hit, d_count, d_dist, d_ws, ws_bytes, stream, descent, early_exit, capped, 0);
    case 6: return launch_kx<MODE, STATS, 6>(A, B, d_poses, N, d_hit, d_count, d_dist, d_ws, ws_bytes, stream, descent, early_exit, capped, 0);
    case 10: return launch_kx<MODE, STATS, 10>(A, B, d_poses, N, d_hit, d_count, d_dist, d_ws, ws_bytes, stream, descent, early_exit, capped, 0);
  }
  return set_error(CBVH_EINVAL, "bad k-DOP");
}

}  // namespace cbvh

using namespace cbvh;

extern "C" {

const char* cbvh_last_error(void) { return g_err; }

void cbvh_set_kernel_events(void* start, void* stop) {
  g_ev_start = static_cast<cudaEvent_t>(start);
  g_ev_stop = static_cast<cudaEvent_t>(stop);
}
int cbvh_last_launch_count(void) { return g_launches; }

int cbvh_bind(const uint8_t* h_blob, size_t bytes, const void* d_blob, cbvh_bvh* out) {
  if (!h_blob || !d_blob || !out) return set_error(CBVH_EINVAL, "null argument");
  if ((reinterpret_cast<uintptr_t>(d_blob) & 255) != 0) return set_error(CBVH_EINVAL, "device blob must be 256-byte aligned");
  cbvh_header h;
  int rc = parse_header(h_blob, bytes, &h);
  if (rc) return rc;
  // Topology validation (O(n)): children strictly after their parent (no
  // cycles, guaranteed by the builder's treelet numbering) and inside the node
  // array, leaf triangle ranges inside the soup — a corrupted blob must fail
  // here, not loop or fault on the device.  (CBVH_SKIP_BLOB_VALIDATION=1 is a
  // test hook for the checked build's device-side checks.)
  const char* skip = std::getenv("CBVH_SKIP_BLOB_VALIDATION");
  if (!(skip && skip[0] == '1')) {
    const uint8_t* tp = h_blob + h.off_topo;
    auto topo_at = [&](uint64_t n) { uint32_t w; std::memcpy(&w, tp + 4ull * n, 4); return w; };
    const bool padded = (h.flags & CBVH_FLAG_ALIGNED_TREELETS) != 0;
    uint64_t real = 0;
    for (uint32_t n = 0; n < h.num_nodes; ++n) {
      const uint32_t w = topo_at(n);
      if (padded && w == kPadTopo) continue;  // padding slot: checked unreferenced below
      ++real;
      if (w & kLeafBit) {
        const uint64_t first = w & 0x1FFFFFFFu, cnt = ((w >> 29) & 3u) + 1;
        if (first + cnt > h.num_tris || cnt > h.leaf_size) return set_error(CBVH_EBLOB, "bad leaf triangle range");
      } else {
        const uint64_t first = w & 0x0FFFFFFFu, cnt = ((w >> 28) & 7u) + 1;
        if (first <= n || first + cnt > h.num_nodes || cnt < 2 || cnt > h.branching)
          return set_error(CBVH_EBLOB, "bad child range");
        if (padded)
          for (uint64_t k = first; k < first + cnt; ++k)
            if (topo_at(k) == kPadTopo) return set_error(CBVH_EBLOB, "child in a padding slot");
      }
    }
    if (real != h.real_nodes || (padded && topo_at(0) == kPadTopo)) return set_error(CBVH_EBLOB, "bad node count");
    if (h.flags & CBVH_FLAG_ZERO_SUPPRESSED) {
      // block regions in order, inside the codes section, each holding its
      // T masks (6 bits) and the fields they announce
      const uint64_t T = h.treelet_nodes, nblocks = h.num_nodes / T, wb = h.code_width / 8;
      const uint8_t* tab = h_blob + h.off_blocks;
      uint32_t prev = 0;
      for (uint64_t b = 0; b < nblocks; ++b) {
        uint32_t o0, o1;
        std::memcpy(&o0, tab + 4 * b, 4);
        std::memcpy(&o1, tab + 4 * (b + 1), 4);
        if (o0 != prev || o1 < o0 || 16ull * o1 > h.off_blocks - h.off_codes) return set_error(CBVH_EBLOB, "bad code regions");
        prev = o1;
        const uint8_t* r = h_blob + h.off_codes + 16ull * o0;
        uint64_t need = T;
        for (uint64_t j = 0; j < T; ++j) {
          if (r[j] > 63u || (r[j] && topo_at(b * T + j) == kPadTopo)) return set_error(CBVH_EBLOB, "bad presence mask");
          need += wb * (uint64_t)__builtin_popcount(r[j]);
        }
        if (need > 16ull * (o1 - o0)) return set_error(CBVH_EBLOB, "bad code regions");
      }
    }
  }
  std::memset(out, 0, sizeof *out);
  out->d_blob = d_blob;
  out->bytes = bytes;
  out->h = h;
  std::memcpy(&out->root_topo, h_blob + h.off_topo, 4);
  if (h.layout != CBVH_LAYOUT_DELTA) {
    // absolute layouts: the root's own stored box, as fp32 bit patterns
    float m = 0.f;
    for (int k = 0; k < 6; ++k) {
      float v;
      if (h.layout == CBVH_LAYOUT_FP32) {
        std::memcpy(&v, h_blob + h.off_codes + 4 * k, 4);
      } else {
        uint16_t hv;
        std::memcpy(&hv, h_blob + h.off_codes + 2 * k, 2);
        const int e = (hv >> 10) & 31, mm = hv & 1023;
        double d = e == 0 ? std::ldexp((double)mm, -24) : std::ldexp((double)(mm + 1024), e - 25);
        v = (float)((hv & 0x8000) ? -d : d);
      }
      std::memcpy(&out->root_decoded[k], &v, 4);
      m = std::fmax(m, std::fabs(v));
    }
    out->max_abs_coord = m;
    return CBVH_OK;
  }
  // node 0 is coded against the header root box (the anchor of treelet 0)
  // and, for a k-DOP, against the axis table's root intervals.  Stored fields:
  // lo of the k/2 axes, then hi (4-bit fields two per byte, low nibble first).
  const int nax = (int)h.kdop / 2;
  const uint8_t* c = h_blob + h.off_codes;
  const bool zs = (h.flags & CBVH_FLAG_ZERO_SUPPRESSED) != 0;
  auto field = [&](int f) -> uint32_t {
    if (zs) {  // node 0 = slot 0 of block 0 (region offset 0): mask byte, then its non-zero fields
      const uint32_t m = c[0];
      if (!((m >> f) & 1u)) return 0u;
      const uint8_t* x = c + h.treelet_nodes + (h.code_width / 8) * __builtin_popcount(m & ((1u << f) - 1u));
      return h.code_width == 16 ? (uint32_t)x[0] | ((uint32_t)x[1] << 8) : x[0];
    }
    if (h.code_width == 16) { uint16_t x; std::memcpy(&x, c + 2 * f, 2); return x; }
    if (h.code_width == 8) return c[f];
    return (c[f / 2] >> (4 * (f % 2))) & 15u;
  };
  auto decode = [&](int64_t lo, int64_t hi, uint32_t qlo, uint32_t qhi, int32_t* dlo, int32_t* dhi) {
    const int64_t E = hi - lo;
    if (E < 0 || E >= (1ll << 23)) return false;
    int bl = 0;
    while ((E >> bl) > 0) ++bl;
    const int s = bl - (int)h.bits > 0 ? bl - (int)h.bits : 0;
    *dlo = (int32_t)(lo + ((int64_t)qlo << s));
    *dhi = (int32_t)(hi - ((int64_t)qhi << s));
    return true;
  };
  for (int a = 0; a < 3; ++a)
    if (!decode(h.root_box[a], h.root_box[3 + a], field(a), field(nax + a), &out->root_decoded[a],
                &out->root_decoded[3 + a]))
      return set_error(CBVH_EBLOB, "bad root box");
  for (int a = 0; a < nax - 3; ++a) {
    const uint8_t* t = h_blob + h.off_axes + 16ull * a;
    int32_t rlo, rhi;
    std::memcpy(&out->axis_origin[a], t, 4);
    std::memcpy(&out->axis_exp[a], t + 4, 4);
    std::memcpy(&rlo, t + 8, 4);
    std::memcpy(&rhi, t + 12, 4);
    if (out->axis_exp[a] < -126 || out->axis_exp[a] > 127 || !std::isfinite(out->axis_origin[a]) || rlo < 0 || rhi >= (1 << 24) ||
        !decode(rlo, rhi, field(3 + a), field(nax + 3 + a), &out->axis_root[2 * a], &out->axis_root[2 * a + 1]))
      return set_error(CBVH_EBLOB, "bad k-DOP axis table");
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
  const int kx = extra_axes(B);
  int w = max_warps(mode == 1 ? 1 : 0, kx);
  if (w <= 0) return 0;
  return workspace_for_warps(w, kx);
}

static int opts_descent(const cbvh_query_opts* o) { return o ? o->descent : CBVH_DESCENT_LARGER; }
static int opts_early(const cbvh_query_opts* o) { return o ? o->early_exit : 0; }
static int opts_capped(const cbvh_query_opts* o) { return o ? o->capped : 0; }
static int opts_stats(const cbvh_query_opts* o) { return o ? o->stats : 0; }
static int opts_stage(const cbvh_query_opts* o) { return o ? o->treelet_staging : 0; }

int collide_batch_ex(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                     uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream, const cbvh_query_opts* o) {
  if (opts_stats(o))
    return launch<0, true>(A, B, d_poses, N, d_hit, d_pair_count, nullptr, d_ws, ws_bytes, stream, opts_descent(o), opts_early(o), opts_capped(o), opts_stage(o));
  return launch<0, false>(A, B, d_poses, N, d_hit, d_pair_count, nullptr, d_ws, ws_bytes, stream, opts_descent(o), opts_early(o), opts_capped(o), opts_stage(o));
}
int distance_batch_ex(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, float* d_min_dist,
                      void* d_ws, size_t ws_bytes, void* stream, const cbvh_query_opts* o) {
  if (opts_stats(o))
    return launch<1, true>(A, B, d_poses, N, nullptr, nullptr, d_min_dist, d_ws, ws_bytes, stream, opts_descent(o), opts_early(o), opts_capped(o), opts_stage(o));
  return launch<1, false>(A, B, d_poses, N, nullptr, nullptr, d_min_dist, d_ws, ws_bytes, stream, opts_descent(o), opts_early(o), opts_capped(o), opts_stage(o));
}
int collide_batch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                  uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream) {
  return collide_batch_ex(A, B, d_poses, N, d_hit, d_pair_count, d_ws, ws_bytes, stream, nullptr);
}
int collide_batch_stats(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, uint8_t* d_hit,
                        uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream) {
  cbvh_query_opts o{CBVH_DESCENT_LARGER, 1, 0, 0, 0};
  return collide_batch_ex(A, B, d_poses, N, d_hit, d_pair_count, d_ws, ws_bytes, stream, &o);
}
int distance_batch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N, float* d_min_dist,
                   void* d_ws, size_t ws_bytes, void* stream) {
  return distance_batch_ex(A, B, d_poses, N, d_min_dist, d_ws, ws_bytes, stream, nullptr);
}
int distance_batch_stats(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                         float* d_min_dist, void* d_ws, size_t ws_bytes, void* stream) {
  cbvh_query_opts o{CBVH_DESCENT_LARGER, 1, 0, 0, 0};
  return distance_batch_ex(A, B, d_poses, N, d_min_dist, d_ws, ws_bytes, stream, &o);
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
  Control ctl;
  cudaError_t e = cudaMemcpyAsync(&ctl, d_ws, sizeof ctl, cudaMemcpyDeviceToHost, st);
  const unsigned long long* v = ctl.stats;
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cbvh_read_stats");
  out->bv_tests = v[0]; out->expansions = v[1]; out->leaf_pairs = v[2]; out->tri_tests = v[3];
  out->nodes_decoded = v[4]; out->record_bytes = v[5]; out->tri_bytes = v[6]; out->spills = v[7];
  const bool timed = ctl.t_end > 0 && ctl.t_start != ~0ull && ctl.t_end >= ctl.t_start;
  out->kernel_ns = timed ? ctl.t_end - ctl.t_start : 0;
  out->tail_ns = (timed && ctl.t_exhausted != ~0ull && ctl.t_end >= ctl.t_exhausted) ? ctl.t_end - ctl.t_exhausted : 0;
  out->dumped = ctl.dumped;
  out->iterations = ctl.iterations;
  out->exact_tests = ctl.exact;
  out->treelet_blocks = ctl.stage_blocks;
  out->treelet_bytes = ctl.stage_bytes;
  out->staged_reads = ctl.stage_reads;
  for (int k = 0; k < 8; ++k)
    out->timeline_ns[k] = (timed && ctl.t_frac[k] != ~0ull && ctl.t_frac[k] >= ctl.t_start) ? ctl.t_frac[k] - ctl.t_start : 0;
  return CBVH_OK;
}

}  // extern "C"
