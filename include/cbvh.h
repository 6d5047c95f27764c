/* cbvh.h — C-ABI of the B200 compressed-BVH collision / proximity library.
 *
 * Paper: arXiv 2012.05348 (compressed BVHs for collision detection & proximity
 * query).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, both under
 * the reference bundle; BJ = BASELINE.json north_star.  The blob layout is
 * documented in DESIGN.md §3.
 *
 * Three calls follow the paper's statement of the problem (BJ):
 *   build_compressed_bvh(mesh, branching, bits) -> blob
 *   collide_batch(bvhA, bvhB, poses[N])         -> per-pose hit flag + colliding-pair count
 *   distance_batch(bvhA, bvhB, poses[N])        -> per-pose minimum separation
 *
 * Conventions
 *   - Every function returns an int status (CBVH_OK = 0, negative = error);
 *     no C++ exception crosses the ABI.  cbvh_last_error() gives a thread-local
 *     message for the last non-zero status of the calling thread.
 *   - Pointers named h_* are host memory, d_* device memory.  The caller owns
 *     every device buffer (blob copy, poses, outputs, workspace) and the
 *     stream; the library never allocates device memory.
 *   - Device calls are stream-ordered and asynchronous (no host sync).  Errors
 *     raised inside a kernel (stack overflow, malformed blob) are written to a
 *     device error word in the workspace and surface through cbvh_check().
 *   - Blobs are immutable; concurrent calls on different streams with
 *     distinct workspaces are safe.
 *   - Poses: fp32 [N][12] row-major [R | t] (row r = R[r][0..2], t[r]);
 *     world = R x_A + t; the environment B is static at identity (S:34-38,
 *     SURVEY §8(c) reading 14).
 */
#ifndef CBVH_H_
#define CBVH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CBVH_OK = 0,
  CBVH_EINVAL = -1,     /* bad argument: B not in {2,4,8}, bits not in [2,16], T < B, c not in [1,4], N not in [0, 2^30), null ptr */
  CBVH_EMESH = -2,      /* empty mesh, index out of range, non-finite vertex, too many triangles (> 2^29) */
  CBVH_EBLOB = -3,      /* bad magic / version / size / section offsets */
  CBVH_ECUDA = -4,      /* a CUDA runtime call failed (message in cbvh_last_error) */
  CBVH_ENOMEM = -5,     /* host allocation failed */
  CBVH_EWORKSPACE = -6, /* workspace too small (see cbvh_workspace_bytes) */
  CBVH_EOVERFLOW = -7,  /* device traversal stack overflow (reported by cbvh_check) */
  CBVH_EINTERNAL = -8   /* checked build only: a device bounds check failed (reported by cbvh_check) */
};

/* ------------------------------------------------------------------ build */

typedef struct {
  const float* vertices;     /* host, fp32 xyz, row-major [num_vertices][3] */
  int64_t num_vertices;
  const int32_t* triangles;  /* host, [num_triangles][3] vertex indices */
  int64_t num_triangles;
} cbvh_mesh;

/* Node box layouts.  DELTA is the paper's compressed layout
 * (b-bit corrections vs the decoded parent, §III.B / P:105); FP16 and
 * FP32 store absolute boxes — binary16 rounded outward (§III.A) and
 * exact single precision — for the paper's half-vs-float comparison. */
enum { CBVH_LAYOUT_DELTA = 0, CBVH_LAYOUT_FP16 = 1, CBVH_LAYOUT_FP32 = 2 };

typedef struct {
  int treelet_nodes; /* T: nodes per treelet ("clustering BVHs into smaller parts"); default 32; must be >= branching */
  int leaf_size;     /* c: max triangles per leaf, 1..4; default 4 */
  int layout;        /* CBVH_LAYOUT_*; default CBVH_LAYOUT_DELTA (bits is ignored for FP16 / FP32) */
  int kdop;          /* k of the k-DOP bounding volumes (Table I): 0 or 6 = AABB (default), 14, 18, 26;
                        k > 6 requires CBVH_LAYOUT_DELTA and is supported for the static model B */
  int align_treelets; /* non-zero: whole treelets are packed next-fit into T-slot blocks (node id = block T +
                        offset; no treelet straddles a block; unused slots are padding), so a treelet block
                        is one aligned, fixed-size span of the topology and code arrays that the traversal
                        can stage in shared memory.  Needs the delta AABB layout and a
                        power-of-two T in [4, 64] */
  int zero_suppress;  /* non-zero: integer-compressed corrections ("compress it using integer compression
                        method"): per treelet block, a presence mask per node and only its non-zero fields
                        (implies align_treelets; delta AABB layout, bits > 4).  Decoded from the staged
                        block, so queries on such blobs stage treelets */
} cbvh_build_opts;

/* Build the compressed BVH of one mesh ("splitting the models and wrap it
 * recursively"; P:103-105 treelets + "delta to the parent nodes"
 * "quantify BV as integer").
 *   branching: B in {2, 4, 8} — recursive binary equal-count median splits on
 *              the longest centroid axis (ties by triangle index)
 *              collapsed into B-ary nodes.
 *   bits:      b in [2, 16] — each node stores 6 inward b-bit corrections
 *              against its parent's DECODED lattice box (DESIGN.md
 *              §3.2).  Stored in 4/8/16-bit fields (b <= 4 / <= 8 / <= 16).
 *   opts:      nullable (defaults T = 32, c = 4).
 * On success *blob is a library-owned host buffer of *blob_bytes bytes, to be
 * released with cbvh_free_blob.  Deterministic: same input -> identical bytes.
 * Errors: CBVH_EINVAL, CBVH_EMESH, CBVH_ENOMEM. */
int build_compressed_bvh(const cbvh_mesh* mesh, int branching, int bits, const cbvh_build_opts* opts,
                         uint8_t** blob, size_t* blob_bytes);
void cbvh_free_blob(uint8_t* blob);

/* Parsed blob header (host copy).  Lattice: world/local coordinate of lattice
 * index k on axis a is origin[a] + k * 2^lattice_exp. */
typedef struct {
  uint32_t branching, bits, treelet_nodes, leaf_size, code_width;
  uint32_t num_nodes, num_tris, num_treelets, depth, num_leaves;
  int32_t lattice_exp;
  float origin[3];
  int32_t root_box[6]; /* lattice lo xyz, hi xyz of the root */
  uint64_t off_topo, off_codes, off_treelets, off_tris, off_tri_index, total_bytes;
  uint32_t layout;     /* CBVH_LAYOUT_* */
  uint32_t kdop;       /* 6 (AABB) or 14 / 18 / 26 */
  uint64_t off_axes;   /* k-DOP axis table: per extra axis {fp32 origin, int32 exp, int32 root lo, root hi} */
  uint32_t flags;      /* CBVH_FLAG_* */
  uint32_t real_nodes; /* nodes of the tree (num_nodes counts node slots, padding included) */
  uint64_t off_blocks; /* zero-suppressed codes: per-block region offsets (u32, 16-byte units from off_codes) */
} cbvh_header;

/* cbvh_header.flags */
enum { CBVH_FLAG_ALIGNED_TREELETS = 1, CBVH_FLAG_ZERO_SUPPRESSED = 2 };

typedef struct {
  cbvh_header h;
  uint64_t bvh_bytes;      /* topo + codes + treelet table: the compressed hierarchy */
  uint64_t tri_bytes;      /* leaf-ordered fp32 triangle soup (48 B / triangle: 9 floats + 3 pads) */
  double bytes_per_node;   /* bvh_bytes / num_nodes */
  double code_bytes_per_node; /* the BV descriptor alone: k * code_width / 8 (AABB: 3 / 6 / 12 delta, 12 fp16, 24 fp32) */
} cbvh_info;

/* Validate and describe a host blob.  Errors: CBVH_EINVAL (null), CBVH_EBLOB. */
int cbvh_blob_info(const uint8_t* h_blob, size_t bytes, cbvh_info* out);

/* ------------------------------------------------------------------ device */

/* A blob bound to its device copy.  d_blob must hold the same bytes as h_blob
 * (the caller uploads it, e.g. into a torch uint8 tensor, 256-B aligned). */
typedef struct {
  const void* d_blob;
  size_t bytes;
  cbvh_header h;
  /* filled by cbvh_bind from the host copy: */
  uint32_t root_topo;      /* topology word of node 0 */
  int32_t root_decoded[6]; /* node 0 decoded against the header root box */
  float max_abs_coord;     /* max |coordinate| of the decoded root box (fp32 slack scale) */
  /* k-DOP (kdop > 6): per extra slab axis a < kdop/2 - 3, the axis lattice
   * (coordinate of index k along the direction: axis_origin[a] + k * 2^axis_exp[a])
   * and node 0 decoded against the axis-table root interval */
  float axis_origin[10];
  int32_t axis_exp[10];
  int32_t axis_root[20];   /* lo, hi per axis */
} cbvh_bvh;

/* Parse h_blob and bind it to d_blob.  Errors: CBVH_EINVAL, CBVH_EBLOB. */
int cbvh_bind(const uint8_t* h_blob, size_t bytes, const void* d_blob, cbvh_bvh* out);

/* Device workspace needed by collide_batch (mode 0) / distance_batch (mode 1)
 * on the current device: control words, stats counters and per-warp stack
 * spill areas.  Independent of N.  Returns 0 if the device query fails. */
size_t cbvh_workspace_bytes(const cbvh_bvh* A, const cbvh_bvh* B, int64_t N, int mode);

/* collide_batch — Algorithm 1 per pose, exhaustive (no early exit):
 * d_pair_count[i] = number of (A-triangle, B-triangle) pairs whose closed
 * triangles intersect under pose i; d_hit[i] = (d_pair_count[i] > 0).
 *   d_poses:      device fp32 [N][12] (see conventions)
 *   d_hit:        device uint8 [N]   (written)
 *   d_pair_count: device uint32 [N]  (written)
 *   d_ws:         device workspace of ws_bytes >= cbvh_workspace_bytes(...)
 *   stream:       cudaStream_t (as void*), 0 = legacy default stream
 * N = 0 is a no-op.  Errors (synchronous): CBVH_EINVAL, CBVH_EWORKSPACE,
 * CBVH_ECUDA (launch failure).  Asynchronous: see cbvh_check.
 * Execution: init + up to 8 traversal phases on `stream`, chained with
 * programmatic dependent launches (each kernel waits for its predecessor in
 * the stream before touching its data; work queued on `stream` before or
 * after the call is ordered as usual).  Blobs in the default format (delta
 * layout, b = 8, not zero-suppressed) with default options — and the fp16 /
 * fp32 layouts, 4- / 16-bit fields and the hit-only option — run kernels with
 * the format compiled in; results do not depend on which kernel runs. */
int collide_batch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                  uint8_t* d_hit, uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream);

/* distance_batch — separation-distance variant:
 * d_min_dist[i] = min over triangle pairs of the Euclidean distance under
 * pose i (0 when any pair intersects), fp32.  Arguments as collide_batch.
 * Launches init, one dive kernel (a beam search that seeds each pose's best
 * with a real triangle-pair distance; R26) and the traversal
 * phases, all on `stream`.  Accuracy: within 1e-5 relative of the fp64
 * distance of the fp32 inputs (candidates below 0.05 x (|t| + extents) are
 * re-evaluated in fp64). */
int distance_batch(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                   float* d_min_dist, void* d_ws, size_t ws_bytes, void* stream);

/* Query options (nullable everywhere; null = defaults). */
enum {
  /* Descend only the node whose box is larger (sum of extents) when both
   * are internal; Alg. 1's other cases unchanged.  Same result, far fewer
   * BV tests when the models differ in scale.  Default. */
  CBVH_DESCENT_LARGER = 1,
  /* Alg. 1 verbatim: descend both nodes, test the cross product
   * of their children. */
  CBVH_DESCENT_SIMULTANEOUS = 0
};
typedef struct {
  int descent;    /* CBVH_DESCENT_* */
  int stats;      /* non-zero: accumulate cbvh_stats in the workspace (slower) */
  int early_exit; /* collide only: stop each pose at its first colliding pair ("early_exit").
                     d_hit stays exact; d_pair_count becomes a lower bound (>= 1 iff hit). */
  int capped;     /* distance only: on entry d_min_dist[i] holds a cap c_i (e.g. a clearance
                     threshold or the previous frame's distance); on return d_min_dist[i] =
                     min(distance_i, c_i), exact whenever distance_i < c_i.  Node pairs whose
                     lower bound reaches the cap are pruned from the start (S:397-405 prune
                     rule with best initialised to c_i instead of +inf).  NaN caps act as
                     +inf, negative caps as 0.  Ignored by collide. */
  int treelet_staging; /* 0 (auto): stage treelet blocks in shared memory when a blob has aligned treelets
                          (cbvh_build_opts.align_treelets); 1: require it (CBVH_EINVAL otherwise); -1: never.
                          AABB blobs only; results are identical either way. */
} cbvh_query_opts;

/* collide_batch / distance_batch with options (opts may be null). */
int collide_batch_ex(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                     uint8_t* d_hit, uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream,
                     const cbvh_query_opts* opts);
int distance_batch_ex(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                      float* d_min_dist, void* d_ws, size_t ws_bytes, void* stream,
                      const cbvh_query_opts* opts);

/* Stats counters gathered by the *_stats variants. */
typedef struct {
  uint64_t bv_tests;        /* child-pair BV tests (Alg. 1 "if a_i and b_j intersect") */
  uint64_t expansions;      /* node pairs popped and expanded */
  uint64_t leaf_pairs;      /* (leafA, leafB) pairs reaching checkPrimitives */
  uint64_t tri_tests;       /* triangle-pair tests */
  uint64_t nodes_decoded;   /* child boxes decoded (records fetched) */
  uint64_t record_bytes;    /* compressed bytes of those records (4 B topo + 6w/8 B codes each) */
  uint64_t tri_bytes;       /* algorithmic triangle bytes: 36 B x triangles loaded (box-leaf filters + leaf phase) */
  uint64_t spills;          /* stack spill events */
  uint64_t kernel_ns;       /* traversal kernel span (first warp start .. last warp end), globaltimer */
  uint64_t tail_ns;         /* span from pose-cursor exhaustion to the last warp's end (load-imbalance tail) */
  uint64_t dumped;          /* items handed to a later load-balancing phase (continuations) */
  uint64_t timeline_ns[8];  /* when the pose cursor passed k/8 of N (ns after the kernel start) */
  uint64_t iterations;      /* warp expansion passes; bv_tests / (32 x iterations) = lane utilisation */
  uint64_t exact_tests;     /* triangle pairs past the leaf phase's cheap culls: exact Möller / distance evaluations */
  uint64_t treelet_blocks;  /* treelet staging: blocks copied into shared memory */
  uint64_t treelet_bytes;   /* treelet staging: their bytes (16-byte loads) */
  uint64_t staged_reads;    /* treelet staging: child records decoded from shared memory */
} cbvh_stats;

/* Same as collide_batch / distance_batch but also accumulate cbvh_stats in
 * the workspace (slower; used to count BV-pair tests for the metric). */
int collide_batch_stats(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                        uint8_t* d_hit, uint32_t* d_pair_count, void* d_ws, size_t ws_bytes, void* stream);
int distance_batch_stats(const cbvh_bvh* A, const cbvh_bvh* B, const float* d_poses, int64_t N,
                         float* d_min_dist, void* d_ws, size_t ws_bytes, void* stream);

/* Synchronize the stream and return the device error word of the last call
 * that used d_ws (CBVH_OK or CBVH_EOVERFLOW / CBVH_EBLOB), or CBVH_ECUDA. */
int cbvh_check(const void* d_ws, void* stream);

/* Synchronize the stream and copy the stats counters out of d_ws. */
int cbvh_read_stats(const void* d_ws, cbvh_stats* out, void* stream);

/* Number of kernel launches the last collide_batch/distance_batch issued on
 * this thread (for the bench's gpu_launches count). */
int cbvh_last_launch_count(void);

/* Observability: when non-null, the next collide/distance calls on this
 * thread record `start` (cudaEvent_t) just before the traversal kernel and
 * `stop` just after it, on the call's stream — used by bench.py to time the
 * dominant kernel alone.  Pass nulls to disable. */
void cbvh_set_kernel_events(void* start, void* stop);

/* Thread-local message for the last non-zero status. */
const char* cbvh_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CBVH_H_ */
