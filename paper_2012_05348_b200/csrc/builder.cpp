// builder.cpp — host-side BVH builder, integer-lattice quantizer,
// predictor–corrector encoder and treelet packer (BJ subsystem (1)).
//
// Paper mapping (P:n = PAPER.md line n, S:n = SPEC.md line n):
//   * "By splitting the models and wrap it recursively": equal-count
//     median split on the longest centroid axis, ties by triangle index
//     (S:178); for B = 4 / 8 the binary median splits are applied
//     log2(B) times and collapsed into one B-ary node (reading R8).
//   * "quantify BV as integer" and "predictors based on the delta to
//     the parent nodes": every box lives on a per-tree power-of-two
//     integer lattice; a node stores 6 inward b-bit corrections against its
//     parent's DECODED box, step 2^s with
//     s = max(0, bitlen(E) - b), E the parent's lattice extent (reading R3).
//   * "clustering BVHs into a smaller parts ('treelet')": greedy
//     BFS packing of sibling groups into treelets of at most T nodes; each
//     treelet header stores the absolute box its first sibling group is coded
//     against, so any treelet decodes from its own bytes.
//
// The blob layout is DESIGN.md §3; the device side reads it in cbvh_device.cu.

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <new>
#include <string>
#include <vector>

#include "../../include/cbvh.h"
#include "cbvh_internal.h"

namespace cbvh {

namespace {

struct BNode {
  double lo[3], hi[3];
  std::vector<int> children;
  int tri_begin = 0, tri_end = 0;  // range into the permutation (leaves)
  int depth = 0;
};

struct Builder {
  const float* V;
  const int32_t* T;
  int64_t nt;
  int B, c;
  std::vector<int> perm;
  std::vector<double> cen;  // centroids [nt*3]
  std::vector<BNode> nodes;

  double centroid(int t, int a) const { return cen[3 * (size_t)t + a]; }

  void fit(int b, int e, double* lo, double* hi) const {
    for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
    for (int k = b; k < e; ++k) {
      int t = perm[k];
      for (int v = 0; v < 3; ++v)
        for (int a = 0; a < 3; ++a) {
          double x = (double)V[3 * (int64_t)T[3 * (int64_t)t + v] + a];
          lo[a] = std::min(lo[a], x);
          hi[a] = std::max(hi[a], x);
        }
    }
  }

  // One binary median split of perm[b, e) on the longest centroid axis.
  int median_split(int b, int e) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = b; k < e; ++k)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], centroid(perm[k], a));
        hi[a] = std::max(hi[a], centroid(perm[k], a));
      }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
      if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
    std::sort(perm.begin() + b, perm.begin() + e, [&](int x, int y) {
      double cx = centroid(x, ax), cy = centroid(y, ax);
      return cx < cy || (cx == cy && x < y);
    });
    return b + (e - b) / 2;
  }

  void split(int b, int e, int levels, std::vector<std::pair<int, int>>& out) {
    if (levels == 0 || e - b <= c) { out.push_back({b, e}); return; }
    int m = median_split(b, e);
    split(b, m, levels - 1, out);
    split(m, e, levels - 1, out);
  }

  int build(int b, int e, int depth) {
    int id = (int)nodes.size();
    nodes.emplace_back();
    fit(b, e, nodes[id].lo, nodes[id].hi);
    nodes[id].depth = depth;
    if (e - b <= c) { nodes[id].tri_begin = b; nodes[id].tri_end = e; return id; }
    int levels = (B == 2) ? 1 : (B == 4) ? 2 : 3;
    std::vector<std::pair<int, int>> parts;
    split(b, e, levels, parts);
    std::vector<int> ch;
    for (auto& p : parts) ch.push_back(build(p.first, p.second, depth + 1));
    nodes[id].children = ch;
    return id;
  }
};

inline int bitlen64(int64_t x) { int n = 0; while (x > 0) { ++n; x >>= 1; } return n; }

// Smallest lattice exponent whose cell 2^e is at least 2^-30 of |origin|, so
// origin + k 2^e moves with every k in fp64 (and the lattice search loops
// terminate) even for a zero-extent mesh.
inline int min_cell_exp(double origin_abs) {
  if (!(origin_abs > 0)) return -100;
  return std::max(-100, std::ilogb(origin_abs) - 30);
}

template <class X> void put(std::vector<uint8_t>& buf, size_t off, X x) { std::memcpy(&buf[off], &x, sizeof(X)); }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// Directed rounding to IEEE binary16 by search over the sorted table of all
// finite half values (obviously correct; used once per node at build time).
static const std::vector<std::pair<double, uint16_t>>& half_table() {
  static std::vector<std::pair<double, uint16_t>> t;
  if (t.empty()) {
    for (uint32_t h = 0; h < 65536; ++h) {
      const uint32_t e = (h >> 10) & 31u, m = h & 1023u;
      if (e == 31) continue;  // inf / nan
      double v = e == 0 ? std::ldexp((double)m, -24) : std::ldexp((double)(m | 1024u), (int)e - 25);
      if (h & 0x8000u) v = -v;
      t.push_back({v, (uint16_t)h});
    }
    std::sort(t.begin(), t.end(), [](const std::pair<double, uint16_t>& a, const std::pair<double, uint16_t>& b) {
      return a.first < b.first || (a.first == b.first && a.second < b.second);
    });
  }
  return t;
}

bool half_round(double x, bool up, uint16_t* out) {
  const auto& t = half_table();
  if (up) {  // smallest half >= x
    auto it = std::lower_bound(t.begin(), t.end(), x, [](const std::pair<double, uint16_t>& a, double v) { return a.first < v; });
    if (it == t.end()) return false;
    *out = it->second;
  } else {   // largest half <= x
    auto it = std::upper_bound(t.begin(), t.end(), x, [](double v, const std::pair<double, uint16_t>& a) { return v < a.first; });
    if (it == t.begin()) return false;
    *out = (--it)->second;
  }
  return true;
}

int build_blob(const cbvh_mesh* mesh, int branching, int bits, const cbvh_build_opts* opts,
               std::vector<uint8_t>& out) {
  if (!mesh) return set_error(CBVH_EINVAL, "mesh is null");
  if (branching != 2 && branching != 4 && branching != 8) return set_error(CBVH_EINVAL, "branching must be 2, 4 or 8");
  if (bits < 2 || bits > 16) return set_error(CBVH_EINVAL, "bits must be in [2, 16]");
  int T = opts ? opts->treelet_nodes : 32;
  int c = opts ? opts->leaf_size : 4;
  if (T < branching || T > (1 << 20)) return set_error(CBVH_EINVAL, "treelet_nodes must be >= branching");
  if (c < 1 || c > 4) return set_error(CBVH_EINVAL, "leaf_size must be in [1, 4]");
  const int layout = opts ? opts->layout : CBVH_LAYOUT_DELTA;
  const int kdop = (opts && opts->kdop) ? opts->kdop : 6;
  if (kdop != 6 && kdop != 14 && kdop != 18 && kdop != 26) return set_error(CBVH_EINVAL, "kdop must be 6, 14, 18 or 26");
  if (kdop != 6 && layout != CBVH_LAYOUT_DELTA) return set_error(CBVH_EINVAL, "k-DOPs use the delta layout");
  if (layout != CBVH_LAYOUT_DELTA && layout != CBVH_LAYOUT_FP16 && layout != CBVH_LAYOUT_FP32)
    return set_error(CBVH_EINVAL, "layout must be CBVH_LAYOUT_DELTA, _FP16 or _FP32");
  const bool aligned = opts && (opts->align_treelets || opts->zero_suppress);
  const bool zs = opts && opts->zero_suppress;
  if (zs && (bits <= 4 || layout != CBVH_LAYOUT_DELTA || kdop != 6))
    return set_error(CBVH_EINVAL, "zero_suppress needs the delta AABB layout with 8- or 16-bit fields (bits > 4)");
  if (aligned && (T < 4 || T > 64 || (T & (T - 1)) || layout != CBVH_LAYOUT_DELTA || kdop != 6))
    return set_error(CBVH_EINVAL, "align_treelets needs the delta AABB layout and a power-of-two T in [4, 64]");
  if (!mesh->vertices || !mesh->triangles) return set_error(CBVH_EINVAL, "null mesh arrays");
  const int64_t nv = mesh->num_vertices, nt = mesh->num_triangles;
  if (nt <= 0 || nv <= 0) return set_error(CBVH_EMESH, "empty mesh");
  if (nt >= (int64_t(1) << 29)) return set_error(CBVH_EMESH, "too many triangles (max 2^29 - 1)");
  for (int64_t i = 0; i < 3 * nt; ++i)
    if (mesh->triangles[i] < 0 || mesh->triangles[i] >= nv) return set_error(CBVH_EMESH, "triangle index out of range");
  for (int64_t i = 0; i < 3 * nv; ++i)
    if (!std::isfinite(mesh->vertices[i])) return set_error(CBVH_EMESH, "non-finite vertex");

  Builder bd;
  bd.V = mesh->vertices; bd.T = mesh->triangles; bd.nt = nt; bd.B = branching; bd.c = c;
  bd.perm.resize(nt);
  bd.cen.resize(3 * (size_t)nt);
  for (int64_t t = 0; t < nt; ++t) {
    bd.perm[t] = (int)t;
    for (int a = 0; a < 3; ++a) {
      double s = 0;
      for (int v = 0; v < 3; ++v) s += (double)mesh->vertices[3 * (int64_t)mesh->triangles[3 * t + v] + a];
      bd.cen[3 * t + a] = s / 3.0;
    }
  }
  bd.build(0, (int)nt, 0);
  const int n = (int)bd.nodes.size();
  if (n >= (1 << 28)) return set_error(CBVH_EMESH, "too many nodes (max 2^28 - 1)");

  // ---- integer lattice (reading R3): origin = root lo (fp32 values), cell 2^e
  const BNode& root = bd.nodes[0];
  double ext = 0;
  for (int a = 0; a < 3; ++a) ext = std::max(ext, root.hi[a] - root.lo[a]);
  int e = (ext > 0) ? (int)std::ceil(std::log2(ext)) - 22 : -100;
  e = std::max(-100, std::min(100, e));
  while (std::ldexp(ext, -e) > double(1 << 22)) ++e;  // guard log2 rounding
  float origin[3] = {(float)root.lo[0], (float)root.lo[1], (float)root.lo[2]};
  // the cell must stay resolvable next to the origin (origin + k 2^e distinct
  // in fp64): a mesh whose extent is tiny or zero against its distance from
  // 0 (a point, a sliver far out) gets a coarser lattice instead of a cell
  // below the origin's ulp
  e = std::max(e, min_cell_exp(std::max(std::fabs(origin[0]), std::max(std::fabs(origin[1]), std::fabs(origin[2])))));
  // x - origin can round in fp64 when |x| << |origin| (e.g. x ~ 1e-17), so
  // the floor/ceil estimate is corrected until origin + k 2^e (exact in fp64
  // for these magnitudes) lies on the conservative side of x.
  auto lat_at = [&](int64_t k, int a) { return (double)origin[a] + std::ldexp((double)k, e); };
  auto lat_lo = [&](double x, int a) {
    int64_t k = (int64_t)std::floor(std::ldexp(x - (double)origin[a], -e));
    while (lat_at(k, a) > x) --k;
    while (lat_at(k + 1, a) <= x) ++k;
    return k;
  };
  auto lat_hi = [&](double x, int a) {
    int64_t k = (int64_t)std::ceil(std::ldexp(x - (double)origin[a], -e));
    while (lat_at(k, a) < x) ++k;
    while (lat_at(k - 1, a) >= x) --k;
    return k;
  };

  std::vector<int64_t> lbox(6 * (size_t)n);  // exact boxes on the lattice (conservative)
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      lbox[6 * i + a] = lat_lo(bd.nodes[i].lo[a], a);
      lbox[6 * i + 3 + a] = lat_hi(bd.nodes[i].hi[a], a);
    }
  int64_t rootbox[6];
  for (int k = 0; k < 6; ++k) rootbox[k] = lbox[k];

  // ---- predictor–corrector codes, top-down against DECODED parents
  std::vector<int64_t> dec(6 * (size_t)n);
  std::vector<uint16_t> code(6 * (size_t)n, 0);
  for (int k = 0; k < 6; ++k) dec[k] = rootbox[k];  // root == anchor -> zero codes
  {
    std::vector<int> stack = {0};
    while (!stack.empty()) {
      int p = stack.back(); stack.pop_back();
      for (int ch : bd.nodes[p].children) {
        for (int a = 0; a < 3; ++a) {
          int64_t Plo = dec[6 * p + a], Phi = dec[6 * p + 3 + a];
          int64_t Clo = lbox[6 * ch + a], Chi = lbox[6 * ch + 3 + a];
          if (Clo < Plo || Chi > Phi) return set_error(CBVH_EMESH, "internal: child not inside decoded parent");
          int s = std::max(0, bitlen64(Phi - Plo) - bits);
          int64_t qlo = (Clo - Plo) >> s, qhi = (Phi - Chi) >> s;
          if (qlo >= (1 << bits) || qhi >= (1 << bits)) return set_error(CBVH_EMESH, "internal: correction overflow");
          code[6 * ch + a] = (uint16_t)qlo;
          code[6 * ch + 3 + a] = (uint16_t)qhi;
          dec[6 * ch + a] = Plo + (qlo << s);
          dec[6 * ch + 3 + a] = Phi - (qhi << s);
        }
        stack.push_back(ch);
      }
    }
  }

  // ---- k-DOP (Table I): k/2 - 3 extra slab directions,
  // each on its own lattice (origin = fp32 floor of the root's min projection,
  // cell 2^e_a), coded like the box axes against the decoded parent.
  const int nx = kdop / 2 - 3;
  std::vector<std::array<int, 3>> xdir;
  if (kdop == 14 || kdop == 26) xdir.insert(xdir.end(), {{1, 1, 1}, {1, 1, -1}, {1, -1, 1}, {-1, 1, 1}});
  if (kdop == 18 || kdop == 26)
    xdir.insert(xdir.end(), {{1, 1, 0}, {1, -1, 0}, {1, 0, 1}, {1, 0, -1}, {0, 1, 1}, {0, 1, -1}});
  std::vector<int64_t> xdec(2 * (size_t)nx * n), xcode_v(2 * (size_t)nx * n, 0);
  std::vector<float> xorigin(nx);
  std::vector<int> xexp(nx);
  std::vector<int64_t> xroot(2 * (size_t)nx);
  if (nx > 0) {
    // exact projections (integer directions: sums of <= 3 fp32 values, exact
    // in fp64), per node bottom-up (children have larger build ids)
    std::vector<double> plo((size_t)nx * n, INFINITY), phi((size_t)nx * n, -INFINITY);
    for (int i = n - 1; i >= 0; --i) {
      const BNode& nd = bd.nodes[i];
      if (nd.children.empty()) {
        for (int k = nd.tri_begin; k < nd.tri_end; ++k)
          for (int v = 0; v < 3; ++v) {
            const float* x = &mesh->vertices[3 * (int64_t)mesh->triangles[3 * (int64_t)bd.perm[k] + v]];
            for (int a = 0; a < nx; ++a) {
              const double d = xdir[a][0] * (double)x[0] + xdir[a][1] * (double)x[1] + xdir[a][2] * (double)x[2];
              plo[(size_t)a * n + i] = std::min(plo[(size_t)a * n + i], d);
              phi[(size_t)a * n + i] = std::max(phi[(size_t)a * n + i], d);
            }
          }
      } else {
        for (int ch : nd.children)
          for (int a = 0; a < nx; ++a) {
            plo[(size_t)a * n + i] = std::min(plo[(size_t)a * n + i], plo[(size_t)a * n + ch]);
            phi[(size_t)a * n + i] = std::max(phi[(size_t)a * n + i], phi[(size_t)a * n + ch]);
          }
      }
    }
    for (int a = 0; a < nx; ++a) {
      const double rlo = plo[(size_t)a * n], rhi = phi[(size_t)a * n];
      float o = (float)rlo;
      if ((double)o > rlo) o = std::nextafter(o, -INFINITY);
      const double ex = rhi - (double)o;
      int ea = ex > 0 ? (int)std::ceil(std::log2(ex)) - 22 : -100;
      ea = std::max(-100, std::min(100, ea));
      while (std::ldexp(ex, -ea) > double(1 << 22)) ++ea;
      ea = std::max(ea, min_cell_exp(std::fabs(o)));
      xorigin[a] = o;
      xexp[a] = ea;
      auto at = [&](int64_t k) { return (double)o + std::ldexp((double)k, ea); };
      auto llo = [&](double x) {
        int64_t k = (int64_t)std::floor(std::ldexp(x - (double)o, -ea));
        while (at(k) > x) --k;
        while (at(k + 1) <= x) ++k;
        return k;
      };
      auto lhi = [&](double x) {
        int64_t k = (int64_t)std::ceil(std::ldexp(x - (double)o, -ea));
        while (at(k) < x) ++k;
        while (at(k - 1) >= x) --k;
        return k;
      };
      std::vector<int64_t> L(2 * (size_t)n);
      for (int i = 0; i < n; ++i) {
        L[2 * i] = llo(plo[(size_t)a * n + i]);
        L[2 * i + 1] = lhi(phi[(size_t)a * n + i]);
      }
      xroot[2 * a] = L[0];
      xroot[2 * a + 1] = L[1];
      xdec[((size_t)a * n + 0) * 2] = L[0];
      xdec[((size_t)a * n + 0) * 2 + 1] = L[1];
      std::vector<int> stack = {0};
      while (!stack.empty()) {
        int pn = stack.back(); stack.pop_back();
        for (int ch : bd.nodes[pn].children) {
          const int64_t Plo = xdec[((size_t)a * n + pn) * 2], Phi = xdec[((size_t)a * n + pn) * 2 + 1];
          const int64_t Clo = L[2 * ch], Chi = L[2 * ch + 1];
          if (Clo < Plo || Chi > Phi) return set_error(CBVH_EMESH, "internal: k-DOP child not inside decoded parent");
          const int sh = std::max(0, bitlen64(Phi - Plo) - bits);
          const int64_t qlo = (Clo - Plo) >> sh, qhi = (Phi - Chi) >> sh;
          if (qlo >= (1 << bits) || qhi >= (1 << bits)) return set_error(CBVH_EMESH, "internal: correction overflow");
          xcode_v[((size_t)a * n + ch) * 2] = qlo;
          xcode_v[((size_t)a * n + ch) * 2 + 1] = qhi;
          xdec[((size_t)a * n + ch) * 2] = Plo + (qlo << sh);
          xdec[((size_t)a * n + ch) * 2 + 1] = Phi - (qhi << sh);
          stack.push_back(ch);
        }
      }
    }
  }

  // ---- greedy BFS treelet packing of sibling groups (reading R6)
  struct Group { int parent; std::vector<int> nodes; };
  struct Treelet { int64_t anchor[6]; int first, count; };
  std::vector<Treelet> treelets;
  std::vector<int> new_id(n, -1), order;
  order.reserve(n);
  std::deque<Group> roots;
  roots.push_back(Group{-1, {0}});
  while (!roots.empty()) {
    Group g0 = roots.front(); roots.pop_front();
    Treelet tl;
    for (int k = 0; k < 6; ++k) tl.anchor[k] = (g0.parent < 0) ? rootbox[k] : dec[6 * g0.parent + k];
    tl.first = (int)order.size();
    int count = 0;
    std::deque<Group> bfs;
    bfs.push_back(g0);
    while (!bfs.empty()) {
      Group g = bfs.front(); bfs.pop_front();
      if (count + (int)g.nodes.size() > T) { roots.push_back(g); continue; }
      for (int x : g.nodes) { new_id[x] = (int)order.size(); order.push_back(x); }
      count += (int)g.nodes.size();
      for (int x : g.nodes)
        if (!bd.nodes[x].children.empty()) bfs.push_back(Group{x, bd.nodes[x].children});
    }
    tl.count = count;
    treelets.push_back(tl);
  }

  // aligned treelets: whole treelets are packed next-fit, in creation order,
  // into T-slot blocks (node id = block * T + offset); a treelet never
  // straddles a block boundary and the slots a block does not fill are
  // padding.  A block is the unit the traversal stages in shared memory.
  int nslots = n;
  if (aligned) {
    int fill = 0, block = 0;
    for (auto& tl : treelets) {
      if (fill + tl.count > T) { ++block; fill = 0; }
      const int first = block * T + fill;
      for (int j = 0; j < tl.count; ++j) new_id[order[tl.first + j]] = first + j;
      tl.first = first;
      fill += tl.count;
    }
    nslots = (block + 1) * T;
  }
  // node id -> original node (-1: a padding slot)
  std::vector<int> slot_node(nslots, -1);
  for (int x = 0; x < n; ++x) slot_node[new_id[x]] = x;

  // ---- triangle soup in leaf order of the new numbering
  std::vector<uint32_t> topo(nslots, kPadTopo), tri_index;
  std::vector<float> soup;
  tri_index.reserve(nt);
  soup.reserve(12 * (size_t)nt);
  int depth = 0, leaves = 0;
  for (int nid = 0; nid < nslots; ++nid) {
    if (slot_node[nid] < 0) continue;
    const BNode& nd = bd.nodes[slot_node[nid]];
    depth = std::max(depth, nd.depth);
    if (nd.children.empty()) {
      ++leaves;
      uint32_t first = (uint32_t)tri_index.size(), cnt = (uint32_t)(nd.tri_end - nd.tri_begin);
      // 48-byte records: v0 v1 v2 (xyz fp32) + 3 pad floats that carry the
      // leaf's slab — a tighter bound of its triangles than its box (used by
      // the device's box-vs-leaf test): record 0's pad = unit slab normal n
      // (area-weighted mean of the triangle normals, fp32), record 1's pad =
      // (dmin, dmax, 0) = the range of n.v over the leaf's vertices, computed
      // in fp64 with the fp32 n and rounded outward (single-triangle leaves
      // carry no range: the device takes it from the triangle's vertices).
      double nsum[3] = {0, 0, 0};
      std::vector<std::array<double, 3>> lv;
      for (int k = nd.tri_begin; k < nd.tri_end; ++k) {
        int t = bd.perm[k];
        tri_index.push_back((uint32_t)t);
        double w[3][3];
        for (int v = 0; v < 3; ++v)
          for (int a = 0; a < 3; ++a) {
            float x = mesh->vertices[3 * (int64_t)mesh->triangles[3 * (int64_t)t + v] + a];
            soup.push_back(x);
            w[v][a] = (double)x;
          }
        for (int z = 0; z < 3; ++z) soup.push_back(0.0f);
        for (int v = 0; v < 3; ++v) lv.push_back({w[v][0], w[v][1], w[v][2]});
        double e1[3] = {w[1][0] - w[0][0], w[1][1] - w[0][1], w[1][2] - w[0][2]};
        double e2[3] = {w[2][0] - w[0][0], w[2][1] - w[0][1], w[2][2] - w[0][2]};
        nsum[0] += e1[1] * e2[2] - e1[2] * e2[1];
        nsum[1] += e1[2] * e2[0] - e1[0] * e2[2];
        nsum[2] += e1[0] * e2[1] - e1[1] * e2[0];
      }
      double len = std::sqrt(nsum[0] * nsum[0] + nsum[1] * nsum[1] + nsum[2] * nsum[2]);
      float nf[3] = {0.f, 0.f, 1.f};
      if (len > 0)
        for (int a = 0; a < 3; ++a) nf[a] = (float)(nsum[a] / len);
      double dmin = INFINITY, dmax = -INFINITY;
      for (const auto& v : lv) {
        const double d = (double)nf[0] * v[0] + (double)nf[1] * v[1] + (double)nf[2] * v[2];
        dmin = std::min(dmin, d);
        dmax = std::max(dmax, d);
      }
      float fmin_ = (float)dmin, fmax_ = (float)dmax;
      if ((double)fmin_ > dmin) fmin_ = std::nextafter(fmin_, -INFINITY);
      if ((double)fmax_ < dmax) fmax_ = std::nextafter(fmax_, INFINITY);
      float* rec0 = &soup[12 * (size_t)first];
      rec0[9] = nf[0]; rec0[10] = nf[1]; rec0[11] = nf[2];
      if (cnt > 1) {
        float* rec1 = &soup[12 * ((size_t)first + 1)];
        rec1[9] = fmin_; rec1[10] = fmax_; rec1[11] = 0.0f;
      }
      topo[nid] = 0x80000000u | ((cnt - 1) << 29) | first;
    } else {
      uint32_t first = (uint32_t)new_id[nd.children[0]], cnt = (uint32_t)nd.children.size();
      for (uint32_t k = 0; k < cnt; ++k)
        if (new_id[nd.children[k]] != (int)(first + k)) return set_error(CBVH_EMESH, "internal: sibling group split");
      topo[nid] = ((cnt - 1) << 28) | first;
    }
  }

  // ---- serialize
  const uint32_t w = layout == CBVH_LAYOUT_FP32 ? 32u : layout == CBVH_LAYOUT_FP16 ? 16u
                   : bits <= 4 ? 4u : bits <= 8 ? 8u : 16u;
  const int nax = kdop / 2;
  const size_t code_bytes_node = 2 * (size_t)nax * w / 8;
  // zero-suppressed codes (integer compression): per
  // T-slot block a 16-byte aligned region = T field-presence masks (bit f:
  // field f is non-zero) followed by the non-zero fields of the block's
  // nodes in node and field order (w/8 bytes each); a table of region
  // offsets (u32, 16-byte units from off_codes, one per block plus the end)
  std::vector<uint8_t> zcodes;
  std::vector<uint32_t> zoff;
  if (zs) {
    const int nblocks = nslots / T;
    for (int b = 0; b < nblocks; ++b) {
      zoff.push_back((uint32_t)(zcodes.size() / 16));
      const size_t base = zcodes.size();
      zcodes.resize(base + T, 0);
      for (int j = 0; j < T; ++j) {
        const int on = slot_node[(size_t)b * T + j];
        if (on < 0) continue;
        const uint16_t* q = &code[6 * (size_t)on];
        uint8_t mask = 0;
        for (int f = 0; f < 6; ++f) {
          if (!q[f]) continue;
          mask |= (uint8_t)(1u << f);
          zcodes.push_back((uint8_t)(q[f] & 255u));
          if (w == 16) zcodes.push_back((uint8_t)(q[f] >> 8));
        }
        zcodes[base + j] = mask;
      }
      zcodes.resize((zcodes.size() + 15) / 16 * 16, 0);
    }
    zoff.push_back((uint32_t)(zcodes.size() / 16));
  }
  size_t off_topo = 256;
  size_t off_codes = align256(off_topo + 4 * (size_t)nslots);
  size_t off_blocks = zs ? align256(off_codes + zcodes.size()) : 0;
  size_t off_axes = zs ? align256(off_blocks + 4 * zoff.size()) : align256(off_codes + code_bytes_node * (size_t)nslots);
  size_t off_treelets = align256(off_axes + 16 * (size_t)nx);
  size_t off_tris = align256(off_treelets + 32 * treelets.size());
  size_t off_tri_index = align256(off_tris + 48 * (size_t)nt);
  size_t total = align256(off_tri_index + 4 * (size_t)nt);
  try {
    out.assign(total, 0);
  } catch (const std::bad_alloc&) {
    return set_error(CBVH_ENOMEM, "blob allocation failed");
  }
  std::memcpy(&out[0], "CBVH", 4);
  put<uint32_t>(out, 4, 5u);
  put<uint32_t>(out, 8, (uint32_t)branching);
  put<uint32_t>(out, 12, (uint32_t)bits);
  put<uint32_t>(out, 16, (uint32_t)T);
  put<uint32_t>(out, 20, (uint32_t)c);
  put<uint32_t>(out, 24, w);
  put<uint32_t>(out, 28, (uint32_t)nslots);
  put<uint32_t>(out, 32, (uint32_t)nt);
  put<uint32_t>(out, 36, (uint32_t)treelets.size());
  put<uint32_t>(out, 40, (uint32_t)depth);
  put<uint32_t>(out, 44, (uint32_t)leaves);
  put<int32_t>(out, 48, e);
  for (int a = 0; a < 3; ++a) put<float>(out, 52 + 4 * a, origin[a]);
  for (int k = 0; k < 6; ++k) put<int32_t>(out, 64 + 4 * k, (int32_t)rootbox[k]);
  put<uint64_t>(out, 88, off_topo);
  put<uint64_t>(out, 96, off_codes);
  put<uint64_t>(out, 104, off_treelets);
  put<uint64_t>(out, 112, off_tris);
  put<uint64_t>(out, 120, off_tri_index);
  put<uint64_t>(out, 128, total);
  put<uint32_t>(out, 136, (uint32_t)layout);
  put<uint32_t>(out, 140, (uint32_t)kdop);
  put<uint64_t>(out, 144, off_axes);
  put<uint32_t>(out, 152, (aligned ? CBVH_FLAG_ALIGNED_TREELETS : 0u) | (zs ? CBVH_FLAG_ZERO_SUPPRESSED : 0u));
  put<uint32_t>(out, 156, (uint32_t)n);
  put<uint64_t>(out, 160, off_blocks);
  if (zs) {
    std::memcpy(&out[off_codes], zcodes.data(), zcodes.size());
    std::memcpy(&out[off_blocks], zoff.data(), 4 * zoff.size());
  }
  for (int a = 0; a < nx; ++a) {
    const size_t o = off_axes + 16 * (size_t)a;
    put<float>(out, o, xorigin[a]);
    put<int32_t>(out, o + 4, xexp[a]);
    put<int32_t>(out, o + 8, (int32_t)xroot[2 * a]);
    put<int32_t>(out, o + 12, (int32_t)xroot[2 * a + 1]);
  }
  std::memcpy(&out[off_topo], topo.data(), 4 * (size_t)nslots);
  for (int nid = 0; nid < nslots && !zs; ++nid) {
    if (slot_node[nid] < 0) continue;  // padding: zero codes
    const int on = slot_node[nid];
    const uint16_t* q = &code[6 * (size_t)on];
    uint8_t* dst = &out[off_codes + code_bytes_node * nid];
    const BNode& nd = bd.nodes[on];
    if (layout == CBVH_LAYOUT_FP32) {
      // absolute boxes: min/max of fp32 coordinates are fp32 values (exact)
      for (int a = 0; a < 3; ++a) {
        put<float>(out, off_codes + code_bytes_node * nid + 4 * a, (float)nd.lo[a]);
        put<float>(out, off_codes + code_bytes_node * nid + 12 + 4 * a, (float)nd.hi[a]);
      }
    } else if (layout == CBVH_LAYOUT_FP16) {
      // binary16 (§III.A), rounded outward: lo down, hi up
      for (int a = 0; a < 3; ++a) {
        uint16_t hl, hh;
        if (!half_round(nd.lo[a], false, &hl) || !half_round(nd.hi[a], true, &hh))
          return set_error(CBVH_EMESH, "coordinate outside the binary16 range");
        put<uint16_t>(out, off_codes + code_bytes_node * nid + 2 * a, hl);
        put<uint16_t>(out, off_codes + code_bytes_node * nid + 6 + 2 * a, hh);
      }
    } else {
      // fields lo[0..nax) then hi[0..nax): box axes x, y, z, then the k-DOP axes
      std::vector<uint32_t> f(2 * (size_t)nax);
      for (int a = 0; a < 3; ++a) { f[a] = q[a]; f[nax + a] = q[3 + a]; }
      for (int a = 0; a < nx; ++a) {
        f[3 + a] = (uint32_t)xcode_v[((size_t)a * n + on) * 2];
        f[nax + 3 + a] = (uint32_t)xcode_v[((size_t)a * n + on) * 2 + 1];
      }
      if (w == 16) {
        for (size_t k = 0; k < f.size(); ++k) { const uint16_t v = (uint16_t)f[k]; std::memcpy(dst + 2 * k, &v, 2); }
      } else if (w == 8) {
        for (size_t k = 0; k < f.size(); ++k) dst[k] = (uint8_t)f[k];
      } else {
        for (size_t k = 0; k < f.size(); k += 2) dst[k / 2] = (uint8_t)((f[k] & 15u) | ((f[k + 1] & 15u) << 4));
      }
    }
  }
  for (size_t k = 0; k < treelets.size(); ++k) {
    size_t o = off_treelets + 32 * k;
    for (int j = 0; j < 6; ++j) put<int32_t>(out, o + 4 * j, (int32_t)treelets[k].anchor[j]);
    put<uint32_t>(out, o + 24, (uint32_t)treelets[k].first);
    put<uint32_t>(out, o + 28, (uint32_t)treelets[k].count);
  }
  std::memcpy(&out[off_tris], soup.data(), 48 * (size_t)nt);
  std::memcpy(&out[off_tri_index], tri_index.data(), 4 * (size_t)nt);
  return CBVH_OK;
}

int parse_header(const uint8_t* p, size_t bytes, cbvh_header* h) {
  if (!p || !h) return set_error(CBVH_EINVAL, "null blob or header");
  if (bytes < 256 || std::memcmp(p, "CBVH", 4) != 0) return set_error(CBVH_EBLOB, "bad magic");
  auto u32 = [&](size_t o) { uint32_t x; std::memcpy(&x, p + o, 4); return x; };
  auto u64 = [&](size_t o) { uint64_t x; std::memcpy(&x, p + o, 8); return x; };
  if (u32(4) != 5) return set_error(CBVH_EBLOB, "unsupported blob version");
  h->layout = u32(136);
  if (h->layout > 2) return set_error(CBVH_EBLOB, "bad layout");
  h->kdop = u32(140);
  h->off_axes = u64(144);
  h->flags = u32(152);
  h->real_nodes = u32(156);
  h->off_blocks = u64(160);
  if (h->flags & ~(uint32_t)(CBVH_FLAG_ALIGNED_TREELETS | CBVH_FLAG_ZERO_SUPPRESSED))
    return set_error(CBVH_EBLOB, "unknown header flags");
  if (h->kdop != 6 && h->kdop != 14 && h->kdop != 18 && h->kdop != 26) return set_error(CBVH_EBLOB, "bad k");
  if (h->kdop != 6 && h->layout != CBVH_LAYOUT_DELTA) return set_error(CBVH_EBLOB, "k-DOP with an absolute layout");
  h->branching = u32(8); h->bits = u32(12); h->treelet_nodes = u32(16); h->leaf_size = u32(20);
  h->code_width = u32(24); h->num_nodes = u32(28); h->num_tris = u32(32); h->num_treelets = u32(36);
  h->depth = u32(40); h->num_leaves = u32(44);
  std::memcpy(&h->lattice_exp, p + 48, 4);
  std::memcpy(h->origin, p + 52, 12);
  std::memcpy(h->root_box, p + 64, 24);
  h->off_topo = u64(88); h->off_codes = u64(96); h->off_treelets = u64(104);
  h->off_tris = u64(112); h->off_tri_index = u64(120); h->total_bytes = u64(128);
  if (h->total_bytes != bytes) return set_error(CBVH_EBLOB, "blob size does not match header");
  if (h->branching != 2 && h->branching != 4 && h->branching != 8) return set_error(CBVH_EBLOB, "bad branching");
  if (h->bits < 2 || h->bits > 16) return set_error(CBVH_EBLOB, "bad bits");
  const uint32_t want_w = h->layout == CBVH_LAYOUT_FP32 ? 32u : h->layout == CBVH_LAYOUT_FP16 ? 16u
                        : h->bits <= 4 ? 4u : h->bits <= 8 ? 8u : 16u;
  if (h->code_width != want_w) return set_error(CBVH_EBLOB, "bad code width");
  if (h->num_nodes == 0 || h->num_tris == 0 || h->num_nodes >= (1u << 28) || h->num_tris >= (1u << 29))
    return set_error(CBVH_EBLOB, "bad counts");
  const uint64_t cb = (uint64_t)h->kdop * h->code_width / 8;
  const bool zs = (h->flags & CBVH_FLAG_ZERO_SUPPRESSED) != 0;
  if (zs && (!(h->flags & CBVH_FLAG_ALIGNED_TREELETS) || h->code_width < 8 || h->kdop != 6))
    return set_error(CBVH_EBLOB, "bad zero-suppressed layout");
  // zero-suppressed: codes section [off_codes, off_blocks), then the block
  // offset table (num_nodes / T + 1 words) up to off_axes
  const uint64_t code_end = zs ? h->off_blocks : h->off_codes + cb * h->num_nodes;
  if (zs && (h->off_blocks < h->off_codes || (h->off_blocks & 15) ||
             h->off_blocks + 4ull * (h->num_nodes / h->treelet_nodes + 1) > h->off_axes))
    return set_error(CBVH_EBLOB, "bad section offsets");
  if (h->off_topo < 256 || h->off_topo + 4ull * h->num_nodes > h->off_codes ||
      code_end > h->off_axes || h->off_axes + 16ull * (h->kdop / 2 - 3) > h->off_treelets ||
      h->off_treelets + 32ull * h->num_treelets > h->off_tris ||
      h->off_tris + 48ull * h->num_tris > h->off_tri_index ||
      h->off_tri_index + 4ull * h->num_tris > h->total_bytes)
    return set_error(CBVH_EBLOB, "bad section offsets");
  if ((h->off_topo | h->off_codes | h->off_tris) & 15) return set_error(CBVH_EBLOB, "misaligned sections");
  if (h->real_nodes == 0 || h->real_nodes > h->num_nodes) return set_error(CBVH_EBLOB, "bad node count");
  if ((h->flags & CBVH_FLAG_ALIGNED_TREELETS) &&
      (h->treelet_nodes > 64 || (h->treelet_nodes & (h->treelet_nodes - 1)) || h->layout != CBVH_LAYOUT_DELTA ||
       h->kdop != 6 || h->num_nodes % h->treelet_nodes != 0))
    return set_error(CBVH_EBLOB, "bad aligned-treelet layout");
  if (!(h->flags & CBVH_FLAG_ALIGNED_TREELETS) && h->real_nodes != h->num_nodes)
    return set_error(CBVH_EBLOB, "bad node count");
  return CBVH_OK;
}

}  // namespace cbvh

extern "C" {

int build_compressed_bvh(const cbvh_mesh* mesh, int branching, int bits, const cbvh_build_opts* opts,
                         uint8_t** blob, size_t* blob_bytes) {
  if (!blob || !blob_bytes) return cbvh::set_error(CBVH_EINVAL, "null output pointer");
  *blob = nullptr; *blob_bytes = 0;
  std::vector<uint8_t> out;
  int rc;
  try {
    rc = cbvh::build_blob(mesh, branching, bits, opts, out);
  } catch (const std::bad_alloc&) {
    return cbvh::set_error(CBVH_ENOMEM, "allocation failed during build");
  } catch (...) {
    return cbvh::set_error(CBVH_EMESH, "unexpected failure during build");
  }
  if (rc != CBVH_OK) return rc;
  uint8_t* p = (uint8_t*)std::malloc(out.size());
  if (!p) return cbvh::set_error(CBVH_ENOMEM, "blob allocation failed");
  std::memcpy(p, out.data(), out.size());
  *blob = p;
  *blob_bytes = out.size();
  return CBVH_OK;
}

void cbvh_free_blob(uint8_t* blob) { std::free(blob); }

int cbvh_blob_info(const uint8_t* h_blob, size_t bytes, cbvh_info* out) {
  if (!h_blob || !out) return cbvh::set_error(CBVH_EINVAL, "null argument");
  int rc = cbvh::parse_header(h_blob, bytes, &out->h);
  if (rc) return rc;
  const cbvh_header& h = out->h;
  // the hierarchy the traversal reads: topology words and codes of every node
  // slot (aligned treelets include their padding slots) and the k-DOP axis
  // table; the treelet table (anchors) is build metadata the device never
  // reads, so it is not counted
  out->bvh_bytes = 4ull * h.num_nodes + ((uint64_t)h.kdop * h.code_width / 8) * h.num_nodes + 16ull * (h.kdop / 2 - 3);
  if (h.flags & CBVH_FLAG_ZERO_SUPPRESSED) {
    // the packed regions and their offset table
    const uint64_t nblocks = h.num_nodes / h.treelet_nodes;
    uint32_t end;
    std::memcpy(&end, h_blob + h.off_blocks + 4 * nblocks, 4);
    out->bvh_bytes = 4ull * h.num_nodes + 16ull * end + 4ull * (nblocks + 1);
  }
  out->tri_bytes = 48ull * h.num_tris;
  out->bytes_per_node = (double)out->bvh_bytes / (double)h.real_nodes;
  out->code_bytes_per_node = (double)h.kdop * h.code_width / 8.0;
  return CBVH_OK;
}

}  // extern "C"
