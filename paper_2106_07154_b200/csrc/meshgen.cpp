// Host mesh generators for the B200 LTS3 path (see include/mswm_host.h).
//
// The spherical generator restates the reference's icosahedral pipeline,
// proj/src/mesh_topology.cpp:38-64 (subdivision) and
// proj/src/mesh_build.cpp:185-366 (dualisation, geometry, kites, weights),
// producing bitwise-identical tables.  It replaces the reference's
// unordered_map edge lookups with sort-based first-encounter numbering and
// per-triangle-corner edge ids, which keeps the reference's id order while
// scaling to level 11 (126M edges).  The planar generator builds a periodic
// triangular lattice and runs the same topological dualisation; only the
// metric terms are planar.  Compiled without FP contraction
// (-ffp-contract=off) so every expression rounds like the reference build.

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mswm_host.h"

namespace {

thread_local std::string g_last_error;

// --- host threads -----------------------------------------------------------
// The builder's per-element loops run on all host cores (MSWM_HOST_THREADS
// overrides); every element's arithmetic is unchanged, so the tables are
// bitwise those of the serial build.
int host_threads() {
  static const int n = [] {
    if (const char* e = std::getenv("MSWM_HOST_THREADS")) return std::max(1, std::atoi(e));
    return std::max(1, int(std::thread::hardware_concurrency()));
  }();
  return n;
}

// f(lo, hi) over [0, n) in contiguous chunks; the first exception is rethrown.
template <class F>
void par_for(int64_t n, F&& f, int64_t grain = 16384) {
  const int64_t T = std::min<int64_t>(host_threads(), std::max<int64_t>(1, n / grain));
  if (T <= 1) {
    if (n > 0) f(int64_t(0), n);
    return;
  }
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> th;
  for (int64_t k = 0; k < T; ++k)
    th.emplace_back([&, k] {
      try {
        f(n * k / T, n * (k + 1) / T);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

// Sample sort on all host threads: sorted chunks, splitters from a sorted
// sample, every chunk cut at the splitters, each bucket gathered and sorted.
template <class T>
void par_sort(std::vector<T>& v) {
  const int64_t n = int64_t(v.size());
  const int64_t C = std::min<int64_t>(host_threads(), std::max<int64_t>(1, n / 65536));
  if (C <= 1) {
    std::sort(v.begin(), v.end());
    return;
  }
  std::vector<int64_t> b(size_t(C) + 1);
  for (int64_t k = 0; k <= C; ++k) b[k] = n * k / C;
  par_for(C, [&](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) std::sort(v.begin() + b[k], v.begin() + b[k + 1]);
  }, 1);
  const int64_t S = 64 * C;
  std::vector<T> sample(S);
  for (int64_t q = 0; q < S; ++q) sample[q] = v[(n - 1) * q / (S - 1)];
  std::sort(sample.begin(), sample.end());
  std::vector<T> split(size_t(C) - 1);
  for (int64_t j = 1; j < C; ++j) split[j - 1] = sample[S * j / C];
  // cut[k][j]: start of bucket j in chunk k
  std::vector<int64_t> cut(size_t(C) * (C + 1));
  par_for(C, [&](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) {
      cut[k * (C + 1)] = b[k];
      for (int64_t j = 1; j < C; ++j)
        cut[k * (C + 1) + j] = std::lower_bound(v.begin() + cut[k * (C + 1) + j - 1],
                                                v.begin() + b[k + 1], split[j - 1]) - v.begin();
      cut[k * (C + 1) + C] = b[k + 1];
    }
  }, 1);
  std::vector<int64_t> out(size_t(C) + 1, 0);
  for (int64_t j = 0; j < C; ++j) {
    int64_t m = 0;
    for (int64_t k = 0; k < C; ++k) m += cut[k * (C + 1) + j + 1] - cut[k * (C + 1) + j];
    out[j + 1] = out[j] + m;
  }
  std::vector<T> tmp(v.size());
  par_for(C, [&](int64_t lo, int64_t hi) {
    for (int64_t j = lo; j < hi; ++j) {
      int64_t at = out[j];
      for (int64_t k = 0; k < C; ++k) {
        const int64_t x = cut[k * (C + 1) + j], y = cut[k * (C + 1) + j + 1];
        std::copy(v.begin() + x, v.begin() + y, tmp.begin() + at);
        at += y - x;
      }
      std::sort(tmp.begin() + out[j], tmp.begin() + out[j + 1]);
    }
  }, 1);
  v.swap(tmp);
}

struct V3 {
  double x, y, z;
};
inline V3 add(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(const V3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(const V3& a) { return std::sqrt(dot(a, a)); }
inline V3 unit(const V3& a) {
  const double n = norm(a);
  return {a.x / n, a.y / n, a.z / n};
}
// geometry.hpp:33-35
inline double arc(const V3& a, const V3& b) { return std::atan2(norm(cross(a, b)), dot(a, b)); }
// geometry.hpp:39-43
inline double sph_tri_area(const V3& a, const V3& b, const V3& c) {
  const double num = dot(a, cross(b, c));
  const double den = 1.0 + dot(a, b) + dot(b, c) + dot(a, c);
  return 2.0 * std::atan2(num, den);
}
// geometry.hpp:53-58
inline V3 great_circle_meet(const V3& a1, const V3& a2, const V3& b1, const V3& b2) {
  V3 p = unit(cross(cross(a1, a2), cross(b1, b2)));
  if (dot(p, add(add(add(a1, a2), b1), b2)) < 0.0) p = scale(p, -1.0);
  return p;
}

using Tri = std::array<int32_t, 3>;

struct Triangulation {
  std::vector<V3> pts;
  std::vector<Tri> tris;
};

// Sort-based first-encounter numbering of the undirected sides of a
// triangle list.  side s = 3*t + k joins tris[t][k] and tris[t][(k+1)%3].
// Returns side_id[s] in [0, n_unique), ids assigned in ascending order of
// each side's first occurrence -- the order an insertion-ordered hash map
// (the reference's edge_of / midpoint maps) produces.
std::vector<int32_t> number_sides(const std::vector<Tri>& tris, int64_t* n_unique,
                                  std::vector<uint8_t>* first = nullptr) {
  const int64_t ns = int64_t(tris.size()) * 3;
  struct KS {
    uint64_t key;
    int64_t s;
    bool operator<(const KS& o) const { return key != o.key ? key < o.key : s < o.s; }
  };
  std::vector<KS> ks(ns);
  par_for(int64_t(tris.size()), [&](int64_t lo, int64_t hi) {
    for (int64_t t = lo; t < hi; ++t)
      for (int k = 0; k < 3; ++k) {
        uint64_t a = uint32_t(tris[t][k]), b = uint32_t(tris[t][(k + 1) % 3]);
        if (a > b) std::swap(a, b);
        ks[3 * t + k] = {(a << 32) | b, 3 * t + k};
      }
  });
  par_sort(ks);
  // rep[s] = first side with the same key (the run head: sorted by (key, s))
  std::vector<int64_t> rep(ns);
  for (int64_t i = 0; i < ns;) {
    int64_t j = i;
    while (j < ns && ks[j].key == ks[i].key) ++j;
    for (int64_t q = i; q < j; ++q) rep[ks[q].s] = ks[i].s;
    i = j;
  }
  std::vector<KS>().swap(ks);
  std::vector<int32_t> id(ns, -1);
  int64_t next = 0;
  for (int64_t s = 0; s < ns; ++s)
    if (rep[s] == s) id[s] = int32_t(next++);
  par_for(ns, [&](int64_t lo, int64_t hi) {
    for (int64_t s = lo; s < hi; ++s) id[s] = id[rep[s]];
  });
  if (first) {
    first->assign(ns, 0);
    par_for(ns, [&](int64_t lo, int64_t hi) {
      for (int64_t s = lo; s < hi; ++s) (*first)[s] = rep[s] == s;
    });
  }
  *n_unique = next;
  return id;
}

// mesh_topology.cpp:13-36 -- the base icosahedron, CCW seen from outside.
Triangulation icosahedron() {
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  const double s = 1.0 / std::sqrt(1.0 + phi * phi);
  const double a = s, b = phi * s;
  Triangulation t;
  const double P[12][3] = {{-a, b, 0}, {a, b, 0},  {-a, -b, 0}, {a, -b, 0},
                           {0, -a, b}, {0, a, b},  {0, -a, -b}, {0, a, -b},
                           {b, 0, -a}, {b, 0, a},  {-b, 0, -a}, {-b, 0, a}};
  for (auto& p : P) t.pts.push_back({p[0], p[1], p[2]});
  const int F[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},  {0, 7, 10}, {0, 10, 11},
                        {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                        {3, 9, 4},  {3, 4, 2},  {3, 2, 6},  {3, 6, 8},  {3, 8, 9},
                        {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},  {9, 8, 1}};
  for (auto& f : F) {
    Tri tri{f[0], f[1], f[2]};
    const V3 &p0 = t.pts[tri[0]], &p1 = t.pts[tri[1]], &p2 = t.pts[tri[2]];
    if (dot(p0, cross(sub(p1, p0), sub(p2, p0))) < 0.0) std::swap(tri[1], tri[2]);
    t.tris.push_back(tri);
  }
  return t;
}

// mesh_topology.cpp:38-64 -- 4:1 split, midpoints normalised.
Triangulation subdivide(int level) {
  Triangulation t = icosahedron();
  for (int l = 0; l < level; ++l) {
    int64_t n_mid = 0;
    std::vector<uint8_t> first;
    const std::vector<int32_t> sid = number_sides(t.tris, &n_mid, &first);
    const int32_t base = int32_t(t.pts.size());
    t.pts.resize(size_t(base + n_mid));
    std::vector<Tri> next(t.tris.size() * 4);
    // a midpoint from its first triangle (the reference's insertion order
    // fixes only its id; add is commutative, so any side gives the same bits)
    par_for(int64_t(t.tris.size()), [&](int64_t lo, int64_t hi) {
      for (int64_t tt = lo; tt < hi; ++tt) {
        const Tri f = t.tris[tt];
        int32_t m[3];
        for (int k = 0; k < 3; ++k) {
          const int32_t id = sid[3 * tt + k];
          if (first[3 * tt + k]) t.pts[base + id] = unit(add(t.pts[f[k]], t.pts[f[(k + 1) % 3]]));
          m[k] = base + id;
        }
        const int32_t ab = m[0], bc = m[1], ca = m[2];
        next[4 * tt + 0] = {f[0], ab, ca};
        next[4 * tt + 1] = {f[1], bc, ab};
        next[4 * tt + 2] = {f[2], ca, bc};
        next[4 * tt + 3] = {ab, bc, ca};
      }
    });
    t.tris.swap(next);
  }
  return t;
}

}  // namespace

struct mswm_mesh {
  int spherical = 1;
  double radius = 1.0, width = 0.0, height = 0.0;
  int32_t nC = 0, nE = 0, nV = 0;
  std::vector<int32_t> cell_offset, cell_edges, cell_vertices, cell_cells;
  std::vector<int32_t> edge_cells, edge_vertices, vertex_cells, vertex_edges;
  std::vector<int32_t> ee_offset, edge_edges;
  std::vector<int8_t> edge_cell_sign, edge_vertex_sign;
  std::vector<double> edge_len, edge_dual_len, cell_area, vertex_area, vertex_kite, edge_weight;
  std::vector<double> kite_area;
  std::vector<double> cell_xyz, vertex_xyz, edge_xyz;

  int ring(int32_t c) const { return cell_offset[c + 1] - cell_offset[c]; }
  double cell_sign(int32_t e, int32_t c) const {
    return edge_cells[2 * e] == c ? double(edge_cell_sign[2 * e]) : double(edge_cell_sign[2 * e + 1]);
  }
  double vertex_sign(int32_t e, int32_t v) const {
    return edge_vertices[2 * e] == v ? double(edge_vertex_sign[2 * e])
                                     : double(edge_vertex_sign[2 * e + 1]);
  }
  int slot_of_edge(int32_t c, int32_t e) const {
    const int off = cell_offset[c], m = ring(c);
    for (int j = 0; j < m; ++j)
      if (cell_edges[off + j] == e) return j;
    throw std::runtime_error("edge " + std::to_string(e) + " missing from ring of cell " +
                             std::to_string(c));
  }
};

namespace {

// Topology of the dual of a closed triangulation (mesh_build.cpp:185-260):
// edges in first-encounter order with ascending edge_cells / edge_vertices,
// counterclockwise cell rings starting at the smallest neighbour id, vertex
// tables rotated so the smallest cell leads, then the edge stencil and the
// orientation signs.
void dualise_topology(const Triangulation& tri, mswm_mesh& m, bool check_euler) {
  const int64_t nT = int64_t(tri.tris.size());
  const int32_t nP = int32_t(tri.pts.size());
  int64_t nE = 0;
  const std::vector<int32_t> side_edge = number_sides(tri.tris, &nE);
  m.nC = nP;
  m.nV = int32_t(nT);
  m.nE = int32_t(nE);
  m.edge_cells.assign(2 * nE, -1);
  m.edge_vertices.assign(2 * nE, -1);
  for (int64_t t = 0; t < nT; ++t)
    for (int k = 0; k < 3; ++k) {
      const int32_t a = tri.tris[t][k], b = tri.tris[t][(k + 1) % 3];
      if (a == b || a < 0 || a >= nP || b < 0 || b >= nP)
        throw std::runtime_error("triangle " + std::to_string(t) + " has invalid corners");
      const int32_t e = side_edge[3 * t + k];
      if (m.edge_cells[2 * e] < 0) {
        m.edge_cells[2 * e] = std::min(a, b);
        m.edge_cells[2 * e + 1] = std::max(a, b);
        m.edge_vertices[2 * e] = int32_t(t);
      } else {
        if (m.edge_vertices[2 * e + 1] != -1)
          throw std::runtime_error("edge borders more than 2 triangles");
        m.edge_vertices[2 * e + 1] = int32_t(t);
      }
    }
  for (int64_t e = 0; e < nE; ++e) {
    if (m.edge_vertices[2 * e + 1] == -1) throw std::runtime_error("open edge (mesh not closed)");
    if (m.edge_vertices[2 * e] > m.edge_vertices[2 * e + 1])
      std::swap(m.edge_vertices[2 * e], m.edge_vertices[2 * e + 1]);
  }
  if (check_euler && nE != int64_t(nP) + nT - 2)
    throw std::runtime_error("Euler identity violated");

  // Fans (mesh_build.cpp:38-88): succ entries per corner in triangle order.
  std::vector<int32_t> deg(nP, 0);
  for (const Tri& f : tri.tris)
    for (int v : f) ++deg[v];
  m.cell_offset.assign(size_t(nP) + 1, 0);
  for (int32_t i = 0; i < nP; ++i) m.cell_offset[i + 1] = m.cell_offset[i] + deg[i];
  const int64_t total = m.cell_offset[nP];
  struct Succ {
    int32_t p, q, t, corner_edge;
  };
  std::vector<Succ> succ(total);
  std::vector<int32_t> fill(nP, 0);
  for (int64_t t = 0; t < nT; ++t) {
    const Tri& f = tri.tris[t];
    for (int k = 0; k < 3; ++k) {
      const int32_t i = f[k];
      succ[m.cell_offset[i] + fill[i]++] = {f[(k + 1) % 3], f[(k + 2) % 3], int32_t(t),
                                            side_edge[3 * t + k]};
    }
  }
  m.cell_edges.assign(total, -1);
  m.cell_vertices.assign(total, -1);
  m.cell_cells.assign(total, -1);
  par_for(nP, [&](int64_t lo, int64_t hi) {
  for (int32_t i = int32_t(lo); i < int32_t(hi); ++i) {
    const int32_t mm = deg[i], off = m.cell_offset[i];
    if (mm < 3) throw std::runtime_error("degenerate Voronoi cell " + std::to_string(i));
    const Succ* s = succ.data() + off;
    int32_t start = s[0].p;
    for (int k = 1; k < mm; ++k) start = std::min(start, s[k].p);
    int32_t cur = start;
    for (int j = 0; j < mm; ++j) {
      int found = -1;
      for (int k = 0; k < mm; ++k)
        if (s[k].p == cur) {
          found = k;
          break;
        }
      if (found < 0) throw std::runtime_error("non-manifold fan around cell " + std::to_string(i));
      m.cell_cells[off + j] = cur;
      m.cell_vertices[off + j] = s[found].t;
      m.cell_edges[off + j] = s[found].corner_edge;  // the side (i, cur) of triangle t
      cur = s[found].q;
    }
    if (cur != start) throw std::runtime_error("fan does not close around cell " + std::to_string(i));
  }
  });

  // Vertex tables, smallest cell first (mesh_build.cpp:249-258).
  m.vertex_cells.assign(3 * nT, -1);
  m.vertex_edges.assign(3 * nT, -1);
  par_for(nT, [&](int64_t lo, int64_t hi) {
  for (int64_t v = lo; v < hi; ++v) {
    Tri f = tri.tris[v];
    int rot = 0;
    while (f[0] > f[1] || f[0] > f[2]) {
      f = {f[1], f[2], f[0]};
      ++rot;
    }
    for (int k = 0; k < 3; ++k) {
      m.vertex_cells[3 * v + k] = f[k];
      m.vertex_edges[3 * v + k] = side_edge[3 * v + (k + rot) % 3];
    }
  }
  });

  // Edge stencil (mesh_build.cpp:133-154): both cells' rings, lower cell
  // first, each walked counterclockwise starting just after e.
  m.ee_offset.assign(size_t(nE) + 1, 0);
  for (int64_t e = 0; e < nE; ++e)
    m.ee_offset[e + 1] =
        m.ee_offset[e] + m.ring(m.edge_cells[2 * e]) + m.ring(m.edge_cells[2 * e + 1]) - 2;
  m.edge_edges.assign(m.ee_offset[nE], -1);
  par_for(nE, [&](int64_t lo, int64_t hi) {
  for (int64_t e = lo; e < hi; ++e) {
    int pos = m.ee_offset[e];
    for (int side = 0; side < 2; ++side) {
      const int32_t c = m.edge_cells[2 * e + side];
      const int off = m.cell_offset[c], mm = m.ring(c);
      const int p = m.slot_of_edge(c, int32_t(e));
      for (int k = 1; k < mm; ++k) m.edge_edges[pos++] = m.cell_edges[off + (p + k) % mm];
    }
  }
  });

  // Orientation signs (mesh_build.cpp:156-183).
  m.edge_cell_sign.assign(2 * nE, 0);
  m.edge_vertex_sign.assign(2 * nE, 0);
  par_for(nE, [&](int64_t lo, int64_t hi) {
  for (int64_t e = lo; e < hi; ++e) {
    m.edge_cell_sign[2 * e] = -1;
    m.edge_cell_sign[2 * e + 1] = +1;
    const int32_t c0 = m.edge_cells[2 * e];
    const int p = m.slot_of_edge(c0, int32_t(e));
    const int32_t after = m.cell_vertices[m.cell_offset[c0] + p];
    if (after == m.edge_vertices[2 * e]) {
      m.edge_vertex_sign[2 * e] = -1;
      m.edge_vertex_sign[2 * e + 1] = +1;
    } else if (after == m.edge_vertices[2 * e + 1]) {
      m.edge_vertex_sign[2 * e] = +1;
      m.edge_vertex_sign[2 * e + 1] = -1;
    } else {
      throw std::runtime_error("edge ring vertex does not match its endpoints");
    }
  }
  });
}

// vertex_kite (mesh_build.cpp:330-341) and TRiSK weights (:343-362), from
// kite_area / cell_area already filled in.
void finish_kites_and_weights(mswm_mesh& m) {
  m.vertex_kite.assign(size_t(3) * m.nV, 0.0);
  par_for(m.nV, [&](int64_t lo, int64_t hi) {
  for (int32_t v = int32_t(lo); v < int32_t(hi); ++v)
    for (int k = 0; k < 3; ++k) {
      const int32_t c = m.vertex_cells[3 * v + k];
      const int off = m.cell_offset[c], mm = m.ring(c);
      int slot = -1;
      for (int j = 0; j < mm; ++j)
        if (m.cell_vertices[off + j] == v) {
          slot = j;
          break;
        }
      if (slot < 0) throw std::runtime_error("vertex missing from ring of its cell");
      m.vertex_kite[3 * v + k] = m.kite_area[off + slot];
    }
  });
  m.edge_weight.assign(m.edge_edges.size(), 0.0);
  par_for(m.nE, [&](int64_t lo, int64_t hi) {
  for (int32_t e = int32_t(lo); e < int32_t(hi); ++e) {
    int pos = m.ee_offset[e];
    for (int side = 0; side < 2; ++side) {
      const int32_t c = m.edge_cells[2 * e + side];
      const int off = m.cell_offset[c], mm = m.ring(c);
      const int p = m.slot_of_edge(c, e);
      const double anchor = m.vertex_sign(e, m.cell_vertices[off + p]);
      double frac = 0.0;
      for (int k = 1; k < mm; ++k) {
        frac += m.kite_area[off + (p + k - 1) % mm] / m.cell_area[c];
        const int32_t ep = m.cell_edges[off + (p + k) % mm];
        m.edge_weight[pos++] = m.cell_sign(ep, c) * anchor * (frac - 0.5);
      }
    }
  }
  });
}

void put3(std::vector<double>& dst, int64_t i, const V3& p) {
  dst[3 * i] = p.x;
  dst[3 * i + 1] = p.y;
  dst[3 * i + 2] = p.z;
}
V3 get3(const std::vector<double>& src, int64_t i) { return {src[3 * i], src[3 * i + 1], src[3 * i + 2]}; }

// Spherical metric terms (mesh_build.cpp:262-328).
void sphere_geometry(const Triangulation& tri, mswm_mesh& m, double R) {
  const double R2 = R * R;
  m.cell_xyz.assign(size_t(3) * m.nC, 0.0);
  par_for(m.nC, [&](int64_t lo, int64_t hi) {
    for (int32_t i = int32_t(lo); i < int32_t(hi); ++i) put3(m.cell_xyz, i, unit(tri.pts[i]));
  });
  m.vertex_xyz.assign(size_t(3) * m.nV, 0.0);
  m.vertex_area.assign(m.nV, 0.0);
  par_for(m.nV, [&](int64_t lo, int64_t hi) {
  for (int32_t v = int32_t(lo); v < int32_t(hi); ++v) {
    const V3 a = get3(m.cell_xyz, m.vertex_cells[3 * v]);
    const V3 b = get3(m.cell_xyz, m.vertex_cells[3 * v + 1]);
    const V3 c = get3(m.cell_xyz, m.vertex_cells[3 * v + 2]);
    V3 cc = cross(sub(b, a), sub(c, a));
    const double len = norm(cc);
    if (len < 1e-15) throw std::runtime_error("degenerate circumcenter at vertex " + std::to_string(v));
    cc = scale(cc, 1.0 / len);
    if (dot(cc, add(add(a, b), c)) < 0.0) cc = scale(cc, -1.0);
    put3(m.vertex_xyz, v, cc);
    const double area = sph_tri_area(a, b, c) * R2;
    if (!(area > 0.0)) throw std::runtime_error("non-positive vertex area at " + std::to_string(v));
    m.vertex_area[v] = area;
  }
  });
  m.edge_xyz.assign(size_t(3) * m.nE, 0.0);
  m.edge_len.assign(m.nE, 0.0);
  m.edge_dual_len.assign(m.nE, 0.0);
  par_for(m.nE, [&](int64_t lo, int64_t hi) {
  for (int32_t e = int32_t(lo); e < int32_t(hi); ++e) {
    const V3 c0 = get3(m.cell_xyz, m.edge_cells[2 * e]);
    const V3 c1 = get3(m.cell_xyz, m.edge_cells[2 * e + 1]);
    const V3 v0 = get3(m.vertex_xyz, m.edge_vertices[2 * e]);
    const V3 v1 = get3(m.vertex_xyz, m.edge_vertices[2 * e + 1]);
    put3(m.edge_xyz, e, great_circle_meet(c0, c1, v0, v1));
    m.edge_len[e] = arc(v0, v1) * R;
    m.edge_dual_len[e] = arc(c0, c1) * R;
    if (!(m.edge_len[e] > R * 1e-14) || !(m.edge_dual_len[e] > R * 1e-14))
      throw std::runtime_error("zero-length edge " + std::to_string(e));
  }
  });
  const int64_t total = m.cell_offset[m.nC];
  m.kite_area.assign(total, 0.0);
  m.cell_area.assign(m.nC, 0.0);
  par_for(m.nC, [&](int64_t lo, int64_t hi) {
  for (int32_t i = int32_t(lo); i < int32_t(hi); ++i) {
    const int off = m.cell_offset[i], mm = m.ring(i);
    const V3 xi = get3(m.cell_xyz, i);
    double acc = 0.0;
    for (int j = 0; j < mm; ++j) {
      const V3 xe = get3(m.edge_xyz, m.cell_edges[off + j]);
      const V3 xv = get3(m.vertex_xyz, m.cell_vertices[off + j]);
      const V3 xe1 = get3(m.edge_xyz, m.cell_edges[off + (j + 1) % mm]);
      const double kite = (sph_tri_area(xi, xe, xv) + sph_tri_area(xi, xv, xe1)) * R2;
      m.kite_area[off + j] = kite;
      acc += kite;
    }
    if (!(acc > 0.0)) throw std::runtime_error("non-positive cell area at " + std::to_string(i));
    m.cell_area[i] = acc;
  }
  });
}

// --- planar periodic hexagonal mesh ---------------------------------------

struct Torus {
  double W, H;
  // minimum-image difference b - a
  V3 delta(const V3& a, const V3& b) const {
    double dx = b.x - a.x, dy = b.y - a.y;
    dx -= W * std::round(dx / W);
    dy -= H * std::round(dy / H);
    return {dx, dy, 0.0};
  }
  V3 wrap(V3 p) const {
    p.x -= W * std::floor(p.x / W);
    p.y -= H * std::floor(p.y / H);
    return p;
  }
};

inline double cross2(const V3& a, const V3& b) { return a.x * b.y - a.y * b.x; }
inline double len2(const V3& a) { return std::sqrt(a.x * a.x + a.y * a.y); }

mswm_mesh* build_planar(int nx, int ny, double dc) {
  if (nx < 4 || ny < 4 || (ny % 2) != 0) throw std::runtime_error("planar hex mesh needs nx,ny >= 4 and even ny");
  if (!(dc > 0.0)) throw std::runtime_error("cell spacing must be positive");
  const double dy = dc * std::sqrt(3.0) / 2.0;
  Torus T{nx * dc, ny * dy};
  Triangulation tri;
  tri.pts.resize(size_t(nx) * ny);
  auto id = [&](int i, int j) {
    i = ((i % nx) + nx) % nx;
    j = ((j % ny) + ny) % ny;
    return int32_t(j * nx + i);
  };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) tri.pts[id(i, j)] = {(i + 0.5 * (j & 1)) * dc, j * dy, 0.0};
  // Two triangles per lattice point, both counterclockwise: the up-triangle
  // (c, E, NE) and the down-triangle (c, NE, NW).
  tri.tris.reserve(size_t(2) * nx * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int odd = j & 1;
      const int32_t c = id(i, j), E = id(i + 1, j);
      const int32_t NE = id(i + odd, j + 1), NW = id(i + odd - 1, j + 1);
      tri.tris.push_back({c, E, NE});
      tri.tris.push_back({c, NE, NW});
    }

  auto* m = new mswm_mesh();
  m->spherical = 0;
  m->width = T.W;
  m->height = T.H;
  dualise_topology(tri, *m, /*check_euler=*/false);

  m->cell_xyz.assign(size_t(3) * m->nC, 0.0);
  for (int32_t i = 0; i < m->nC; ++i) put3(m->cell_xyz, i, tri.pts[i]);
  m->vertex_xyz.assign(size_t(3) * m->nV, 0.0);
  m->vertex_area.assign(m->nV, 0.0);
  for (int32_t v = 0; v < m->nV; ++v) {
    const V3 a = tri.pts[tri.tris[v][0]];
    const V3 ab = T.delta(a, tri.pts[tri.tris[v][1]]);
    const V3 ac = T.delta(a, tri.pts[tri.tris[v][2]]);
    // circumcentre of (0, ab, ac) relative to a
    const double d = 2.0 * cross2(ab, ac);
    const double b2 = ab.x * ab.x + ab.y * ab.y, c2 = ac.x * ac.x + ac.y * ac.y;
    const V3 cc{(ac.y * b2 - ab.y * c2) / d, (ab.x * c2 - ac.x * b2) / d, 0.0};
    put3(m->vertex_xyz, v, T.wrap(add(a, cc)));
    const double area = 0.5 * cross2(ab, ac);
    if (!(area > 0.0)) throw std::runtime_error("non-positive triangle area");
    m->vertex_area[v] = area;
  }
  m->edge_xyz.assign(size_t(3) * m->nE, 0.0);
  m->edge_len.assign(m->nE, 0.0);
  m->edge_dual_len.assign(m->nE, 0.0);
  for (int32_t e = 0; e < m->nE; ++e) {
    const V3 c0 = get3(m->cell_xyz, m->edge_cells[2 * e]);
    const V3 c1 = get3(m->cell_xyz, m->edge_cells[2 * e + 1]);
    const V3 v0 = get3(m->vertex_xyz, m->edge_vertices[2 * e]);
    const V3 v1 = get3(m->vertex_xyz, m->edge_vertices[2 * e + 1]);
    const V3 dcc = T.delta(c0, c1);
    put3(m->edge_xyz, e, T.wrap(add(c0, scale(dcc, 0.5))));
    m->edge_len[e] = len2(T.delta(v0, v1));
    m->edge_dual_len[e] = len2(dcc);
  }
  const int64_t total = m->cell_offset[m->nC];
  m->kite_area.assign(total, 0.0);
  m->cell_area.assign(m->nC, 0.0);
  for (int32_t i = 0; i < m->nC; ++i) {
    const int off = m->cell_offset[i], mm = m->ring(i);
    const V3 xi = get3(m->cell_xyz, i);
    double acc = 0.0;
    for (int j = 0; j < mm; ++j) {
      const V3 xe = T.delta(xi, get3(m->edge_xyz, m->cell_edges[off + j]));
      const V3 xv = T.delta(xi, get3(m->vertex_xyz, m->cell_vertices[off + j]));
      const V3 xe1 = T.delta(xi, get3(m->edge_xyz, m->cell_edges[off + (j + 1) % mm]));
      const double kite = 0.5 * cross2(xe, xv) + 0.5 * cross2(xv, xe1);
      m->kite_area[off + j] = kite;
      acc += kite;
    }
    if (!(acc > 0.0)) throw std::runtime_error("non-positive cell area");
    m->cell_area[i] = acc;
  }
  finish_kites_and_weights(*m);
  return m;
}

mswm_mesh* build_sphere(int level, double radius) {
  if (level < 0 || level > 12) throw std::runtime_error("icosahedral level must be in [0, 12]");
  if (!(radius > 0.0)) throw std::runtime_error("sphere radius must be positive");
  Triangulation tri = subdivide(level);
  auto* m = new mswm_mesh();
  m->spherical = 1;
  m->radius = radius;
  try {
    dualise_topology(tri, *m, /*check_euler=*/true);
    sphere_geometry(tri, *m, radius);
    finish_kites_and_weights(*m);
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

// Hilbert index of (x, y) on an n x n grid (n a power of two).
uint64_t hilbert2(uint32_t n, uint32_t x, uint32_t y) {
  uint64_t d = 0;
  for (uint32_t s = n / 2; s > 0; s /= 2) {
    const uint32_t rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
    d += uint64_t(s) * s * ((3u * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = n - 1 - x;
        y = n - 1 - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}

// Space-filling-curve cell order: 2-D Hilbert on the plane; on the sphere a
// Hilbert curve per cube face (faces visited so consecutive faces share an
// edge).  Only the internal memory layout of the CUDA path depends on it.
void locality_order(const mswm_mesh& m, int32_t* order) {
  const uint32_t n = 1u << 20;
  std::vector<std::pair<uint64_t, int32_t>> key(m.nC);
  par_for(m.nC, [&](int64_t lo, int64_t hi) {
  for (int32_t i = int32_t(lo); i < int32_t(hi); ++i) {
    const double* p = &m.cell_xyz[3 * size_t(i)];
    uint64_t k;
    if (!m.spherical) {
      const uint32_t x = uint32_t(std::min(double(n - 1), std::max(0.0, p[0] / m.width * n)));
      const uint32_t y = uint32_t(std::min(double(n - 1), std::max(0.0, p[1] / m.height * n)));
      k = hilbert2(n, x, y);
    } else {
      const double ax = std::fabs(p[0]), ay = std::fabs(p[1]), az = std::fabs(p[2]);
      int face;
      double u, v;
      if (ax >= ay && ax >= az) {
        face = p[0] > 0 ? 0 : 3;
        u = p[1] / ax;
        v = p[2] / ax;
      } else if (ay >= az) {
        face = p[1] > 0 ? 1 : 4;
        u = p[2] / ay;
        v = p[0] / ay;
      } else {
        face = p[2] > 0 ? 2 : 5;
        u = p[0] / az;
        v = p[1] / az;
      }
      const uint32_t x = uint32_t(std::min(double(n - 1), std::max(0.0, (u + 1.0) * 0.5 * n)));
      const uint32_t y = uint32_t(std::min(double(n - 1), std::max(0.0, (v + 1.0) * 0.5 * n)));
      k = (uint64_t(face) << 40) | hilbert2(n, x, y);
    }
    key[i] = {k, i};
  }
  });
  par_sort(key);
  for (int32_t k = 0; k < m.nC; ++k) order[k] = key[k].second;
}

}  // namespace

extern "C" {

int mswm_mesh_locality_order(const mswm_mesh* m, int32_t* cell_order) {
  if (!m || !cell_order) return MSWM_E_USAGE;
  locality_order(*m, cell_order);
  return MSWM_OK;
}

const char* mswm_host_last_error(void) { return g_last_error.c_str(); }

mswm_mesh* mswm_mesh_icosahedral(int level, double radius) {
  try {
    return build_sphere(level, radius);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return nullptr;
  }
}

mswm_mesh* mswm_mesh_planar_hex(int nx, int ny, double dc) {
  try {
    return build_planar(nx, ny, dc);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return nullptr;
  }
}

void mswm_mesh_free(mswm_mesh* m) { delete m; }

int mswm_mesh_get_sizes(const mswm_mesh* m, mswm_mesh_sizes* out) {
  if (!m || !out) return MSWM_E_USAGE;
  out->n_cells = m->nC;
  out->n_edges = m->nE;
  out->n_vertices = m->nV;
  out->n_ring = m->cell_offset.empty() ? 0 : m->cell_offset.back();
  out->n_stencil = m->ee_offset.empty() ? 0 : m->ee_offset.back();
  return MSWM_OK;
}

int mswm_mesh_get_desc(const mswm_mesh* m, mswm_mesh_desc* d) {
  if (!m || !d) return MSWM_E_USAGE;
  d->n_cells = m->nC;
  d->n_edges = m->nE;
  d->n_vertices = m->nV;
  d->cell_offset = m->cell_offset.data();
  d->cell_edges = m->cell_edges.data();
  d->cell_vertices = m->cell_vertices.data();
  d->cell_cells = m->cell_cells.data();
  d->edge_cells = m->edge_cells.data();
  d->edge_vertices = m->edge_vertices.data();
  d->vertex_cells = m->vertex_cells.data();
  d->vertex_edges = m->vertex_edges.data();
  d->edge_edge_offset = m->ee_offset.data();
  d->edge_edges = m->edge_edges.data();
  d->edge_cell_sign = m->edge_cell_sign.data();
  d->edge_vertex_sign = m->edge_vertex_sign.data();
  d->edge_len = m->edge_len.data();
  d->edge_dual_len = m->edge_dual_len.data();
  d->cell_area = m->cell_area.data();
  d->vertex_area = m->vertex_area.data();
  d->vertex_kite = m->vertex_kite.data();
  d->edge_weight = m->edge_weight.data();
  return MSWM_OK;
}

int mswm_mesh_get_geometry(const mswm_mesh* m, const double** cell_xyz, const double** vertex_xyz,
                           const double** edge_xyz, const double** kite_area) {
  if (!m) return MSWM_E_USAGE;
  if (cell_xyz) *cell_xyz = m->cell_xyz.data();
  if (vertex_xyz) *vertex_xyz = m->vertex_xyz.data();
  if (edge_xyz) *edge_xyz = m->edge_xyz.data();
  if (kite_area) *kite_area = m->kite_area.data();
  return MSWM_OK;
}

int mswm_mesh_get_domain(const mswm_mesh* m, int* spherical, double* radius, double* width,
                         double* height) {
  if (!m) return MSWM_E_USAGE;
  if (spherical) *spherical = m->spherical;
  if (radius) *radius = m->radius;
  if (width) *width = m->width;
  if (height) *height = m->height;
  return MSWM_OK;
}

}  // extern "C"
