// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product, and links
// nothing of the product (the timed reference arm of bench.py maps only this).
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/
// proj/src/*.cpp compiled by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests and bench.py's CPU-baseline leg drive the reference's own hot
// path: make_regions (regions.cpp:164-171), SerialEvaluator /
// ThreadedEvaluator (integrators.cpp:297-364, rank_pool.cpp:61-176),
// shallow_water_tendencies (operators.cpp:22-118), Stepper
// (integrators.cpp:462-778) and the partitioner (partition.cpp:172-403).
// Meshes either come from the reference generator or are loaded from the
// product's tables (mswm_mesh_desc), which is how planar meshes -- which the
// sphere-only reference cannot generate -- reach the reference hot path.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "mswm/errors.hpp"
#include "mswm/harness.hpp"
#include "mswm/integrators.hpp"
#include "mswm/mesh.hpp"
#include "mswm/operators.hpp"
#include "mswm/partition.hpp"
#include "mswm/rank_pool.hpp"
#include "mswm/regions.hpp"
#include "mswm_cuda.h"

#include "ref_shim.hpp"

using namespace mswm_shim;

namespace {

std::vector<int> union_sets(const RegionMap& map, unsigned mask, bool cells) {
  static const unsigned cbits[6] = {kCellsFinePlain, kCellsUF1, kCellsUF2,
                                    kCellsIf1,       kCellsIf2, kCellsCoarse};
  static const unsigned ebits[5] = {kEdgesFinePlain, kEdgesUFine, kEdgesIf1, kEdgesIf2,
                                    kEdgesCoarse};
  const std::vector<int>* cl[6] = {&map.cells_fine_plain, &map.cells_uf1, &map.cells_uf2,
                                   &map.cells_if1,        &map.cells_if2, &map.cells_coarse};
  const std::vector<int>* el[5] = {&map.edges_fine, &map.edges_ufine, &map.edges_if1,
                                   &map.edges_if2, &map.edges_coarse};
  std::vector<int> out;
  if (cells) {
    for (int g = 0; g < 6; ++g)
      if (mask & cbits[g]) out.insert(out.end(), cl[g]->begin(), cl[g]->end());
  } else {
    for (int g = 0; g < 5; ++g)
      if (mask & ebits[g]) out.insert(out.end(), el[g]->begin(), el[g]->end());
  }
  std::sort(out.begin(), out.end());
  return out;
}

}  // namespace

extern "C" {

// ---- meshes -----------------------------------------------------------------

void* ref_mesh_icosahedral(int level, double radius, char* err, int errlen) {
  VoronoiMesh* out = nullptr;
  guarded(err, errlen, nullptr, [&] {
    out = new VoronoiMesh(build_voronoi_mesh(subdivide_icosahedron(level), radius));
  });
  return out;
}

void* ref_mesh_icosphere(int level, int lloyd, double radius, char* err, int errlen) {
  VoronoiMesh* out = nullptr;
  guarded(err, errlen, nullptr,
          [&] { out = new VoronoiMesh(generate_icosphere_mesh(level, lloyd, radius)); });
  return out;
}

// Load the hot-path tables (and optionally positions / kites) into a
// VoronoiMesh.  Positions are only used by reference diagnostics.
void* ref_mesh_from_desc(const mswm_mesh_desc* d, const double* cell_xyz,
                         const double* vertex_xyz, const double* edge_xyz,
                         const double* kite_area) {
  auto* m = new VoronoiMesh();
  m->n_cells = d->n_cells;
  m->n_edges = d->n_edges;
  m->n_vertices = d->n_vertices;
  const int nC = d->n_cells, nE = d->n_edges, nV = d->n_vertices;
  const int ring = d->cell_offset[nC], sten = d->edge_edge_offset[nE];
  m->cell_offset.assign(d->cell_offset, d->cell_offset + nC + 1);
  m->cell_edges.assign(d->cell_edges, d->cell_edges + ring);
  m->cell_vertices.assign(d->cell_vertices, d->cell_vertices + ring);
  m->cell_cells.assign(d->cell_cells, d->cell_cells + ring);
  m->edge_cells.resize(nE);
  m->edge_vertices.resize(nE);
  m->edge_cell_sign.resize(nE);
  m->edge_vertex_sign.resize(nE);
  for (int e = 0; e < nE; ++e) {
    m->edge_cells[e] = {d->edge_cells[2 * e], d->edge_cells[2 * e + 1]};
    m->edge_vertices[e] = {d->edge_vertices[2 * e], d->edge_vertices[2 * e + 1]};
    m->edge_cell_sign[e] = {d->edge_cell_sign[2 * e], d->edge_cell_sign[2 * e + 1]};
    m->edge_vertex_sign[e] = {d->edge_vertex_sign[2 * e], d->edge_vertex_sign[2 * e + 1]};
  }
  m->vertex_cells.resize(nV);
  m->vertex_edges.resize(nV);
  m->vertex_kite.resize(nV);
  for (int v = 0; v < nV; ++v)
    for (int k = 0; k < 3; ++k) {
      m->vertex_cells[v][k] = d->vertex_cells[3 * v + k];
      m->vertex_edges[v][k] = d->vertex_edges[3 * v + k];
      m->vertex_kite[v][k] = d->vertex_kite[3 * v + k];
    }
  m->edge_edge_offset.assign(d->edge_edge_offset, d->edge_edge_offset + nE + 1);
  m->edge_edges.assign(d->edge_edges, d->edge_edges + sten);
  m->edge_weight.assign(d->edge_weight, d->edge_weight + sten);
  m->edge_len.assign(d->edge_len, d->edge_len + nE);
  m->edge_dual_len.assign(d->edge_dual_len, d->edge_dual_len + nE);
  m->cell_area.assign(d->cell_area, d->cell_area + nC);
  m->vertex_area.assign(d->vertex_area, d->vertex_area + nV);
  if (kite_area) m->kite_area.assign(kite_area, kite_area + ring);
  auto load3 = [](std::vector<Vec3>& dst, const double* src, int n) {
    dst.resize(n);
    if (src)
      for (int i = 0; i < n; ++i) dst[i] = {src[3 * i], src[3 * i + 1], src[3 * i + 2]};
  };
  load3(m->cell_xyz, cell_xyz, nC);
  load3(m->vertex_xyz, vertex_xyz, nV);
  load3(m->edge_xyz, edge_xyz, nE);
  return m;
}

void ref_mesh_free(void* m) { delete static_cast<VoronoiMesh*>(m); }

void ref_mesh_sizes(void* mp, int64_t out[5]) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  out[0] = m->n_cells;
  out[1] = m->n_edges;
  out[2] = m->n_vertices;
  out[3] = m->cell_offset.back();
  out[4] = m->edge_edge_offset.back();
}

// Views into the VoronoiMesh storage (std::array<int,2> etc. are contiguous).
void ref_mesh_desc(void* mp, mswm_mesh_desc* d) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  d->n_cells = m->n_cells;
  d->n_edges = m->n_edges;
  d->n_vertices = m->n_vertices;
  d->cell_offset = m->cell_offset.data();
  d->cell_edges = m->cell_edges.data();
  d->cell_vertices = m->cell_vertices.data();
  d->cell_cells = m->cell_cells.data();
  d->edge_cells = m->edge_cells.data()->data();
  d->edge_vertices = m->edge_vertices.data()->data();
  d->vertex_cells = m->vertex_cells.data()->data();
  d->vertex_edges = m->vertex_edges.data()->data();
  d->edge_edge_offset = m->edge_edge_offset.data();
  d->edge_edges = m->edge_edges.data();
  d->edge_cell_sign = m->edge_cell_sign.data()->data();
  d->edge_vertex_sign = m->edge_vertex_sign.data()->data();
  d->edge_len = m->edge_len.data();
  d->edge_dual_len = m->edge_dual_len.data();
  d->cell_area = m->cell_area.data();
  d->vertex_area = m->vertex_area.data();
  d->vertex_kite = m->vertex_kite.data()->data();
  d->edge_weight = m->edge_weight.data();
}

void ref_mesh_geometry(void* mp, const double** cell_xyz, const double** vertex_xyz,
                       const double** edge_xyz, const double** kite_area) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  *cell_xyz = &m->cell_xyz.data()->x;
  *vertex_xyz = &m->vertex_xyz.data()->x;
  *edge_xyz = &m->edge_xyz.data()->x;
  *kite_area = m->kite_area.data();
}

// Re-derive the stencil and orientation signs with the reference's own
// routines (mesh_build.cpp:133-183): pins the product's planar builder.
int ref_mesh_rederive(void* mp, char* err, int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  return guarded(err, errlen, nullptr, [&] {
    rebuild_edge_stencil(*m);
    assign_orientation_signs(*m);
  });
}

int ref_mesh_validate(void* mp, char* err, int errlen) {
  return guarded(err, errlen, nullptr, [&] { validate_mesh(*static_cast<VoronoiMesh*>(mp)); });
}

double ref_total_mass(void* mp, const double* h) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  CellField f(m->n_cells);
  std::copy(h, h + m->n_cells, f.data.begin());
  return total_mass(*m, f);
}

double ref_total_energy(void* mp, const double* h, const double* u, const double* b, double g) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  State st(m->n_cells, m->n_edges);
  std::copy(h, h + m->n_cells, st.h.data.begin());
  std::copy(u, u + m->n_edges, st.u.data.begin());
  CellField bf(m->n_cells);
  std::copy(b, b + m->n_cells, bf.data.begin());
  return total_energy(*m, st, bf, g);
}

// rp may be null (no region map)
int ref_courant(void* mp, void* rp, const double* u, double dt, int M, double* out, char* err,
                int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  return guarded(err, errlen, nullptr, [&] {
    EdgeField uf(m->n_edges);
    std::copy(u, u + m->n_edges, uf.data.begin());
    const CourantNumbers c = courant_numbers(*m, static_cast<const RegionMap*>(rp), uf, dt, M);
    out[0] = c.fine;
    out[1] = c.coarse;
  });
}

// ---- regions ----------------------------------------------------------------

void* ref_regions_make(void* mp, const uint8_t* fine_mask, int width, char* err, int errlen,
                       int* n_warnings) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  RegionMap* out = nullptr;
  int rc = guarded(err, errlen, nullptr, [&] {
    std::vector<std::string> warn;
    out = new RegionMap(make_regions(*m, [&](int i) { return fine_mask[i] != 0; }, width, &warn));
    if (n_warnings) *n_warnings = int(warn.size());
  });
  (void)rc;
  return out;
}

void ref_regions_free(void* r) { delete static_cast<RegionMap*>(r); }

void ref_regions_labels(void* rp, uint8_t* cell_label, uint8_t* cell_sub, uint8_t* edge_label) {
  auto* r = static_cast<RegionMap*>(rp);
  for (size_t i = 0; i < r->cell_label.size(); ++i) {
    cell_label[i] = uint8_t(r->cell_label[i]);
    cell_sub[i] = uint8_t(r->cell_sublabel[i]);
  }
  for (size_t e = 0; e < r->edge_label.size(); ++e) edge_label[e] = uint8_t(r->edge_label[e]);
}

int64_t ref_regions_group(void* rp, int g, int32_t* ids) {
  auto* r = static_cast<RegionMap*>(rp);
  const std::vector<int>* L[11] = {&r->cells_fine_plain, &r->cells_uf1,  &r->cells_uf2,
                                   &r->cells_if1,        &r->cells_if2,  &r->cells_coarse,
                                   &r->edges_fine,       &r->edges_ufine, &r->edges_if1,
                                   &r->edges_if2,        &r->edges_coarse};
  if (g < 0 || g > 10) return -1;
  if (ids) std::copy(L[g]->begin(), L[g]->end(), ids);
  return int64_t(L[g]->size());
}

int ref_regions_validate(void* mp, void* rp) {
  return int(validate_regions(*static_cast<VoronoiMesh*>(mp), *static_cast<RegionMap*>(rp))
                 .violations.size());
}

// validate_regions on a copy of the map with the given labels (lists rebuilt
// from them): the number of violations, messages joined by '\n' in msgs.
int ref_regions_validate_labels(void* mp, void* rp, const uint8_t* cell_label,
                                const uint8_t* cell_sub, const uint8_t* edge_label, char* msgs,
                                int len) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  RegionMap r = *static_cast<RegionMap*>(rp);
  for (int i = 0; i < m->n_cells; ++i) {
    r.cell_label[i] = CellRegion(cell_label[i]);
    r.cell_sublabel[i] = CellSub(cell_sub[i]);
  }
  for (int e = 0; e < m->n_edges; ++e) r.edge_label[e] = EdgeRegion(edge_label[e]);
  r.rebuild_groups(m->n_cells, m->n_edges);
  const RegionReport rep = validate_regions(*m, r);
  std::string all;
  for (const auto& v : rep.violations) all += v + "\n";
  if (msgs && len > 0) {
    std::strncpy(msgs, all.c_str(), size_t(len) - 1);
    msgs[len - 1] = 0;
  }
  return int(rep.violations.size());
}

// ---- evaluators -------------------------------------------------------------

// nranks == 0: SerialEvaluator.  nranks >= 1: ThreadedEvaluator over
// partition_multiconstraint(build_cell_graph(mesh, map), nranks, seed) and
// make_block_plan -- the reference's emulated-rank path (mswm.cpp:319-323).
void* ref_eval_create(void* mp, void* rp, const double* b, const double* f, double gravity,
                      int nranks, uint64_t seed, int replication, char* err, int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  auto* r = static_cast<RegionMap*>(rp);
  Evaluator* out = nullptr;
  guarded(err, errlen, nullptr, [&] {
    auto ev = std::make_unique<Evaluator>();
    ev->mesh = m;
    ev->map = r;
    ev->b = CellField(m->n_cells);
    ev->f = VertexField(m->n_vertices);
    std::copy(b, b + m->n_cells, ev->b.data.begin());
    std::copy(f, f + m->n_vertices, ev->f.data.begin());
    ev->gravity = gravity;
    ev->replication = replication;
    if (nranks <= 0) {
      ev->ev = std::make_unique<SerialEvaluator>(*m, r, ev->b, ev->f, gravity, replication);
    } else {
      if (!r) throw UsageError("threaded evaluator needs a region map");
      const CellGraph g = build_cell_graph(*m, r);
      const std::vector<int> labels = partition_multiconstraint(g, nranks, seed, nullptr);
      ev->plan = std::make_unique<PartitionPlan>(make_block_plan(*m, *r, labels, nranks));
      ev->ev = std::make_unique<ThreadedEvaluator>(*m, *r, *ev->plan, ev->b, ev->f, gravity,
                                                   replication);
    }
    out = ev.release();
  });
  return out;
}

void ref_eval_free(void* e) { delete static_cast<Evaluator*>(e); }

int ref_eval(void* ep, const double* h, const double* u, unsigned mask, double* dh, double* du,
             char* err, int errlen, int* dry_vertex) {
  auto* e = static_cast<Evaluator*>(ep);
  return guarded(err, errlen, dry_vertex, [&] { e->ev->eval(h, u, mask, dh, du); });
}

// Closure sets of one masked evaluation, straight from TendencyScratch
// after shallow_water_tendencies (operators.cpp:30-58), in discovery order.
int ref_closure(void* ep, const double* h, const double* u, unsigned mask, int kind, int32_t* ids,
                int64_t* n, char* err, int errlen) {
  auto* e = static_cast<Evaluator*>(ep);
  return guarded(err, errlen, nullptr, [&] {
    std::vector<int> cells, edges;
    if (e->map) {
      cells = union_sets(*e->map, mask, true);
      edges = union_sets(*e->map, mask, false);
    } else {
      cells.resize(e->mesh->n_cells);
      std::iota(cells.begin(), cells.end(), 0);
      edges.resize(e->mesh->n_edges);
      std::iota(edges.begin(), edges.end(), 0);
    }
    TendencyScratch s;
    s.bind(*e->mesh);
    std::vector<double> dh(e->mesh->n_cells), du(e->mesh->n_edges);
    shallow_water_tendencies(*e->mesh, h, u, e->b.ptr(), e->f.ptr(), e->gravity, {cells, edges},
                             dh.data(), du.data(), s, 1);
    const std::vector<int>* L[4] = {&s.flux_ids, &s.qt_ids, &s.cell_ids, &s.vertex_ids};
    if (kind < 0 || kind > 3) throw UsageError("closure kind out of range");
    *n = int64_t(L[kind]->size());
    if (ids) std::copy(L[kind]->begin(), L[kind]->end(), ids);
  });
}

// ---- stepper ----------------------------------------------------------------

void* ref_stepper_create(void* ep) {
  auto* e = static_cast<Evaluator*>(ep);
  auto* s = new StepperBox();
  s->mesh = e->mesh;
  s->stepper = std::make_unique<Stepper>(*e->mesh, e->map, *e->ev, &s->ledger, e->replication);
  return s;
}

void ref_stepper_free(void* s) { delete static_cast<StepperBox*>(s); }

// n_steps of Stepper::step on (h,u,time) in place; *seconds = wall time of
// the stepping loop alone (steady_clock, like harness.cpp:181-194).
int ref_step(void* sp, int scheme, double* h, double* u, double* time, double dt, int M,
             int64_t n_steps, char* err, int errlen, int* dry_vertex, double* seconds) {
  auto* s = static_cast<StepperBox*>(sp);
  return guarded(err, errlen, dry_vertex, [&] {
    State st(s->mesh->n_cells, s->mesh->n_edges);
    std::copy(h, h + s->mesh->n_cells, st.h.data.begin());
    std::copy(u, u + s->mesh->n_edges, st.u.data.begin());
    st.time = *time;
    SchemeConfig cfg;
    cfg.scheme = Scheme(scheme);
    cfg.dt = dt;
    cfg.substeps = M;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      for (int64_t k = 0; k < n_steps; ++k) s->stepper->step(st, cfg);
    } catch (...) {
      if (seconds)
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      throw;
    }
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::copy(st.h.data.begin(), st.h.data.end(), h);
    std::copy(st.u.data.begin(), st.u.data.end(), u);
    *time = st.time;
  });
}

void ref_ledger(void* sp, int64_t cell[16], int64_t edge[16], int64_t* steps) {
  auto* s = static_cast<StepperBox*>(sp);
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) {
      cell[4 * r + k] = s->ledger.cell_evals[r][k];
      edge[4 * r + k] = s->ledger.edge_evals[r][k];
    }
  if (steps) *steps = s->ledger.steps_taken;
}

int ref_lts_coeffs(int order, int stage, int k, int M, double out[3], char* err, int errlen) {
  return guarded(err, errlen, nullptr, [&] {
    const LtsCoeffs c = lts_interp_coeffs(order, stage, k, M);
    out[0] = c.w_old;
    out[1] = c.w_first;
    out[2] = c.w_second;
  });
}

// ---- partition / block plan (the multi-rank analogue) -----------------------

int ref_partition(void* mp, void* rp, int nparts, uint64_t seed, int32_t* labels, char* err,
                  int errlen) {
  return guarded(err, errlen, nullptr, [&] {
    const CellGraph g =
        build_cell_graph(*static_cast<VoronoiMesh*>(mp), static_cast<RegionMap*>(rp));
    const std::vector<int> l = partition_multiconstraint(g, nparts, seed, nullptr);
    std::copy(l.begin(), l.end(), labels);
  });
}

void* ref_block_plan(void* mp, void* rp, const int32_t* labels, int nranks, char* err,
                     int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  PartitionPlan* out = nullptr;
  guarded(err, errlen, nullptr, [&] {
    std::vector<int> l(labels, labels + m->n_cells);
    out = new PartitionPlan(make_block_plan(*m, *static_cast<RegionMap*>(rp), l, nranks));
  });
  return out;
}

void ref_block_plan_free(void* p) { delete static_cast<PartitionPlan*>(p); }

// which: 0 owned cells, 1 owned edges, 2 halo cells, 3 halo edges
int64_t ref_block_plan_list(void* pp, int block, int which, int32_t* ids) {
  auto* p = static_cast<PartitionPlan*>(pp);
  const std::vector<std::vector<int>>* L[4] = {&p->owned_cells, &p->owned_edges, &p->halo_cells,
                                               &p->halo_edges};
  if (block < 0 || block >= p->n_blocks || which < 0 || which > 3) return -1;
  const auto& v = (*L[which])[block];
  if (ids) std::copy(v.begin(), v.end(), ids);
  return int64_t(v.size());
}

// init_tc5 with the default TestCaseConfig (harness.cpp:35-72).
int ref_init_tc5(void* mp, double* h, double* u, double* b, double* f, char* err, int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  return guarded(err, errlen, nullptr, [&] {
    const Tc5Init init = init_tc5(*m, TestCaseConfig{});
    std::copy(init.state.h.data.begin(), init.state.h.data.end(), h);
    std::copy(init.state.u.data.begin(), init.state.u.data.end(), u);
    std::copy(init.b.data.begin(), init.b.data.end(), b);
    std::copy(init.f.data.begin(), init.f.data.end(), f);
  });
}

// convergence_study (harness.cpp:243-309) on TC5 with the default test case:
// out = err_h[n], err_u[n], then slope_h, slope_u, monotone_h, monotone_u.
int ref_convergence_study(void* mp, void* rp, int scheme, int M, const double* dts, int n,
                          double duration, double* out, char* err, int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  auto* r = static_cast<RegionMap*>(rp);
  return guarded(err, errlen, nullptr, [&] {
    const ConvergenceResult cr = convergence_study(*m, r, Scheme(scheme), M,
                                                   std::vector<double>(dts, dts + n), duration,
                                                   TestCaseConfig{});
    for (int k = 0; k < n; ++k) {
      out[k] = cr.err_h[k];
      out[n + k] = cr.err_u[k];
    }
    out[2 * n] = cr.slope_h;
    out[2 * n + 1] = cr.slope_u;
    out[2 * n + 2] = cr.monotone_h ? 1.0 : 0.0;
    out[2 * n + 3] = cr.monotone_u ? 1.0 : 0.0;
  });
}

}  // extern "C"
