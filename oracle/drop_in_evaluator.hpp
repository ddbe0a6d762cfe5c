// The reference-side binding a maintainer adds to use the B200 path from the
// unmodified reference code: a mswm::TendencyEvaluator (the reference's one
// compute boundary, proj/include/mswm/integrators.hpp:68-73) implemented over
// the C ABI of include/mswm_cuda.h.  Drop it in wherever the reference
// constructs an evaluator (harness.cpp:151-158) and the reference's own
// Stepper (integrators.cpp:412-575) runs on the GPU, one eval() per stage.
//
// In this repository it is compiled (test infrastructure, oracle/Makefile)
// into oracle/_ref together with the reference sources, so the GPU tests can
// drive the reference's Stepper through it (tests/test_gpu_parity.py).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "mswm/errors.hpp"
#include "mswm/integrators.hpp"
#include "mswm/ledger.hpp"
#include "mswm/mesh.hpp"
#include "mswm/regions.hpp"
#include "mswm_cuda.h"

namespace mswm {

// SoA views of a VoronoiMesh for the C ABI (mesh.hpp:31-68 are contiguous
// std::vector / std::array storage, so no copies are needed).
inline mswm_mesh_desc cuda_mesh_desc(const VoronoiMesh& m) {
  mswm_mesh_desc d{};
  d.n_cells = m.n_cells;
  d.n_edges = m.n_edges;
  d.n_vertices = m.n_vertices;
  d.cell_offset = m.cell_offset.data();
  d.cell_edges = m.cell_edges.data();
  d.cell_vertices = m.cell_vertices.data();
  d.cell_cells = m.cell_cells.data();
  d.edge_cells = m.edge_cells.data()->data();
  d.edge_vertices = m.edge_vertices.data()->data();
  d.vertex_cells = m.vertex_cells.data()->data();
  d.vertex_edges = m.vertex_edges.data()->data();
  d.edge_edge_offset = m.edge_edge_offset.data();
  d.edge_edges = m.edge_edges.data();
  d.edge_cell_sign = m.edge_cell_sign.data()->data();
  d.edge_vertex_sign = m.edge_vertex_sign.data()->data();
  d.edge_len = m.edge_len.data();
  d.edge_dual_len = m.edge_dual_len.data();
  d.cell_area = m.cell_area.data();
  d.vertex_area = m.vertex_area.data();
  d.vertex_kite = m.vertex_kite.data()->data();
  d.edge_weight = m.edge_weight.data();
  return d;
}

// Maps a C-ABI status to the reference's exception (errors.hpp:9-49).
inline void cuda_check(int rc, const mswm_cuda_ctx* ctx) {
  if (rc == MSWM_OK) return;
  const std::string msg = mswm_cuda_last_error(ctx);
  switch (rc) {
    case MSWM_E_CONFIG: throw ConfigError(msg);
    case MSWM_E_USAGE: throw UsageError(msg);
    case MSWM_E_TOPOLOGY: throw TopologyError(msg);
    case MSWM_E_DRY_VERTEX: throw DryVertexError(msg, mswm_cuda_dry_vertex(ctx, nullptr));
    default: throw Error(msg);
  }
}

class CudaEvaluator : public TendencyEvaluator {
 public:
  // Same arguments as SerialEvaluator (integrators.hpp:79-81).  The map's
  // labels are re-derived on the device from the fine cells of `map`
  // (bit-exact with make_regions), so masks mean the same groups.
  CudaEvaluator(const VoronoiMesh& mesh, const RegionMap* map, const CellField& b,
                const VertexField& f_vertex, double gravity, int device = 0,
                const int32_t* cell_order = nullptr) {
    const mswm_mesh_desc d = cuda_mesh_desc(mesh);
    if (mswm_cuda_create(&d, device, cell_order, &ctx_) != MSWM_OK)
      throw Error(std::string("mswm_cuda_create: ") + mswm_cuda_last_error(nullptr));
    cuda_check(mswm_cuda_set_fields(ctx_, b.ptr(), f_vertex.ptr(), gravity), ctx_);
    if (map) {
      std::vector<uint8_t> fine(mesh.n_cells);
      for (int i = 0; i < mesh.n_cells; ++i) fine[i] = map->cell_label[i] == CellRegion::Fine;
      cuda_check(mswm_cuda_set_regions(ctx_, fine.data(), map->interface_width, nullptr,
                                       nullptr, nullptr, nullptr, nullptr),
                 ctx_);
    }
  }
  ~CudaEvaluator() override { mswm_cuda_destroy(ctx_); }
  CudaEvaluator(const CudaEvaluator&) = delete;
  CudaEvaluator& operator=(const CudaEvaluator&) = delete;

  void eval(const double* h, const double* u, unsigned mask, double* dh, double* du) override {
    cuda_check(mswm_cuda_eval(ctx_, h, u, mask, dh, du), ctx_);
  }

  mswm_cuda_ctx* context() { return ctx_; }

 private:
  mswm_cuda_ctx* ctx_ = nullptr;
};

// The device-resident counterpart of Stepper (integrators.hpp:136-160):
// same step entry points and the same ledger, but the whole coarse step --
// every stage, prediction, accumulation and correction -- runs on the GPU as
// one graph replay (mswm_cuda_step) instead of one eval() per stage.  The
// caller's State is uploaded, stepped and downloaded per call; advance()
// runs n steps between one upload and one download.  Errors map to the
// reference's exceptions (ConfigError for dt <= 0 / M < 1 / missing map,
// DryVertexError with its step, integrators.cpp:413-421, harness.cpp:183-190).
class CudaStepper {
 public:
  CudaStepper(const VoronoiMesh& mesh, const RegionMap* map, const CellField& b,
              const VertexField& f_vertex, double gravity, WorkLedger* ledger,
              int replication = 1, int device = 0, const int32_t* cell_order = nullptr)
      : ledger_(ledger), n_cells_(mesh.n_cells), n_edges_(mesh.n_edges) {
    const mswm_mesh_desc d = cuda_mesh_desc(mesh);
    if (mswm_cuda_create(&d, device, cell_order, &ctx_) != MSWM_OK)
      throw Error(std::string("mswm_cuda_create: ") + mswm_cuda_last_error(nullptr));
    try {
      cuda_check(mswm_cuda_set_fields(ctx_, b.ptr(), f_vertex.ptr(), gravity), ctx_);
      cuda_check(mswm_cuda_set_replication(ctx_, replication), ctx_);
      if (map) {
        std::vector<uint8_t> fine(mesh.n_cells);
        for (int i = 0; i < mesh.n_cells; ++i) fine[i] = map->cell_label[i] == CellRegion::Fine;
        cuda_check(mswm_cuda_set_regions(ctx_, fine.data(), map->interface_width, nullptr,
                                         nullptr, nullptr, nullptr, nullptr),
                   ctx_);
      }
    } catch (...) {
      mswm_cuda_destroy(ctx_);
      throw;
    }
  }
  ~CudaStepper() { mswm_cuda_destroy(ctx_); }
  CudaStepper(const CudaStepper&) = delete;
  CudaStepper& operator=(const CudaStepper&) = delete;

  void ssprk_step(int order, State& state, double dt) {
    if (order != 2 && order != 3) throw UsageError("SSPRK order must be 2 or 3");
    run(order == 2 ? MSWM_SSPRK2 : MSWM_SSPRK3, state, dt, 1, 1);
  }
  void rk4_step(State& state, double dt) { run(MSWM_RK4, state, dt, 1, 1); }
  void lts_step(int order, State& state, double dt, int substeps) {
    if (order != 2 && order != 3) throw UsageError("LTS order must be 2 or 3");
    run(order == 2 ? MSWM_LTS2 : MSWM_LTS3, state, dt, substeps, 1);
  }
  void step(State& state, const SchemeConfig& cfg) { advance(state, cfg, 1); }

  // n_steps of cfg.scheme with the state resident on the GPU in between.
  void advance(State& state, const SchemeConfig& cfg, int64_t n_steps) {
    run(scheme_of(cfg.scheme), state, cfg.dt, cfg.substeps, n_steps);
  }

  mswm_cuda_ctx* context() { return ctx_; }

 private:
  static int scheme_of(Scheme s) {
    switch (s) {
      case Scheme::SSPRK2: return MSWM_SSPRK2;
      case Scheme::SSPRK3: return MSWM_SSPRK3;
      case Scheme::RK4: return MSWM_RK4;
      case Scheme::LTS2: return MSWM_LTS2;
      case Scheme::LTS3: return MSWM_LTS3;
    }
    throw UsageError("unknown scheme");
  }

  void run(int scheme, State& st, double dt, int M, int64_t n) {
    if (st.h.size() != std::size_t(n_cells_) || st.u.size() != std::size_t(n_edges_))
      throw UsageError("state size does not match the mesh");
    cuda_check(mswm_cuda_state_upload(ctx_, st.h.ptr(), st.u.ptr(), st.time), ctx_);
    int64_t c0[16], e0[16], s0 = 0;
    cuda_check(mswm_cuda_ledger(ctx_, c0, e0, &s0), ctx_);
    cuda_check(mswm_cuda_step(ctx_, scheme, dt, M, n, 1), ctx_);
    cuda_check(mswm_cuda_state_download(ctx_, st.h.ptr(), st.u.ptr(), &st.time), ctx_);
    if (!ledger_) return;
    int64_t c1[16], e1[16], s1 = 0;
    cuda_check(mswm_cuda_ledger(ctx_, c1, e1, &s1), ctx_);
    for (int r = 0; r < kLedgerRegionCount; ++r)
      for (int k = 0; k < kLedgerStageCount; ++k) {
        ledger_->add_cells(r, k, c1[4 * r + k] - c0[4 * r + k]);
        ledger_->add_edges(r, k, e1[4 * r + k] - e0[4 * r + k]);
      }
  }

  WorkLedger* ledger_;
  mswm_cuda_ctx* ctx_ = nullptr;
  int n_cells_, n_edges_;
};

}  // namespace mswm
