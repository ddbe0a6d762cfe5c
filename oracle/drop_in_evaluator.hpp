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

}  // namespace mswm
