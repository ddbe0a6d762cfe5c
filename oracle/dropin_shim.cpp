// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// The C++ drop-in exercised from Python: an evaluator handle of the
// reference shim (libmswm_ref.so) whose TendencyEvaluator is
// mswm::CudaEvaluator (drop_in_evaluator.hpp, over the C ABI of
// libmswm_cuda.so).  Kept out of libmswm_ref.so so the timed reference arm
// never maps a product library.

#include <algorithm>
#include <memory>

#include "drop_in_evaluator.hpp"
#include "ref_shim.hpp"

using namespace mswm_shim;

extern "C" {

// The drop-in: the reference's own Stepper driving the GPU through
// mswm::CudaEvaluator (drop_in_evaluator.hpp) -- one C-ABI eval() per stage.
void* ref_cuda_eval_create(void* mp, void* rp, const double* b, const double* f, double gravity,
                           int device, char* err, int errlen) {
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
    ev->ev = std::make_unique<CudaEvaluator>(*m, r, ev->b, ev->f, gravity, device);
    out = ev.release();
  });
  return out;
}

// The C++ CudaStepper (drop_in_evaluator.hpp): the device-resident Stepper.
struct CudaStepperBox {
  const VoronoiMesh* mesh;
  CellField b;
  VertexField f;
  WorkLedger ledger;
  std::unique_ptr<CudaStepper> stepper;
};

void* ref_cuda_stepper_create(void* mp, void* rp, const double* b, const double* f,
                              double gravity, int replication, int device, char* err,
                              int errlen) {
  auto* m = static_cast<VoronoiMesh*>(mp);
  auto* r = static_cast<RegionMap*>(rp);
  CudaStepperBox* out = nullptr;
  guarded(err, errlen, nullptr, [&] {
    auto box = std::make_unique<CudaStepperBox>();
    box->mesh = m;
    box->b = CellField(m->n_cells);
    box->f = VertexField(m->n_vertices);
    std::copy(b, b + m->n_cells, box->b.data.begin());
    std::copy(f, f + m->n_vertices, box->f.data.begin());
    box->stepper = std::make_unique<CudaStepper>(*m, r, box->b, box->f, gravity, &box->ledger,
                                                 replication, device);
    out = box.release();
  });
  return out;
}

void ref_cuda_stepper_free(void* s) { delete static_cast<CudaStepperBox*>(s); }

// per_call = 1: n_steps calls of CudaStepper::step (state up / down each);
// 0: one CudaStepper::advance over n_steps.
int ref_cuda_stepper_run(void* sp, int scheme, double* h, double* u, double* time, double dt,
                         int M, int64_t n_steps, int per_call, char* err, int errlen,
                         int* dry_vertex) {
  auto* s = static_cast<CudaStepperBox*>(sp);
  return guarded(err, errlen, dry_vertex, [&] {
    State st(s->mesh->n_cells, s->mesh->n_edges);
    std::copy(h, h + s->mesh->n_cells, st.h.data.begin());
    std::copy(u, u + s->mesh->n_edges, st.u.data.begin());
    st.time = *time;
    SchemeConfig cfg;
    cfg.scheme = Scheme(scheme);
    cfg.dt = dt;
    cfg.substeps = M;
    if (per_call) {
      for (int64_t k = 0; k < n_steps; ++k) s->stepper->step(st, cfg);
    } else {
      s->stepper->advance(st, cfg, n_steps);
    }
    std::copy(st.h.data.begin(), st.h.data.end(), h);
    std::copy(st.u.data.begin(), st.u.data.end(), u);
    *time = st.time;
  });
}

void ref_cuda_stepper_ledger(void* sp, int64_t cell[16], int64_t edge[16]) {
  auto* s = static_cast<CudaStepperBox*>(sp);
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) {
      cell[4 * r + k] = s->ledger.cell_evals[r][k];
      edge[4 * r + k] = s->ledger.edge_evals[r][k];
    }
}

}  // extern "C"
