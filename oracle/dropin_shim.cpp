// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// The C++ drop-in exercised from Python: an evaluator handle of the
// reference shim (libmswm_ref.so) whose TendencyEvaluator is
// mswm::CudaEvaluator (drop_in_evaluator.hpp, over the C ABI of
// libmswm_cuda.so).  Kept out of libmswm_ref.so so the timed reference arm
// never maps a product library.

#include <algorithm>

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

}  // extern "C"
