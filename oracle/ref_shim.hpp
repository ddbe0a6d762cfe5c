// ORACLE / TEST INFRASTRUCTURE ONLY -- shared by the reference shim
// (ref_shim.cpp -> oracle/_ref/libmswm_ref.so, the pure reference) and the
// drop-in shim (dropin_shim.cpp -> oracle/_ref/libmswm_dropin.so, the
// reference's Stepper over mswm::CudaEvaluator).
#pragma once

#include <cstring>
#include <memory>
#include <string>

#include "mswm/errors.hpp"
#include "mswm/fields.hpp"
#include "mswm/integrators.hpp"
#include "mswm/ledger.hpp"
#include "mswm/mesh.hpp"
#include "mswm/partition.hpp"
#include "mswm/regions.hpp"
#include "mswm_cuda.h"

namespace mswm_shim {

using namespace mswm;

inline void put_err(char* buf, int n, const std::string& s) {
  if (!buf || n <= 0) return;
  std::strncpy(buf, s.c_str(), size_t(n - 1));
  buf[n - 1] = 0;
}

// Runs f, translating reference exceptions into mswm_status codes.
template <class F>
int guarded(char* err, int errlen, int* dry_vertex, F&& f) {
  try {
    f();
    return MSWM_OK;
  } catch (const DryVertexError& e) {
    if (dry_vertex) *dry_vertex = e.vertex;
    put_err(err, errlen, e.what());
    return MSWM_E_DRY_VERTEX;
  } catch (const ConfigError& e) {
    put_err(err, errlen, e.what());
    return MSWM_E_CONFIG;
  } catch (const UsageError& e) {
    put_err(err, errlen, e.what());
    return MSWM_E_USAGE;
  } catch (const TopologyError& e) {
    put_err(err, errlen, e.what());
    return MSWM_E_TOPOLOGY;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return MSWM_E_CONFIG;
  }
}

// An evaluator and the fields it references (TendencyEvaluator keeps
// references, integrators.hpp:88-91); ref_eval_free deletes it through the
// virtual destructor whichever library made it.
struct Evaluator {
  const VoronoiMesh* mesh;
  const RegionMap* map;
  CellField b;
  VertexField f;
  double gravity;
  int replication = 1;  // SerialEvaluator / ThreadedEvaluator / Stepper cost replication
  std::unique_ptr<PartitionPlan> plan;
  std::unique_ptr<TendencyEvaluator> ev;
};

struct StepperBox {
  WorkLedger ledger;
  std::unique_ptr<Stepper> stepper;
  const VoronoiMesh* mesh;
};

}  // namespace mswm_shim
