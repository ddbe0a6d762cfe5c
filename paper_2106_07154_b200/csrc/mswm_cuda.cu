// C ABI of the B200 LTS3 / TRiSK path (include/mswm_cuda.h).
//
// One context = one GPU, one CUDA stream, the mesh tables in internal
// numbering, the device-resident state and the LTS workspace.  Evaluations
// are three kernels (A: PV + K on the closure, B: (F, q~) on the edge
// closure, C: dh/du on the output lists with the stage update fused);
// coarse steps are captured once into a CUDA graph per (scheme, dt, M) and
// replayed.
//
// Device schedule of one LTS3 coarse step (reference:
// proj/src/integrators.cpp:412-575).  The reference keeps 18 full-size
// stage arrays and copies/zeroes most of them every step (:488-519); here
// the stage arrays alias (ha == state, hb == h1, hc == h2) and only the
// I1/I2 values the predictions and the correction read are saved, which
// removes every O(n) copy.  This is exact because (i) no evaluation reads a
// stage value that the aliasing changes (the stencil reaches one cell ring
// for h and the ring edges of that ring for u, so step 2 never reads fine
// cells beyond UF1 and step 4 never reads anything closer to the fine
// region than Interface2), and (ii) every element's arithmetic is the
// reference's expression, evaluated once.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <atomic>
#include <thread>
#include <tuple>
#include <type_traits>
#include <vector>

#include "kernels.cuh"
#include "mswm_cuda.h"

using namespace mswm_dev;

namespace {

thread_local std::string g_create_error;

struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw Error(MSWM_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));   \
  } while (0)

template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  DArr() = default;
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  DArr(DArr&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DArr& operator=(DArr&& o) noexcept {
    if (this != &o) {
      if (p) cudaFree(p);
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DArr() {
    if (p) cudaFree(p);
  }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count) {
      cudaError_t e = cudaMalloc(&p, count * sizeof(T));
      if (e != cudaSuccess)
        throw Error(MSWM_E_NOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                      " bytes: " + cudaGetErrorString(e));
    }
  }
  void upload(const std::vector<T>& h, cudaStream_t s) {
    alloc(h.size());
    if (n) CK(cudaMemcpyAsync(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void zero(cudaStream_t s) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

inline int nblk(int64_t n, int b = kBlock) { return int((n + b - 1) / b); }

// MSWM_DEBUG_MEM=1: host resident set at setup milestones (stderr)
void debug_mem(const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("MSWM_DEBUG_MEM");
    return e && e[0] == '1';
  }();
  if (!on) return;
  long pages = 0, rss = 0;
  if (FILE* f = std::fopen("/proc/self/statm", "r")) {
    if (std::fscanf(f, "%ld %ld", &pages, &rss) != 2) rss = 0;
    std::fclose(f);
  }
  std::fprintf(stderr, "[mswm mem] %-40s rss %.2f GB\n", what, double(rss) * 4096.0 / (1 << 30));
}

__global__ void k_fill_af(int32_t n, const double* __restrict__ f, double2* __restrict__ af) {
  const int32_t v = blockIdx.x * kBlock + threadIdx.x;
  if (v < n) af[v].y = f[v];
}

// Output lists and closure lists of one mask (operators.cpp:35-58).
struct MaskPlan {
  unsigned mask = 0;
  const int32_t* cells = nullptr;  // device, group-concatenated
  int32_t nc = 0, csplit = 0;
  const int32_t* edges = nullptr;
  int32_t ne = 0, esplit = 0;
  DArr<int32_t> own_cells, own_edges;  // storage when not aliasing the group buffer
  DArr<int32_t> vclos, kclos, eclos, fclos, qclos;
  int32_t nv = 0, nk = 0, nec = 0, nf = 0, nq = 0;
  // launch sets: a contiguous range plus a short list (see make_span) or a
  // dense superset; no index-list traffic for ranges, coalesced access
  bool dense_v = false, dense_k = false, dense_fq = false, dense_out = false;
  struct HSpan {
    int32_t base = 0, n_range = 0, n_list = 0;
    const int32_t* list = nullptr;
    DArr<int32_t> own;
    Span dev() const { return Span{base, n_range, list, n_list}; }
    int64_t n() const { return int64_t(n_range) + n_list; }
  } sv, sk, se, sc_out, se_out;
  DArr<uint32_t> vmask;  // closure bitmask for the dense dry-vertex check
  // chunk schedules of kernels A and C (kernels.cuh ChunkMap) and, for the
  // ping-pong order (MSWM_MIX bit 4), their reversals and kernel B's
  DArr<int32_t> cmapA, cmapC, cmapA_r, cmapB_r, cmapC_r;
  std::vector<int32_t> host_cells, host_edges;  // original ids, same order as device lists
  // drop-in eval I/O (mswm_cuda_eval): the h / u entries the evaluation
  // reads, original ids on the host and internal ids on the device (built on
  // first use)
  bool io_ready = false;
  std::vector<int32_t> io_rc_orig, io_re_orig;
  DArr<int32_t> io_rc, io_re;
  // outputs in ascending original id (the host scatter streams): original
  // ids on the host, internal ids on the device
  std::vector<int32_t> io_oc_orig, io_oe_orig;
  DArr<int32_t> io_oc, io_oe;
};

// Halo exchange plan of one rank: per peer slot, the owned values it sends
// and the halo values it receives, as flat codes into the (h, u) arrays
// (code >= 0: cell id, code < 0: ~edge id) and offsets into one send and one
// receive buffer.
struct Halo {
  std::vector<int> peer;
  std::vector<int64_t> soff, scnt, roff, rcnt;
  std::vector<int32_t> h_scode, h_rcode;  // host copies (per-mask subsets)
  DArr<int32_t> scode, rcode;
  DArr<double> sbuf, rbuf;
  int64_t ns = 0, nr = 0;
  // peer-store transport (mswm_cuda_peer_*): this halo's receive region in the
  // context's arena (two halves of pstride doubles) and, per peer slot, where
  // this rank's values go in the neighbour's arena
  double* prbuf = nullptr;
  int64_t pstride = 0;
  std::vector<PeerSlot> h_pslots;
  DArr<PeerSlot> pslots;
  DArr<uint8_t> sslot;  // peer slot of every send item
  bool active() const { return !peer.empty(); }
};

// NCCL, resolved at run time from the process's libnccl.so.2 (the one torch
// already loaded, if any), so the library has no link-time NCCL dependency.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  // optional (NCCL >= 2.18): a second communicator for the forked coarse step
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = "libnccl.so.2 not found";
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd &&
           a.Send && a.Recv && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks the p2p API";
    return a;
  }();
  if (!api.ok) throw Error(MSWM_E_NCCL, "NCCL unavailable: " + api.why);
  return api;
}

void nccl_check(ncclResult_t r) {
  if (r != ncclSuccess) throw Error(MSWM_E_NCCL, std::string("NCCL: ") + nccl().GetErrorString(r));
}

struct EvalRecord {
  cudaEvent_t start, stop;
  int64_t nc, ne;
};

}  // namespace

struct mswm_cuda_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t ls = nullptr;  // launch stream (== stream, or a group's stream while capturing)
  // multi-rank: this context is rank `rank` of `n_ranks`, owning part of the mesh
  int rank = 0, n_ranks = 1;
  Halo halo;
  // per-mask restrictions of `halo` to what that evaluation reads (SURVEY
  // §8(e)); masks without one exchange the full halo
  std::map<unsigned, Halo> halo_mask;
  ncclComm_t nccl_comm = nullptr;
  ncclComm_t nccl_comm2 = nullptr;  // the concurrent coarse step's exchanges (ncclCommSplit)
  bool nccl_warm = false;           // p2p connections to every neighbour set up (warm_nccl)
  // in-process group over a one-rank NCCL communicator (owned by the group,
  // mswm_cuda_group_nccl_loopback): halo copies as NCCL send/recv to self
  ncclComm_t loop_comm = nullptr, loop_comm2 = nullptr;
  // peer-store transport: one arena per rank -- flag words [channel][rank],
  // then every halo's double-buffered receive region -- exported to the
  // neighbours (CUDA IPC between processes, plain pointers inside a group)
  int transport = 0;  // 0: NCCL / device copies, 1: peer stores
  DArr<unsigned char> arena;
  std::vector<unsigned char*> peer_base;  // neighbours' arenas as mapped here, by rank
  std::vector<char> peer_ipc;             // opened with cudaIpcOpenMemHandle (to close)
  DArr<unsigned long long> xchan;         // per channel: exchanges done, block arrivals
  DArr<int> xerr;                         // 1 + rank of a neighbour that did not signal
  // how long a wait polls for a neighbour's flag (MSWM_PEER_TIMEOUT_MS): long
  // enough for start-up skew between processes, finite so a dead rank
  // becomes an error
  unsigned long long peer_budget_ns = 60000ull * 1000000ull;
  DArr<int32_t> d_peers;
  std::string last_error;
  int32_t nC = 0, nE = 0, nV = 0, deg_max = 0, sten_max = 0;
  bool identity = true;
  std::vector<int32_t> c_new2old, e_new2old, v_new2old, c_old2new, e_old2new, v_old2new;
  std::vector<double> h_cell_area;  // original order (total_mass)

  // device mesh
  DArr<int32_t> c_edge, c_vert, c_nbr, v_cell, v_edge, v_orig, e_sten;
  DArr<uint2> e_st16;
  DArr<double2> e_coef2, v_af;
  DArr<int2> c_edge2, v_ce;
  DArr<uint4> v_rec, c_rec;      // 16-bit index records (kernels.cuh DevMesh)
  DArr<uint2> e_cv16;
  DArr<uint32_t> e_c16;
  bool pack16 = false;
  int64_t n_wide16[3] = {0, 0, 0};  // vertices, cells, edges with an offset outside int16
  uint32_t rq[5] = {0}, rf[5] = {0};  // base ratios: ce, ve, cv, ev, ec
  int64_t n_sten_wide = 0;
  DArr<uint8_t> c_deg, c_sbits, v_sbits, e_nst;
  DArr<double> c_area, v_kite, v_area, e_len, e_ld, e_dual, e_invd, b, f;
  // streamed kernels run a resident grid (persist_ctas CTAs per SM, 8 =
  // full occupancy at 32 registers) looping over their elements: 3.7 % faster
  // C4 steps than one CTA per 256 elements (CTA churn capped occupancy at
  // ~70 %); MSWM_PERSIST=0 restores one element per thread
  int persist_ctas[3] = {2048 / kSBlock, 2048 / kSBlock, 2048 / kSBlock}, n_sm = 148;  // A, B, C
  // chunk schedules of the two-part launches (MSWM_MIX): bit 0 kernel A, bit
  // 1 kernel C interleaved in proportion; bits 2 / 3 windowed.  Measured on C4
  // (profiles/r2_s4_mix_sweep_c4.log): A interleaved gains ~1.5 % of the step
  // (u and h are read once instead of twice), C interleaved loses ~2 %.
  // C windowed gains ~2 % (its cell pass finds the window's (F, q~) in L2:
  // profiles/r2_s4_mix_windows_sweep_c4.log); A windowed does not.
  // Bit 4: ping-pong directions (A forward, B backward, C forward, the next
  // evaluation mirrored): ~0.5 % (profiles/r2_s4_mix_pingpong_sweep_c4.log).
  int mix = 25;
  // window mode: part-0 elements per window (C4: 64 windows of 164k cells,
  // ~80 MB of traffic each, inside L2), or a fixed window count (MSWM_MIX_WIN)
  int flip_main = 0, flip_side = 0;  // ping-pong direction of the next evaluation
  int mix_window_elems = 163840;
  int mix_windows = 0;
  DArr<int2> e_cells, e_verts;
  double gravity = 9.80616;
  bool have_fields = false;

  // state + workspace (internal order)
  DArr<double> H, U, H1, U1, H2, U2, A1h, A1u, A2h, A2u, A3h, A3u, S0h, S0u, S1h, S1u, S2h, S2u;
  DArr<double> T1h, T1u, T2h, T2u;  // RK4 / SSPRK stage buffers
  DArr<double> Dh, Du;              // eval ABI outputs
  DArr<double> pv, K;
  DArr<double2> FQ;
  // concurrent LTS3 coarse step (enqueue_lts3, MSWM_FORK): a second launch
  // stream, its own intermediates, and the "band" -- coarse elements the
  // substep evaluations read as h_old, which the coarse step parks in
  // T1h / T1u until the substeps are done
  cudaStream_t ls2 = nullptr, lsh = nullptr;  // coarse step (low), substeps (high priority)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join_h = nullptr;
  // resident CTAs per SM of the concurrent coarse step (A, B, C): 3/4 of an SM
  int fork_ctas[3] = {1536 / kSBlock, 1536 / kSBlock, 1536 / kSBlock};
  DArr<double> pv2, K2;
  DArr<double2> FQ2;
  DArr<uint32_t> band_cbits, band_ebits;
  DArr<int32_t> band_cells, band_edges;
  int32_t n_band_c = 0, n_band_e = 0;
  int fork_state = 0;  // 0 not prepared, 1 ready, -1 not eligible
  int replication = 1;  // SchemeConfig::replication (operators.cpp:60)
  // interior / boundary split of ranked evaluations (plan_part)
  bool bnd_ready = false;
  DArr<uint8_t> cbnd, ebnd;
  cudaStream_t lx = nullptr;         // halo exchanges overlapping the interior evaluation
  int overlap_level = 0;             // 1: steps 1-2, 2: every evaluation (MSWM_OVERLAP)
  cudaEvent_t ev_x0 = nullptr, ev_x1 = nullptr;
  cudaStream_t stream_of_capture = nullptr;
  DArr<int32_t> d_c_n2o, d_e_n2o;  // internal -> original ids (device permutes)
  DArr<double> io_h, io_u;          // staging for permuted uploads / downloads
  double* pin = nullptr;            // pinned host staging of mswm_cuda_eval (packed reads / outputs)
  size_t pin_n = 0;
  DArr<double> io_pack;             // its device twin
  double time = 0.0;
  // dry-vertex flag: (step << 32 | original vertex), ~0 = none; set by kernel
  // A, cleared only after a synchronous check has reported it
  DArr<unsigned long long> dry_flag;
  DArr<int64_t> step_ctr;  // device copy of steps_issued (k_step_counter)
  int last_dry_vertex = -1;
  int64_t last_dry_step = 0;  // 1-based step of the batch it happened in, 0: an eval call
  int64_t steps_issued = 0;
  // step batches issued since the flag was last consumed: (first global step, count)
  std::vector<std::pair<int64_t, int64_t>> batches;

  // regions
  bool have_regions = false;
  int width = 1;
  DArr<uint8_t> cell_label, cell_sub, edge_label;
  DArr<int32_t> cell_groups, edge_groups;  // group-concatenated ascending lists
  DArr<uint8_t> ckey, ekey;                // GroupBit index per cell / edge (-6)
  int64_t gsize[11] = {0};
  int64_t goff[11] = {0};  // offset of group g inside its buffer
  DArr<int32_t> all_cells, all_edges;  // identity lists (no regions)

  std::map<unsigned, std::unique_ptr<MaskPlan>> plans;

  // ledger (ledger.hpp:25-60)
  int64_t ledger_cell[4][4] = {{0}}, ledger_edge[4][4] = {{0}}, ledger_steps = 0;

  // graphs, one per (scheme, dt, M, profiling); profiled graphs own the
  // events bracketing each evaluation
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    std::vector<EvalRecord> records;
    int64_t kernels = 0;  // kernel nodes per step
  };
  std::map<std::tuple<int, double, int, int>, Graph> graphs;
  int profiling = 0;  // 1: every evaluation bracketed by events, 2: only the first large one
  std::vector<EvalRecord>* capture_records = nullptr;  // set while capturing
  int64_t launches = 0;                               // kernels enqueued (capture counting)
  int64_t last_kernels_per_step = 0;
  const std::vector<EvalRecord>* last_records = nullptr;

  // configuration generation: bumped whenever captured graphs may hold stale
  // pointers or arguments (plans, halos, fields, communicators); group graphs
  // (mswm_cuda_group) compare it to recapture
  uint64_t gen = 0;

  void drop_graphs() {
    ++gen;
    for (auto& kv : graphs) {
      cudaGraphExecDestroy(kv.second.exec);
      for (auto& r : kv.second.records) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
      }
    }
    graphs.clear();
    last_records = nullptr;
  }

  ~mswm_cuda_ctx() {
    drop_graphs();
    for (size_t r = 0; r < peer_base.size(); ++r)
      if (peer_base[r] && peer_ipc[r]) cudaIpcCloseMemHandle(peer_base[r]);
    if (nccl_comm2) nccl().CommDestroy(nccl_comm2);
    if (nccl_comm) nccl().CommDestroy(nccl_comm);
    if (ls2) cudaStreamDestroy(ls2);
    if (lsh) cudaStreamDestroy(lsh);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_join_h) cudaEventDestroy(ev_join_h);
    if (lx) cudaStreamDestroy(lx);
    if (ev_x0) cudaEventDestroy(ev_x0);
    if (ev_x1) cudaEventDestroy(ev_x1);
    if (stream) cudaStreamDestroy(stream);
    if (pin) cudaFreeHost(pin);
  }

  DevMesh dev() const {
    DevMesh M;
    M.nC = nC;
    M.nE = nE;
    M.nV = nV;
    M.deg_max = deg_max;
    M.sten_max = sten_max;
    M.c_edge = c_edge.p;
    M.c_deg = c_deg.p;
    M.c_sbits = c_sbits.p;
    M.c_area = c_area.p;
    M.v_cell = v_cell.p;
    M.v_edge = v_edge.p;
    M.v_kite = v_kite.p;
    M.v_sbits = v_sbits.p;
    M.v_area = v_area.p;
    M.v_orig = v_orig.p;
    M.e_cells = e_cells.p;
    M.e_verts = e_verts.p;
    M.e_len = e_len.p;
    M.e_ld = e_ld.p;
    M.e_dual = e_dual.p;
    M.e_invd = e_invd.p;
    M.e_nst = e_nst.p;
    M.e_sten = e_sten.p;
    M.e_st16 = e_st16.p;
    M.e_coef2 = e_coef2.p;
    M.c_edge2 = c_edge2.p;
    M.v_ce = v_ce.p;
    M.v_af = v_af.p;
    M.v_rec = pack16 ? v_rec.p : nullptr;
    M.c_rec = pack16 && c_rec.p ? c_rec.p : nullptr;
    M.e_cv16 = pack16 ? e_cv16.p : nullptr;
    M.e_c16 = pack16 ? e_c16.p : nullptr;
    M.rq_ce = rq[0]; M.rf_ce = rf[0];
    M.rq_ve = rq[1]; M.rf_ve = rf[1];
    M.rq_cv = rq[2]; M.rf_cv = rf[2];
    M.rq_ev = rq[3]; M.rf_ev = rf[3];
    M.rq_ec = rq[4]; M.rf_ec = rf[4];
    M.b = b.p;
    M.f = f.p;
    M.g = gravity;
    return M;
  }
};

namespace {

// ---------------------------------------------------------------------------
// helpers

// host twin of kernels.cuh pbase: q * x + floor(x * f / 2^32), mod 2^32
int32_t pbase_host(int32_t x, uint32_t q, uint32_t f) {
  return int32_t(q * uint32_t(x) + uint32_t((uint64_t(uint32_t(x)) * f) >> 32));
}

void check_ctx(mswm_cuda_ctx* c) {
  if (!c) throw Error(MSWM_E_USAGE, "null context");
  CK(cudaSetDevice(c->device));
}

// Host permutation helpers: internal array from original-order input.
template <class T>
std::vector<T> to_internal(const mswm_cuda_ctx* c, const T* src, const std::vector<int32_t>& n2o,
                           size_t n) {
  std::vector<T> out(n);
  if (c->identity)
    std::copy(src, src + n, out.begin());
  else
    for (size_t i = 0; i < n; ++i) out[i] = src[n2o[i]];
  return out;
}

// Upload an original-order array into a device buffer in internal order.
// Cell and edge fields are permuted on the device (H2D into a staging
// buffer, then a gather kernel); vertex fields (set once) on the host.
void upload_field(mswm_cuda_ctx* c, DArr<double>& dst, const double* src,
                  const std::vector<int32_t>& n2o, size_t n) {
  if (dst.n != n) dst.alloc(n);
  if (c->identity) {
    CK(cudaMemcpyAsync(dst.p, src, n * 8, cudaMemcpyHostToDevice, c->stream));
    return;
  }
  DArr<double>* stage = nullptr;
  const int32_t* perm = nullptr;
  if (&n2o == &c->c_new2old) {
    stage = &c->io_h;
    perm = c->d_c_n2o.p;
  } else if (&n2o == &c->e_new2old) {
    stage = &c->io_u;
    perm = c->d_e_n2o.p;
  }
  if (stage) {
    CK(cudaMemcpyAsync(stage->p, src, n * 8, cudaMemcpyHostToDevice, c->stream));
    k_gather_perm<<<nblk(int64_t(n)), kBlock, 0, c->stream>>>(int32_t(n), perm, stage->p, dst.p);
    CK(cudaGetLastError());
    return;
  }
  std::vector<double> tmp = to_internal(c, src, n2o, n);
  CK(cudaMemcpyAsync(dst.p, tmp.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

void download_field(mswm_cuda_ctx* c, const DArr<double>& src, double* dst,
                    const std::vector<int32_t>& n2o, size_t n) {
  if (c->identity) {
    CK(cudaMemcpyAsync(dst, src.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return;
  }
  const bool cells = &n2o == &c->c_new2old;
  DArr<double>& stage = cells ? c->io_h : c->io_u;
  const int32_t* perm = cells ? c->d_c_n2o.p : c->d_e_n2o.p;
  k_scatter_perm<<<nblk(int64_t(n)), kBlock, 0, c->stream>>>(int32_t(n), perm, src.p, stage.p);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(dst, stage.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// Order-preserving compaction of key[0..n) into G ascending groups.
// Returns group sizes; out receives group g at offset sum_{h<g} size_h.
std::vector<int64_t> compact(mswm_cuda_ctx* c, const uint8_t* d_key, int32_t n, int G,
                             DArr<int32_t>& out) {
  const int32_t nb = std::max(1, int32_t((int64_t(n) + kCompactTile - 1) / kCompactTile));
  DArr<int32_t> counts;
  counts.alloc(size_t(G) * nb);
  DArr<int64_t> totals, gbase;
  totals.alloc(G);
  gbase.alloc(G);
  k_compact_count<<<nb, kBlock, 0, c->stream>>>(d_key, n, G, counts.p, nb);
  CK(cudaGetLastError());
  k_compact_scan<<<1, kBlock, 0, c->stream>>>(counts.p, nb, G, totals.p);
  CK(cudaGetLastError());
  std::vector<int64_t> sizes(G), base(G);
  CK(cudaMemcpyAsync(sizes.data(), totals.p, G * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int64_t acc = 0;
  for (int g = 0; g < G; ++g) {
    base[g] = acc;
    acc += sizes[g];
  }
  out.alloc(size_t(std::max<int64_t>(acc, 1)));
  CK(cudaMemcpyAsync(gbase.p, base.data(), G * 8, cudaMemcpyHostToDevice, c->stream));
  k_compact_scatter<<<nb, kBlock, 0, c->stream>>>(d_key, n, G, counts.p, nb, gbase.p, out.p);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return sizes;
}

// ---------------------------------------------------------------------------
// create

// f(lo, hi) over [0, n) on the host cores (the drop-in eval's pack and
// scatter loops: independent elements).
template <class F>
void host_par_for(int64_t n, F&& f) {
  static const int64_t T = std::max(1u, std::thread::hardware_concurrency());
  const int64_t t = std::min<int64_t>(T, std::max<int64_t>(1, n / (1 << 18)));
  if (t <= 1) {
    if (n > 0) f(int64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t k = 1; k < t; ++k) th.emplace_back([&, k] { f(n * k / t, n * (k + 1) / t); });
  f(0, n / t);
  for (auto& x : th) x.join();
}

// Internal numbering.  Cells follow `cell_order` (a space-filling curve from
// the caller, or the input order); edges are sorted by the internal ids of
// their two cells (min, max) and vertices by their three, so every gather of
// the kernels lands near the element that issues it.  Per-element
// arithmetic does not depend on the numbering (slot orders, edge_cells
// order and stencil order are carried verbatim), so results are bitwise
// independent of it (SURVEY.md §0 finding 5).
struct OrderKey {
  uint32_t a, b, cc;
};

void make_orders(mswm_cuda_ctx* c, const mswm_mesh_desc* d, const int32_t* cell_order) {
  const int32_t nC = d->n_cells, nE = d->n_edges, nV = d->n_vertices;
  c->c_new2old.resize(nC);
  c->e_new2old.resize(nE);
  c->v_new2old.resize(nV);
  c->c_old2new.assign(nC, -1);
  for (int32_t k = 0; k < nC; ++k) {
    const int32_t i = cell_order ? cell_order[k] : k;
    if (i < 0 || i >= nC || c->c_old2new[i] != -1)
      throw Error(MSWM_E_USAGE, "cell_order is not a permutation of the cells");
    c->c_old2new[i] = k;
    c->c_new2old[k] = i;
  }
  const auto& r = c->c_old2new;
  // Edges by (min cell, max cell, id) and vertices by (their three cells
  // ascending, id) in internal cell ids: a bucket pass on the smallest cell
  // (an element lands in the bucket of one of its <= kMaxDeg-ring cells) and
  // an insertion sort inside each bucket -- linear, parallel over the cells,
  // the order a comparison sort of the full keys gives.
  auto bucket_sort = [&](int32_t n, auto&& key_of, std::vector<int32_t>& new2old,
                         std::vector<int32_t>& old2new) {
    // key_of(x) -> {a, b, c}: a = bucket (smallest cell), (b, c) the rest of the key
    using K = OrderKey;
    std::vector<K> key(static_cast<size_t>(n));
    host_par_for(n, [&](int64_t lo, int64_t hi) {
      for (int64_t x = lo; x < hi; ++x) key[size_t(x)] = key_of(int32_t(x));
    });
    std::vector<int32_t> start(size_t(nC) + 1, 0);
    for (int32_t x = 0; x < n; ++x) ++start[size_t(key[size_t(x)].a) + 1];
    for (int32_t i = 0; i < nC; ++i) start[size_t(i) + 1] += start[size_t(i)];
    std::vector<int32_t> fill(start.begin(), start.end() - 1);
    for (int32_t x = 0; x < n; ++x) new2old[size_t(fill[key[size_t(x)].a]++)] = x;  // ascending id
    host_par_for(nC, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        const int32_t b0 = start[size_t(i)], b1 = start[size_t(i) + 1];
        for (int32_t p = b0 + 1; p < b1; ++p) {
          const int32_t x = new2old[size_t(p)];
          const K kx = key[size_t(x)];
          int32_t q = p;
          while (q > b0) {
            const int32_t y = new2old[size_t(q) - 1];
            const K ky = key[size_t(y)];
            if (std::tie(ky.b, ky.cc, y) <= std::tie(kx.b, kx.cc, x)) break;
            new2old[size_t(q)] = y;
            --q;
          }
          new2old[size_t(q)] = x;
        }
      }
    });
    old2new.assign(size_t(n), 0);
    host_par_for(n, [&](int64_t lo, int64_t hi) {
      for (int64_t k = lo; k < hi; ++k) old2new[size_t(new2old[size_t(k)])] = int32_t(k);
    });
  };
  bucket_sort(
      nE,
      [&](int32_t e) {
        uint32_t a = uint32_t(r[d->edge_cells[2 * e]]), b = uint32_t(r[d->edge_cells[2 * e + 1]]);
        if (a > b) std::swap(a, b);
        return OrderKey{a, b, 0u};
      },
      c->e_new2old, c->e_old2new);
  bucket_sort(
      nV,
      [&](int32_t v) {
        uint32_t x[3] = {uint32_t(r[d->vertex_cells[3 * v]]), uint32_t(r[d->vertex_cells[3 * v + 1]]),
                         uint32_t(r[d->vertex_cells[3 * v + 2]])};
        std::sort(x, x + 3);
        return OrderKey{x[0], x[1], x[2]};
      },
      c->v_new2old, c->v_old2new);
  bool ident = true;
  for (int32_t k = 0; k < nC && ident; ++k) ident = c->c_new2old[k] == k;
  for (int32_t k = 0; k < nE && ident; ++k) ident = c->e_new2old[k] == k;
  for (int32_t k = 0; k < nV && ident; ++k) ident = c->v_new2old[k] == k;
  c->identity = ident;
}


void build_tables(mswm_cuda_ctx* c, const mswm_mesh_desc* d, const int32_t* cell_order) {
  const int32_t nC = d->n_cells, nE = d->n_edges, nV = d->n_vertices;
  if (nC <= 0 || nE <= 0 || nV <= 0) throw Error(MSWM_E_TOPOLOGY, "empty mesh");
  auto need = [](bool ok, const std::string& what) {
    if (!ok) throw Error(MSWM_E_TOPOLOGY, what);
  };
  need(d->cell_offset && d->cell_edges && d->cell_vertices && d->cell_cells && d->edge_cells &&
           d->edge_vertices && d->vertex_cells && d->vertex_edges && d->edge_edge_offset &&
           d->edge_edges && d->edge_cell_sign && d->edge_vertex_sign && d->edge_len &&
           d->edge_dual_len && d->cell_area && d->vertex_area && d->vertex_kite && d->edge_weight,
       "mesh descriptor has a null table");
  c->nC = nC;
  c->nE = nE;
  c->nV = nV;
  int deg_max = 0;
  for (int32_t i = 0; i < nC; ++i) {
    const int deg = d->cell_offset[i + 1] - d->cell_offset[i];
    need(deg >= 3 && deg <= kMaxDeg, "cell " + std::to_string(i) + " ring size out of [3, 8]");
    deg_max = std::max(deg_max, deg);
  }
  int sten_max = 0;
  for (int32_t e = 0; e < nE; ++e) {
    const int n = d->edge_edge_offset[e + 1] - d->edge_edge_offset[e];
    need(n >= 0 && n <= kMaxSten, "edge " + std::to_string(e) + " stencil too long");
    sten_max = std::max(sten_max, n);
  }
  for (int64_t k = 0; k < 2 * int64_t(nE); ++k)
    need(d->edge_cells[k] >= 0 && d->edge_cells[k] < nC && d->edge_vertices[k] >= 0 &&
             d->edge_vertices[k] < nV,
         "edge table id out of range");
  for (int64_t k = 0; k < 3 * int64_t(nV); ++k)
    need(d->vertex_cells[k] >= 0 && d->vertex_cells[k] < nC && d->vertex_edges[k] >= 0 &&
             d->vertex_edges[k] < nE,
         "vertex table id out of range");
  c->deg_max = deg_max;
  c->sten_max = sten_max;
  make_orders(c, d, cell_order);
  const auto& cn = c->c_new2old;
  const auto& en = c->e_new2old;
  const auto& vn = c->v_new2old;
  const auto& co = c->c_old2new;
  const auto& eo = c->e_old2new;
  const auto& vo = c->v_old2new;

  if (const char* pe = std::getenv("MSWM_PERSIST")) {  // "n" or "a,b,c"
    int v[3];
    const int k = std::sscanf(pe, "%d,%d,%d", &v[0], &v[1], &v[2]);
    for (int j = 0; j < 3; ++j) c->persist_ctas[j] = std::max(0, k == 3 ? v[j] : v[0]);
  }
  CK(cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, c->device));

  // cells
  std::vector<int32_t> c_edge(size_t(deg_max) * nC, 0), c_vert(size_t(deg_max) * nC, 0),
      c_nbr(size_t(deg_max) * nC, 0);
  std::vector<uint8_t> c_deg(nC), c_sbits(nC, 0);
  std::vector<double> c_area(nC);
  // the per-element loops below run on all host cores (independent elements,
  // every thread writes its own range); an id out of range is recorded and
  // raised after the join
  std::atomic<int> bad_ring{0}, bad_sten{0};
  host_par_for(nC, [&](int64_t lo, int64_t hi) {
    for (int32_t ni = int32_t(lo); ni < int32_t(hi); ++ni) {
      const int32_t i = cn[ni];
      const int off = d->cell_offset[i], deg = d->cell_offset[i + 1] - off;
      c_deg[ni] = uint8_t(deg);
      c_area[ni] = d->cell_area[i];
      for (int j = 0; j < deg; ++j) {
        const int32_t e = d->cell_edges[off + j], v = d->cell_vertices[off + j],
                      nb = d->cell_cells[off + j];
        if (!(e >= 0 && e < nE && v >= 0 && v < nV && nb >= 0 && nb < nC)) {
          bad_ring = 1;
          continue;
        }
        c_edge[size_t(j) * nC + ni] = eo[e];
        c_vert[size_t(j) * nC + ni] = vo[v];
        c_nbr[size_t(j) * nC + ni] = co[nb];
        // cell_sign(e, i) (mesh.hpp:89-92)
        const int8_t sg = d->edge_cells[2 * e] == i ? d->edge_cell_sign[2 * e] : d->edge_cell_sign[2 * e + 1];
        if (sg < 0) c_sbits[ni] |= uint8_t(1u << j);
      }
    }
  });
  need(!bad_ring, "ring id out of range");
  c->h_cell_area.assign(d->cell_area, d->cell_area + nC);
  // vertices
  std::vector<int32_t> v_cell(size_t(3) * nV), v_edge(size_t(3) * nV), v_orig(nV);
  std::vector<double> v_kite(size_t(3) * nV), v_area(nV);
  std::vector<uint8_t> v_sbits(nV, 0);
  host_par_for(nV, [&](int64_t lo, int64_t hi) {
    for (int32_t nv = int32_t(lo); nv < int32_t(hi); ++nv) {
      const int32_t v = vn[nv];
      v_orig[nv] = v;
      v_area[nv] = d->vertex_area[v];
      for (int k = 0; k < 3; ++k) {
        const int32_t cc = d->vertex_cells[3 * v + k], e = d->vertex_edges[3 * v + k];
        v_cell[size_t(k) * nV + nv] = co[cc];
        v_edge[size_t(k) * nV + nv] = eo[e];
        v_kite[size_t(k) * nV + nv] = d->vertex_kite[3 * v + k];
        // vertex_sign(e, v) (mesh.hpp:93-96)
        const int8_t sg =
            d->edge_vertices[2 * e] == v ? d->edge_vertex_sign[2 * e] : d->edge_vertex_sign[2 * e + 1];
        if (sg < 0) v_sbits[nv] |= uint8_t(1u << k);
      }
    }
  });
  // edges
  std::vector<int2> e_cells(nE), e_verts(nE);
  std::vector<double> e_len(nE), e_ld(nE), e_dual(nE), e_invd(nE);
  std::vector<uint8_t> e_nst;
  std::vector<int32_t> e_sten;
  // built directly in their packed layouts (no int32 / f64 staging copies:
  // C5's tables are ~10 GB each on the host)
  std::vector<uint2> e_st16p;     // [(W+1)/2][nE] u32 word pairs, W = n_words
  std::vector<double2> e_coef2;   // [(sten_max+1)/2][nE] coefficient pairs
  const int n_words = (std::max(sten_max, 1) + 1) / 2;
  // 16-bit stencil offsets (kernels.cuh item_out_edge); MSWM_ST16=0 keeps the
  // int32 table only (A/B runs)
  if (const char* me = std::getenv("MSWM_MIX")) c->mix = std::atoi(me);
  if (const char* me = std::getenv("MSWM_MIX_WIN")) c->mix_windows = std::max(1, std::atoi(me));
  const char* s16 = std::getenv("MSWM_ST16");
  const bool use16 = sten_max < 0x80 && !(s16 && s16[0] == '0');
  // 16-bit index records (kernels.cuh DevMesh: v_rec, c_rec, e_cv16, e_c16);
  // MSWM_PACK16=0 keeps the int32 tables only (A/B runs)
  const char* p16 = std::getenv("MSWM_PACK16");
  c->pack16 = !(p16 && p16[0] == '0');
  {
    const int64_t n_of[3] = {nC, nE, nV};  // 0 cells, 1 edges, 2 vertices
    const int pairs[5][2] = {{0, 1}, {2, 1}, {0, 2}, {1, 2}, {1, 0}};  // (to, from)
    for (int k = 0; k < 5; ++k) {
      const uint64_t num = uint64_t(n_of[pairs[k][0]]), den = uint64_t(n_of[pairs[k][1]]);
      c->rq[k] = uint32_t(num / den);
      c->rf[k] = uint32_t(((num % den) << 32) / den);
    }
  }
  // offset of id from the base of x under ratio k; 0x8000 (and a wide flag)
  // when it does not fit
  auto off16 = [&](int32_t id, int32_t x, int k, bool& wide) -> uint32_t {
    const int32_t base = pbase_host(x, c->rq[k], c->rf[k]);
    const int64_t dd = int64_t(id) - base;
    if (dd < -32767 || dd > 32767) {
      wide = true;
      return 0x8000u;
    }
    return uint32_t(dd) & 0xFFFFu;
  };
  std::vector<uint2> e_cv16;
  std::vector<uint32_t> e_c16;
  if (c->pack16) {
    e_cv16.resize(nE);
    e_c16.resize(nE);
  }
  e_nst.resize(nE);
  e_sten.assign(size_t(std::max(sten_max, 1)) * nE, 0);
  e_coef2.assign(size_t((std::max(sten_max, 1) + 1) / 2) * nE, make_double2(0.0, 0.0));
  if (use16) e_st16p.assign(size_t((n_words + 1) / 2) * nE, make_uint2(0u, 0u));
  std::atomic<int64_t> wide_edges{0};
  host_par_for(nE, [&](int64_t lo, int64_t hi) {
    int64_t n_wide_local = 0;
    for (int32_t ne = int32_t(lo); ne < int32_t(hi); ++ne) {
      const int32_t e = en[ne];
      const int32_t c0 = d->edge_cells[2 * e], c1 = d->edge_cells[2 * e + 1];
      const int32_t v0 = d->edge_vertices[2 * e], v1 = d->edge_vertices[2 * e + 1];
      e_cells[ne] = make_int2(co[c0], co[c1]);
      e_verts[ne] = make_int2(vo[v0], vo[v1]);
      const double l = d->edge_len[e], dd = d->edge_dual_len[e];
      e_len[ne] = l;
      e_dual[ne] = dd;
      e_ld[ne] = l * dd;              // operators.cpp:70, first product
      const double inv_d = 1.0 / dd;  // operators.cpp:103
      e_invd[ne] = inv_d;
      const int off = d->edge_edge_offset[e], n = d->edge_edge_offset[e + 1] - off;
      e_nst[ne] = uint8_t(n);
      if (c->pack16) {
        bool wc = false, wv = false;
        const uint32_t a = off16(e_cells[ne].x, ne, 0, wc), b2 = off16(e_cells[ne].y, ne, 0, wc);
        const uint32_t x = off16(e_verts[ne].x, ne, 1, wv), y = off16(e_verts[ne].y, ne, 1, wv);
        e_cv16[ne] = make_uint2(a | b2 << 16, x | y << 16);
        e_c16[ne] = a | b2 << 16;
        // ten-entry stencils use five of the six words of the e_st16 row: the
        // sixth carries (c0, c1) for kernel C
        if (use16 && sten_max == kFastSten) e_st16p[size_t(2) * nE + ne].y = a | b2 << 16;
        if (wc) e_nst[ne] |= 0x40;
        n_wide_local += wc || wv;
      }
      for (int j = 0; j < n; ++j) {
        const int32_t e2 = d->edge_edges[off + j];
        if (!(e2 >= 0 && e2 < nE)) {
          bad_sten = 1;
          continue;
        }
        e_sten[size_t(j) * nE + ne] = eo[e2];
        const int32_t dlt = eo[e2] - ne;
        if (dlt < INT16_MIN || dlt > INT16_MAX)
          e_nst[ne] |= 0x80;
        else if (use16) {
          // entry j -> word j/2 (half j&1) -> pair word/2 (component word&1)
          uint2& pw = e_st16p[size_t(j / 4) * nE + ne];
          ((j / 2) & 1 ? pw.y : pw.x) |= (uint32_t(dlt) & 0xFFFFu) << (16 * (j & 1));
        }
        // operators.cpp:109: weights[j] * (edge_len[e2] * inv_d), the first
        // two factors of the stencil term -- mesh constants.
        double2& cp = e_coef2[size_t(j / 2) * nE + ne];
        (j & 1 ? cp.y : cp.x) = d->edge_weight[off + j] * (d->edge_len[e2] * inv_d);
      }
    }
    wide_edges += n_wide_local;
  });
  need(!bad_sten, "stencil id out of range");
  c->n_wide16[2] += wide_edges;
  cudaStream_t s = c->stream;
  // upload, then release the host copy at once (C5's tables total tens of GB
  // on the host; keeping them all alive until the end ran the box out of
  // memory)
  auto put = [&](auto& dst, auto& vec) {
    dst.upload(vec, s);
    CK(cudaStreamSynchronize(s));
    std::remove_reference_t<decltype(vec)>().swap(vec);
  };
  put(c->e_coef2, e_coef2);
  c->n_sten_wide = 0;
  for (const uint8_t x : e_nst) c->n_sten_wide += x >> 7;
  put(c->e_st16, e_st16p);
  put(c->e_sten, e_sten);
  put(c->e_nst, e_nst);
  if (c->pack16) {
    put(c->e_cv16, e_cv16);
    put(c->e_c16, e_c16);
  }
  {
    // packed copies (kernels.cuh DevMesh): pairs of slots / entries per load
    std::vector<int2> c_edge2(size_t((deg_max + 1) / 2) * nC, make_int2(0, 0));
    host_par_for(nC, [&](int64_t lo, int64_t hi) {
      for (int j = 0; j < deg_max; ++j)
        for (int32_t i = int32_t(lo); i < int32_t(hi); ++i) {
          int2& p = c_edge2[size_t(j / 2) * nC + i];
          (j & 1 ? p.y : p.x) = c_edge[size_t(j) * nC + i];
        }
    });
    put(c->c_edge2, c_edge2);
    std::vector<int2> v_ce(size_t(3) * nV);
    host_par_for(nV, [&](int64_t lo, int64_t hi) {
      for (int32_t v = int32_t(lo); v < int32_t(hi); ++v)
        for (int k = 0; k < 3; ++k)
          v_ce[size_t(k) * nV + v] = make_int2(v_cell[size_t(k) * nV + v], v_edge[size_t(k) * nV + v]);
    });
    put(c->v_ce, v_ce);
    // 16-bit index records of vertices and cells (e_cv16 / e_c16 above)
    if (c->pack16) {
      std::vector<uint4> v_rec(nV);
      std::atomic<int64_t> wide_v{0};
      host_par_for(nV, [&](int64_t lo, int64_t hi) {
        int64_t nw = 0;
        for (int32_t v = int32_t(lo); v < int32_t(hi); ++v) {
          bool w = false;
          uint32_t o[6];
          for (int k = 0; k < 3; ++k) {
            o[k] = off16(v_cell[size_t(k) * nV + v], v, 2, w);
            o[3 + k] = off16(v_edge[size_t(k) * nV + v], v, 3, w);
          }
          nw += w;
          v_rec[v] = make_uint4(o[0] | o[1] << 16, o[2] | o[3] << 16, o[4] | o[5] << 16,
                                uint32_t(v_sbits[v]) | (w ? 0x80u : 0u));
        }
        wide_v += nw;
      });
      c->n_wide16[0] += wide_v;
      put(c->v_rec, v_rec);
      if (deg_max == kFastDeg) {
        std::vector<uint4> c_rec(nC);
        std::atomic<int64_t> wide_c{0};
        host_par_for(nC, [&](int64_t lo, int64_t hi) {
          int64_t nw = 0;
          for (int32_t i = int32_t(lo); i < int32_t(hi); ++i) {
            bool w = false;
            uint32_t o[6];
            for (int j = 0; j < 6; ++j)
              o[j] = j < c_deg[i] ? off16(c_edge[size_t(j) * nC + i], i, 4, w) : 0u;
            nw += w;
            c_rec[i] = make_uint4(o[0] | o[1] << 16, o[2] | o[3] << 16, o[4] | o[5] << 16,
                                  uint32_t(c_deg[i]) | (w ? 0x80u : 0u) | uint32_t(c_sbits[i]) << 8);
          }
          wide_c += nw;
        });
        c->n_wide16[1] += wide_c;
        put(c->c_rec, c_rec);
      }
    }
    std::vector<double2> v_af(nV);
    for (int32_t v = 0; v < nV; ++v) v_af[v] = make_double2(v_area[v], 0.0);  // f_v: set_fields
    put(c->v_af, v_af);
  }
  put(c->c_edge, c_edge);
  put(c->c_vert, c_vert);
  put(c->c_nbr, c_nbr);
  put(c->c_deg, c_deg);
  put(c->c_sbits, c_sbits);
  put(c->c_area, c_area);
  put(c->v_cell, v_cell);
  put(c->v_edge, v_edge);
  put(c->v_orig, v_orig);
  put(c->v_kite, v_kite);
  put(c->v_area, v_area);
  put(c->v_sbits, v_sbits);
  put(c->e_cells, e_cells);
  put(c->e_verts, e_verts);
  put(c->e_len, e_len);
  put(c->e_ld, e_ld);
  put(c->e_dual, e_dual);
  put(c->e_invd, e_invd);
  CK(cudaStreamSynchronize(s));  // host vectors die here

  // state + workspace, zero-initialised
  DArr<double>* cellbufs[] = {&c->H, &c->H1, &c->H2, &c->A1h, &c->A2h, &c->A3h, &c->S0h,
                              &c->S1h, &c->S2h, &c->T1h, &c->T2h, &c->Dh, &c->K};
  DArr<double>* edgebufs[] = {&c->U, &c->U1, &c->U2, &c->A1u, &c->A2u, &c->A3u, &c->S0u,
                              &c->S1u, &c->S2u, &c->T1u, &c->T2u, &c->Du};
  for (auto* bptr : cellbufs) {
    bptr->alloc(nC);
    bptr->zero(s);
  }
  for (auto* bptr : edgebufs) {
    bptr->alloc(nE);
    bptr->zero(s);
  }
  c->pv.alloc(nV);
  c->pv.zero(s);
  c->FQ.alloc(nE);
  c->FQ.zero(s);
  if (!c->identity) {
    c->d_c_n2o.upload(c->c_new2old, s);
    c->d_e_n2o.upload(c->e_new2old, s);
    c->io_h.alloc(nC);
    c->io_u.alloc(nE);
    CK(cudaStreamSynchronize(s));
  }
  c->b.alloc(nC);
  c->b.zero(s);
  c->f.alloc(nV);
  c->f.zero(s);
  c->dry_flag.alloc(1);
  CK(cudaMemsetAsync(c->dry_flag.p, 0xFF, 8, s));
  c->step_ctr.alloc(1);
  c->step_ctr.zero(s);
  // identity lists for evaluation without regions
  std::vector<int32_t> ic(nC), ie(nE);
  std::iota(ic.begin(), ic.end(), 0);
  std::iota(ie.begin(), ie.end(), 0);
  c->all_cells.upload(ic, s);
  c->all_edges.upload(ie, s);
  CK(cudaStreamSynchronize(s));
}

// Synchronise and consume the dry-vertex flag: if kernel A hit a dry vertex
// since the last check, clear the flag and throw DryVertexError with the step
// ("during step k of n" of the batch it happened in, harness.cpp:183-190).
void check_dry(mswm_cuda_ctx* c, const char* who = nullptr) {
  unsigned long long v = ~0ull;
  int xe = 0;
  CK(cudaMemcpyAsync(&v, c->dry_flag.p, 8, cudaMemcpyDeviceToHost, c->stream));
  if (c->xerr.p) CK(cudaMemcpyAsync(&xe, c->xerr.p, sizeof(xe), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->xerr.p) {
    if (xe) {
      CK(cudaMemsetAsync(c->xerr.p, 0, sizeof(xe), c->stream));
      CK(cudaStreamSynchronize(c->stream));
      throw Error(MSWM_E_NCCL, "peer-store halo exchange: rank " + std::to_string(xe - 1) +
                                   " did not signal within the poll budget");
    }
  }
  const auto batches = std::move(c->batches);
  c->batches.clear();
  if (v == ~0ull) return;
  CK(cudaMemsetAsync(c->dry_flag.p, 0xFF, 8, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->last_dry_vertex = int(uint32_t(v & 0xFFFFFFFFu));
  const int64_t gstep = int64_t(v >> 32);
  std::string msg = (who ? std::string(who) + ": " : std::string()) + "vertex " +
                    std::to_string(c->last_dry_vertex) + " has non-positive thickness";
  c->last_dry_step = 0;
  for (const auto& b : batches)
    if (gstep > b.first && gstep <= b.first + b.second) {
      c->last_dry_step = gstep - b.first;
      msg += " (during step " + std::to_string(gstep - b.first) + " of " + std::to_string(b.second) + ")";
    }
  throw Error(MSWM_E_DRY_VERTEX, msg);
}

// ---------------------------------------------------------------------------
// mask plans

void invalidate(mswm_cuda_ctx* c) {
  c->plans.clear();
  c->bnd_ready = false;
  c->drop_graphs();
  c->fork_state = 0;  // the band depends on the plans
}

// Launch set for a sorted id list: its longest run of consecutive ids as a
// range plus the rest as a list when the run holds >= 90 % of the ids (the
// region-major layout makes every LTS set such a range), else a dense
// superset [0, universe) when the list covers >= `dense_frac` of it (the
// kernels filter outputs by group key and dry vertices by bitmask), else the
// plain list.
void make_span(mswm_cuda_ctx* c, const int32_t* d_list, int32_t n, int32_t universe,
               double dense_frac, MaskPlan::HSpan& out) {
  out = MaskPlan::HSpan();
  if (n <= 0) return;
  std::vector<int32_t> h(n);
  CK(cudaMemcpyAsync(h.data(), d_list, size_t(n) * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::sort(h.begin(), h.end());
  int32_t best_lo = 0, best_len = 1;
  for (int32_t k = 0; k < n;) {
    int32_t j = k + 1;
    while (j < n && h[j] == h[j - 1] + 1) ++j;
    if (j - k > best_len) {
      best_len = j - k;
      best_lo = k;
    }
    k = j;
  }
  if (best_len >= int64_t(n) * 9 / 10) {
    out.base = h[best_lo];
    out.n_range = best_len;
    std::vector<int32_t> rest;
    rest.reserve(size_t(n - best_len));
    rest.insert(rest.end(), h.begin(), h.begin() + best_lo);
    rest.insert(rest.end(), h.begin() + best_lo + best_len, h.end());
    out.n_list = int32_t(rest.size());
    if (!rest.empty()) {
      out.own.upload(rest, c->stream);
      out.list = out.own.p;
    }
    return;
  }
  if (double(n) >= dense_frac * universe) {
    out.n_range = universe;
    return;
  }
  out.own.upload(h, c->stream);
  out.list = out.own.p;
  out.n_list = n;
}

void finish_plan(mswm_cuda_ctx* c, MaskPlan* p, double out_dense_frac);
std::vector<int32_t> chunk_map(int64_t n0, int64_t n1, int mode, int n_windows);

MaskPlan& plan_for(mswm_cuda_ctx* c, unsigned mask) {
  auto it = c->plans.find(mask);
  if (it != c->plans.end()) return *it->second;
  if (mask & ~unsigned(MSWM_MASK_ALL)) throw Error(MSWM_E_USAGE, "mask has unknown group bits");
  auto p = std::make_unique<MaskPlan>();
  p->mask = mask;
  debug_mem("plan_for: start");
  cudaStream_t s = c->stream;
  if (!c->have_regions) {
    // integrators.cpp:139-142
    if (mask != MSWM_MASK_ALL)
      throw Error(MSWM_E_USAGE, "partial evaluation masks require a region map on the evaluator");
    p->cells = c->all_cells.p;
    p->nc = p->csplit = c->nC;
    p->edges = c->all_edges.p;
    p->ne = p->esplit = c->nE;
  } else {
    // Segment 0 = fine groups (bits 0-2 / 6-7), segment 1 = the rest.
    // Group buffers are [g0 | g1 | ... ], so a run of consecutive set bits
    // aliases a contiguous range; otherwise the groups are concatenated.
    auto build = [&](int g0, int g1, DArr<int32_t>& groups, DArr<int32_t>& own,
                     const int32_t*& list, int32_t& n, int32_t& split, int fine_last) {
      std::vector<int> sel;
      for (int g = g0; g <= g1; ++g)
        if (mask & (1u << g)) sel.push_back(g);
      n = 0;
      split = 0;
      for (int g : sel) {
        n += int32_t(c->gsize[g]);
        if (g <= fine_last) split += int32_t(c->gsize[g]);
      }
      bool contiguous = true;
      for (size_t k = 1; k < sel.size(); ++k) contiguous &= sel[k] == sel[k - 1] + 1;
      if (sel.empty()) {
        list = nullptr;
      } else if (contiguous) {
        list = groups.p + c->goff[sel[0]];
      } else {
        own.alloc(size_t(std::max(n, 1)));
        int64_t pos = 0;
        for (int g : sel) {
          if (c->gsize[g])
            CK(cudaMemcpyAsync(own.p + pos, groups.p + c->goff[g], c->gsize[g] * 4,
                               cudaMemcpyDeviceToDevice, s));
          pos += c->gsize[g];
        }
        list = own.p;
      }
    };
    build(0, 5, c->cell_groups, p->own_cells, p->cells, p->nc, p->csplit, 2);
    build(6, 10, c->edge_groups, p->own_edges, p->edges, p->ne, p->esplit, 7);
  }
  finish_plan(c, p.get(), 0.5);
  auto& slot = c->plans[mask];
  slot = std::move(p);
  debug_mem("plan_for: done");
  return *slot;
}

// Closures, launch spans and host id lists of a plan whose output lists are
// set.  out_dense_frac > 1: the output spans are never dense supersets (a
// part plan must not touch the other part's outputs).
void finish_plan(mswm_cuda_ctx* c, MaskPlan* p, double out_dense_frac) {
  cudaStream_t s = c->stream;
  // Closure marks (operators.cpp:35-58) and their compaction.
  DArr<uint8_t> mf, mq, mk, mv, key;
  mf.alloc(c->nE);
  mq.alloc(c->nE);
  mk.alloc(c->nC);
  mv.alloc(c->nV);
  mf.zero(s);
  mq.zero(s);
  mk.zero(s);
  mv.zero(s);
  if (p->nc + p->ne > 0) {
    k_mark_closure<<<nblk(int64_t(p->nc) + p->ne), kBlock, 0, s>>>(
        c->dev(), c->c_vert.p, p->cells, p->nc, p->edges, p->ne, mf.p, mq.p, mk.p, mv.p);
    CK(cudaGetLastError());
  }
  key.alloc(std::max(c->nE, std::max(c->nC, c->nV)));
  k_union_key<<<nblk(c->nE), kBlock, 0, s>>>(c->nE, mf.p, mq.p, key.p);
  p->nec = int32_t(compact(c, key.p, c->nE, 1, p->eclos)[0]);
  k_flag_key<<<nblk(c->nE), kBlock, 0, s>>>(c->nE, mf.p, key.p);
  p->nf = int32_t(compact(c, key.p, c->nE, 1, p->fclos)[0]);
  k_flag_key<<<nblk(c->nE), kBlock, 0, s>>>(c->nE, mq.p, key.p);
  p->nq = int32_t(compact(c, key.p, c->nE, 1, p->qclos)[0]);
  k_flag_key<<<nblk(c->nC), kBlock, 0, s>>>(c->nC, mk.p, key.p);
  p->nk = int32_t(compact(c, key.p, c->nC, 1, p->kclos)[0]);
  k_flag_key<<<nblk(c->nV), kBlock, 0, s>>>(c->nV, mv.p, key.p);
  p->nv = int32_t(compact(c, key.p, c->nV, 1, p->vclos)[0]);
  debug_mem("plan_for: closures");
  p->dense_v = p->nv >= int64_t(c->nV) * 85 / 100;
  p->dense_k = p->nk >= int64_t(c->nC) * 85 / 100;
  p->dense_fq = p->nec >= int64_t(c->nE) * 85 / 100;
  p->dense_out = int64_t(p->nc) + p->ne >= (int64_t(c->nC) + c->nE) / 2;
  make_span(c, p->vclos.p, p->nv, c->nV, 0.85, p->sv);
  make_span(c, p->kclos.p, p->nk, c->nC, 0.85, p->sk);
  make_span(c, p->eclos.p, p->nec, c->nE, 0.85, p->se);
  make_span(c, p->cells, p->nc, c->nC, out_dense_frac, p->sc_out);
  make_span(c, p->edges, p->ne, c->nE, out_dense_frac, p->se_out);
  debug_mem("plan_for: spans");
  // supersets need the closure bitmask for the dry check
  if (p->sv.n() > p->nv) p->dense_v = true;
  if (p->dense_v && p->nv < c->nV) {
    p->vmask.alloc((size_t(c->nV) + 31) / 32);
    k_pack_bits<<<nblk((int64_t(c->nV) + 31) / 32), kBlock, 0, s>>>(c->nV, mv.p, p->vmask.p);
    CK(cudaGetLastError());
  }
  // chunk schedules of the two-part launches (MSWM_MIX: bits 0 / 1 kernel A /
  // C interleaved, bits 2 / 3 windowed)
  {
    const int ma = (c->mix & 4) ? 2 : (c->mix & 1) ? 1 : 0, mc = (c->mix & 8) ? 2 : (c->mix & 2) ? 1 : 0;
    auto windows = [&](int64_t n0) {
      return c->mix_windows > 0 ? c->mix_windows
                                : int(std::max<int64_t>(1, (n0 + c->mix_window_elems - 1) / c->mix_window_elems));
    };
    const std::vector<int32_t> a = chunk_map(p->sv.n(), p->sk.n(), ma, windows(p->sv.n()));
    const std::vector<int32_t> o = chunk_map(p->sc_out.n(), p->se_out.n(), mc, windows(p->sc_out.n()));
    if (!a.empty()) p->cmapA.upload(a, s);
    if (!o.empty()) p->cmapC.upload(o, s);
    if (c->mix & 16) {
      // reversed schedules: a kernel that starts where its producer just
      // finished finds that stretch of the producer's output still in L2
      auto rev = [&](std::vector<int32_t> m, int64_t n0, int64_t n1, DArr<int32_t>& out) {
        if (m.empty()) {  // part 0's chunks, then part 1's
          for (int64_t k = 0; k < nblk(n0, kSBlock); ++k) m.push_back(int32_t(k * kSBlock));
          for (int64_t k = 0; k < nblk(n1, kSBlock); ++k) m.push_back(int32_t(n0 + k * kSBlock));
        }
        std::reverse(m.begin(), m.end());
        if (!m.empty()) out.upload(m, s);
      };
      rev(a, p->sv.n(), p->sk.n(), p->cmapA_r);
      rev(o, p->sc_out.n(), p->se_out.n(), p->cmapC_r);
      rev({}, p->se.n(), 0, p->cmapB_r);
    }
  }
  // host copies of the output lists (original ids) for the eval ABI
  p->host_cells.resize(p->nc);
  p->host_edges.resize(p->ne);
  if (p->nc)
    CK(cudaMemcpyAsync(p->host_cells.data(), p->cells, size_t(p->nc) * 4, cudaMemcpyDeviceToHost, s));
  if (p->ne)
    CK(cudaMemcpyAsync(p->host_edges.data(), p->edges, size_t(p->ne) * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!c->identity) {
    for (auto& i : p->host_cells) i = c->c_new2old[i];
    for (auto& e : p->host_edges) e = c->e_new2old[e];
  }
}

// Boundary flags of a rank's outputs (k_taint_*, k_mark_boundary): the
// outputs whose evaluation reads a halo value, directly or through PV, psi
// or (F, q~).
void ensure_boundary(mswm_cuda_ctx* c) {
  if (c->bnd_ready) return;
  cudaStream_t s = c->stream;
  DArr<uint8_t> tv, tf, tp;
  tv.alloc(c->nV);
  tf.alloc(c->nE);
  tp.alloc(c->nC);
  c->cbnd.alloc(c->nC);
  c->ebnd.alloc(c->nE);
  const DevMesh M = c->dev();
  k_taint_vertices<<<nblk(c->nV), kBlock, 0, s>>>(M, c->ckey.p, c->ekey.p, tv.p);
  k_taint_fp<<<nblk(int64_t(c->nE) + c->nC), kBlock, 0, s>>>(M, c->ckey.p, c->ekey.p, tv.p, tf.p,
                                                              tp.p);
  k_mark_boundary<<<nblk(int64_t(c->nC) + c->nE), kBlock, 0, s>>>(M, tf.p, tp.p, c->cbnd.p,
                                                                   c->ebnd.p);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  c->bnd_ready = true;
}

// The interior (part 1: reads no halo value) or boundary (part 2) outputs of
// a mask, as a plan of their own.
MaskPlan& plan_part(mswm_cuda_ctx* c, unsigned mask, int part) {
  const unsigned key = mask | (unsigned(part) << 16);
  auto it = c->plans.find(key);
  if (it != c->plans.end()) return *it->second;
  plan_for(c, mask);  // validates the mask
  ensure_boundary(c);
  auto p = std::make_unique<MaskPlan>();
  p->mask = mask;
  cudaStream_t s = c->stream;
  const uint8_t want = part == 2 ? 1 : 0;
  DArr<uint8_t> k;
  k.alloc(std::max(c->nC, c->nE));
  k_part_key<<<nblk(c->nC), kBlock, 0, s>>>(c->nC, c->ckey.p, 0, mask, 5, c->cbnd.p, want, k.p);
  CK(cudaGetLastError());
  p->nc = int32_t(compact(c, k.p, c->nC, 1, p->own_cells)[0]);
  p->cells = p->nc ? p->own_cells.p : nullptr;
  k_part_key<<<nblk(c->nE), kBlock, 0, s>>>(c->nE, c->ekey.p, 6, mask, 4, c->ebnd.p, want, k.p);
  CK(cudaGetLastError());
  p->ne = int32_t(compact(c, k.p, c->nE, 1, p->own_edges)[0]);
  p->edges = p->ne ? p->own_edges.p : nullptr;
  finish_plan(c, p.get(), 2.0);
  auto& slot = c->plans[key];
  slot = std::move(p);
  return *slot;
}

// ---------------------------------------------------------------------------
// one tendency evaluation = kernels A, B, C on the stream

// Grid of a streamed kernel: one element per thread, or at most
// `persist_ctas` CTAs per SM looping over the elements (MSWM_PERSIST).
int sgrid(const mswm_cuda_ctx* c, int64_t n, int kernel) {
  const int64_t b = nblk(n, kSBlock);
  const int p = c->persist_ctas[kernel];
  return int(p > 0 ? std::min<int64_t>(b, int64_t(p) * c->n_sm) : b);
}

// Chunk schedule of a two-part launch (kernels.cuh ChunkMap) for parts of n0
// and n1 elements.  mode 1: the parts' chunks interleaved in proportion (part
// 0's chunk count among the first q chunks = floor(q C0 / (C0 + C1))); mode 2:
// n_windows windows along the curve, each running its part-1 chunks and then
// its part-0 chunks.  Empty: part 0, then part 1 (no map).
std::vector<int32_t> chunk_map(int64_t n0, int64_t n1, int mode, int n_windows) {
  std::vector<int32_t> m;
  const int64_t C0 = nblk(n0, kSBlock), C1 = nblk(n1, kSBlock);
  if (mode == 0 || C0 == 0 || C1 == 0) return m;
  m.reserve(size_t(C0 + C1));
  auto part0 = [&](int64_t k) { m.push_back(int32_t(k * kSBlock)); };
  auto part1 = [&](int64_t k) { m.push_back(int32_t(n0 + k * kSBlock)); };
  if (mode == 1) {
    const int64_t T = C0 + C1;
    int64_t k0 = 0, k1 = 0;
    for (int64_t q = 0; q < T; ++q) {
      if ((q + 1) * C0 / T > q * C0 / T)
        part0(k0++);
      else
        part1(k1++);
    }
  } else {
    const int64_t nw = std::max(1, n_windows);
    const int64_t w0 = (C0 + nw - 1) / nw, w1 = (C1 + nw - 1) / nw;
    for (int64_t k0 = 0, k1 = 0; k0 < C0 || k1 < C1;) {
      for (int64_t j = 0; j < w1 && k1 < C1; ++j) part1(k1++);
      for (int64_t j = 0; j < w0 && k0 < C0; ++j) part0(k0++);
    }
  }
  return m;
}

Op op_none() {
  Op o;
  std::memset(&o, 0, sizeof(o));
  o.kind = OP_NONE;
  return o;
}

// Where a launch_eval goes: stream and intermediates (null: the context's).
struct Side {
  cudaStream_t s;
  double* pv;
  double* K;
  double2* FQ;
  int ctas_per_sm[3];  // resident-grid size of kernels A, B, C (0: default)
};

void launch_eval_once(mswm_cuda_ctx* c, const MaskPlan& p, const double* h, const double* u,
                      const Op cop[2], const Op eop[2], const PredArgs* pred,
                      const Side* side) {
  cudaStream_t s = side ? side->s : c->ls;
  double* const pv = side ? side->pv : c->pv.p;
  double* const Kp = side ? side->K : c->K.p;
  double2* const FQ = side ? side->FQ : c->FQ.p;
  auto grid = [&](int64_t n, int kernel) {
    const int g = sgrid(c, n, kernel);
    return side && side->ctas_per_sm[kernel] > 0 ? std::min(g, side->ctas_per_sm[kernel] * c->n_sm)
                                                 : g;
  };
  if (pred && int64_t(pred->nc) + pred->ne > 0) {
    k_predict<<<nblk(int64_t(pred->nc) + pred->ne), kBlock, 0, s>>>(pred->clist, pred->nc,
        pred->elist, pred->ne, pred->c0, pred->c1, pred->c2, pred->hs0, pred->hs1, pred->hs2,
        pred->hdst, pred->us0, pred->us1, pred->us2, pred->udst);
    CK(cudaGetLastError());
    ++c->launches;
  }
  const DevMesh M = c->dev();
  // ping-pong order (MSWM_MIX bit 4): A forward, B backward, C forward, and
  // the next evaluation on this stream mirrored (A backward from where C ended)
  bool flip = false;
  if (c->mix & 16) {
    int& par = side ? c->flip_side : c->flip_main;
    flip = par != 0;
    par ^= 1;
  }
  EvalRecord* rec = nullptr;
  if (c->capture_records &&
      (c->profiling != 2 || (c->capture_records->empty() &&
                             2 * (int64_t(p.nc) + p.ne) >= int64_t(c->nC) + c->nE))) {
    EvalRecord r;
    CK(cudaEventCreate(&r.start));
    CK(cudaEventCreate(&r.stop));
    c->capture_records->push_back(r);
    rec = &c->capture_records->back();
    rec->nc = p.nc;
    rec->ne = p.ne;
    CK(cudaEventRecordWithFlags(rec->start, s, cudaEventRecordExternal));
  }
  const Span vs = p.sv.dev(), ks = p.sk.dev(), es = p.se.dev();
  const int64_t na = p.sv.n() + p.sk.n();
  if (na > 0) {
    const DArr<int32_t>& ma = flip ? p.cmapA_r : p.cmapA;
    k_vertex_cell<<<grid(na, 0), kSBlock, 0, s>>>(M, h, u, vs, ks, pv, Kp, c->dry_flag.p,
        c->step_ctr.p, p.vmask.p, ChunkMap{ma.p, int32_t(ma.n)});
    CK(cudaGetLastError());
    ++c->launches;
  }
  if (p.se.n() > 0) {
    // ping-pong: B runs against A's direction, C against B's
    const DArr<int32_t>* mb = (c->mix & 16) && !flip ? &p.cmapB_r : nullptr;
    k_edge_fq<<<grid(p.se.n(), 1), kSBlock, 0, s>>>(M, h, u, pv, es, FQ,
        mb ? ChunkMap{mb->p, int32_t(mb->n)} : ChunkMap{nullptr, 0});
    CK(cudaGetLastError());
    ++c->launches;
  }
  const int64_t nout = p.sc_out.n() + p.se_out.n();
  if (nout > 0) {
    OutArgs a;
    std::memset(&a, 0, sizeof(a));
    a.cs = p.sc_out.dev();
    a.es = p.se_out.dev();
    a.mask = p.mask;
    a.ckey = c->have_regions ? c->ckey.p : nullptr;
    a.ekey = c->have_regions ? c->ekey.p : nullptr;
    a.cop[0] = cop[0];
    a.cop[1] = cop[1];
    a.eop[0] = eop[0];
    a.eop[1] = eop[1];
    const DArr<int32_t>& mc = flip ? p.cmapC_r : p.cmapC;
    a.cm = ChunkMap{mc.p, int32_t(mc.n)};
    k_out<<<grid(nout, 2), kSBlock, 0, s>>>(M, h, Kp, FQ, a);
    CK(cudaGetLastError());
    ++c->launches;
  }
  if (rec) CK(cudaEventRecordWithFlags(rec->stop, s, cudaEventRecordExternal));
}

// Op factories (cells use h-arrays, edges u-arrays)
Op mk_op(int kind, double* dst, const double* y0 = nullptr, double c0 = 0, const double* y1 = nullptr,
         double c1 = 0, double c2 = 0, double* acc = nullptr, int first = 0,
         const double* a1 = nullptr, const double* a2 = nullptr) {
  Op o = op_none();
  o.kind = kind;
  o.dst = dst;
  o.y0 = y0;
  o.c0 = c0;
  o.y1 = y1;
  o.c1 = c1;
  o.c2 = c2;
  o.acc = acc;
  o.first = first;
  o.a1 = a1;
  o.a2 = a2;
  return o;
}

// One masked evaluation with its fused stage update.  With a replication
// factor R > 1 (SchemeConfig::replication, operators.cpp:60: the kernel
// arithmetic repeated to emulate more vertical layers) the three kernels run
// R times; the first R - 1 passes store into the eval scratch (Dh / Du) and
// only the last applies the stage update, so results are unchanged.
void launch_eval(mswm_cuda_ctx* c, const MaskPlan& p, const double* h, const double* u,
                 const Op cop[2], const Op eop[2], const PredArgs* pred = nullptr,
                 const Side* side = nullptr) {
  for (int r = 1; r < c->replication; ++r) {
    const Op so[2] = {mk_op(OP_STORE, c->Dh.p), mk_op(OP_STORE, c->Dh.p)};
    const Op se[2] = {mk_op(OP_STORE, c->Du.p), mk_op(OP_STORE, c->Du.p)};
    launch_eval_once(c, p, h, u, so, se, r == 1 ? pred : nullptr, side);
  }
  launch_eval_once(c, p, h, u, cop, eop, c->replication > 1 ? nullptr : pred, side);
}

// ---------------------------------------------------------------------------
// ledger (Stepper::tally, integrators.cpp:302-335)

void tally(mswm_cuda_ctx* c, unsigned mask, int stage) {
  const int64_t L = c->replication;  // counts scale with the replication (integrators.cpp:304)
  if (!c->have_regions) {
    if (mask & MSWM_CELLS_ALL) c->ledger_cell[0][stage] += L * c->nC;
    if (mask & MSWM_EDGES_ALL) c->ledger_edge[0][stage] += L * c->nE;
    return;
  }
  static const int cell_region[6] = {0, 0, 0, 1, 2, 3};
  static const int edge_region[5] = {0, 0, 1, 2, 3};
  for (int g = 0; g < 6; ++g)
    if (mask & (1u << g)) c->ledger_cell[cell_region[g]][stage] += L * c->gsize[g];
  for (int g = 0; g < 5; ++g)
    if (mask & (1u << (6 + g))) c->ledger_edge[edge_region[g]][stage] += L * c->gsize[6 + g];
}

constexpr unsigned kMaskCoarseOnly = MSWM_CELLS_COARSE | MSWM_EDGES_COARSE;
constexpr unsigned kMaskIfCoarse = MSWM_CELLS_IF1 | MSWM_CELLS_IF2 | MSWM_CELLS_COARSE |
                                   MSWM_EDGES_IF1 | MSWM_EDGES_IF2 | MSWM_EDGES_COARSE;
constexpr unsigned kMaskStep1 = kMaskIfCoarse | MSWM_CELLS_UF1 | MSWM_CELLS_UF2 | MSWM_EDGES_UFINE;
constexpr unsigned kMaskSub = MSWM_CELLS_FINE_PLAIN | MSWM_CELLS_UF1 | MSWM_CELLS_UF2 |
                              MSWM_CELLS_IF1 | MSWM_CELLS_IF2 | MSWM_EDGES_FINE_PLAIN |
                              MSWM_EDGES_UFINE | MSWM_EDGES_IF1 | MSWM_EDGES_IF2;

// lts_interp_coeffs (integrators.cpp:186-212)
void lts_coeffs(int order, int stage, int k, int M, double out[3]) {
  const double kd = k, Md = M;
  double x = 0.0, xt = 0.0;
  switch (stage) {
    case 1:
      x = kd / Md;
      xt = (order == 3) ? (kd * kd) / (Md * Md) : 0.0;
      break;
    case 2:
      x = (kd + 1.0) / Md;
      xt = (order == 3) ? (kd * (kd + 2.0)) / (Md * Md) : 0.0;
      break;
    default:
      x = (2.0 * kd + 1.0) / (2.0 * Md);
      xt = (2.0 * kd * kd + 2.0 * kd + 1.0) / (2.0 * Md * Md);
      break;
  }
  out[0] = 1.0 - x - xt;
  out[1] = x - xt;
  out[2] = 2.0 * xt;
}

// The I1 / I1 u I2 lists: groups 3-4 (cells) and 8-9 (edges) are
// contiguous in the group buffers.
struct IfLists {
  const int32_t *c, *e;
  int32_t nc, nc1, ne, ne1;
};
IfLists if_lists(mswm_cuda_ctx* c) {
  IfLists L;
  L.c = c->cell_groups.p + c->goff[3];
  L.nc1 = int32_t(c->gsize[3]);
  L.nc = int32_t(c->gsize[3] + c->gsize[4]);
  L.e = c->edge_groups.p + c->goff[8];
  L.ne1 = int32_t(c->gsize[8]);
  L.ne = int32_t(c->gsize[8] + c->gsize[9]);
  return L;
}

void launch_predict(mswm_cuda_ctx* c, int stage, int k, int M, double* hdst, double* udst,
                    int order = 3) {
  const IfLists L = if_lists(c);
  double w[3];
  lts_coeffs(order, stage, k, M, w);
  const int64_t n = int64_t(L.nc1) + L.ne1;
  if (n == 0) return;
  const bool o3 = order == 3;
  k_predict<<<nblk(n), kBlock, 0, c->ls>>>(L.c, L.nc1, L.e, L.ne1, w[0], w[1], w[2], c->S0h.p,
      c->S1h.p, o3 ? c->S2h.p : nullptr, hdst, c->S0u.p, c->S1u.p, o3 ? c->S2u.p : nullptr, udst);
  CK(cudaGetLastError());
  ++c->launches;
}

PredArgs make_pred(mswm_cuda_ctx* c, int stage, int k, int M, double* hdst, double* udst,
                   int order = 3) {
  const IfLists L = if_lists(c);
  double w[3];
  lts_coeffs(order, stage, k, M, w);
  PredArgs pa;
  pa.clist = L.c;
  pa.nc = L.nc1;
  pa.elist = L.e;
  pa.ne = L.ne1;
  pa.c0 = w[0];
  pa.c1 = w[1];
  pa.c2 = w[2];
  pa.hs0 = c->S0h.p;
  pa.hs1 = c->S1h.p;
  pa.hs2 = order == 3 ? c->S2h.p : nullptr;
  pa.us0 = c->S0u.p;
  pa.us1 = c->S1u.p;
  pa.us2 = order == 3 ? c->S2u.p : nullptr;
  pa.hdst = hdst;
  pa.udst = udst;
  return pa;
}

// ---------------------------------------------------------------------------
// Halo exchange (multi-rank).  Before every evaluation each rank refreshes
// the halo copies of the (h, u) stage arrays the evaluation reads -- the
// device form of ThreadedEvaluator's per-eval copy-in (rank_pool.cpp:133-135).
// Transports: NCCL point-to-point between processes (one GPU each), or, for
// an in-process group of rank contexts on one device, device-to-device
// copies.  Both are stream-ordered and capturable in the step graph.

using ArrSel = DArr<double> mswm_cuda_ctx::*;

// MSWM_HALO_DRYRUN=1: timing aid for one rank of a partition stepped alone
// on one GPU (scripts/rank_timing.py) -- exchanges pack and unpack but skip
// the transfer; the receive buffers keep the halo values of the uploaded
// state, so the (wrong) results stay physical.
bool halo_dry_run() {
  static const bool on = [] {
    const char* e = std::getenv("MSWM_HALO_DRYRUN");
    return e && e[0] == '1';
  }();
  return on;
}

Halo& halo_for(mswm_cuda_ctx* c, unsigned mask) {
  auto it = c->halo_mask.find(mask);
  return it == c->halo_mask.end() ? c->halo : it->second;
}

bool restricted(const std::vector<mswm_cuda_ctx*>& cs) {
  for (auto* c : cs)
    if (!c->halo_mask.empty()) return true;
  return false;
}

// `preds` (one per member, or null): the next stage's interface-1
// prediction, fused into the unpack launch (k_unpack_pred).
void exchange(std::vector<mswm_cuda_ctx*>& cs, ArrSel hs, ArrSel us, unsigned mask,
              bool second_comm = false, const std::vector<PredArgs>* preds = nullptr) {
  bool any = false;
  for (auto* c : cs) any |= c->halo.active();
  if (!any) {
    if (preds) throw Error(MSWM_E_USAGE, "fused prediction without a halo exchange");
    return;
  }
  if (cs[0]->transport == 1 && !(cs.size() == 1 && halo_dry_run())) {
    // peer stores: pack into the neighbours' buffers and signal; wait and
    // unpack.  Both launch on every rank for every exchange (the protocol's
    // neighbourhood barrier, kernels.cuh), also with nothing to move.
    const int ch = second_comm ? 1 : 0;
    for (auto* c : cs) {
      Halo& x = halo_for(c, mask);
      if (c->transport != 1 || !x.pslots.p) throw Error(MSWM_E_USAGE, "peer transport not enabled on every rank");
      k_push<<<unsigned(std::max<int64_t>(1, nblk(x.ns))), kBlock, 0, c->ls>>>(x.ns, x.scode.p,
          x.sslot.p, (c->*hs).p, (c->*us).p, x.pslots.p, int(x.peer.size()), ch * c->n_ranks,
          c->xchan.p + 2 * ch);
      CK(cudaGetLastError());
      ++c->launches;
    }
    for (size_t m = 0; m < cs.size(); ++m) {
      mswm_cuda_ctx* c = cs[m];
      Halo& x = halo_for(c, mask);
      PredArgs pa;
      std::memset(&pa, 0, sizeof(pa));
      if (preds) pa = (*preds)[m];
      const int64_t np = int64_t(pa.nc) + pa.ne;
      k_wait_unpack<<<unsigned(std::max<int64_t>(1, nblk(x.nr + np))), kBlock, 0, c->ls>>>(x.nr,
          x.rcode.p, x.prbuf, x.pstride, (c->*hs).p, (c->*us).p, pa,
          reinterpret_cast<const unsigned long long*>(c->arena.p) + ch * c->n_ranks, c->d_peers.p,
          int(x.peer.size()), c->xchan.p + 2 * ch, c->xerr.p, c->peer_budget_ns);
      CK(cudaGetLastError());
      ++c->launches;
    }
    return;
  }
  for (auto* c : cs) {
    Halo& x = halo_for(c, mask);
    if (x.ns > 0) {
      k_pack<<<nblk(x.ns), kBlock, 0, c->ls>>>(x.ns, x.scode.p, (c->*hs).p, (c->*us).p, x.sbuf.p);
      CK(cudaGetLastError());
      ++c->launches;
    }
  }
  if (cs.size() == 1 && halo_dry_run()) {
    // timing aid only (results are wrong): one rank of a partition stepped
    // alone on one GPU -- pack and unpack run, the transfer is skipped
  } else if (cs.size() == 1) {
    mswm_cuda_ctx* c = cs[0];
    Halo& x = halo_for(c, mask);
    if (!c->nccl_comm) throw Error(MSWM_E_USAGE, "halo set but no communicator (mswm_cuda_comm_init)");
    // the forked coarse step exchanges on its own stream: a communicator of
    // its own keeps the two streams' NCCL operations independent
    ncclComm_t comm = second_comm ? c->nccl_comm2 : c->nccl_comm;
    if (!comm) throw Error(MSWM_E_NCCL, "no second communicator for the concurrent coarse step");
    nccl_check(nccl().GroupStart());
    for (size_t j = 0; j < x.peer.size(); ++j) {
      if (x.scnt[j])
        nccl_check(nccl().Send(x.sbuf.p + x.soff[j], size_t(x.scnt[j]), ncclFloat64, x.peer[j],
                               comm, c->ls));
      if (x.rcnt[j])
        nccl_check(nccl().Recv(x.rbuf.p + x.roff[j], size_t(x.rcnt[j]), ncclFloat64, x.peer[j],
                               comm, c->ls));
    }
    nccl_check(nccl().GroupEnd());
  } else if (cs[0]->loop_comm) {
    // in-process group over a one-rank communicator: every halo copy is an
    // NCCL send to self matched, in issue order, by the receive after it --
    // the NCCL transport's calls, buffers and graph capture on one GPU
    ncclComm_t comm = second_comm ? cs[0]->loop_comm2 : cs[0]->loop_comm;
    nccl_check(nccl().GroupStart());
    for (auto* c : cs) {
      Halo& x = halo_for(c, mask);
      for (size_t j = 0; j < x.peer.size(); ++j) {
        if (!x.rcnt[j]) continue;
        mswm_cuda_ctx* src = cs[x.peer[j]];
        const Halo& y = halo_for(src, mask);
        size_t k = 0;
        while (k < y.peer.size() && y.peer[k] != c->rank) ++k;
        if (k == y.peer.size() || y.scnt[k] != x.rcnt[j])
          throw Error(MSWM_E_USAGE, "inconsistent halo plans between ranks " +
                                        std::to_string(c->rank) + " and " + std::to_string(x.peer[j]));
        nccl_check(nccl().Send(y.sbuf.p + y.soff[k], size_t(x.rcnt[j]), ncclFloat64, 0, comm, c->ls));
        nccl_check(nccl().Recv(x.rbuf.p + x.roff[j], size_t(x.rcnt[j]), ncclFloat64, 0, comm, c->ls));
      }
    }
    nccl_check(nccl().GroupEnd());
  } else {
    // in-process group: member index == rank
    for (auto* c : cs) {
      Halo& x = halo_for(c, mask);
      for (size_t j = 0; j < x.peer.size(); ++j) {
        if (!x.rcnt[j]) continue;
        mswm_cuda_ctx* src = cs[x.peer[j]];
        const Halo& y = halo_for(src, mask);
        size_t k = 0;
        while (k < y.peer.size() && y.peer[k] != c->rank) ++k;
        if (k == y.peer.size() || y.scnt[k] != x.rcnt[j])
          throw Error(MSWM_E_USAGE, "inconsistent halo plans between ranks " +
                                        std::to_string(c->rank) + " and " + std::to_string(x.peer[j]));
        CK(cudaMemcpyAsync(x.rbuf.p + x.roff[j], y.sbuf.p + y.soff[k], size_t(x.rcnt[j]) * 8,
                           cudaMemcpyDeviceToDevice, c->ls));
      }
    }
  }
  for (size_t m = 0; m < cs.size(); ++m) {
    mswm_cuda_ctx* c = cs[m];
    Halo& x = halo_for(c, mask);
    const PredArgs* pa = preds ? &(*preds)[m] : nullptr;
    const int64_t np = pa ? int64_t(pa->nc) + pa->ne : 0;
    if (np > 0) {
      k_unpack_pred<<<nblk(x.nr + np), kBlock, 0, c->ls>>>(x.nr, x.rcode.p, x.rbuf.p, (c->*hs).p,
          (c->*us).p, *pa);
      CK(cudaGetLastError());
      ++c->launches;
    } else if (x.nr > 0) {
      k_unpack<<<nblk(x.nr), kBlock, 0, c->ls>>>(x.nr, x.rcode.p, x.rbuf.p, (c->*hs).p, (c->*us).p);
      CK(cudaGetLastError());
      ++c->launches;
    }
  }
}

// An evaluation preceded by its halo exchange.  With ranks (and
// MSWM_OVERLAP unset or 1) the exchange runs on a side stream while the
// interior outputs -- those whose closure reads no halo value -- evaluate,
// and the boundary outputs follow once the halo has landed: the transfer
// hides behind the interior work.  Both parts are pure functions of their
// inputs, so the split changes no bits.  `eval(c, plan)` launches one
// member's evaluation with its fused stage update.
// The split costs a launch-latency floor for the boundary part (~10 us per
// evaluation, measured on the 8-way C4 partition, scripts/rank_timing.py),
// about what it hides of a small exchange: it pays on the large
// evaluations (steps 1 and 2, big_eval) and is used for the substeps only
// with MSWM_OVERLAP=2.
template <class F>
void exchange_eval(std::vector<mswm_cuda_ctx*>& cs, ArrSel hs, ArrSel us, unsigned mask,
                   bool big_eval, F&& eval, const std::vector<PredArgs>* preds = nullptr) {
  bool halos = false;
  for (auto* c : cs) halos |= c->halo.active();
  mswm_cuda_ctx* const c0 = cs[0];
  if (!halos || !c0->lx || (!big_eval && c0->overlap_level < 2)) {
    exchange(cs, hs, us, mask, false, preds);
    for (auto* c : cs) eval(c, plan_for(c, mask));
    return;
  }
  cudaStream_t main = c0->ls;
  CK(cudaEventRecord(c0->ev_x0, main));
  CK(cudaStreamWaitEvent(c0->lx, c0->ev_x0, 0));
  for (auto* c : cs) c->ls = c0->lx;
  exchange(cs, hs, us, mask, false, preds);
  CK(cudaEventRecord(c0->ev_x1, c0->lx));
  for (auto* c : cs) c->ls = main;
  for (auto* c : cs) eval(c, plan_part(c, mask, 1));
  CK(cudaStreamWaitEvent(main, c0->ev_x1, 0));
  for (auto* c : cs) eval(c, plan_part(c, mask, 2));
}

void prepare_overlap(mswm_cuda_ctx* c) {
  if (!c->halo.active() || c->lx) return;
  const char* e = std::getenv("MSWM_OVERLAP");
  if (e && e[0] == '0') return;
  c->overlap_level = (e && e[0] == '2') ? 2 : 1;
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&c->lx, cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&c->ev_x0, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_x1, cudaEventDisableTiming));
}

// One LTS3 coarse step (see the file header for the aliasing argument) for
// every rank context of the executor.
// The LTS3 coarse step (step 4) runs concurrently with the substeps when
// one context steps alone on the streamed path: it reads (h2, u2) only on
// coarse and interface-2 elements and h_old only on its own outputs, none of
// which the substeps write; the substeps read h_old on a thin band of
// coarse elements next to interface 2, which step 4 therefore writes to
// T1h / T1u (Op::alt) and k_copy_band moves into the state after the join.
// Separate intermediates (pv2, K2, FQ2) keep the two evaluations apart.
// MSWM_FORK=0 keeps the sequential order.  Bitwise either way (evaluations
// are pure functions of their inputs).
void prepare_fork(mswm_cuda_ctx* c) {
  if (c->fork_state != 0) return;
  c->fork_state = -1;
  const char* fe = std::getenv("MSWM_FORK");
  if ((fe && fe[0] == '0') || !c->have_regions) return;
  if (c->halo.active()) {
    // ranks: the coarse step's exchange runs on the fork stream concurrently
    // with the substeps' exchanges, so both need buffers of their own
    // (per-mask restricted halos) and, between processes, the second
    // communicator
    if (!c->halo_mask.count(kMaskSub) || !c->halo_mask.count(kMaskCoarseOnly)) return;
    if (c->nccl_comm && !c->nccl_comm2) return;
  }
  MaskPlan& ps = plan_for(c, kMaskSub);
  MaskPlan& pc = plan_for(c, kMaskCoarseOnly);
  if (const char* fc = std::getenv("MSWM_FORK_CTAS")) {  // "n" or "a,b,c"
    int v[3];
    const int k = std::sscanf(fc, "%d,%d,%d", &v[0], &v[1], &v[2]);
    for (int j = 0; j < 3; ++j) c->fork_ctas[j] = std::max(0, k == 3 ? v[j] : v[0]);
  }
  cudaStream_t s = c->stream;
  DArr<uint8_t> cr, er;
  cr.alloc(c->nC);
  er.alloc(c->nE);
  cr.zero(s);
  er.zero(s);
  const int64_t n = int64_t(ps.nv) + ps.nk + ps.nf + ps.ne;
  if (n > 0) {
    k_mark_reads<<<nblk(n), kBlock, 0, s>>>(c->dev(), ps.vclos.p, ps.nv, ps.kclos.p, ps.nk,
                                            ps.fclos.p, ps.nf, ps.edges, ps.ne, cr.p, er.p);
    CK(cudaGetLastError());
  }
  std::vector<uint8_t> hc(c->nC), he(c->nE), kc(c->nC), ke(c->nE);
  CK(cudaMemcpyAsync(hc.data(), cr.p, size_t(c->nC), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(he.data(), er.p, size_t(c->nE), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(kc.data(), c->ckey.p, size_t(c->nC), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ke.data(), c->ekey.p, size_t(c->nE), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // ranks: the substeps' exchanges also read h_old / u_old (the state) on
  // the owned elements they send
  if (c->halo.active()) {
    const Halo& xs = halo_for(c, kMaskSub);
    for (const int32_t code : xs.h_scode) {
      if (code >= 0) hc[code] = 1;
      else he[~code] = 1;
    }
  }
  std::vector<int32_t> bc, be;
  std::vector<uint32_t> cb((size_t(c->nC) + 31) / 32, 0u), eb((size_t(c->nE) + 31) / 32, 0u);
  for (int32_t i = 0; i < c->nC; ++i)
    if (hc[i] && kc[i] == 5) {  // read by a substep, written by step 4 (coarse)
      bc.push_back(i);
      cb[i >> 5] |= 1u << (i & 31);
    }
  for (int32_t e = 0; e < c->nE; ++e)
    if (he[e] && ke[e] == 4) {
      be.push_back(e);
      eb[e >> 5] |= 1u << (e & 31);
    }
  c->band_cbits.upload(cb, s);
  c->band_ebits.upload(eb, s);
  c->band_cells.upload(bc, s);
  c->band_edges.upload(be, s);
  c->n_band_c = int32_t(bc.size());
  c->n_band_e = int32_t(be.size());
  c->pv2.alloc(c->nV);
  c->pv2.zero(s);
  c->K2.alloc(c->nC);
  c->K2.zero(s);
  c->FQ2.alloc(c->nE);
  c->FQ2.zero(s);
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  if (!c->ls2) CK(cudaStreamCreateWithPriority(&c->ls2, cudaStreamNonBlocking, lo));
  if (!c->lsh) CK(cudaStreamCreateWithPriority(&c->lsh, cudaStreamNonBlocking, hi));
  if (!c->ev_fork) CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  if (!c->ev_join) CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  if (!c->ev_join_h) CK(cudaEventCreateWithFlags(&c->ev_join_h, cudaEventDisableTiming));
  CK(cudaStreamSynchronize(s));
  c->fork_state = 1;
}

void enqueue_lts3(std::vector<mswm_cuda_ctx*>& cs, double dt, int M) {
  const double delta = dt / M;
  bool fuse_pred = true;
  for (auto* c : cs) fuse_pred &= !c->halo.active();
  const double third = 1.0 / 3.0, two3 = 2.0 / 3.0;
  using C = mswm_cuda_ctx;
  // Step 1 (:483-487): h1 = h_old + dt*dh on UF1 u UF2 u I1 u I2 u C.
  exchange_eval(cs, &C::H, &C::U, kMaskStep1, true, [&](mswm_cuda_ctx* c, const MaskPlan& p) {
    double *H = c->H.p, *U = c->U.p, *H1 = c->H1.p, *U1 = c->U1.p;
    Op co[2] = {mk_op(OP_EULER, H1, H, dt), mk_op(OP_EULER, H1, H, dt)};
    Op eo[2] = {mk_op(OP_EULER, U1, U, dt), mk_op(OP_EULER, U1, U, dt)};
    launch_eval(c, p, H, U, co, eo);
  });
  // Step 2 (:491-500): h2 = 0.75 h_old + 0.25 h1 + (0.25 dt) dh on I u C.
  exchange_eval(cs, &C::H1, &C::U1, kMaskIfCoarse, true, [&](mswm_cuda_ctx* c, const MaskPlan& p) {
    double *H = c->H.p, *U = c->U.p, *H1 = c->H1.p, *U1 = c->U1.p, *H2 = c->H2.p, *U2 = c->U2.p;
    const double cr = 0.25 * dt;
    Op co[2] = {mk_op(OP_WCOMB, H2, H, 0.75, H1, 0.25, cr), mk_op(OP_WCOMB, H2, H, 0.75, H1, 0.25, cr)};
    Op eo[2] = {mk_op(OP_WCOMB, U2, U, 0.75, U1, 0.25, cr), mk_op(OP_WCOMB, U2, U, 0.75, U1, 0.25, cr)};
    launch_eval(c, p, H1, U1, co, eo);
  });
  // Step 4 forked onto the second stream (prepare_fork); with ranks, its
  // (restricted) halo exchange of h2/u2 rides on that stream too.  The
  // streams and events of member 0 serve the whole group.
  bool fork = true;
  for (auto* c : cs) fork &= c->fork_state == 1;
  mswm_cuda_ctx* const c0 = cs[0];
  cudaStream_t capture_stream = c0->ls;
  if (fork) {
    CK(cudaEventRecord(c0->ev_fork, capture_stream));
    CK(cudaStreamWaitEvent(c0->ls2, c0->ev_fork, 0));
    for (auto* c : cs) c->ls = c0->ls2;
    if (restricted(cs)) exchange(cs, &C::H2, &C::U2, kMaskCoarseOnly, true);
    for (auto* c : cs) {
      const double cr = two3 * dt;
      double *H = c->H.p, *U = c->U.p, *H2 = c->H2.p, *U2 = c->U2.p;
      Op co = mk_op(OP_WCOMB, H, H, third, H2, two3, cr);
      Op eo = mk_op(OP_WCOMB, U, U, third, U2, two3, cr);
      co.alt = c->T1h.p;
      co.altbits = c->band_cbits.p;
      eo.alt = c->T1u.p;
      eo.altbits = c->band_ebits.p;
      Op cos[2] = {co, co}, eos[2] = {eo, eo};
      const Side side{c0->ls2, c->pv2.p, c->K2.p, c->FQ2.p,
                      {c->fork_ctas[0], c->fork_ctas[1], c->fork_ctas[2]}};
      launch_eval(c, plan_for(c, kMaskCoarseOnly), H2, U2, cos, eos, nullptr, &side);
    }
    CK(cudaEventRecord(c0->ev_join, c0->ls2));
    // the substeps on the high-priority stream: their CTAs take SM slots
    // ahead of the coarse step's as slots free up
    CK(cudaStreamWaitEvent(c0->lsh, c0->ev_fork, 0));
    for (auto* c : cs) c->ls = c0->lsh;
  }
  // Substep prologue: save I1 u I2 old values, I1 stage values, predict
  // stage 1 of substep 0 into the state (ha == state).
  for (auto* c : cs) {
    const IfLists L = if_lists(c);
    double w[3];
    lts_coeffs(3, 1, 0, M, w);
    const int64_t n = int64_t(L.nc) + L.ne;
    if (n > 0) {
      k_save_predict<<<nblk(n), kBlock, 0, c->ls>>>(L.c, L.nc, L.nc1, L.e, L.ne, L.ne1, w[0], w[1],
          w[2], c->H.p, c->H1.p, c->H2.p, c->S0h.p, c->S1h.p, c->S2h.p, c->U.p, c->U1.p, c->U2.p,
          c->S0u.p, c->S1u.p, c->S2u.p);
      CK(cudaGetLastError());
      ++c->launches;
    }
  }
  for (int k = 0; k < M; ++k) {
    const int first = k == 0;
    // stage 1: fine hb = ha + delta*d; interfaces acc1 += d   (:521-531)
    // predictions ride in the evaluation's launch unless a halo exchange
    // has to propagate them first (multi-rank)
    // ranks: each stage's exchange carries the next stage's prediction in its
    // unpack launch (k_unpack_pred; substep 0's stage 1 is the prologue's)
    std::vector<PredArgs> pred2, pred3, pred1n;
    if (!fuse_pred)
      for (auto* c : cs) {
        pred2.push_back(make_pred(c, 2, k, M, c->H1.p, c->U1.p));
        pred3.push_back(make_pred(c, 3, k, M, c->H2.p, c->U2.p));
        if (k + 1 < M) pred1n.push_back(make_pred(c, 1, k + 1, M, c->H.p, c->U.p));
      }
    exchange_eval(cs, &C::H, &C::U, kMaskSub, false, [&](mswm_cuda_ctx* c, const MaskPlan& p) {
      const PredArgs pa = make_pred(c, 1, k, M, c->H.p, c->U.p);
      Op co[2] = {mk_op(OP_EULER, c->H1.p, c->H.p, delta),
                  mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A1h.p, first)};
      Op eo[2] = {mk_op(OP_EULER, c->U1.p, c->U.p, delta),
                  mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A1u.p, first)};
      launch_eval(c, p, c->H.p, c->U.p, co, eo, (k > 0 && fuse_pred) ? &pa : nullptr);
    }, fuse_pred ? nullptr : &pred2);
    // stage 2: fine hc = 0.75 ha + 0.25 hb + (0.25 delta) d; acc2 += d   (:532-541)
    exchange_eval(cs, &C::H1, &C::U1, kMaskSub, false, [&](mswm_cuda_ctx* c, const MaskPlan& p) {
      const PredArgs pa = make_pred(c, 2, k, M, c->H1.p, c->U1.p);
      const double cr = 0.25 * delta;
      Op co[2] = {mk_op(OP_WCOMB, c->H2.p, c->H.p, 0.75, c->H1.p, 0.25, cr),
                  mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A2h.p, first)};
      Op eo[2] = {mk_op(OP_WCOMB, c->U2.p, c->U.p, 0.75, c->U1.p, 0.25, cr),
                  mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A2u.p, first)};
      launch_eval(c, p, c->H1.p, c->U1.p, co, eo, fuse_pred ? &pa : nullptr);
    }, fuse_pred ? nullptr : &pred3);
    // stage 3: fine ha = 1/3 ha + 2/3 hc + (2/3 delta) d; acc3 += d, and on
    // the last substep the interface correction (:542-553, :231-274).
    exchange_eval(cs, &C::H2, &C::U2, kMaskSub, false, [&](mswm_cuda_ctx* c, const MaskPlan& p) {
      const PredArgs pa = make_pred(c, 3, k, M, c->H2.p, c->U2.p);
      const double cr = two3 * delta;
      Op co[2], eo[2];
      co[0] = mk_op(OP_WCOMB, c->H.p, c->H.p, third, c->H2.p, two3, cr);
      eo[0] = mk_op(OP_WCOMB, c->U.p, c->U.p, third, c->U2.p, two3, cr);
      if (k < M - 1) {
        co[1] = mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A3h.p, first);
        eo[1] = mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A3u.p, first);
      } else {
        co[1] = mk_op(OP_ACC_CORR, c->H.p, c->S0h.p, delta, nullptr, 1.0 / 6.0, two3, c->A3h.p,
                      first, c->A1h.p, c->A2h.p);
        eo[1] = mk_op(OP_ACC_CORR, c->U.p, c->S0u.p, delta, nullptr, 1.0 / 6.0, two3, c->A3u.p,
                      first, c->A1u.p, c->A2u.p);
      }
      launch_eval(c, p, c->H2.p, c->U2.p, co, eo, fuse_pred ? &pa : nullptr);
    }, (fuse_pred || k + 1 == M) ? nullptr : &pred1n);
  }
  // Step 4 (:557-563): coarse h = 1/3 h_old + 2/3 h2 + (2/3 dt) dh, in place.
  // With full halos the H2/U2 copies are current (the last exchange
  // refreshed them; only fine/I1 entries, never read here, changed since);
  // restricted halos refreshed only the substep's read set.
  if (fork) {
    CK(cudaEventRecord(c0->ev_join_h, c0->lsh));
    for (auto* c : cs) c->ls = capture_stream;
    CK(cudaStreamWaitEvent(capture_stream, c0->ev_join_h, 0));
    CK(cudaStreamWaitEvent(capture_stream, c0->ev_join, 0));
    for (auto* c : cs) {
      const int64_t nb = int64_t(c->n_band_c) + c->n_band_e;
      if (nb > 0) {
        k_copy_band<<<nblk(nb), kBlock, 0, c->ls>>>(c->band_cells.p, c->n_band_c, c->T1h.p, c->H.p,
            c->band_edges.p, c->n_band_e, c->T1u.p, c->U.p);
        CK(cudaGetLastError());
        ++c->launches;
      }
    }
    return;
  }
  if (restricted(cs)) exchange(cs, &C::H2, &C::U2, kMaskCoarseOnly);
  for (auto* c : cs) {
    const double cr = two3 * dt;
    double *H = c->H.p, *U = c->U.p, *H2 = c->H2.p, *U2 = c->U2.p;
    Op co[2] = {mk_op(OP_WCOMB, H, H, third, H2, two3, cr), mk_op(OP_WCOMB, H, H, third, H2, two3, cr)};
    Op eo[2] = {mk_op(OP_WCOMB, U, U, third, U2, two3, cr), mk_op(OP_WCOMB, U, U, third, U2, two3, cr)};
    launch_eval(c, plan_for(c, kMaskCoarseOnly), H2, U2, co, eo);
  }
}

// One LTS2 coarse step (Stepper::lts_step(2, ...), integrators.cpp:412-575
// with order 2) on the LTS3 aliasing: ha = state, hb = h1.  Step 2 -- the
// coarse finalisation h = 0.5 h_old + 0.5 h1 + (0.5 dt) dh -- runs after the
// substeps, in place: it reads h1 only on interface-2 / coarse elements,
// which the substeps never write, and the substeps read the state's coarse
// entries as h_old, which it overwrites.  Evaluations are pure functions of
// their inputs, so the reordering changes no bits.
void enqueue_lts2(std::vector<mswm_cuda_ctx*>& cs, double dt, int M) {
  const double delta = dt / M;
  bool fuse_pred = true;
  for (auto* c : cs) fuse_pred &= !c->halo.active();
  using C = mswm_cuda_ctx;
  // Step 1 (:483-487): h1 = h_old + dt*dh on I1 u I2 u C.
  exchange(cs, &C::H, &C::U, kMaskIfCoarse);
  for (auto* c : cs) {
    double *H = c->H.p, *U = c->U.p, *H1 = c->H1.p, *U1 = c->U1.p;
    Op co[2] = {mk_op(OP_EULER, H1, H, dt), mk_op(OP_EULER, H1, H, dt)};
    Op eo[2] = {mk_op(OP_EULER, U1, U, dt), mk_op(OP_EULER, U1, U, dt)};
    launch_eval(c, plan_for(c, kMaskIfCoarse), H, U, co, eo);
  }
  // Substep prologue: save I1 u I2 old values and I1 stage-1 values, predict
  // stage 1 of substep 0 (two-term) into the state.
  for (auto* c : cs) {
    const IfLists L = if_lists(c);
    double w[3];
    lts_coeffs(2, 1, 0, M, w);
    const int64_t n = int64_t(L.nc) + L.ne;
    if (n > 0) {
      k_save_predict<<<nblk(n), kBlock, 0, c->ls>>>(L.c, L.nc, L.nc1, L.e, L.ne, L.ne1, w[0], w[1],
          w[2], c->H.p, c->H1.p, nullptr, c->S0h.p, c->S1h.p, nullptr, c->U.p, c->U1.p, nullptr,
          c->S0u.p, c->S1u.p, nullptr);
      CK(cudaGetLastError());
      ++c->launches;
    }
  }
  for (int k = 0; k < M; ++k) {
    const int first = k == 0;
    // stage 1: fine hb = ha + delta*d; interfaces acc1 += d   (:521-531)
    if (k > 0 && !fuse_pred)
      for (auto* c : cs) launch_predict(c, 1, k, M, c->H.p, c->U.p, 2);
    exchange(cs, &C::H, &C::U, kMaskSub);
    for (auto* c : cs) {
      const PredArgs pa = make_pred(c, 1, k, M, c->H.p, c->U.p, 2);
      Op co[2] = {mk_op(OP_EULER, c->H1.p, c->H.p, delta),
                  mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A1h.p, first)};
      Op eo[2] = {mk_op(OP_EULER, c->U1.p, c->U.p, delta),
                  mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A1u.p, first)};
      launch_eval(c, plan_for(c, kMaskSub), c->H.p, c->U.p, co, eo,
                  (k > 0 && fuse_pred) ? &pa : nullptr);
    }
    // stage 2: fine ha = 0.5 ha + 0.5 hb + (0.5 delta) d; acc2 += d, and on
    // the last substep the interface correction (:532-541 order 2, :231-274)
    if (!fuse_pred)
      for (auto* c : cs) launch_predict(c, 2, k, M, c->H1.p, c->U1.p, 2);
    exchange(cs, &C::H1, &C::U1, kMaskSub);
    for (auto* c : cs) {
      const PredArgs pa = make_pred(c, 2, k, M, c->H1.p, c->U1.p, 2);
      const double cr = 0.5 * delta;
      Op co[2], eo[2];
      co[0] = mk_op(OP_WCOMB, c->H.p, c->H.p, 0.5, c->H1.p, 0.5, cr);
      eo[0] = mk_op(OP_WCOMB, c->U.p, c->U.p, 0.5, c->U1.p, 0.5, cr);
      if (k < M - 1) {
        co[1] = mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A2h.p, first);
        eo[1] = mk_op(OP_ACC, nullptr, nullptr, 0, nullptr, 0, 0, c->A2u.p, first);
      } else {
        co[1] = mk_op(OP_ACC_CORR2, c->H.p, c->S0h.p, delta, nullptr, 0.5, 0, c->A2h.p, first,
                      c->A1h.p);
        eo[1] = mk_op(OP_ACC_CORR2, c->U.p, c->S0u.p, delta, nullptr, 0.5, 0, c->A2u.p, first,
                      c->A1u.p);
      }
      launch_eval(c, plan_for(c, kMaskSub), c->H1.p, c->U1.p, co, eo, fuse_pred ? &pa : nullptr);
    }
  }
  // Step 2 (:491-497): coarse h = 0.5 h_old + 0.5 h1 + (0.5 dt) dh, in place.
  // With full halos the H1/U1 copies are current (the last exchange
  // refreshed them and only the state changed since); restricted halos
  // refreshed only the substep's read set.
  if (restricted(cs)) exchange(cs, &C::H1, &C::U1, kMaskCoarseOnly);
  for (auto* c : cs) {
    const double cr = 0.5 * dt;
    double *H = c->H.p, *U = c->U.p, *H1 = c->H1.p, *U1 = c->U1.p;
    Op co[2] = {mk_op(OP_WCOMB, H, H, 0.5, H1, 0.5, cr), mk_op(OP_WCOMB, H, H, 0.5, H1, 0.5, cr)};
    Op eo[2] = {mk_op(OP_WCOMB, U, U, 0.5, U1, 0.5, cr), mk_op(OP_WCOMB, U, U, 0.5, U1, 0.5, cr)};
    launch_eval(c, plan_for(c, kMaskCoarseOnly), H1, U1, co, eo);
  }
}

void tally_lts2(mswm_cuda_ctx* c, int M) {
  tally(c, kMaskIfCoarse, 0);
  tally(c, kMaskCoarseOnly, 1);
  for (int k = 0; k < M; ++k) {
    tally(c, kMaskSub, 0);
    tally(c, kMaskSub, 1);
  }
}

void tally_lts3(mswm_cuda_ctx* c, int M) {
  tally(c, kMaskStep1, 0);
  tally(c, kMaskIfCoarse, 1);
  for (int k = 0; k < M; ++k) {
    tally(c, kMaskSub, 0);
    tally(c, kMaskSub, 1);
    tally(c, kMaskSub, 2);
  }
  tally(c, kMaskCoarseOnly, 2);
}

// RK4 (integrators.cpp:370-410) with ping-pong stage buffers.
void enqueue_rk4(std::vector<mswm_cuda_ctx*>& cs, double dt) {
  using C = mswm_cuda_ctx;
  const double half = 0.5 * dt, sixth = dt / 6.0;
  auto both = [](Op o) { return std::array<Op, 2>{o, o}; };
  struct St {
    ArrSel rh, ru, wh, wu;
    int kind;
    double c0;
  };
  const St stages[4] = {{&C::H, &C::U, &C::T1h, &C::T1u, OP_RK4_FIRST, half},
                        {&C::T1h, &C::T1u, &C::T2h, &C::T2u, OP_RK4_MID, half},
                        {&C::T2h, &C::T2u, &C::T1h, &C::T1u, OP_RK4_MID, dt},
                        {&C::T1h, &C::T1u, &C::H, &C::U, OP_RK4_LAST, sixth}};
  // every stage reads one buffer pair and writes another (or, last, the
  // state at its own outputs only): the exchange of the read pair can
  // overlap the interior evaluation (exchange_eval)
  for (const St& st : stages) {
    exchange_eval(cs, st.rh, st.ru, MSWM_MASK_ALL, true, [&](mswm_cuda_ctx* c, const MaskPlan& p) {
      auto co = both(mk_op(st.kind, (c->*st.wh).p, c->H.p, st.c0, nullptr, 0, 0, c->A1h.p));
      auto eo = both(mk_op(st.kind, (c->*st.wu).p, c->U.p, st.c0, nullptr, 0, 0, c->A1u.p));
      launch_eval(c, p, (c->*st.rh).p, (c->*st.ru).p, co.data(), eo.data());
    });
  }
}

// SSPRK2/3 (integrators.cpp:337-368).
void enqueue_ssprk(std::vector<mswm_cuda_ctx*>& cs, int order, double dt) {
  using C = mswm_cuda_ctx;
  auto both = [](Op o) { return std::array<Op, 2>{o, o}; };
  exchange(cs, &C::H, &C::U, MSWM_MASK_ALL);
  for (auto* c : cs) {
    auto co = both(mk_op(OP_EULER, c->T1h.p, c->H.p, dt));
    auto eo = both(mk_op(OP_EULER, c->T1u.p, c->U.p, dt));
    launch_eval(c, plan_for(c, MSWM_MASK_ALL), c->H.p, c->U.p, co.data(), eo.data());
  }
  exchange(cs, &C::T1h, &C::T1u, MSWM_MASK_ALL);
  if (order == 2) {
    for (auto* c : cs) {
      const double cr = 0.5 * dt;
      auto co = both(mk_op(OP_WCOMB, c->H.p, c->H.p, 0.5, c->T1h.p, 0.5, cr));
      auto eo = both(mk_op(OP_WCOMB, c->U.p, c->U.p, 0.5, c->T1u.p, 0.5, cr));
      launch_eval(c, plan_for(c, MSWM_MASK_ALL), c->T1h.p, c->T1u.p, co.data(), eo.data());
    }
    return;
  }
  for (auto* c : cs) {
    const double cr = 0.25 * dt;
    auto co = both(mk_op(OP_WCOMB, c->T2h.p, c->H.p, 0.75, c->T1h.p, 0.25, cr));
    auto eo = both(mk_op(OP_WCOMB, c->T2u.p, c->U.p, 0.75, c->T1u.p, 0.25, cr));
    launch_eval(c, plan_for(c, MSWM_MASK_ALL), c->T1h.p, c->T1u.p, co.data(), eo.data());
  }
  exchange(cs, &C::T2h, &C::T2u, MSWM_MASK_ALL);
  for (auto* c : cs) {
    const double cr = (2.0 / 3.0) * dt;
    auto co = both(mk_op(OP_WCOMB, c->H.p, c->H.p, 1.0 / 3.0, c->T2h.p, 2.0 / 3.0, cr));
    auto eo = both(mk_op(OP_WCOMB, c->U.p, c->U.p, 1.0 / 3.0, c->T2u.p, 2.0 / 3.0, cr));
    launch_eval(c, plan_for(c, MSWM_MASK_ALL), c->T2h.p, c->T2u.p, co.data(), eo.data());
  }
}

void enqueue_step(std::vector<mswm_cuda_ctx*>& cs, int scheme, double dt, int M) {
  for (auto* c : cs) {
    k_step_counter<<<1, 1, 0, c->ls>>>(c->step_ctr.p);
    CK(cudaGetLastError());
    ++c->launches;
  }
  switch (scheme) {
    case MSWM_LTS3: enqueue_lts3(cs, dt, M); break;
    case MSWM_LTS2: enqueue_lts2(cs, dt, M); break;
    case MSWM_RK4: enqueue_rk4(cs, dt); break;
    case MSWM_SSPRK3: enqueue_ssprk(cs, 3, dt); break;
    case MSWM_SSPRK2: enqueue_ssprk(cs, 2, dt); break;
    default: throw Error(MSWM_E_CONFIG, "scheme not supported on the device path");
  }
}

void tally_step(mswm_cuda_ctx* c, int scheme, int M) {
  switch (scheme) {
    case MSWM_LTS3: tally_lts3(c, M); break;
    case MSWM_LTS2: tally_lts2(c, M); break;
    case MSWM_RK4:
      for (int s = 0; s < 4; ++s) tally(c, MSWM_MASK_ALL, s);
      break;
    case MSWM_SSPRK3:
      for (int s = 0; s < 3; ++s) tally(c, MSWM_MASK_ALL, s);
      break;
    case MSWM_SSPRK2:
      for (int s = 0; s < 2; ++s) tally(c, MSWM_MASK_ALL, s);
      break;
  }
  ++c->ledger_steps;
}

void check_step_args(mswm_cuda_ctx* c, int scheme, double dt, int M, int64_t n_steps) {
  if (!(dt > 0.0)) throw Error(MSWM_E_CONFIG, "time step must be positive");
  if (n_steps < 0) throw Error(MSWM_E_USAGE, "negative step count");
  if (scheme == MSWM_LTS3 || scheme == MSWM_LTS2) {
    if (M < 1) throw Error(MSWM_E_CONFIG, "substep count must be >= 1");
    if (!c->have_regions) throw Error(MSWM_E_CONFIG, "local time stepping requires a region map");
  } else if (scheme != MSWM_RK4 && scheme != MSWM_SSPRK3 && scheme != MSWM_SSPRK2) {
    throw Error(MSWM_E_CONFIG, "unknown scheme");
  }
  if (!c->have_fields) throw Error(MSWM_E_USAGE, "set_fields must be called before stepping");
}

// Capture one step of every context in `cs` on `stream` into a graph.
// One eager one-double send / receive with every neighbour on each
// communicator, so NCCL sets its point-to-point connections up (allocations,
// handshakes) before the exchanges are captured into the step graph.
void warm_nccl(mswm_cuda_ctx* c) {
  if (c->nccl_warm || !c->nccl_comm || !c->halo.active()) return;
  const size_t np = c->halo.peer.size();
  DArr<double> buf;
  buf.alloc(2 * np);
  buf.zero(c->stream);
  for (ncclComm_t comm : {c->nccl_comm, c->nccl_comm2}) {
    if (!comm) continue;
    nccl_check(nccl().GroupStart());
    for (size_t j = 0; j < np; ++j) {
      nccl_check(nccl().Send(buf.p + j, 1, ncclFloat64, c->halo.peer[j], comm, c->stream));
      nccl_check(nccl().Recv(buf.p + np + j, 1, ncclFloat64, c->halo.peer[j], comm, c->stream));
    }
    nccl_check(nccl().GroupEnd());
  }
  CK(cudaStreamSynchronize(c->stream));
  c->nccl_warm = true;
}

mswm_cuda_ctx::Graph capture_step(std::vector<mswm_cuda_ctx*>& cs, cudaStream_t stream, int scheme,
                                  double dt, int M, bool profile) {
  if (cs.size() == 1 && cs[0]->transport == 0 && !halo_dry_run()) warm_nccl(cs[0]);
  // Build every plan outside the capture (plan construction synchronises).
  for (auto* c : cs) {
    if (scheme == MSWM_LTS3 || scheme == MSWM_LTS2) {
      if (scheme == MSWM_LTS3) plan_for(c, kMaskStep1);
      plan_for(c, kMaskIfCoarse);
      plan_for(c, kMaskSub);
      plan_for(c, kMaskCoarseOnly);
      if (scheme == MSWM_LTS3) prepare_fork(c);
      prepare_overlap(c);
      if (c->halo.active() && scheme == MSWM_LTS3) {
        // part plans are built outside the capture too
        for (unsigned m : {kMaskStep1, kMaskIfCoarse, kMaskSub}) {
          plan_part(c, m, 1);
          plan_part(c, m, 2);
        }
      }
    } else {
      plan_for(c, MSWM_MASK_ALL);
      prepare_overlap(c);
      if (c->halo.active() && scheme == MSWM_RK4) {
        plan_part(c, MSWM_MASK_ALL, 1);
        plan_part(c, MSWM_MASK_ALL, 2);
      }
    }
  }
  mswm_cuda_ctx::Graph gr;
  cudaGraph_t g = nullptr;
  for (auto* c : cs) {
    c->ls = stream;
    c->launches = 0;
  }
  cs[0]->capture_records = profile ? &gr.records : nullptr;
  debug_mem("capture_step: plans built");
  CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_step(cs, scheme, dt, M);
  } catch (...) {
    for (auto* c : cs) {
      c->ls = c->stream;
      c->capture_records = nullptr;
    }
    cudaStreamEndCapture(stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  for (auto* c : cs) {
    gr.kernels += c->launches;
    c->ls = c->stream;
    c->capture_records = nullptr;
  }
  CK(cudaStreamEndCapture(stream, &g));
  debug_mem("capture_step: captured");
  // per-node priorities (the concurrent coarse step / substeps, enqueue_lts3)
  cudaError_t e = cudaGraphInstantiate(&gr.exec, g, cudaGraphInstantiateFlagUseNodePriority);
  debug_mem("capture_step: instantiated");
  cudaGraphDestroy(g);
  if (e != cudaSuccess) throw Error(MSWM_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  return gr;
}

cudaGraphExec_t graph_for(mswm_cuda_ctx* c, int scheme, double dt, int M) {
  const auto key = std::make_tuple(scheme, dt, (scheme == MSWM_LTS3 || scheme == MSWM_LTS2) ? M : 0, int(c->profiling));
  auto it = c->graphs.find(key);
  if (it != c->graphs.end()) {
    c->last_records = &it->second.records;
    c->last_kernels_per_step = it->second.kernels;
    return it->second.exec;
  }
  std::vector<mswm_cuda_ctx*> cs{c};
  auto& slot = c->graphs[key];
  slot = capture_step(cs, c->stream, scheme, dt, M, c->profiling);
  c->last_records = &slot.records;
  c->last_kernels_per_step = slot.kernels;
  return slot.exec;
}

// ---------------------------------------------------------------------------
// regions on device (regions.cpp:14-171)

int set_regions_impl(mswm_cuda_ctx* c, const uint8_t* fine_mask, int width, uint8_t* cell_label,
                     uint8_t* cell_sub, uint8_t* edge_label, int64_t* group_size, int* warnings) {
  if (width < 1) throw Error(MSWM_E_CONFIG, "interface width must be >= 1");
  if (!fine_mask) throw Error(MSWM_E_USAGE, "fine mask is null");
  cudaStream_t s = c->stream;
  const int32_t nC = c->nC, nE = c->nE;
  // dist = 0 for fine cells, -1 elsewhere (internal order)
  std::vector<int32_t> dist0(nC);
  int64_t n_fine = 0;
  for (int32_t ni = 0; ni < nC; ++ni) {
    const bool fine = fine_mask[c->c_new2old[ni]] != 0;
    dist0[ni] = fine ? 0 : -1;
    n_fine += fine;
  }
  if (n_fine == 0) throw Error(MSWM_E_CONFIG, "fine predicate selects no cells");
  if (n_fine == nC)
    throw Error(MSWM_E_CONFIG, "fine predicate selects every cell; no room for interface layers");
  invalidate(c);
  c->have_regions = false;
  DArr<int32_t> dist, counters;
  dist.upload(dist0, s);
  counters.alloc(size_t(2 * width) + 1);
  counters.zero(s);
  const DevMesh M = c->dev();
  for (int level = 1; level <= 2 * width; ++level) {
    k_bfs_layer<<<nblk(nC), kBlock, 0, s>>>(M, c->c_nbr.p, dist.p, level, counters.p + level);
    CK(cudaGetLastError());
  }
  std::vector<int32_t> cnt(size_t(2 * width) + 1);
  CK(cudaMemcpyAsync(cnt.data(), counters.p, cnt.size() * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int64_t n_layers = 0;
  for (int layer = 1; layer <= 2 * width; ++layer) {
    if (cnt[layer] == 0)
      throw Error(MSWM_E_CONFIG, "interface layer " + std::to_string(layer) +
                                     " is empty; the non-fine region is too small for width " +
                                     std::to_string(width));
    n_layers += cnt[layer];
  }
  if (n_fine + n_layers == nC)
    throw Error(MSWM_E_CONFIG, "interface layers exhaust the non-fine cells; no coarse region left");
  c->cell_label.alloc(nC);
  c->cell_sub.alloc(nC);
  c->edge_label.alloc(nE);
  k_cell_labels<<<nblk(nC), kBlock, 0, s>>>(nC, dist.p, width, c->cell_label.p, c->cell_sub.p);
  k_underline<<<nblk(nC), kBlock, 0, s>>>(M, c->c_nbr.p, c->cell_label.p, c->cell_sub.p, 1);
  k_underline<<<nblk(nC), kBlock, 0, s>>>(M, c->c_nbr.p, c->cell_label.p, c->cell_sub.p, 2);
  DArr<uint8_t>& ckey = c->ckey;
  DArr<uint8_t>& ekey = c->ekey;
  ckey.alloc(nC);
  ekey.alloc(nE);
  k_edge_labels_and_keys<<<nblk(std::max(nC, nE)), kBlock, 0, s>>>(M, c->cell_label.p, c->cell_sub.p,
                                                                   c->edge_label.p, ckey.p, ekey.p);
  CK(cudaGetLastError());
  // Warp-ballot compaction into the 11 ascending group lists.
  std::vector<int64_t> cs = compact(c, ckey.p, nC, 6, c->cell_groups);
  std::vector<int64_t> es = compact(c, ekey.p, nE, 5, c->edge_groups);
  int64_t off = 0;
  for (int g = 0; g < 6; ++g) {
    c->gsize[g] = cs[g];
    c->goff[g] = off;
    off += cs[g];
  }
  off = 0;
  for (int g = 0; g < 5; ++g) {
    c->gsize[6 + g] = es[g];
    c->goff[6 + g] = off;
    off += es[g];
  }
  c->width = width;
  c->have_regions = true;
  // Outputs in original order.
  if (cell_label || cell_sub || edge_label) {
    std::vector<uint8_t> cl(nC), cb(nC), el(nE);
    CK(cudaMemcpyAsync(cl.data(), c->cell_label.p, nC, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(cb.data(), c->cell_sub.p, nC, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(el.data(), c->edge_label.p, nE, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int32_t ni = 0; ni < nC; ++ni) {
      if (cell_label) cell_label[c->c_new2old[ni]] = cl[ni];
      if (cell_sub) cell_sub[c->c_new2old[ni]] = cb[ni];
    }
    if (edge_label)
      for (int32_t ne = 0; ne < nE; ++ne) edge_label[c->e_new2old[ne]] = el[ne];
  }
  if (group_size)
    for (int g = 0; g < 11; ++g) group_size[g] = c->gsize[g];
  if (warnings) {
    // label_underline_fine warnings (regions.cpp:131-138)
    *warnings = c->gsize[1] == 0 ? 1 : (c->gsize[2] == 0 ? 2 : (c->gsize[0] == 0 ? 4 : 0));
  }
  return MSWM_OK;
}

template <class F>
int guard(mswm_cuda_ctx* c, F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    if (c) c->last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    if (c) c->last_error = "host allocation failed";
    return MSWM_E_NOMEM;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what();
    return MSWM_E_CONFIG;
  }
}

}  // namespace


// ===========================================================================
// C ABI

extern "C" {

int mswm_cuda_create(const mswm_mesh_desc* mesh, int device, const int32_t* cell_order,
                     mswm_cuda_ctx** out) {
  if (!out) return MSWM_E_USAGE;
  *out = nullptr;
  auto c = std::make_unique<mswm_cuda_ctx>();
  try {
    if (!mesh) throw Error(MSWM_E_USAGE, "null mesh descriptor");
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->ls = c->stream;
    build_tables(c.get(), mesh, cell_order);
  } catch (const Error& e) {
    g_create_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return MSWM_E_NOMEM;
  }
  *out = c.release();
  return MSWM_OK;
}

void mswm_cuda_destroy(mswm_cuda_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

const char* mswm_cuda_last_error(const mswm_cuda_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : g_create_error.c_str();
}

int mswm_cuda_set_fields(mswm_cuda_ctx* c, const double* b, const double* f_vertex, double gravity) {
  return guard(c, [&] {
    check_ctx(c);
    if (!b || !f_vertex) throw Error(MSWM_E_USAGE, "null field");
    upload_field(c, c->b, b, c->c_new2old, c->nC);
    upload_field(c, c->f, f_vertex, c->v_new2old, c->nV);
    if (c->nV) {  // (A_v, f_v) pairs of kernel A
      k_fill_af<<<nblk(c->nV), kBlock, 0, c->stream>>>(c->nV, c->f.p, c->v_af.p);
      CK(cudaGetLastError());
    }
    c->gravity = gravity;
    c->have_fields = true;
    CK(cudaStreamSynchronize(c->stream));
    invalidate(c);  // gravity is a graph kernel argument
    return int(MSWM_OK);
  });
}

int mswm_cuda_set_regions(mswm_cuda_ctx* c, const uint8_t* fine_mask, int interface_width,
                          uint8_t* cell_label, uint8_t* cell_sublabel, uint8_t* edge_label,
                          int64_t group_size[11], int* warnings) {
  return guard(c, [&] {
    check_ctx(c);
    return set_regions_impl(c, fine_mask, interface_width, cell_label, cell_sublabel, edge_label,
                            group_size, warnings);
  });
}

int mswm_cuda_get_group(mswm_cuda_ctx* c, int group, int32_t* ids) {
  return guard(c, [&] {
    check_ctx(c);
    if (!c->have_regions) throw Error(MSWM_E_USAGE, "no regions");
    if (group < 0 || group > 10) throw Error(MSWM_E_USAGE, "group index out of range");
    const int64_t n = c->gsize[group];
    if (!ids || n == 0) return int(MSWM_OK);
    const DArr<int32_t>& buf = group < 6 ? c->cell_groups : c->edge_groups;
    CK(cudaMemcpyAsync(ids, buf.p + c->goff[group], size_t(n) * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!c->identity) {
      const auto& n2o = group < 6 ? c->c_new2old : c->e_new2old;
      for (int64_t k = 0; k < n; ++k) ids[k] = n2o[ids[k]];
      std::sort(ids, ids + n);
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_get_closure(mswm_cuda_ctx* c, unsigned mask, int kind, int32_t* ids, int64_t* n) {
  return guard(c, [&] {
    check_ctx(c);
    MaskPlan& p = plan_for(c, mask);
    const DArr<int32_t>* L = nullptr;
    int64_t cnt = 0;
    const std::vector<int32_t>* n2o = nullptr;
    switch (kind) {
      case MSWM_CLOSURE_FLUX: L = &p.fclos; cnt = p.nf; n2o = &c->e_new2old; break;
      case MSWM_CLOSURE_QT: L = &p.qclos; cnt = p.nq; n2o = &c->e_new2old; break;
      case MSWM_CLOSURE_K: L = &p.kclos; cnt = p.nk; n2o = &c->c_new2old; break;
      case MSWM_CLOSURE_PV: L = &p.vclos; cnt = p.nv; n2o = &c->v_new2old; break;
      default: throw Error(MSWM_E_USAGE, "closure kind out of range");
    }
    if (n) *n = cnt;
    if (ids && cnt) {
      CK(cudaMemcpyAsync(ids, L->p, size_t(cnt) * 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (!c->identity) {
        for (int64_t k = 0; k < cnt; ++k) ids[k] = (*n2o)[ids[k]];
        std::sort(ids, ids + cnt);
      }
    }
    return int(MSWM_OK);
  });
}

// Read set of a mask plan for the drop-in eval (k_mark_reads over its
// closure lists, operators.cpp:61-86) as original / internal id lists.
void build_eval_io(mswm_cuda_ctx* c, MaskPlan& p) {
  if (p.io_ready) return;
  cudaStream_t s = c->stream;
  DArr<uint8_t> cr, er;
  cr.alloc(c->nC);
  er.alloc(c->nE);
  cr.zero(s);
  er.zero(s);
  const int64_t n = int64_t(p.nv) + p.nk + p.nf + p.ne;
  if (n > 0) {
    k_mark_reads<<<nblk(n), kBlock, 0, s>>>(c->dev(), p.vclos.p, p.nv, p.kclos.p, p.nk, p.fclos.p,
                                            p.nf, p.edges, p.ne, cr.p, er.p);
    CK(cudaGetLastError());
  }
  std::vector<uint8_t> hc(c->nC), he(c->nE);
  CK(cudaMemcpyAsync(hc.data(), cr.p, size_t(c->nC), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(he.data(), er.p, size_t(c->nE), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<int32_t> ci, ei;
  p.io_rc_orig.clear();
  p.io_re_orig.clear();
  for (int32_t o = 0; o < c->nC; ++o) {
    const int32_t ni = c->identity ? o : c->c_old2new[o];
    if (hc[ni]) {
      p.io_rc_orig.push_back(o);
      ci.push_back(ni);
    }
  }
  for (int32_t o = 0; o < c->nE; ++o) {
    const int32_t ni = c->identity ? o : c->e_old2new[o];
    if (he[ni]) {
      p.io_re_orig.push_back(o);
      ei.push_back(ni);
    }
  }
  // inputs always go through pinned staging (packed on all host cores; a
  // pageable copy of the whole array is slower even when the read set is
  // most of the mesh)
  if (!ci.empty()) p.io_rc.upload(ci, s);
  if (!ei.empty()) p.io_re.upload(ei, s);
  auto sorted_out = [&](const std::vector<int32_t>& orig, const std::vector<int32_t>& o2n,
                        std::vector<int32_t>& so, DArr<int32_t>& dev) {
    so = orig;
    std::sort(so.begin(), so.end());
    std::vector<int32_t> ni(so.size());
    for (size_t k = 0; k < so.size(); ++k) ni[k] = c->identity ? so[k] : o2n[so[k]];
    if (!ni.empty()) dev.upload(ni, s);
  };
  sorted_out(p.host_cells, c->c_old2new, p.io_oc_orig, p.io_oc);
  sorted_out(p.host_edges, c->e_old2new, p.io_oe_orig, p.io_oe);
  CK(cudaStreamSynchronize(s));
  p.io_ready = true;
}

void ensure_pin(mswm_cuda_ctx* c, size_t n) {
  if (c->pin_n >= n) return;
  if (c->pin) CK(cudaFreeHost(c->pin));
  c->pin = nullptr;
  c->pin_n = 0;
  CK(cudaMallocHost(&c->pin, n * 8));
  c->pin_n = n;
  c->io_pack.alloc(n);
}

int mswm_cuda_eval(mswm_cuda_ctx* c, const double* h, const double* u, unsigned mask, double* dh,
                   double* du) {
  return guard(c, [&] {
    check_ctx(c);
    if (!h || !u || !dh || !du) throw Error(MSWM_E_USAGE, "null array");
    if (!c->have_fields) throw Error(MSWM_E_USAGE, "set_fields must be called before eval");
    check_dry(c);  // a pending error of an earlier step batch surfaces first
    MaskPlan& p = plan_for(c, mask);
    build_eval_io(c, p);
    cudaStream_t s = c->stream;
    // inputs: only the h / u entries the evaluation reads cross PCIe, packed
    // on the host cores into pinned staging
    if (c->T1h.n != size_t(c->nC)) c->T1h.alloc(c->nC);
    if (c->T1u.n != size_t(c->nE)) c->T1u.alloc(c->nE);
    const size_t nrc = p.io_rc_orig.size();
    const size_t nre = p.io_re_orig.size();
    const size_t nout = size_t(p.nc) + p.ne;
    ensure_pin(c, std::max<size_t>(1, std::max(nrc + nre, nout)));
    if (nrc + nre > 0) {
      double* pin = c->pin;
      const int32_t* rc = p.io_rc_orig.data();
      const int32_t* re = p.io_re_orig.data();
      host_par_for(int64_t(nrc), [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) pin[k] = h[rc[k]];
      });
      host_par_for(int64_t(nre), [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) pin[nrc + k] = u[re[k]];
      });
      CK(cudaMemcpyAsync(c->io_pack.p, c->pin, (nrc + nre) * 8, cudaMemcpyHostToDevice, s));
      if (nrc)
        k_scatter_perm<<<nblk(int64_t(nrc)), kBlock, 0, s>>>(int32_t(nrc), p.io_rc.p, c->io_pack.p,
                                                             c->T1h.p);
      if (nre)
        k_scatter_perm<<<nblk(int64_t(nre)), kBlock, 0, s>>>(int32_t(nre), p.io_re.p,
                                                             c->io_pack.p + nrc, c->T1u.p);
      CK(cudaGetLastError());
    }
    Op co[2] = {mk_op(OP_STORE, c->Dh.p), mk_op(OP_STORE, c->Dh.p)};
    Op eo[2] = {mk_op(OP_STORE, c->Du.p), mk_op(OP_STORE, c->Du.p)};
    launch_eval(c, p, c->T1h.p, c->T1u.p, co, eo);
    // outputs: gathered on the device in the plan's order, one packed copy
    // back, scattered into the caller's arrays; everything else is left
    // untouched (integrators.hpp:63-67)
    if (nout > 0) {
      if (p.nc)
        k_gather_perm<<<nblk(int64_t(p.nc)), kBlock, 0, s>>>(p.nc, p.io_oc.p, c->Dh.p, c->io_pack.p);
      if (p.ne)
        k_gather_perm<<<nblk(int64_t(p.ne)), kBlock, 0, s>>>(p.ne, p.io_oe.p, c->Du.p,
                                                             c->io_pack.p + p.nc);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(c->pin, c->io_pack.p, nout * 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    check_dry(c);
    {
      const double* pin = c->pin;
      const int32_t* oc = p.io_oc_orig.data();
      const int32_t* oe = p.io_oe_orig.data();
      const int64_t nc = p.nc;
      host_par_for(nc, [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) dh[oc[k]] = pin[k];
      });
      host_par_for(int64_t(p.ne), [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) du[oe[k]] = pin[nc + k];
      });
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_state_upload(mswm_cuda_ctx* c, const double* h, const double* u, double time) {
  return guard(c, [&] {
    check_ctx(c);
    if (!h || !u) throw Error(MSWM_E_USAGE, "null array");
    upload_field(c, c->H, h, c->c_new2old, c->nC);
    upload_field(c, c->U, u, c->e_new2old, c->nE);
    c->time = time;
    if (halo_dry_run()) {
      std::vector<Halo*> hs{&c->halo};
      for (auto& kv : c->halo_mask) hs.push_back(&kv.second);
      for (Halo* x : hs)
        if (x->nr > 0) {
          k_pack<<<nblk(x->nr), kBlock, 0, c->stream>>>(x->nr, x->rcode.p, c->H.p, c->U.p, x->rbuf.p);
          CK(cudaGetLastError());
        }
    }
    CK(cudaStreamSynchronize(c->stream));
    return int(MSWM_OK);
  });
}

int mswm_cuda_state_download(mswm_cuda_ctx* c, double* h, double* u, double* time) {
  return guard(c, [&] {
    check_ctx(c);
    if (h) download_field(c, c->H, h, c->c_new2old, c->nC);
    if (u) download_field(c, c->U, u, c->e_new2old, c->nE);
    if (time) *time = c->time;
    check_dry(c);  // the state is written either way; a pending error is reported
    return int(MSWM_OK);
  });
}

int mswm_cuda_step(mswm_cuda_ctx* c, int scheme, double dt, int M, int64_t n_steps, int sync) {
  return guard(c, [&] {
    check_ctx(c);
    check_step_args(c, scheme, dt, M, n_steps);
    // n_steps == 0 prepares: plans built, the step graph captured, nothing launched
    cudaGraphExec_t g = graph_for(c, scheme, dt, M);
    if (n_steps == 0) return int(MSWM_OK);
    c->batches.emplace_back(c->steps_issued, n_steps);
    for (int64_t k = 0; k < n_steps; ++k) {
      CK(cudaGraphLaunch(g, c->stream));
      tally_step(c, scheme, M);
      c->time += dt;
    }
    c->steps_issued += n_steps;
    if (sync) check_dry(c);
    return int(MSWM_OK);
  });
}

int mswm_cuda_ledger(mswm_cuda_ctx* c, int64_t cell_evals[16], int64_t edge_evals[16], int64_t* steps) {
  if (!c) return MSWM_E_USAGE;
  for (int r = 0; r < 4; ++r)
    for (int s = 0; s < 4; ++s) {
      if (cell_evals) cell_evals[4 * r + s] = c->ledger_cell[r][s];
      if (edge_evals) edge_evals[4 * r + s] = c->ledger_edge[r][s];
    }
  if (steps) *steps = c->ledger_steps;
  return MSWM_OK;
}

int mswm_cuda_ledger_reset(mswm_cuda_ctx* c) {
  if (!c) return MSWM_E_USAGE;
  std::memset(c->ledger_cell, 0, sizeof(c->ledger_cell));
  std::memset(c->ledger_edge, 0, sizeof(c->ledger_edge));
  c->ledger_steps = 0;
  return MSWM_OK;
}

int mswm_cuda_dry_vertex(const mswm_cuda_ctx* c, int64_t* step) {
  if (!c) return -1;
  if (step) *step = c->last_dry_step;
  return c->last_dry_vertex;
}

int mswm_cuda_sync(mswm_cuda_ctx* c) {
  return guard(c, [&] {
    check_ctx(c);
    check_dry(c);
    return int(MSWM_OK);
  });
}

void* mswm_cuda_stream(mswm_cuda_ctx* c) { return c ? (void*)c->stream : nullptr; }

int mswm_cuda_set_profiling(mswm_cuda_ctx* c, int enable) {
  return guard(c, [&] {
    check_ctx(c);
    if (enable < 0 || enable > 2) throw Error(MSWM_E_USAGE, "profiling level must be 0, 1 or 2");
    c->profiling = enable;
    return int(MSWM_OK);
  });
}

int mswm_cuda_eval_profile(mswm_cuda_ctx* c, float* eval_ms, int64_t* out_cells, int64_t* out_edges,
                           int cap, int* n) {
  return guard(c, [&] {
    check_ctx(c);
    CK(cudaStreamSynchronize(c->stream));
    const std::vector<EvalRecord> empty;
    const std::vector<EvalRecord>& R = c->last_records ? *c->last_records : empty;
    const int cnt = int(R.size());
    if (n) *n = cnt;
    for (int k = 0; k < cnt && k < cap; ++k) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, R[k].start, R[k].stop));
      if (eval_ms) eval_ms[k] = ms;
      if (out_cells) out_cells[k] = R[k].nc;
      if (out_edges) out_edges[k] = R[k].ne;
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_layout_info(const mswm_cuda_ctx* c, int* kernel_path, int* identity_order) {
  if (!c) return MSWM_E_USAGE;
  if (kernel_path) *kernel_path = 0;
  if (identity_order) *identity_order = c->identity ? 1 : 0;
  return MSWM_OK;
}

int mswm_cuda_stencil_info(const mswm_cuda_ctx* c, int* offsets16, int64_t* n_wide) {
  if (!c) return MSWM_E_USAGE;
  if (offsets16) *offsets16 = c->e_st16.p ? 1 : 0;
  if (n_wide) *n_wide = c->n_sten_wide;
  return MSWM_OK;
}

int mswm_cuda_index_info(const mswm_cuda_ctx* c, int* packed16, int64_t* n_wide_vertices,
                         int64_t* n_wide_cells, int64_t* n_wide_edges) {
  if (!c) return MSWM_E_USAGE;
  if (packed16) *packed16 = (c->pack16 ? 1 : 0) | (c->c_rec.p ? 2 : 0);
  if (n_wide_vertices) *n_wide_vertices = c->n_wide16[0];
  if (n_wide_cells) *n_wide_cells = c->n_wide16[1];
  if (n_wide_edges) *n_wide_edges = c->n_wide16[2];
  return MSWM_OK;
}

int mswm_cuda_kernels_per_step(mswm_cuda_ctx* c, int64_t* n) {
  if (!c || !n) return MSWM_E_USAGE;
  *n = c->last_kernels_per_step;
  return MSWM_OK;
}

int mswm_cuda_set_replication(mswm_cuda_ctx* c, int replication) {
  return guard(c, [&] {
    check_ctx(c);
    // integrators.cpp:128-129
    if (replication < 1) throw Error(MSWM_E_CONFIG, "cost replication factor must be >= 1");
    if (replication != c->replication) {
      c->replication = replication;
      c->drop_graphs();
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_schedule_info(const mswm_cuda_ctx* c, int* concurrent_coarse) {
  if (!c || !concurrent_coarse) return MSWM_E_USAGE;
  *concurrent_coarse = c->fork_state == 0 ? -1 : (c->fork_state == 1 ? 1 : 0);
  return MSWM_OK;
}

// Per-cell diagnostics terms of the device state; exact: sequential sums in
// ascending caller cell id on the host (the reference's order), else the
// fixed-shape device sum.
void diagnostics(mswm_cuda_ctx* c, bool exact, double* mass, double* energy) {
  cudaStream_t s = c->stream;
  DArr<double> mt, et;
  mt.alloc(c->nC);
  et.alloc(c->nC);
  const uint8_t* ckey = (c->have_regions && c->n_ranks > 1) ? c->ckey.p : nullptr;
  k_cell_diag<<<nblk(c->nC), kBlock, 0, s>>>(c->dev(), c->H.p, c->U.p, ckey, mt.p, et.p);
  CK(cudaGetLastError());
  if (exact) {
    std::vector<double> hm(c->nC), he(c->nC);
    CK(cudaMemcpyAsync(hm.data(), mt.p, size_t(c->nC) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(he.data(), et.p, size_t(c->nC) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double m = 0.0, e = 0.0;
    for (int32_t i = 0; i < c->nC; ++i) {  // harness.cpp:103, :110-122: ascending id
      const int32_t k = c->identity ? i : c->c_old2new[i];
      m += hm[k];
      e += he[k];
    }
    if (mass) *mass = m;
    if (energy) *energy = e;
    return;
  }
  const int32_t chunk = 8192;
  const int32_t nb = (c->nC + chunk - 1) / chunk;
  DArr<double> part, tot;
  part.alloc(2 * size_t(nb));
  tot.alloc(2);
  k_sum_chunks<<<nb, kBlock, 0, s>>>(c->nC, chunk, mt.p, part.p);
  k_sum_chunks<<<nb, kBlock, 0, s>>>(c->nC, chunk, et.p, part.p + nb);
  k_sum_chunks<<<1, kBlock, 0, s>>>(nb, nb, part.p, tot.p);
  k_sum_chunks<<<1, kBlock, 0, s>>>(nb, nb, part.p + nb, tot.p + 1);
  CK(cudaGetLastError());
  double r[2];
  CK(cudaMemcpyAsync(r, tot.p, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (mass) *mass = r[0];
  if (energy) *energy = r[1];
}

int mswm_cuda_total_mass(mswm_cuda_ctx* c, double* mass) {
  return guard(c, [&] {
    check_ctx(c);
    if (!mass) throw Error(MSWM_E_USAGE, "null output");
    diagnostics(c, true, mass, nullptr);
    return int(MSWM_OK);
  });
}

int mswm_cuda_diagnostics(mswm_cuda_ctx* c, int exact, double* mass, double* energy) {
  return guard(c, [&] {
    check_ctx(c);
    if (!c->have_fields) throw Error(MSWM_E_USAGE, "set_fields must be called first");
    diagnostics(c, exact != 0, mass, energy);
    return int(MSWM_OK);
  });
}

int mswm_cuda_courant(mswm_cuda_ctx* c, double dt, int M, double* fine, double* coarse) {
  return guard(c, [&] {
    check_ctx(c);
    if (M < 1) throw Error(MSWM_E_USAGE, "substep count must be >= 1");  // integrators.cpp:636
    cudaStream_t s = c->stream;
    DArr<unsigned long long> out;
    out.alloc(2);
    out.zero(s);
    const uint8_t* ekey = c->have_regions ? c->ekey.p : nullptr;
    k_courant<<<nblk(c->nE), kBlock, 0, s>>>(c->dev(), c->U.p, ekey, dt, dt / M, out.p);
    CK(cudaGetLastError());
    unsigned long long r[2];
    CK(cudaMemcpyAsync(r, out.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double v[2];
    std::memcpy(v, r, 16);
    if (fine) *fine = v[0];
    if (coarse) *coarse = ekey ? v[1] : v[0];
    return int(MSWM_OK);
  });
}

// ---- multi-rank --------------------------------------------------------------

int mswm_cuda_halo_reach(mswm_cuda_ctx* c, const int32_t* rank_of_cell, int n_ranks,
                         uint64_t* cell_reach, uint64_t* edge_reach, uint64_t* vertex_reach) {
  return guard(c, [&] {
    check_ctx(c);
    if (!rank_of_cell) throw Error(MSWM_E_USAGE, "rank_of_cell is null");
    if (n_ranks < 1 || n_ranks > 64) throw Error(MSWM_E_USAGE, "n_ranks must lie in [1, 64]");
    cudaStream_t s = c->stream;
    std::vector<int32_t> r(c->nC);
    for (int32_t ni = 0; ni < c->nC; ++ni) {
      const int32_t q = rank_of_cell[c->identity ? ni : c->c_new2old[ni]];
      if (q < 0 || q >= n_ranks) throw Error(MSWM_E_USAGE, "rank out of range");
      r[ni] = q;
    }
    DArr<int32_t> dr;
    dr.upload(r, s);
    DArr<uint64_t> a, b, er, vr;
    a.alloc(c->nC);
    b.alloc(c->nC);
    er.alloc(c->nE);
    vr.alloc(c->nV);
    const DevMesh M = c->dev();
    k_reach_init<<<nblk(c->nC), kBlock, 0, s>>>(c->nC, dr.p, a.p);
    k_reach_hop<<<nblk(c->nC), kBlock, 0, s>>>(M, c->c_nbr.p, a.p, b.p);
    k_reach_hop<<<nblk(c->nC), kBlock, 0, s>>>(M, c->c_nbr.p, b.p, a.p);
    k_reach_ev<<<nblk(int64_t(c->nE) + c->nV), kBlock, 0, s>>>(M, a.p, er.p, vr.p);
    CK(cudaGetLastError());
    auto down = [&](const DArr<uint64_t>& d, uint64_t* out, int32_t n, const std::vector<int32_t>& n2o) {
      if (!out) return;
      std::vector<uint64_t> h(n);
      CK(cudaMemcpyAsync(h.data(), d.p, size_t(n) * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int32_t k = 0; k < n; ++k) out[c->identity ? k : n2o[k]] = h[k];
    };
    down(a, cell_reach, c->nC, c->c_new2old);
    down(er, edge_reach, c->nE, c->e_new2old);
    down(vr, vertex_reach, c->nV, c->v_new2old);
    return int(MSWM_OK);
  });
}

int mswm_cuda_partition(mswm_cuda_ctx* c, const int32_t* sweep_order, int n_parts,
                        int32_t* rank_of_cell, int32_t* edge_owner) {
  return guard(c, [&] {
    check_ctx(c);
    if (!sweep_order) throw Error(MSWM_E_USAGE, "sweep_order is null");
    if (!c->have_regions || !c->cell_label.p || !c->edge_label.p)
      throw Error(MSWM_E_USAGE, "partition needs the region map of mswm_cuda_set_regions");
    const int32_t nC = c->nC, nE = c->nE;
    if (n_parts < 1 || n_parts > nC) throw Error(MSWM_E_USAGE, "n_parts out of range");
    cudaStream_t s = c->stream;
    // sweep in internal ids (and a permutation check)
    std::vector<int32_t> ord(nC);
    {
      std::vector<uint8_t> seen(nC, 0);
      for (int32_t k = 0; k < nC; ++k) {
        const int32_t x = sweep_order[k];
        if (x < 0 || x >= nC || seen[x]) throw Error(MSWM_E_USAGE, "sweep_order is not a permutation");
        seen[x] = 1;
        ord[k] = c->identity ? x : c->c_old2new[x];
      }
    }
    DArr<int32_t> d_ord, lst, rank, owner, bad;
    DArr<uint8_t> key;
    d_ord.upload(ord, s);
    key.alloc(nC);
    k_part_class<<<nblk(nC), kBlock, 0, s>>>(nC, d_ord.p, c->cell_label.p, key.p);
    CK(cudaGetLastError());
    const std::vector<int64_t> t = compact(c, key.p, nC, 3, lst);
    rank.alloc(nC);
    k_part_assign<<<nblk(nC), kBlock, 0, s>>>(nC, lst.p, d_ord.p, t[0], t[1], t[2], n_parts,
                                              rank.p);
    owner.alloc(nE);
    const int32_t none = INT32_MAX;
    bad.alloc(1);
    CK(cudaMemcpyAsync(bad.p, &none, 4, cudaMemcpyHostToDevice, s));
    k_part_edge_owner<<<nblk(nE), kBlock, 0, s>>>(c->dev(), c->cell_label.p, c->edge_label.p,
                                                  rank.p, owner.p, bad.p);
    CK(cudaGetLastError());
    int32_t first_bad = none;
    CK(cudaMemcpyAsync(&first_bad, bad.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (first_bad != none)
      throw Error(MSWM_E_TOPOLOGY, "edge " + std::to_string(c->e_new2old[first_bad]) +
                                       " has no adjacent cell of its own region class");
    auto down = [&](const DArr<int32_t>& d, int32_t* out, int32_t n, const std::vector<int32_t>& n2o) {
      if (!out) return;
      std::vector<int32_t> h(n);
      CK(cudaMemcpyAsync(h.data(), d.p, size_t(n) * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int32_t k = 0; k < n; ++k) out[c->identity ? k : n2o[k]] = h[k];
    };
    down(rank, rank_of_cell, nC, c->c_new2old);
    down(owner, edge_owner, nE, c->e_new2old);
    return int(MSWM_OK);
  });
}

int mswm_cuda_set_labels(mswm_cuda_ctx* c, const uint8_t* cell_label, const uint8_t* cell_sub,
                         const uint8_t* edge_label, const uint8_t* cell_owned,
                         const uint8_t* edge_owned, int interface_width) {
  return guard(c, [&] {
    check_ctx(c);
    if (!cell_label || !cell_sub || !edge_label) throw Error(MSWM_E_USAGE, "null label array");
    if (interface_width < 1) throw Error(MSWM_E_CONFIG, "interface width must be >= 1");
    const int32_t nC = c->nC, nE = c->nE;
    std::vector<uint8_t> ck(nC), ek(nE);
    for (int32_t ni = 0; ni < nC; ++ni) {
      const int32_t i = c->c_new2old[ni];
      const uint8_t l = cell_label[i], sb = cell_sub[i];
      if (l > 3 || sb > 2 || (l != 0 && sb != 0)) throw Error(MSWM_E_USAGE, "invalid cell label");
      ck[ni] = (cell_owned && !cell_owned[i]) ? 0xFF : (l == 0 ? sb : uint8_t(l + 2));
    }
    for (int32_t ne = 0; ne < nE; ++ne) {
      const int32_t e = c->e_new2old[ne];
      if (edge_label[e] > 4) throw Error(MSWM_E_USAGE, "invalid edge label");
      ek[ne] = (edge_owned && !edge_owned[e]) ? 0xFF : edge_label[e];
    }
    invalidate(c);
    c->ckey.upload(ck, c->stream);
    c->ekey.upload(ek, c->stream);
    std::vector<int64_t> cs = compact(c, c->ckey.p, nC, 6, c->cell_groups);
    std::vector<int64_t> es = compact(c, c->ekey.p, nE, 5, c->edge_groups);
    int64_t off = 0;
    for (int g = 0; g < 6; ++g) {
      c->gsize[g] = cs[g];
      c->goff[g] = off;
      off += cs[g];
    }
    off = 0;
    for (int g = 0; g < 5; ++g) {
      c->gsize[6 + g] = es[g];
      c->goff[6 + g] = off;
      off += es[g];
    }
    c->width = interface_width;
    c->have_regions = true;
    return int(MSWM_OK);
  });
}

int mswm_cuda_validate_labels(mswm_cuda_ctx* c, const uint8_t* cell_label, const uint8_t* cell_sub,
                              const uint8_t* edge_label, int interface_width, int64_t counts[6],
                              int32_t first[6]) {
  return guard(c, [&] {
    check_ctx(c);
    if (!cell_label || !counts || !first) throw Error(MSWM_E_USAGE, "null label or output array");
    if (interface_width < 1) throw Error(MSWM_E_CONFIG, "interface width must be >= 1");
    const int32_t nC = c->nC, nE = c->nE;
    const int w = interface_width;
    cudaStream_t s = c->stream;
    // labels in internal order; dist = 0 on the label-0 set, -1 elsewhere
    std::vector<uint8_t> cl(nC), cb(cell_sub ? nC : 0), el(edge_label ? nE : 0);
    std::vector<int32_t> dist0(nC);
    host_par_for(nC, [&](int64_t lo, int64_t hi) {
      for (int64_t ni = lo; ni < hi; ++ni) {
        const int32_t i = c->c_new2old[ni];
        cl[ni] = cell_label[i];
        if (cell_sub) cb[ni] = cell_sub[i];
        dist0[ni] = cell_label[i] == 0 ? 0 : -1;
      }
    });
    if (edge_label)
      host_par_for(nE, [&](int64_t lo, int64_t hi) {
        for (int64_t ne = lo; ne < hi; ++ne) el[ne] = edge_label[c->e_new2old[ne]];
      });
    DArr<uint8_t> d_cl, d_cb, d_el;
    DArr<int32_t> dist, layer_count, d_first, ident_c;
    DArr<unsigned long long> d_count;
    d_cl.upload(cl, s);
    if (cell_sub) d_cb.upload(cb, s);
    if (edge_label) d_el.upload(el, s);
    dist.upload(dist0, s);
    layer_count.alloc(size_t(2 * w) + 1);
    layer_count.zero(s);
    const DevMesh M = c->dev();
    for (int level = 1; level <= 2 * w; ++level) {
      k_bfs_layer<<<nblk(nC), kBlock, 0, s>>>(M, c->c_nbr.p, dist.p, level, layer_count.p + level);
      CK(cudaGetLastError());
    }
    const int32_t *n2o_c = c->d_c_n2o.p, *n2o_e = c->d_e_n2o.p;
    if (c->identity) {
      std::vector<int32_t> id(size_t(std::max(nC, nE)));
      for (size_t k = 0; k < id.size(); ++k) id[k] = int32_t(k);
      ident_c.upload(id, s);
      n2o_c = n2o_e = ident_c.p;
    }
    d_count.alloc(VK_COUNT);
    d_count.zero(s);
    std::vector<int32_t> f0(VK_COUNT, INT32_MAX);
    d_first.upload(f0, s);
    k_validate_labels<<<nblk(std::max(nC, nE)), kBlock, 0, s>>>(
        M, c->c_nbr.p, dist.p, w, d_cl.p, cell_sub ? d_cb.p : nullptr,
        edge_label ? d_el.p : nullptr, n2o_c, n2o_e, d_count.p, d_first.p);
    CK(cudaGetLastError());
    unsigned long long hc[VK_COUNT];
    int32_t hf[VK_COUNT];
    CK(cudaMemcpyAsync(hc, d_count.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hf, d_first.p, sizeof(hf), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int k = 0; k < VK_COUNT; ++k) {
      counts[k] = int64_t(hc[k]);
      first[k] = hc[k] ? hf[k] : -1;
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_set_halo(mswm_cuda_ctx* c, int rank, int n_ranks, int n_peers, const int32_t* peers,
                       const int64_t* counts, const int32_t* ids) {
  return guard(c, [&] {
    check_ctx(c);
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks || n_peers < 0 || n_peers > n_ranks - 1)
      throw Error(MSWM_E_USAGE, "bad rank / peer counts");
    if (n_peers > 0 && (!peers || !counts || !ids)) throw Error(MSWM_E_USAGE, "null halo arrays");
    Halo h;
    std::vector<int32_t> sc, rc;
    const int32_t* p = ids;
    for (int j = 0; j < n_peers; ++j) {
      const int64_t nsc = counts[4 * j], nse = counts[4 * j + 1], nrc = counts[4 * j + 2],
                    nre = counts[4 * j + 3];
      if (peers[j] < 0 || peers[j] >= n_ranks || peers[j] == rank)
        throw Error(MSWM_E_USAGE, "bad peer rank");
      h.peer.push_back(peers[j]);
      h.soff.push_back(int64_t(sc.size()));
      h.scnt.push_back(nsc + nse);
      for (int64_t k = 0; k < nsc; ++k) {
        if (p[k] < 0 || p[k] >= c->nC) throw Error(MSWM_E_USAGE, "halo cell id out of range");
        sc.push_back(c->c_old2new[p[k]]);
      }
      p += nsc;
      for (int64_t k = 0; k < nse; ++k) {
        if (p[k] < 0 || p[k] >= c->nE) throw Error(MSWM_E_USAGE, "halo edge id out of range");
        sc.push_back(~c->e_old2new[p[k]]);
      }
      p += nse;
      h.roff.push_back(int64_t(rc.size()));
      h.rcnt.push_back(nrc + nre);
      for (int64_t k = 0; k < nrc; ++k) {
        if (p[k] < 0 || p[k] >= c->nC) throw Error(MSWM_E_USAGE, "halo cell id out of range");
        rc.push_back(c->c_old2new[p[k]]);
      }
      p += nrc;
      for (int64_t k = 0; k < nre; ++k) {
        if (p[k] < 0 || p[k] >= c->nE) throw Error(MSWM_E_USAGE, "halo edge id out of range");
        rc.push_back(~c->e_old2new[p[k]]);
      }
      p += nre;
    }
    h.ns = int64_t(sc.size());
    h.nr = int64_t(rc.size());
    h.scode.upload(sc, c->stream);
    h.rcode.upload(rc, c->stream);
    h.h_scode = std::move(sc);
    h.h_rcode = std::move(rc);
    h.sbuf.alloc(size_t(std::max<int64_t>(h.ns, 1)));
    h.rbuf.alloc(size_t(std::max<int64_t>(h.nr, 1)));
    CK(cudaStreamSynchronize(c->stream));
    c->drop_graphs();
    c->arena.alloc(0);  // the peer-store arena follows the halo plans
    c->transport = 0;
    c->halo = std::move(h);
    c->halo_mask.clear();
    c->rank = rank;
    c->n_ranks = n_ranks;
    return int(MSWM_OK);
  });
}

int mswm_cuda_halo_needs(mswm_cuda_ctx* c, unsigned mask, int64_t* counts, int32_t* pos) {
  return guard(c, [&] {
    check_ctx(c);
    if (!counts) throw Error(MSWM_E_USAGE, "null counts");
    const Halo& x = c->halo;
    MaskPlan& p = plan_for(c, mask);
    cudaStream_t s = c->stream;
    DArr<uint8_t> cr, er;
    cr.alloc(c->nC);
    er.alloc(c->nE);
    cr.zero(s);
    er.zero(s);
    const int64_t n = int64_t(p.nv) + p.nk + p.nf + p.ne;
    if (n > 0) {
      k_mark_reads<<<nblk(n), kBlock, 0, s>>>(c->dev(), p.vclos.p, p.nv, p.kclos.p, p.nk, p.fclos.p,
                                              p.nf, p.edges, p.ne, cr.p, er.p);
      CK(cudaGetLastError());
    }
    std::vector<uint8_t> hc(c->nC), he(c->nE);
    CK(cudaMemcpyAsync(hc.data(), cr.p, size_t(c->nC), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(he.data(), er.p, size_t(c->nE), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int64_t at = 0;
    for (size_t j = 0; j < x.peer.size(); ++j) {
      int64_t k = 0;
      for (int64_t q = 0; q < x.rcnt[j]; ++q) {
        const int32_t code = x.h_rcode[size_t(x.roff[j] + q)];
        if (code >= 0 ? hc[code] : he[~code]) {
          if (pos) pos[at + k] = int32_t(q);
          ++k;
        }
      }
      counts[j] = k;
      at += k;
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_set_halo_mask(mswm_cuda_ctx* c, unsigned mask, const int64_t* send_counts,
                            const int32_t* send_pos, const int64_t* recv_counts,
                            const int32_t* recv_pos) {
  return guard(c, [&] {
    check_ctx(c);
    const Halo& x = c->halo;
    const size_t np = x.peer.size();
    if (np && (!send_counts || !recv_counts)) throw Error(MSWM_E_USAGE, "null halo counts");
    Halo h;
    h.peer = x.peer;
    std::vector<int32_t> sc, rc;
    const int32_t* sp = send_pos;
    const int32_t* rp = recv_pos;
    for (size_t j = 0; j < np; ++j) {
      h.soff.push_back(int64_t(sc.size()));
      h.scnt.push_back(send_counts[j]);
      for (int64_t k = 0; k < send_counts[j]; ++k) {
        if (sp[k] < 0 || sp[k] >= x.scnt[j]) throw Error(MSWM_E_USAGE, "send position out of range");
        sc.push_back(x.h_scode[size_t(x.soff[j] + sp[k])]);
      }
      sp += send_counts[j];
      h.roff.push_back(int64_t(rc.size()));
      h.rcnt.push_back(recv_counts[j]);
      for (int64_t k = 0; k < recv_counts[j]; ++k) {
        if (rp[k] < 0 || rp[k] >= x.rcnt[j]) throw Error(MSWM_E_USAGE, "recv position out of range");
        rc.push_back(x.h_rcode[size_t(x.roff[j] + rp[k])]);
      }
      rp += recv_counts[j];
    }
    h.ns = int64_t(sc.size());
    h.nr = int64_t(rc.size());
    h.scode.upload(sc, c->stream);
    h.rcode.upload(rc, c->stream);
    h.sbuf.alloc(size_t(std::max<int64_t>(h.ns, 1)));
    h.rbuf.alloc(size_t(std::max<int64_t>(h.nr, 1)));
    CK(cudaStreamSynchronize(c->stream));
    h.h_scode = std::move(sc);
    h.h_rcode = std::move(rc);
    c->drop_graphs();
    c->arena.alloc(0);
    c->transport = 0;
    c->halo.prbuf = nullptr;
    for (auto& kv : c->halo_mask) kv.second.prbuf = nullptr;
    c->halo_mask[mask] = std::move(h);
    return int(MSWM_OK);
  });
}


}  // extern "C"

namespace {

constexpr size_t kArenaAlign = 256;
size_t arena_align(size_t n) { return (n + kArenaAlign - 1) / kArenaAlign * kArenaAlign; }

// the context's halos in export order: the full halo (key -1), then the
// per-mask restrictions by ascending mask
std::vector<std::pair<int64_t, Halo*>> peer_halos(mswm_cuda_ctx* c) {
  std::vector<std::pair<int64_t, Halo*>> v;
  v.emplace_back(-1, &c->halo);
  for (auto& kv : c->halo_mask) v.emplace_back(int64_t(kv.first), &kv.second);
  return v;
}

// allocate the arena for the current halo plans (idempotent until they change)
void peer_prepare(mswm_cuda_ctx* c) {
  if (!c->halo.active()) throw Error(MSWM_E_USAGE, "peer transport needs a halo plan (mswm_cuda_set_halo)");
  if (c->arena.p) return;
  size_t off = arena_align(size_t(2) * c->n_ranks * 8);
  std::vector<size_t> at;
  for (auto& kh : peer_halos(c)) {
    at.push_back(off);
    off += arena_align(size_t(2) * std::max<int64_t>(kh.second->nr, 1) * 8);
  }
  c->arena.alloc(off);
  c->arena.zero(c->stream);
  size_t k = 0;
  for (auto& kh : peer_halos(c)) {
    kh.second->prbuf = reinterpret_cast<double*>(c->arena.p + at[k++]);
    kh.second->pstride = std::max<int64_t>(kh.second->nr, 1);
    kh.second->h_pslots.assign(kh.second->peer.size(), PeerSlot{nullptr, 0, nullptr, 0});
  }
  if (const char* e = std::getenv("MSWM_PEER_TIMEOUT_MS"))
    c->peer_budget_ns = std::max(1ll, std::atoll(e)) * 1000000ull;
  c->xchan.alloc(4);
  c->xchan.zero(c->stream);
  c->xerr.alloc(1);
  c->xerr.zero(c->stream);
  std::vector<int32_t> peers(c->halo.peer.begin(), c->halo.peer.end());
  c->d_peers.upload(peers, c->stream);
  for (size_t r = 0; r < c->peer_base.size(); ++r)
    if (c->peer_base[r] && c->peer_ipc[r]) cudaIpcCloseMemHandle(c->peer_base[r]);
  c->peer_base.assign(size_t(c->n_ranks), nullptr);
  c->peer_ipc.assign(size_t(c->n_ranks), 0);
  CK(cudaStreamSynchronize(c->stream));
}

// rows of (mask or -1, sending rank, byte offset, stride bytes, count): where
// each neighbour's values land in this rank's arena
std::vector<int64_t> peer_rows(mswm_cuda_ctx* c) {
  std::vector<int64_t> rows;
  for (auto& kh : peer_halos(c)) {
    const Halo& x = *kh.second;
    for (size_t j = 0; j < x.peer.size(); ++j) {
      rows.push_back(kh.first);
      rows.push_back(x.peer[j]);
      rows.push_back(int64_t(reinterpret_cast<unsigned char*>(x.prbuf + x.roff[j]) - c->arena.p));
      rows.push_back(x.pstride * 8);
      rows.push_back(x.rcnt[j]);
    }
  }
  return rows;
}

void peer_attach(mswm_cuda_ctx* c, int peer_rank, unsigned char* base, bool ipc, const int64_t* rows,
                 int64_t n_rows) {
  if (peer_rank < 0 || peer_rank >= c->n_ranks || peer_rank == c->rank)
    throw Error(MSWM_E_USAGE, "bad peer rank");
  c->peer_base[size_t(peer_rank)] = base;
  c->peer_ipc[size_t(peer_rank)] = ipc;
  for (auto& kh : peer_halos(c)) {
    Halo& x = *kh.second;
    for (size_t j = 0; j < x.peer.size(); ++j) {
      if (x.peer[j] != peer_rank) continue;
      const int64_t* hit = nullptr;
      for (int64_t r = 0; r < n_rows; ++r)
        if (rows[5 * r] == kh.first && rows[5 * r + 1] == c->rank) hit = rows + 5 * r;
      if (!hit || hit[4] != x.scnt[j])
        throw Error(MSWM_E_USAGE, "inconsistent halo plans between ranks " + std::to_string(c->rank) +
                                      " and " + std::to_string(peer_rank));
      x.h_pslots[j] = PeerSlot{reinterpret_cast<double*>(base + hit[2]), hit[3] / 8,
                               reinterpret_cast<unsigned long long*>(base) + c->rank, x.soff[j]};
    }
  }
}

void peer_enable(mswm_cuda_ctx* c, bool on) {
  if (on) {
    if (!c->arena.p) throw Error(MSWM_E_USAGE, "peer transport: export and import first");
    for (auto& kh : peer_halos(c)) {
      Halo& x = *kh.second;
      std::vector<uint8_t> ss(size_t(std::max<int64_t>(x.ns, 1)), 0);
      for (size_t j = 0; j < x.peer.size(); ++j) {
        if (!x.h_pslots[j].dst)
          throw Error(MSWM_E_USAGE, "peer transport: rank " + std::to_string(x.peer[j]) + " not imported");
        for (int64_t k = 0; k < x.scnt[j]; ++k) ss[size_t(x.soff[j] + k)] = uint8_t(j);
      }
      if (x.peer.size() > 255) throw Error(MSWM_E_USAGE, "peer transport: more than 255 neighbours");
      x.pslots.upload(x.h_pslots, c->stream);
      x.sslot.upload(ss, c->stream);
    }
    CK(cudaStreamSynchronize(c->stream));
  }
  c->transport = on ? 1 : 0;
  c->fork_state = 0;
  c->drop_graphs();
}

}  // namespace

extern "C" {

int mswm_cuda_peer_export(mswm_cuda_ctx* c, void* ipc_handle, int64_t* rows, int64_t cap_rows,
                          int64_t* n_rows) {
  return guard(c, [&] {
    check_ctx(c);
    if (!n_rows) throw Error(MSWM_E_USAGE, "null row count");
    peer_prepare(c);
    const std::vector<int64_t> r = peer_rows(c);
    *n_rows = int64_t(r.size() / 5);
    if (rows) {
      if (cap_rows < *n_rows) throw Error(MSWM_E_USAGE, "row buffer too small");
      std::copy(r.begin(), r.end(), rows);
    }
    if (ipc_handle) {
      cudaIpcMemHandle_t hnd;
      CK(cudaIpcGetMemHandle(&hnd, c->arena.p));
      static_assert(sizeof(hnd) == 64, "cudaIpcMemHandle_t is 64 bytes");
      std::memcpy(ipc_handle, &hnd, sizeof(hnd));
    }
    return int(MSWM_OK);
  });
}

int mswm_cuda_peer_import(mswm_cuda_ctx* c, int peer_rank, const void* ipc_handle, const int64_t* rows,
                          int64_t n_rows) {
  return guard(c, [&] {
    check_ctx(c);
    if (!ipc_handle || (n_rows && !rows)) throw Error(MSWM_E_USAGE, "null handle or rows");
    peer_prepare(c);
    if (peer_rank >= 0 && peer_rank < c->n_ranks && c->peer_base[size_t(peer_rank)] &&
        c->peer_ipc[size_t(peer_rank)]) {
      cudaIpcCloseMemHandle(c->peer_base[size_t(peer_rank)]);
      c->peer_base[size_t(peer_rank)] = nullptr;
    }
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, ipc_handle, sizeof(hnd));
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess));
    peer_attach(c, peer_rank, static_cast<unsigned char*>(base), true, rows, n_rows);
    return int(MSWM_OK);
  });
}

int mswm_cuda_peer_enable(mswm_cuda_ctx* c, int on) {
  return guard(c, [&] {
    check_ctx(c);
    peer_enable(c, on != 0);
    return int(MSWM_OK);
  });
}

int mswm_cuda_peer_exchange(mswm_cuda_ctx* c, int phase) {
  return guard(c, [&] {
    check_ctx(c);
    if (c->transport != 1) throw Error(MSWM_E_USAGE, "peer transport not enabled");
    if (phase < 0 || phase > 2)
      throw Error(MSWM_E_USAGE, "phase must be 0 (push), 1 (wait + unpack) or 2 (the same, not awaited)");
    Halo& x = c->halo;
    if (phase == 0) {
      k_push<<<unsigned(std::max<int64_t>(1, nblk(x.ns))), kBlock, 0, c->stream>>>(x.ns, x.scode.p,
          x.sslot.p, c->H.p, c->U.p, x.pslots.p, int(x.peer.size()), 0, c->xchan.p);
    } else {
      PredArgs pa;
      std::memset(&pa, 0, sizeof(pa));
      k_wait_unpack<<<unsigned(std::max<int64_t>(1, nblk(x.nr))), kBlock, 0, c->stream>>>(x.nr,
          x.rcode.p, x.prbuf, x.pstride, c->H.p, c->U.p, pa,
          reinterpret_cast<const unsigned long long*>(c->arena.p), c->d_peers.p, int(x.peer.size()),
          c->xchan.p, c->xerr.p, c->peer_budget_ns);
    }
    CK(cudaGetLastError());
    if (phase != 2) check_dry(c);  // phase 2 returns at once: mswm_cuda_sync reports
    return int(MSWM_OK);
  });
}

int mswm_cuda_nccl_unique_id(void* id_out) {
  try {
    if (!id_out) return MSWM_E_USAGE;
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
    return MSWM_OK;
  } catch (const Error& e) {
    g_create_error = e.what();
    return e.status;
  }
}

int mswm_cuda_comm_init(mswm_cuda_ctx* c, const void* unique_id, int rank, int n_ranks) {
  return guard(c, [&] {
    check_ctx(c);
    if (!unique_id) throw Error(MSWM_E_USAGE, "null unique id");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    if (c->nccl_comm) {
      nccl().CommDestroy(c->nccl_comm);
      c->nccl_comm = nullptr;
    }
    if (c->nccl_comm2) {
      nccl().CommDestroy(c->nccl_comm2);
      c->nccl_comm2 = nullptr;
    }
    c->nccl_warm = false;
    nccl_check(nccl().CommInitRank(&c->nccl_comm, n_ranks, id, rank));
    if (nccl().CommSplit) nccl_check(nccl().CommSplit(c->nccl_comm, 0, rank, &c->nccl_comm2, nullptr));
    c->fork_state = 0;  // the concurrent coarse step may use the new communicators
    c->drop_graphs();
    return int(MSWM_OK);
  });
}

struct mswm_cuda_group {
  std::vector<mswm_cuda_ctx*> members;
  cudaStream_t stream = nullptr;
  ncclComm_t loop = nullptr, loop2 = nullptr;  // one-rank communicators (nccl_loopback)
  std::map<std::tuple<int, double, int>, mswm_cuda_ctx::Graph> graphs;
  std::vector<uint64_t> gens;  // members' configuration generations the graphs were captured at
  std::string last_error;
  void drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
  ~mswm_cuda_group() {
    drop_graphs();
    if (stream) cudaStreamSynchronize(stream);
    if (loop2) nccl().CommDestroy(loop2);
    if (loop) nccl().CommDestroy(loop);
    if (stream) cudaStreamDestroy(stream);
  }
};

int mswm_cuda_group_create(mswm_cuda_ctx* const* members, int n, mswm_cuda_group** out) {
  if (!out || !members || n < 1) return MSWM_E_USAGE;
  *out = nullptr;
  auto g = std::make_unique<mswm_cuda_group>();
  try {
    for (int r = 0; r < n; ++r) {
      if (!members[r]) throw Error(MSWM_E_USAGE, "null member");
      if (members[r]->rank != r || members[r]->n_ranks != n)
        throw Error(MSWM_E_USAGE, "member " + std::to_string(r) + " is not rank " +
                                      std::to_string(r) + " of " + std::to_string(n));
      if (members[r]->device != members[0]->device)
        throw Error(MSWM_E_USAGE, "group members must share a device");
      g->members.push_back(members[r]);
    }
    for (auto* c : g->members) c->loop_comm = c->loop_comm2 = nullptr;  // a previous group's
    CK(cudaSetDevice(members[0]->device));
    CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  } catch (const Error& e) {
    g_create_error = e.what();
    return e.status;
  }
  *out = g.release();
  return MSWM_OK;
}

void mswm_cuda_group_destroy(mswm_cuda_group* g) {
  if (!g) return;
  cudaStreamSynchronize(g->stream);
  delete g;
}

int mswm_cuda_group_step(mswm_cuda_group* g, int scheme, double dt, int M, int64_t n_steps) {
  if (!g) return MSWM_E_USAGE;
  mswm_cuda_ctx* c0 = g->members[0];
  const int rc = guard(c0, [&] {
    check_ctx(c0);
    for (auto* c : g->members) {
      check_step_args(c, scheme, dt, M, n_steps);
      CK(cudaStreamSynchronize(c->stream));  // uploads were issued on member streams
    }
    if (n_steps == 0) return int(MSWM_OK);
    // a member reconfigured since capture (restrict_halos, relabel, fields):
    // its buffers and plans may have moved, so every group graph is stale
    std::vector<uint64_t> now;
    for (auto* c : g->members) now.push_back(c->gen);
    if (now != g->gens) {
      g->drop_graphs();
      g->gens = now;
    }
    const auto key = std::make_tuple(scheme, dt, (scheme == MSWM_LTS3 || scheme == MSWM_LTS2) ? M : 0);
    auto it = g->graphs.find(key);
    if (it == g->graphs.end()) {
      auto gr = capture_step(g->members, g->stream, scheme, dt, M, false);
      it = g->graphs.emplace(key, std::move(gr)).first;
    }
    for (auto* c : g->members) c->batches.emplace_back(c->steps_issued, n_steps);
    for (int64_t k = 0; k < n_steps; ++k) {
      CK(cudaGraphLaunch(it->second.exec, g->stream));
      for (auto* c : g->members) {
        tally_step(c, scheme, M);
        c->time += dt;
      }
    }
    CK(cudaStreamSynchronize(g->stream));
    for (auto* c : g->members) {
      c->steps_issued += n_steps;
      check_dry(c, ("rank " + std::to_string(c->rank)).c_str());
    }
    return int(MSWM_OK);
  });
  if (rc) g->last_error = c0->last_error;
  return rc;
}

int mswm_cuda_group_nccl_loopback(mswm_cuda_group* g) {
  if (!g) return MSWM_E_USAGE;
  mswm_cuda_ctx* c0 = g->members[0];
  const int rc = guard(c0, [&] {
    CK(cudaSetDevice(c0->device));
    if (!g->loop) {
      ncclUniqueId id1, id2;
      nccl_check(nccl().GetUniqueId(&id1));
      nccl_check(nccl().CommInitRank(&g->loop, 1, id1, 0));
      nccl_check(nccl().GetUniqueId(&id2));
      nccl_check(nccl().CommInitRank(&g->loop2, 1, id2, 0));
    }
    for (auto* c : g->members) {
      c->loop_comm = g->loop;
      c->loop_comm2 = g->loop2;
      c->drop_graphs();
    }
    g->drop_graphs();
    return int(MSWM_OK);
  });
  if (rc) g->last_error = c0->last_error;
  return rc;
}

int mswm_cuda_group_peer(mswm_cuda_group* g, int on) {
  if (!g) return MSWM_E_USAGE;
  mswm_cuda_ctx* c0 = g->members[0];
  const int rc = guard(c0, [&] {
    CK(cudaSetDevice(c0->device));
    if (on) {
      for (auto* c : g->members) peer_prepare(c);
      for (auto* c : g->members)
        for (auto* d : g->members) {
          if (c == d) continue;
          bool nb = false;
          for (int p : c->halo.peer) nb |= p == d->rank;
          if (!nb) continue;
          const std::vector<int64_t> rows = peer_rows(d);
          peer_attach(c, d->rank, d->arena.p, false, rows.data(), int64_t(rows.size() / 5));
        }
    }
    for (auto* c : g->members) {
      peer_enable(c, on != 0);
      if (on) c->loop_comm = c->loop_comm2 = nullptr;
    }
    g->drop_graphs();
    return int(MSWM_OK);
  });
  if (rc) g->last_error = c0->last_error;
  return rc;
}

const char* mswm_cuda_group_last_error(const mswm_cuda_group* g) {
  return g ? g->last_error.c_str() : g_create_error.c_str();
}

}  // extern "C"
