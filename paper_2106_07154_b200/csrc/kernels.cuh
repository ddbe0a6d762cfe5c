// sm_100a device kernels of the LTS3 / TRiSK path.
//
// Every kernel keeps the reference's per-element IEEE operation sequence
// (proj/src/operators.cpp:61-116,
// proj/src/integrators.cpp:18-52,186-274,370-410) and is compiled with
// --fmad=false, so results are bitwise equal to the reference.  FP64
// gathers over SoA tables; nothing here is a dense contraction, so there are
// no tensor-core paths.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mswm_dev {

constexpr int kMaxDeg = 8;               // ring size bound (hexagons 6, pentagons 5)
constexpr int kMaxSten = 2 * kMaxDeg - 2;
// hexagon/pentagon meshes (every mesh of BASELINE.json): ring tables of 6
// slots, stencils of at most 10 -- the kernels' straight-line fast paths
constexpr int kFastDeg = 6;
constexpr int kFastSten = 10;
constexpr int kBlock = 256;
// threads per CTA of the three streamed evaluation kernels
#ifndef MSWM_SBLOCK
#define MSWM_SBLOCK 256
#endif
constexpr int kSBlock = MSWM_SBLOCK;
// minimum resident CTAs per SM requested from ptxas (register budget) for
// the streamed kernels; tuned on B200 (profiles/r1_*): a full SM of 2048 threads
#ifndef MSWM_KA_MINB
#define MSWM_KA_MINB (2048 / MSWM_SBLOCK)
#endif
#ifndef MSWM_KOUT_BATCH
#define MSWM_KOUT_BATCH 3   // coefficient pairs per batch
#endif
#ifndef MSWM_KOUT_MINB
#define MSWM_KOUT_MINB (2048 / MSWM_SBLOCK)
#endif
#if MSWM_KA_MINB > 0
#define MSWM_KA_BOUNDS __launch_bounds__(kSBlock, MSWM_KA_MINB)
#else
#define MSWM_KA_BOUNDS __launch_bounds__(kSBlock)
#endif
#if MSWM_KOUT_MINB > 0
#define MSWM_KOUT_BOUNDS __launch_bounds__(kSBlock, MSWM_KOUT_MINB)
#else
#define MSWM_KOUT_BOUNDS __launch_bounds__(kSBlock)
#endif

// Device mesh tables in internal numbering.  Slot-major SoA ([slot][elem])
// so consecutive threads of a warp read consecutive addresses.
struct DevMesh {
  int32_t nC, nE, nV;
  int32_t deg_max, sten_max;
  // cells
  const int32_t* __restrict__ c_edge;    // [deg_max][nC] ring edges
  const uint8_t* __restrict__ c_deg;     // [nC]
  const uint8_t* __restrict__ c_sbits;   // [nC] bit j: cell_sign(ring edge j, i) < 0
  const double* __restrict__ c_area;     // [nC] A_i
  // vertices
  const int32_t* __restrict__ v_cell;    // [3][nV]
  const int32_t* __restrict__ v_edge;    // [3][nV]
  const double* __restrict__ v_kite;     // [3][nV]
  const uint8_t* __restrict__ v_sbits;   // [nV] bit k: vertex_sign(v_edge k, v) < 0
  const double* __restrict__ v_area;     // [nV] A_v
  const int32_t* __restrict__ v_orig;    // [nV] original vertex id (error path only)
  // edges
  const int2* __restrict__ e_cells;      // [nE] (edge_cells[e][0], [1]) in stored order
  const int2* __restrict__ e_verts;      // [nE]
  const double* __restrict__ e_len;      // l_e
  const double* __restrict__ e_ld;       // l_e * d_e (the K product's first rounding)
  const double* __restrict__ e_dual;     // d_e
  const double* __restrict__ e_invd;     // 1.0 / d_e
  const uint8_t* __restrict__ e_nst;     // stencil length; bit 7: some e' - e outside int16
  const int32_t* __restrict__ e_sten;    // [sten_max][nE] edges_on_edge
  const uint2* __restrict__ e_st16;      // [(W+1)/2][nE], W = (sten_max+1)/2 u32 words of
                                         // e' - e as int16 pairs (entry 2k in the low half
                                         // of word k), two words per load (null: int32 only)
  const double2* __restrict__ e_coef2;   // [(sten_max+1)/2][nE] w * (l_{e'} * (1/d_e)) for
                                         // entries (2k, 2k+1): one 16 B load per pair
  // packed copies for the streamed kernels (fewer load instructions, same
  // coalescing: consecutive threads still read consecutive 8/16 B)
  const int2* __restrict__ c_edge2;      // [(deg_max+1)/2][nC] ring edges (2k, 2k+1)
  const int2* __restrict__ v_ce;         // [3][nV] (vertex_cells k, vertex_edges k)
  const double2* __restrict__ v_af;      // [nV] (A_v, f_v)
  // 16-bit index records (null: the int32 tables above only).  Each id is
  // stored as an int16 offset from a base proportional to the issuing
  // element's own id (pbase: edges, cells and vertices follow the same
  // space-filling curve, so an element's neighbours sit near id * n_to /
  // n_from); an element with an offset outside int16 (region seams, ~0.3 %)
  // is flagged "wide", and a warp holding one reads the int32 tables
  // instead (warp-uniform vote: the gathers stay back to back).
  const uint4* __restrict__ v_rec;       // [nV] 3 cells, 3 edges; w: bits 0-2 v_sbits, bit 7 wide
  const uint4* __restrict__ c_rec;       // [nC] 6 ring edges; w: byte 0 deg | wide << 7, byte 1 c_sbits
                                         // (deg_max == 6 meshes only)
  const uint2* __restrict__ e_cv16;      // [nE] (c0, c1), (v0, v1); a half 0x8000: wide
  const uint32_t* __restrict__ e_c16;    // [nE] (c0, c1) for kernel C; wide: e_nst bit 6
                                         // (also in e_st16's sixth word when sten_max == 10)
  uint32_t rq_ce, rf_ce;                 // base ratios n_to / n_from as q + f / 2^32:
  uint32_t rq_ve, rf_ve;                 //   cells per edge, vertices per edge,
  uint32_t rq_cv, rf_cv;                 //   cells per vertex, edges per vertex,
  uint32_t rq_ev, rf_ev;                 //   edges per cell
  uint32_t rq_ec, rf_ec;
  // fields
  const double* __restrict__ b;          // [nC]
  const double* __restrict__ f;          // [nV]
  double g;
};

// base id of a 16-bit offset record (host twin: pbase_host in mswm_cuda.cu)
__device__ __forceinline__ int32_t pbase(int32_t x, uint32_t q, uint32_t f) {
  return int32_t(q * uint32_t(x) + __umulhi(uint32_t(x), f));
}
__device__ __forceinline__ int32_t lo16(uint32_t w) { return int32_t(w << 16) >> 16; }
__device__ __forceinline__ int32_t hi16(uint32_t w) { return int32_t(w) >> 16; }
__device__ __forceinline__ bool has_sentinel16(uint32_t w) {
  return (w & 0xFFFFu) == 0x8000u || (w >> 16) == 0x8000u;
}

// (c0, c1) of edge e from its 16-bit record word
__device__ __forceinline__ int2 c16_cells(const DevMesh& M, int32_t e, uint32_t r) {
  const int32_t bc = pbase(e, M.rq_ce, M.rf_ce);
  return make_int2(bc + lo16(r), bc + hi16(r));
}

// A set of elements: the range [base, base+n_range) followed by list[0..n_list).
struct Span {
  int32_t base, n_range;
  const int32_t* list;
  int32_t n_list;
  __host__ __device__ __forceinline__ int32_t n() const { return n_range + n_list; }
  __device__ __forceinline__ int32_t at(int32_t t) const {
    return t < n_range ? base + t : list[t - n_range];
  }
};

// Chunk schedule of a two-part launch (kernel A: vertices | cells, kernel C:
// cells | edges): map[q] = index of the first element of the q-th kSBlock-sized
// chunk to run (part 0's elements are [0, n0), part 1's [n0, n0 + n1); a chunk
// never straddles the two).  Null: part 0's elements, then part 1's.  The host
// (chunk_map in mswm_cuda.cu) interleaves the parts' chunks in proportion, or
// window by window, so the CTAs resident at any time work on the same stretch
// of the space-filling curve in both parts and the second part's gathers (u,
// h; (F, q~)) hit lines the first part's just brought into L2.
struct ChunkMap {
  const int32_t* map;
  int32_t nq;
};

// Stage epilogue fused into the output kernel (integrators.cpp:18-52,
// 231-274, 370-410).  d is the freshly computed tendency of element i.
enum OpKind : int {
  OP_NONE = 0,
  OP_STORE,        // dst = d
  OP_EULER,        // dst = y0 + c0*d
  OP_WCOMB,        // dst = ((c0*y0) + (c1*y1)) + (c2*d), c2 = w_rhs*dt
  OP_ACC,          // acc = (first ? 0.0 : acc) + d
  OP_ACC_CORR,     // a3 = (first ? 0.0 : acc) + d;
                   // dst = y0 + c0*(((c1*a1) + (c1*a2)) + (c2*a3))
  OP_ACC_CORR2,    // second order: a2 = (first ? 0.0 : acc) + d;
                   // dst = y0 + c0*((c1*a1) + (c1*a2))
  OP_RK4_FIRST,    // acc = d;              dst = y0 + c0*d
  OP_RK4_MID,      // acc = acc + 2.0*d;    dst = y0 + c0*d
  OP_RK4_LAST,     // dst = y0 + c0*(acc + d)
};

struct Op {
  int kind;
  int first;
  double c0, c1, c2;
  double* dst;
  const double* y0;
  const double* y1;
  double* acc;
  const double* a1;
  const double* a2;
  // elements whose bit is set in altbits are written to alt[i] instead of
  // dst[i] (null altbits: never) -- the concurrent coarse step of the LTS3
  // schedule parks the values the substeps still read as h_old
  double* alt;
  const uint32_t* altbits;
};

__device__ __forceinline__ void apply_op(const Op& op_in, int32_t i, double d) {
  Op op = op_in;
  if (op.altbits && ((op.altbits[i >> 5] >> (i & 31)) & 1u)) op.dst = op.alt;
  switch (op.kind) {
    case OP_STORE:
      op.dst[i] = d;
      break;
    case OP_EULER:
      op.dst[i] = op.y0[i] + op.c0 * d;
      break;
    case OP_WCOMB:
      op.dst[i] = op.c0 * op.y0[i] + op.c1 * op.y1[i] + op.c2 * d;
      break;
    case OP_ACC:
      op.acc[i] = (op.first ? 0.0 : op.acc[i]) + d;
      break;
    case OP_ACC_CORR: {
      const double a3 = (op.first ? 0.0 : op.acc[i]) + d;
      op.dst[i] = op.y0[i] + op.c0 * (op.c1 * op.a1[i] + op.c1 * op.a2[i] + op.c2 * a3);
      break;
    }
    case OP_ACC_CORR2: {
      const double a2 = (op.first ? 0.0 : op.acc[i]) + d;
      op.dst[i] = op.y0[i] + op.c0 * (op.c1 * op.a1[i] + op.c1 * a2);
      break;
    }
    case OP_RK4_FIRST:
      op.acc[i] = d;
      op.dst[i] = op.y0[i] + op.c0 * d;
      break;
    case OP_RK4_MID:
      op.acc[i] = op.acc[i] + 2.0 * d;
      op.dst[i] = op.y0[i] + op.c0 * d;
      break;
    case OP_RK4_LAST: {
      const double a = op.acc[i] + d;
      op.dst[i] = op.y0[i] + op.c0 * a;
      break;
    }
    default:
      break;
  }
}

// Ring edge ids (six slots), ring size and sign bits of cell i on a
// deg_max == 6 mesh: from the 16-bit record unless the warp holds a wide cell.
__device__ __forceinline__ void ring_ids(const DevMesh& M, int32_t i, int32_t (&ce)[kFastDeg],
                                         int& deg, uint8_t* sbits = nullptr) {
  bool wide = true;
  if (M.c_rec) {
    const uint4 r = M.c_rec[i];
    deg = int(r.w & 0x7Fu);
    if (sbits) *sbits = uint8_t(r.w >> 8);
    wide = __any_sync(__activemask(), r.w & 0x80u);
    if (!wide) {
      const int32_t be = pbase(i, M.rq_ec, M.rf_ec);
      ce[0] = be + lo16(r.x);
      ce[1] = be + hi16(r.x);
      ce[2] = be + lo16(r.y);
      ce[3] = be + hi16(r.y);
      ce[4] = be + lo16(r.z);
      ce[5] = be + hi16(r.z);
    }
  } else {
    deg = M.c_deg[i];
    if (sbits) *sbits = M.c_sbits[i];
  }
  if (wide) {
#pragma unroll
    for (int k = 0; k < kFastDeg / 2; ++k) {
      const int2 p = M.c_edge2[k * M.nC + i];
      ce[2 * k] = p.x;
      ce[2 * k + 1] = p.y;
    }
  }
}

// ---------------------------------------------------------------------------
// Phase A: potential vorticity on the closure vertices (operators.cpp:74-86)
// and kinetic energy -> Bernoulli potential psi on the closure cells
// (:64-72, :112-113), one launch.
// one element of phase A (t indexes vs then ks)
__device__ __forceinline__ void item_vertex_cell(const DevMesh& M, const double* __restrict__ h,
                                                 const double* __restrict__ u, const Span& vs,
                                                 const Span& ks, double* __restrict__ pv,
                                                 double* __restrict__ K, unsigned long long* __restrict__ dry,
                                                 const int64_t* __restrict__ step_ctr,
                                                 const uint32_t* __restrict__ vmask, int32_t t) {
  // Spans may be supersets of the closure (dense ranges, slabs); the dry
  // check then consults the closure bitmask vmask so only closure vertices
  // raise, as in operators.cpp:74-84.
  const int32_t nv = vs.n();
  if (t < nv) {
    const int32_t v = vs.at(t);
    uint8_t sb;
    int2 ce[3];
    if (M.v_rec) {
      const uint4 r = M.v_rec[v];
      sb = uint8_t(r.w & 7u);
      if (!__any_sync(__activemask(), r.w & 0x80u)) {
        const int32_t bc = pbase(v, M.rq_cv, M.rf_cv), be = pbase(v, M.rq_ev, M.rf_ev);
        ce[0] = make_int2(bc + lo16(r.x), be + hi16(r.y));
        ce[1] = make_int2(bc + hi16(r.x), be + lo16(r.z));
        ce[2] = make_int2(bc + lo16(r.y), be + hi16(r.z));
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) ce[k] = M.v_ce[k * M.nV + v];
      }
    } else {
      sb = M.v_sbits[v];
#pragma unroll
      for (int k = 0; k < 3; ++k) ce[k] = M.v_ce[k * M.nV + v];
    }
    double hv = 0.0, circ = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) hv += M.v_kite[k * M.nV + v] * h[ce[k].x];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double d = M.e_dual[ce[k].y];
      circ += ((sb >> k) & 1 ? -d : d) * u[ce[k].y];
    }
    const double2 af = M.v_af[v];
    hv /= af.x;
    if (!(hv > 0.0)) {
      // (step << 32 | vertex): the earliest step wins, then the lowest id
      // (the reference reports the first dry vertex it meets; the tests
      // only require an adjacent valid id, test_operators.cpp:236-240)
      if (!vmask || ((vmask[v >> 5] >> (v & 31)) & 1u))
        atomicMin(dry, (static_cast<unsigned long long>(*step_ctr) << 32) |
                           static_cast<uint32_t>(M.v_orig[v]));
      pv[v] = 0.0;
      return;
    }
    pv[v] = (af.y + circ / af.x) / hv;
  } else if (t - nv < ks.n()) {
    const int32_t i = ks.at(t - nv);
    int deg;
    double acc = 0.0;
    if (M.deg_max == kFastDeg) {
      // all ring ids first, then all gathers: the loads of one cell are
      // independent and issue back to back (padding slots hold id 0, a
      // valid edge, and are not accumulated)
      int32_t ce[kFastDeg];
      ring_ids(M, i, ce, deg);
#pragma unroll
      for (int j = 0; j < kFastDeg; ++j) {
        const double ue = u[ce[j]];
        const double x = M.e_ld[ce[j]] * ue * ue;
        if (j < deg) acc += x;
      }
    } else {
      deg = M.c_deg[i];
      for (int j = 0; j < deg; ++j) {
        const int32_t e = M.c_edge[j * M.nC + i];
        const double ue = u[e];
        acc += M.e_ld[e] * ue * ue;
      }
    }
    // the Bernoulli potential psi_i = g (h_i + b_i) + K_i (operators.cpp:112-113),
    // formed here once per closure cell instead of twice per output edge
    // in phase C (same operations, same order: bitwise the reference's)
    const double Ki = acc / (4.0 * M.c_area[i]);
    K[i] = M.g * (h[i] + M.b[i]) + Ki;
  }
}

__global__ void MSWM_KA_BOUNDS k_vertex_cell(DevMesh M, const double* __restrict__ h,
                                             const double* __restrict__ u, Span vs, Span ks,
                                             double* __restrict__ pv, double* __restrict__ K,
                                             unsigned long long* __restrict__ dry,
                                             const int64_t* __restrict__ step_ctr,
                                             const uint32_t* __restrict__ vmask, ChunkMap cm) {
  const int32_t n0 = vs.n(), n = n0 + ks.n();
  const int32_t nt = cm.map ? cm.nq * kSBlock : n;
  for (int32_t t = blockIdx.x * kSBlock + threadIdx.x; t < nt; t += gridDim.x * kSBlock) {
    int32_t tt = t;
    if (cm.map) {
      const int32_t base = cm.map[t / kSBlock];
      tt = base + threadIdx.x;
      if (tt >= (base < n0 ? n0 : n)) continue;
    }
    item_vertex_cell(M, h, u, vs, ks, pv, K, dry, step_ctr, vmask, tt);
  }
}

// Phase B: thickness flux F_e (operators.cpp:61-62) and q~_e (:88-89) on the
// union of the flux and q~ closures, packed as (F, q~) so the stencil loop
// of phase C reads both with one 16-byte gather.
// ids of edge e's two cells and two vertices: 16-bit records unless the warp
// holds a wide edge
__device__ __forceinline__ void edge_cv(const DevMesh& M, int32_t e, int2& c, int2& v) {
  bool wide = true;
  if (M.e_cv16) {
    const uint2 r = M.e_cv16[e];
    wide = __any_sync(__activemask(), has_sentinel16(r.x) || has_sentinel16(r.y));
    if (!wide) {
      const int32_t bc = pbase(e, M.rq_ce, M.rf_ce), bv = pbase(e, M.rq_ve, M.rf_ve);
      c = make_int2(bc + lo16(r.x), bc + hi16(r.x));
      v = make_int2(bv + lo16(r.y), bv + hi16(r.y));
    }
  }
  if (wide) {
    c = M.e_cells[e];
    v = M.e_verts[e];
  }
}

__device__ __forceinline__ void item_edge_fq(const DevMesh& M, const double* __restrict__ h,
                                             const double* __restrict__ u,
                                             const double* __restrict__ pv, const Span& es,
                                             double2* __restrict__ FQ, int32_t t) {
  if (t >= es.n()) return;
  const int32_t e = es.at(t);
  int2 c, v;
  edge_cv(M, e, c, v);
  const double F = 0.5 * (h[c.x] + h[c.y]) * u[e];
  const double q = 0.5 * (pv[v.x] + pv[v.y]);
  FQ[e] = make_double2(F, q);
}

// (2 and 4 edges per thread -- more independent loads in flight, 40 registers
// -- measured slower on C4: 6.12 / 6.34 vs 5.93 ms per step,
// profiles/r2_s4_kernelB_unroll_sweep_c4.log)
__global__ void __launch_bounds__(kSBlock) k_edge_fq(DevMesh M, const double* __restrict__ h,
                                                   const double* __restrict__ u,
                                                   const double* __restrict__ pv, Span es,
                                                   double2* __restrict__ FQ, ChunkMap cm) {
  const int32_t n = es.n();
  const int32_t nt = cm.map ? cm.nq * kSBlock : n;
  for (int32_t t = blockIdx.x * kSBlock + threadIdx.x; t < nt; t += gridDim.x * kSBlock) {
    const int32_t tt = cm.map ? cm.map[t / kSBlock] + threadIdx.x : t;
    item_edge_fq(M, h, u, pv, es, FQ, tt);
  }
}

// Phase C: the output tendencies -- dh on out cells (operators.cpp:91-99),
// du on out edges (:101-116) -- with the stage update fused in.  Threads
// [0, nc) take cells, [nc, nc+ne) edges; lists are group-concatenated and
// split into two epilogue segments at csplit / esplit.
struct OutArgs {
  Span cs;               // output cells (a superset is fine: membership from ckey)
  Span es;               // output edges (membership from ekey)
  const uint8_t* ckey;   // GroupBit index per cell (null = every cell, segment 0)
  const uint8_t* ekey;   // GroupBit index - 6 per edge; 0xFF: not an output here
  uint32_t mask;
  Op cop[2];             // segment 0 = fine groups, 1 = the rest
  Op eop[2];
  ChunkMap cm;           // chunk schedule of cells | edges
};

__device__ __forceinline__ void item_out_cell(const DevMesh& M, const double2* __restrict__ FQ,
                                              const OutArgs& a, int32_t i) {
  {
    const int g = a.ckey ? a.ckey[i] : 0;
    if (g > 5 || !((a.mask >> g) & 1u)) return;  // 0xFF: not an output of this rank
    const int seg = g <= 2 ? 0 : 1;
    int deg;
    uint8_t sb;
    double acc = 0.0;
    if (M.deg_max == kFastDeg) {
      int32_t ce[kFastDeg];
      ring_ids(M, i, ce, deg, &sb);
#pragma unroll
      for (int j = 0; j < kFastDeg; ++j) {
        const double l = M.e_len[ce[j]];
        const double x = ((sb >> j) & 1 ? -l : l) * FQ[ce[j]].x;
        if (j < deg) acc += x;
      }
    } else {
      deg = M.c_deg[i];
      sb = M.c_sbits[i];
#pragma unroll
      for (int j = 0; j < kMaxDeg; ++j) {
        if (j < deg) {
          const int32_t e = M.c_edge[j * M.nC + i];
          const double l = M.e_len[e];
          acc += ((sb >> j) & 1 ? -l : l) * FQ[e].x;
        }
      }
    }
    const double dh = -acc / M.c_area[i];
    apply_op(a.cop[seg], i, dh);
  }
}

__device__ __forceinline__ void item_out_edge(const DevMesh& M, const double* __restrict__ K,
                                              const double2* __restrict__ FQ, const OutArgs& a,
                                              int32_t e) {
  {
    const int g = a.ekey ? a.ekey[e] : 0;
    if (g > 4 || !((a.mask >> (6 + g)) & 1u)) return;
    const int seg = g <= 1 ? 0 : 1;
    const double qt_e = FQ[e].y;
    const double inv_d = M.e_invd[e];
    const int nstw = M.e_nst[e];  // bits 0-5 stencil length, 6: e_c16 wide, 7: e_st16 wide
    // (c0, c1) for psi: 16-bit offsets (e_c16, or the spare sixth word of
    // the e_st16 row on ten-entry stencils) unless the warp holds an edge
    // whose offsets do not fit (e_nst bit 6)
    const bool wide_c = !M.e_c16 || __any_sync(__activemask(), nstw & 0x40);
    int2 cc;
    double pvflux = 0.0;
    {
      // Stencil ids as 16-bit offsets from e (20 B/edge instead of 40 B);
      // a warp holding any edge whose offsets do not fit (bit 7 of e_nst:
      // ~1 % of edges, along the curve's seams) reads the int32 table
      // instead.  The vote keeps the path warp-uniform, so the ten gathers
      // stay back to back.
      const int nst = nstw & 0x3f;
      const bool wide = !M.e_st16 || __any_sync(__activemask(), nstw & 0x80);
      if (!wide && M.sten_max == kFastSten) {
        // straight line: three 8 B loads of packed id words, then batches
        // of coefficient pairs (16 B) and (F, q~) gathers, predicated
        // accumulation (padding entries hold valid ids and are skipped)
        uint32_t w[kFastSten / 2 + 1];
#pragma unroll
        for (int k = (kFastSten / 2 + 1) / 2 - 1; k >= 0; --k) {
          const uint2 p = M.e_st16[k * M.nE + e];
          w[2 * k] = p.x;
          w[2 * k + 1] = p.y;
          if (k == (kFastSten / 2 + 1) / 2 - 1)
            cc = wide_c ? M.e_cells[e] : c16_cells(M, e, w[kFastSten / 2]);
        }
#pragma unroll
        for (int j0 = 0; j0 < kFastSten; j0 += 2 * MSWM_KOUT_BATCH) {
          double2 c[MSWM_KOUT_BATCH];
          double2 fq[2 * MSWM_KOUT_BATCH];
#pragma unroll
          for (int b = 0; b < 2 * MSWM_KOUT_BATCH; ++b) {
            const int j = j0 + b;
            if (j < kFastSten) {
              if (!(b & 1)) c[b >> 1] = M.e_coef2[(j >> 1) * M.nE + e];
              const int32_t e2 = e + (j & 1 ? int32_t(w[j >> 1]) >> 16
                                            : int32_t(w[j >> 1] << 16) >> 16);
              fq[b] = FQ[e2];
            }
          }
#pragma unroll
          for (int b = 0; b < 2 * MSWM_KOUT_BATCH; ++b) {
            const int j = j0 + b;
            if (j < kFastSten) {
              const double cj = b & 1 ? c[b >> 1].y : c[b >> 1].x;
              const double x = cj * fq[b].x * (0.5 * (qt_e + fq[b].y));
              if (j < nst) pvflux += x;
            }
          }
        }
      } else if (M.sten_max == kFastSten) {
        // the int32 ids (~9 % of warps on C4), same straight-line batches
        cc = wide_c ? M.e_cells[e] : c16_cells(M, e, M.e_c16[e]);
#pragma unroll
        for (int j0 = 0; j0 < kFastSten; j0 += 2 * MSWM_KOUT_BATCH) {
          double2 c[MSWM_KOUT_BATCH];
          double2 fq[2 * MSWM_KOUT_BATCH];
#pragma unroll
          for (int b = 0; b < 2 * MSWM_KOUT_BATCH; ++b) {
            const int j = j0 + b;
            if (j < kFastSten) {
              if (!(b & 1)) c[b >> 1] = M.e_coef2[(j >> 1) * M.nE + e];
              fq[b] = FQ[M.e_sten[j * M.nE + e]];
            }
          }
#pragma unroll
          for (int b = 0; b < 2 * MSWM_KOUT_BATCH; ++b) {
            const int j = j0 + b;
            if (j < kFastSten) {
              const double cj = b & 1 ? c[b >> 1].y : c[b >> 1].x;
              const double x = cj * fq[b].x * (0.5 * (qt_e + fq[b].y));
              if (j < nst) pvflux += x;
            }
          }
        }
      } else {
        cc = wide_c ? M.e_cells[e] : c16_cells(M, e, M.e_c16[e]);
#pragma unroll
        for (int j = 0; j < kMaxSten; ++j) {
          if (j < nst) {
            const int32_t e2 = M.e_sten[j * M.nE + e];
            const double2 cp = M.e_coef2[(j >> 1) * M.nE + e];
            const double c = j & 1 ? cp.y : cp.x;
            const double2 fq = FQ[e2];
            pvflux += c * fq.x * (0.5 * (qt_e + fq.y));
          }
        }
      }
    }
    const double psi_lo = K[cc.x];  // psi (phase A)
    const double psi_hi = K[cc.y];
    const double du = -pvflux - (psi_lo - psi_hi) * inv_d;
    apply_op(a.eop[seg], e, du);
  }
}

__device__ __forceinline__ void item_out(const DevMesh& M, const double* __restrict__ K,
                                         const double2* __restrict__ FQ, const OutArgs& a,
                                         int32_t t) {
  const int32_t ncs = a.cs.n();
  if (t < ncs)
    item_out_cell(M, FQ, a, a.cs.at(t));
  else if (t - ncs < a.es.n())
    item_out_edge(M, K, FQ, a, a.es.at(t - ncs));
}

__global__ void MSWM_KOUT_BOUNDS k_out(DevMesh M, const double* __restrict__ h,
                                     const double* __restrict__ K,
                                     const double2* __restrict__ FQ, OutArgs a) {
  const int32_t n0 = a.cs.n(), n = n0 + a.es.n();
  const int32_t nt = a.cm.map ? a.cm.nq * kSBlock : n;
  for (int32_t t = blockIdx.x * kSBlock + threadIdx.x; t < nt; t += gridDim.x * kSBlock) {
    int32_t tt = t;
    if (a.cm.map) {
      const int32_t base = a.cm.map[t / kSBlock];
      tt = base + threadIdx.x;
      if (tt >= (base < n0 ? n0 : n)) continue;
    }
    item_out(M, K, FQ, a, tt);
  }
}

// ---------------------------------------------------------------------------
// Interface-1 prediction (integrators.cpp:217-227): order 3
// dst = ((c0*s0) + (c1*s1)) + (c2*s2), order 2 (s2 null) (c0*s0) + (c1*s1),
// on the I1 lists.
__global__ void k_predict(const int32_t* __restrict__ clist, int32_t nc,
                          const int32_t* __restrict__ elist, int32_t ne, double c0, double c1,
                          double c2, const double* __restrict__ hs0, const double* __restrict__ hs1,
                          const double* __restrict__ hs2, double* __restrict__ hdst,
                          const double* __restrict__ us0, const double* __restrict__ us1,
                          const double* __restrict__ us2, double* __restrict__ udst) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nc) {
    const int32_t i = clist[t];
    // second order (hs2 null): w_old*y_old + w_first*y1 (integrators.cpp:221-222)
    hdst[i] = hs2 ? c0 * hs0[i] + c1 * hs1[i] + c2 * hs2[i] : c0 * hs0[i] + c1 * hs1[i];
  } else if (t - nc < ne) {
    const int32_t e = elist[t - nc];
    udst[e] = us2 ? c0 * us0[e] + c1 * us1[e] + c2 * us2[e] : c0 * us0[e] + c1 * us1[e];
  }
}

// Substep prologue: save the values the predictions and the correction
// read (old state on I1 u I2, stage-1/2 values on I1), then write the
// stage-1 prediction of substep 0.  Lists are [I1 | I2].  Second order:
// H2 / U2 null, no second stage value, two-term prediction.
__global__ void k_save_predict(const int32_t* __restrict__ clist, int32_t nc, int32_t nc1,
                               const int32_t* __restrict__ elist, int32_t ne, int32_t ne1,
                               double c0, double c1, double c2, double* __restrict__ H,
                               const double* __restrict__ H1, const double* __restrict__ H2,
                               double* __restrict__ HS0, double* __restrict__ HS1,
                               double* __restrict__ HS2, double* __restrict__ U,
                               const double* __restrict__ U1, const double* __restrict__ U2,
                               double* __restrict__ US0, double* __restrict__ US1,
                               double* __restrict__ US2) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nc) {
    const int32_t i = clist[t];
    const double y0 = H[i];
    HS0[i] = y0;
    if (t < nc1) {
      const double y1 = H1[i];
      HS1[i] = y1;
      if (H2) {
        const double y2 = H2[i];
        HS2[i] = y2;
        H[i] = c0 * y0 + c1 * y1 + c2 * y2;
      } else {
        H[i] = c0 * y0 + c1 * y1;
      }
    }
  } else if (t - nc < ne) {
    const int32_t q = t - nc;
    const int32_t e = elist[q];
    const double y0 = U[e];
    US0[e] = y0;
    if (q < ne1) {
      const double y1 = U1[e];
      US1[e] = y1;
      if (U2) {
        const double y2 = U2[e];
        US2[e] = y2;
        U[e] = c0 * y0 + c1 * y1 + c2 * y2;
      } else {
        U[e] = c0 * y0 + c1 * y1;
      }
    }
  }
}

// Interface-1 prediction as a data structure (for the fused kernel).
struct PredArgs {
  const int32_t *clist, *elist;
  int32_t nc, ne;
  double c0, c1, c2;
  const double *hs0, *hs1, *hs2, *us0, *us1, *us2;
  double *hdst, *udst;
};

__device__ __forceinline__ void item_predict(const PredArgs& p, int32_t t) {
  if (t < p.nc) {
    const int32_t i = p.clist[t];
    p.hdst[i] = p.hs2 ? p.c0 * p.hs0[i] + p.c1 * p.hs1[i] + p.c2 * p.hs2[i]
                      : p.c0 * p.hs0[i] + p.c1 * p.hs1[i];
  } else if (t - p.nc < p.ne) {
    const int32_t e = p.elist[t - p.nc];
    p.udst[e] = p.us2 ? p.c0 * p.us0[e] + p.c1 * p.us1[e] + p.c2 * p.us2[e]
                      : p.c0 * p.us0[e] + p.c1 * p.us1[e];
  }
}

// First node of every step graph: the 1-based index of the coarse step in
// flight since the context was created (dry-vertex reports, harness.cpp:183-190).
__global__ void k_step_counter(int64_t* ctr) { ++*ctr; }

// Halo exchange pack/unpack: code >= 0 is a cell id (h array), code < 0 is
// ~edge id (u array).
__global__ void k_pack(int64_t n, const int32_t* __restrict__ code, const double* __restrict__ h,
                       const double* __restrict__ u, double* __restrict__ buf) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t c = code[k];
  buf[k] = c >= 0 ? h[c] : u[~c];
}
__global__ void k_unpack(int64_t n, const int32_t* __restrict__ code, const double* __restrict__ buf,
                         double* __restrict__ h, double* __restrict__ u) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t c = code[k];
  if (c >= 0)
    h[c] = buf[k];
  else
    u[~c] = buf[k];
}
// Unpack fused with the next stage's interface-1 prediction (ranks: the
// prediction writes the next stage's input array on I1, which neither this
// exchange nor this stage's evaluation touches) -- one launch fewer per
// substep stage on the latency-bound chain.
__global__ void k_unpack_pred(int64_t n, const int32_t* __restrict__ code,
                              const double* __restrict__ buf, double* __restrict__ h,
                              double* __restrict__ u, PredArgs pa) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) {
    const int32_t c = code[k];
    if (c >= 0)
      h[c] = buf[k];
    else
      u[~c] = buf[k];
  } else if (k - n < int64_t(pa.nc) + pa.ne) {
    item_predict(pa, int32_t(k - n));
  }
}

// ---------------------------------------------------------------------------
// Peer-store halo transport: the pack kernel stores straight into the
// receivers' buffers through peer-mapped pointers (CUDA IPC between processes,
// NVLink / NVSwitch peer access; plain pointers inside an in-process group)
// and then raises a flag at every neighbour; the unpack kernel waits for its
// neighbours' flags.  One exchange = two launches and no library call.
//
// Protocol (per channel: 0 = main schedule, 1 = the concurrent coarse stage):
// every rank performs the same sequence of exchanges on a channel, and every
// exchange signals and awaits ALL neighbours (also those it has no data for), so
// an exchange is a neighbourhood barrier.  seq = 1, 2, ... counts the channel's
// exchanges in a device counter (graph replays need no patched arguments);
// receive regions are double buffered on seq & 1: a sender can run at most
// one exchange ahead of a neighbour (it needs that neighbour's flag of
// exchange n + 1, raised after the neighbour's unpack of n in stream order,
// before it may store exchange n + 2 into the half n used).
struct PeerSlot {
  double* dst;                 // the neighbour's receive region for this rank's values (half 0)
  int64_t stride;              // doubles between the two halves of that region
  unsigned long long* flag;    // the neighbour's flag word for (channel 0, this rank)
  int64_t soff;                // first send item of this slot
};

__device__ __forceinline__ unsigned long long ld_flag(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_flag(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// pack + store into the neighbours' buffers + signal.  chan[0] = seq of the
// channel's last finished exchange, chan[1] = block arrival counter (as u64).
__global__ void k_push(int64_t n, const int32_t* __restrict__ code, const uint8_t* __restrict__ sslot,
                       const double* __restrict__ h, const double* __restrict__ u,
                       const PeerSlot* __restrict__ slots, int np, int flag_stride,
                       unsigned long long* chan) {
  __shared__ bool last;
  const unsigned long long seq = chan[0] + 1;
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) {
    const int32_t c = code[k];
    const PeerSlot s = slots[sslot[k]];
    s.dst[int64_t(seq & 1) * s.stride + (k - s.soff)] = c >= 0 ? h[c] : u[~c];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(chan + 1, 1ull) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  // every block's stores are fenced: publish
  __threadfence_system();
  for (int j = threadIdx.x; j < np; j += blockDim.x) st_flag(slots[j].flag + flag_stride, seq);
  if (threadIdx.x == 0) {
    chan[1] = 0;
    chan[0] = seq;
  }
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// wait for every neighbour's flag of this exchange, then unpack (and the
// fused interface-1 prediction, as k_unpack_pred).  flags: this rank's flag
// words of the channel, indexed by rank.  A neighbour that does not answer
// within budget_ns sets *err (1 + its rank; reported as MSWM_E_NCCL by the
// next synchronous call) instead of hanging the device, and once *err is set
// no later wait polls.
__global__ void k_wait_unpack(int64_t n, const int32_t* __restrict__ code, const double* rbuf,
                              int64_t stride, double* __restrict__ h, double* __restrict__ u,
                              PredArgs pa, const unsigned long long* flags,
                              const int32_t* __restrict__ peers, int np,
                              const unsigned long long* chan, int* err,
                              unsigned long long budget_ns) {
  const unsigned long long seq = chan[0];
  if (threadIdx.x < np) {
    const unsigned long long* f = flags + peers[threadIdx.x];
    if (ld_flag(f) < seq) {
      const unsigned long long t0 = global_ns();
      while (ld_flag(f) < seq) {
        __nanosleep(100);
        if (*reinterpret_cast<volatile int*>(err)) break;
        if (global_ns() - t0 > budget_ns) {
          atomicCAS(err, 0, 1 + peers[threadIdx.x]);
          break;
        }
      }
    }
  }
  __syncthreads();
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) {
    const int32_t c = code[k];
    const double v = __ldcg(rbuf + int64_t(seq & 1) * stride + k);
    if (c >= 0)
      h[c] = v;
    else
      u[~c] = v;
  } else if (k - n < int64_t(pa.nc) + pa.ne) {
    item_predict(pa, int32_t(k - n));
  }
}

// Boundary permutations between the caller's numbering and the internal one.
__global__ void k_gather_perm(int32_t n, const int32_t* __restrict__ n2o,
                              const double* __restrict__ src, double* __restrict__ dst) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[n2o[i]];
}
__global__ void k_scatter_perm(int32_t n, const int32_t* __restrict__ n2o,
                               const double* __restrict__ src, double* __restrict__ dst) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[n2o[i]] = src[i];
}


// ---------------------------------------------------------------------------
// Region classification (regions.cpp:14-162) on device.

// One BFS layer: unvisited cells with a neighbour at distance level-1 get
// `level`.  In-place is safe: a cell set to `level` in this launch never
// matches level-1.  Counts the layer.
__global__ void k_bfs_layer(DevMesh M, const int32_t* __restrict__ c_nbr, int32_t* dist, int level,
                            int32_t* counter) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.nC || dist[i] != -1) return;
  const int deg = M.c_deg[i];
  for (int j = 0; j < deg; ++j)
    if (dist[c_nbr[j * M.nC + i]] == level - 1) {
      dist[i] = level;
      atomicAdd(counter, 1);
      return;
    }
}

// labels: 0 fine, 1 interface1, 2 interface2, 3 coarse (regions.hpp:12)
__global__ void k_cell_labels(int32_t nC, const int32_t* __restrict__ dist, int w,
                              uint8_t* __restrict__ label, uint8_t* __restrict__ sub) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nC) return;
  const int d = dist[i];
  label[i] = d == 0 ? 0 : (d >= 1 && d <= w ? 1 : (d > w && d <= 2 * w ? 2 : 3));
  sub[i] = 0;
}

// underline layers (regions.cpp:107-139); pass 1 then pass 2
__global__ void k_underline(DevMesh M, const int32_t* __restrict__ c_nbr,
                            const uint8_t* __restrict__ label, uint8_t* __restrict__ sub, int pass) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.nC || label[i] != 0) return;
  const int deg = M.c_deg[i];
  if (pass == 1) {
    for (int j = 0; j < deg; ++j)
      if (label[c_nbr[j * M.nC + i]] == 1) {
        sub[i] = 1;
        return;
      }
  } else {
    if (sub[i] != 0) return;
    for (int j = 0; j < deg; ++j) {
      const int32_t nb = c_nbr[j * M.nC + i];
      if (label[nb] == 0 && sub[nb] == 1) {
        sub[i] = 2;
        return;
      }
    }
  }
}

__device__ __forceinline__ int cell_rank(uint8_t label, uint8_t sub) {
  return label == 0 ? (sub == 0 ? 0 : 1) : int(label) + 1;
}

// edge labels: fine side wins (regions.cpp:141-162); also the compaction
// keys (GroupBit index) of cells and edges.
__global__ void k_edge_labels_and_keys(DevMesh M, const uint8_t* __restrict__ label,
                                       const uint8_t* __restrict__ sub,
                                       uint8_t* __restrict__ elabel, uint8_t* __restrict__ ckey,
                                       uint8_t* __restrict__ ekey) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < M.nE) {
    const int2 c = M.e_cells[t];
    const int r0 = cell_rank(label[c.x], sub[c.x]);
    const int r1 = cell_rank(label[c.y], sub[c.y]);
    const uint8_t r = uint8_t(r0 < r1 ? r0 : r1);
    elabel[t] = r;
    ekey[t] = r;
  }
  if (t < M.nC) {
    const uint8_t l = label[t], s = sub[t];
    ckey[t] = l == 0 ? s : uint8_t(l + 2);  // 0 plain, 1 uf1, 2 uf2, 3 if1, 4 if2, 5 coarse
  }
}

// validate_regions (regions.cpp:173-288) for label arrays the caller supplies:
// band distances (:213-244), underline sublabels (:247-262, sub null: not
// assigned) and the fine-side-wins edge rule (:265-286, elabel null: not
// assigned).  dist holds the BFS layers 1..2w from the label-0 set (-1:
// farther).  Per check kind the number of offending elements and the lowest
// original id (the one the reference reports first).
enum ValidateKind : int {
  VK_VALUE = 0,    // label / sublabel value out of range, sublabel on a non-fine cell
  VK_IF1,          // Interface1 cell outside distance 1..w
  VK_IF2,          // Interface2 cell outside w+1..2w
  VK_COARSE,       // coarse cell within 2w
  VK_UNDERLINE,    // fine cell with the wrong underline sublabel
  VK_EDGE,         // edge label disagrees with the fine-side-wins rule
  VK_COUNT
};

__device__ __forceinline__ void validate_hit(int kind, int32_t orig, unsigned long long* count,
                                             int32_t* first) {
  atomicAdd(count + kind, 1ull);
  atomicMin(first + kind, orig);
}

__global__ void k_validate_labels(DevMesh M, const int32_t* __restrict__ c_nbr,
                                  const int32_t* __restrict__ dist, int w,
                                  const uint8_t* __restrict__ label, const uint8_t* __restrict__ sub,
                                  const uint8_t* __restrict__ elabel,
                                  const int32_t* __restrict__ c_new2old,
                                  const int32_t* __restrict__ e_new2old,
                                  unsigned long long* count, int32_t* first) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < M.nC) {
    const int l = label[t];
    const int s = sub ? sub[t] : 0;
    const int32_t orig = c_new2old[t];
    if (l > 3 || s > 2 || (l != 0 && s != 0)) {
      validate_hit(VK_VALUE, orig, count, first);
    } else {
      const int d = dist[t] == -1 ? INT32_MAX : dist[t];
      if (l == 1 && (d < 1 || d > w)) validate_hit(VK_IF1, orig, count, first);
      if (l == 2 && (d <= w || d > 2 * w)) validate_hit(VK_IF2, orig, count, first);
      if (l == 3 && d <= 2 * w) validate_hit(VK_COARSE, orig, count, first);
      if (l == 0 && sub) {
        bool touch_i1 = false, touch_uf1 = false;
        const int deg = M.c_deg[t];
        for (int j = 0; j < deg; ++j) {
          const int32_t nb = c_nbr[j * M.nC + t];
          if (label[nb] == 1) touch_i1 = true;
          if (label[nb] == 0 && sub[nb] == 1) touch_uf1 = true;
        }
        const int want = touch_i1 ? 1 : (touch_uf1 ? 2 : 0);
        if (s != want) validate_hit(VK_UNDERLINE, orig, count, first);
      }
    }
  }
  if (elabel && t < M.nE) {
    const int2 c = M.e_cells[t];
    const int r0 = cell_rank(label[c.x], sub ? sub[c.x] : 0);
    const int r1 = cell_rank(label[c.y], sub ? sub[c.y] : 0);
    if (elabel[t] != (r0 < r1 ? r0 : r1)) validate_hit(VK_EDGE, e_new2old[t], count, first);
  }
}

// ---------------------------------------------------------------------------
// Closure marking (operators.cpp:35-58) for one mask's out lists.
// mf: flux marks (ring edges of out cells and of both cells of out edges)
// mq: q~ marks (out edges and ring edges of both cells of out edges)
// mk: K cells (both cells of out edges); mv: PV vertices (their ring vertices)
__global__ void k_mark_closure(DevMesh M, const int32_t* __restrict__ c_vert,
                               const int32_t* __restrict__ clist, int32_t nc,
                               const int32_t* __restrict__ elist, int32_t ne,
                               uint8_t* __restrict__ mf, uint8_t* __restrict__ mq,
                               uint8_t* __restrict__ mk, uint8_t* __restrict__ mv) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nc) {
    const int32_t i = clist[t];
    const int deg = M.c_deg[i];
    for (int j = 0; j < deg; ++j) mf[M.c_edge[j * M.nC + i]] = 1;
  } else if (t - nc < ne) {
    const int32_t e = elist[t - nc];
    mq[e] = 1;
    const int2 cc = M.e_cells[e];
    for (int side = 0; side < 2; ++side) {
      const int32_t i = side ? cc.y : cc.x;
      mk[i] = 1;
      const int deg = M.c_deg[i];
      for (int j = 0; j < deg; ++j) {
        const int32_t e2 = M.c_edge[j * M.nC + i];
        mf[e2] = 1;
        mq[e2] = 1;
        mv[c_vert[j * M.nC + i]] = 1;
      }
    }
  }
}

// Halo plan of a partition (make_block_plan's 2-hop rule, partition.cpp:
// 355-392) for every rank at once: reach[c] = bit set of the ranks whose
// local mesh (owned cells + cells within two hops) holds c.  One OR over the
// ring neighbours per hop; an edge / vertex belongs to the local mesh of every
// rank that holds one of its cells.
__global__ void k_reach_init(int32_t nC, const int32_t* __restrict__ rank_of_cell,
                             uint64_t* __restrict__ reach) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nC) reach[i] = uint64_t(1) << rank_of_cell[i];
}
__global__ void k_reach_hop(DevMesh M, const int32_t* __restrict__ c_nbr,
                            const uint64_t* __restrict__ in, uint64_t* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.nC) return;
  uint64_t r = in[i];
  for (int j = 0; j < M.c_deg[i]; ++j) r |= in[c_nbr[j * M.nC + i]];
  out[i] = r;
}
__global__ void k_reach_ev(DevMesh M, const uint64_t* __restrict__ cr, uint64_t* __restrict__ er,
                           uint64_t* __restrict__ vr) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < M.nE) {
    const int2 c = M.e_cells[t];
    er[t] = cr[c.x] | cr[c.y];
  } else if (t - M.nE < M.nV) {
    const int32_t v = t - M.nE;
    vr[v] = cr[M.v_cell[v]] | cr[M.v_cell[M.nV + v]] | cr[M.v_cell[2 * M.nV + v]];
  }
}

// Partition of the mesh for N ranks (partition.cpp:219-231, 338-353).
// Region class of a cell: 0 fine (incl. underline), 1 coarse, 2 interface
// (partition.cpp:16-25); of an edge: 0 fine / underline fine, 1 coarse, 2
// interfaces (:27-37).
__device__ __forceinline__ uint8_t part_cell_class(uint8_t label) {
  return label == 0 ? 0 : (label == 3 ? 1 : 2);
}
// key[k] = class of the k-th cell of the sweep (ord: internal ids)
__global__ void k_part_class(int32_t n, const int32_t* __restrict__ ord,
                             const uint8_t* __restrict__ label, uint8_t* __restrict__ key) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) key[k] = part_cell_class(label[ord[k]]);
}
// lst: sweep positions grouped by class (ascending inside each, sizes t[3]);
// position p of its class's run goes to part p * N / t (partition.cpp:219-231)
__global__ void k_part_assign(int32_t n, const int32_t* __restrict__ lst,
                              const int32_t* __restrict__ ord, int64_t t0, int64_t t1, int64_t t2,
                              int n_parts, int32_t* __restrict__ rank) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t base = 0, t = t0;
  if (j >= t0 + t1) {
    base = t0 + t1;
    t = t2;
  } else if (j >= t0) {
    base = t0;
    t = t1;
  }
  rank[ord[lst[j]]] = int32_t((int64_t(j) - base) * n_parts / t);
}
// owner of an edge: the rank of its first cell (edge_cells order) whose class
// is the edge's (partition.cpp:338-353); bad = lowest edge without one
__global__ void k_part_edge_owner(DevMesh M, const uint8_t* __restrict__ clabel,
                                  const uint8_t* __restrict__ elabel,
                                  const int32_t* __restrict__ rank, int32_t* __restrict__ owner,
                                  int32_t* __restrict__ bad) {
  const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M.nE) return;
  const uint8_t el = elabel[e];
  const uint8_t ec = el <= 1 ? 0 : (el == 4 ? 1 : 2);
  const int2 c = M.e_cells[e];
  if (part_cell_class(clabel[c.x]) == ec) {
    owner[e] = rank[c.x];
  } else if (part_cell_class(clabel[c.y]) == ec) {
    owner[e] = rank[c.y];
  } else {
    owner[e] = -1;
    atomicMin(bad, e);
  }
}

// Halo dependence of a rank's evaluations (interior / boundary split of the
// multi-rank schedule).  A halo element is one this rank does not own
// (key 0xFF); every value computed from one is "tainted".
// tv[v]: q_v reads h / u of a halo element (operators.cpp:74-86).
__global__ void k_taint_vertices(DevMesh M, const uint8_t* __restrict__ ckey,
                                 const uint8_t* __restrict__ ekey, uint8_t* __restrict__ tv) {
  const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= M.nV) return;
  uint8_t t = 0;
  for (int k = 0; k < 3; ++k)
    t |= (ckey[M.v_cell[k * M.nV + v]] == 0xFF) | (ekey[M.v_edge[k * M.nV + v]] == 0xFF);
  tv[v] = t;
}
// tf[e]: F_e or q~_e is tainted (:61-62, :88-89); tp[i]: psi_i is (:64-72, :112).
__global__ void k_taint_fp(DevMesh M, const uint8_t* __restrict__ ckey,
                           const uint8_t* __restrict__ ekey, const uint8_t* __restrict__ tv,
                           uint8_t* __restrict__ tf, uint8_t* __restrict__ tp) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < M.nE) {
    const int2 c = M.e_cells[t];
    const int2 v = M.e_verts[t];
    tf[t] = (ekey[t] == 0xFF) | (ckey[c.x] == 0xFF) | (ckey[c.y] == 0xFF) | tv[v.x] | tv[v.y];
  } else if (t - M.nE < M.nC) {
    const int32_t i = t - M.nE;
    uint8_t x = ckey[i] == 0xFF;
    for (int j = 0; j < M.c_deg[i]; ++j) x |= ekey[M.c_edge[j * M.nC + i]] == 0xFF;
    tp[i] = x;
  }
}
// Boundary outputs: dh_i reads (F, q~) of its ring (:91-99); du_e reads its
// own q~, (F, q~) of its stencil = the rest of both cells' rings, and psi of
// both cells (:101-116).  Everything else is interior: computable before
// the halo exchange lands.
__global__ void k_mark_boundary(DevMesh M, const uint8_t* __restrict__ tf,
                                const uint8_t* __restrict__ tp, uint8_t* __restrict__ cb,
                                uint8_t* __restrict__ eb) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < M.nC) {
    uint8_t x = 0;
    for (int j = 0; j < M.c_deg[t]; ++j) x |= tf[M.c_edge[j * M.nC + t]];
    cb[t] = x;
  } else if (t - M.nC < M.nE) {
    const int32_t e = t - M.nC;
    const int2 c = M.e_cells[e];
    uint8_t x = tf[e] | tp[c.x] | tp[c.y];
    for (int side = 0; side < 2; ++side) {
      const int32_t i = side ? c.y : c.x;
      for (int j = 0; j < M.c_deg[i]; ++j) x |= tf[M.c_edge[j * M.nC + i]];
    }
    eb[e] = x;
  }
}
// Compaction key of one part of a mask's outputs: owned, in the mask, and
// boundary flag == want.
__global__ void k_part_key(int32_t n, const uint8_t* __restrict__ key, int shift, uint32_t mask,
                           int gmax, const uint8_t* __restrict__ bnd, uint8_t want,
                           uint8_t* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int g = key[i];
  out[i] = (g <= gmax && ((mask >> (shift + g)) & 1u) && bnd[i] == want) ? 0 : 0xFF;
}

// Elements whose h (cells) or u (edges) one masked evaluation reads
// (operators.cpp:61-86 over the closure lists): cells and edges of the PV
// vertices, ring edges of the K cells, flux edges and their cells, and the
// cells of the output edges (psi).  Outputs' own values are the rank's.
__global__ void k_mark_reads(DevMesh M, const int32_t* __restrict__ vl, int32_t nv,
                             const int32_t* __restrict__ kl, int32_t nk,
                             const int32_t* __restrict__ fl, int32_t nf,
                             const int32_t* __restrict__ ol, int32_t no,
                             uint8_t* __restrict__ cread, uint8_t* __restrict__ eread) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nv) {
    const int32_t v = vl[t];
    for (int k = 0; k < 3; ++k) {
      cread[M.v_cell[k * M.nV + v]] = 1;
      eread[M.v_edge[k * M.nV + v]] = 1;
    }
    return;
  }
  t -= nv;
  if (t < nk) {
    const int32_t i = kl[t];
    for (int j = 0; j < M.c_deg[i]; ++j) eread[M.c_edge[j * M.nC + i]] = 1;
    return;
  }
  t -= nk;
  if (t < nf) {
    const int32_t e = fl[t];
    eread[e] = 1;
    cread[M.e_cells[e].x] = 1;
    cread[M.e_cells[e].y] = 1;
    return;
  }
  t -= nf;
  if (t < no) {
    const int32_t e = ol[t];
    cread[M.e_cells[e].x] = 1;
    cread[M.e_cells[e].y] = 1;
  }
}

// key = 0 where either mark is set, 0xFF elsewhere (closure-union key)
__global__ void k_union_key(int32_t n, const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                            uint8_t* __restrict__ key) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = (a[i] | b[i]) ? 0 : 0xFF;
}

// ---------------------------------------------------------------------------
// Diagnostics (harness.cpp:99-123, integrators.cpp:632-659).

// Per-cell terms of total_mass and total_energy in the reference's per-cell
// operation order; cells with ckey 0xFF (not owned by this rank) give 0.
__global__ void k_cell_diag(DevMesh M, const double* __restrict__ h, const double* __restrict__ u,
                            const uint8_t* __restrict__ ckey, double* __restrict__ mass_t,
                            double* __restrict__ energy_t) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.nC) return;
  if (ckey && ckey[i] > 5) {
    mass_t[i] = 0.0;
    energy_t[i] = 0.0;
    return;
  }
  const int deg = M.c_deg[i];
  double k = 0.0;
  for (int j = 0; j < deg; ++j) {
    const int32_t e = M.c_edge[j * M.nC + i];
    const double ue = u[e];
    k += M.e_ld[e] * ue * ue;  // ((l d) u) u
  }
  const double A = M.c_area[i];
  k /= 4.0 * A;
  const double hi = h[i];
  mass_t[i] = A * hi;
  energy_t[i] = A * (hi * k + 0.5 * M.g * hi * (hi + 2.0 * M.b[i]));
}

// Fixed-shape two-level sum (deterministic for a given n, not the
// sequential rounding): block b sums [b*chunk, (b+1)*chunk) as a strided
// per-thread sum and a shared-memory tree; then one block sums the partials.
__global__ void __launch_bounds__(kBlock) k_sum_chunks(int32_t n, int32_t chunk,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ partial) {
  __shared__ double sm[kBlock];
  const int32_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double acc = 0.0;
  for (int32_t i = lo + threadIdx.x; i < hi; i += kBlock) acc += x[i];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kBlock / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sm[0];
}

// Courant numbers: max of step |u_e| / d_e over fine (edge groups 6-7, step
// dt/M) and coarse (8-10, step dt) edges; without regions every edge at dt
// into slot 0.  Non-negative doubles order like their bit patterns, so the
// maxima are exact atomicMax results; NaNs never win (c > target is false).
__global__ void __launch_bounds__(kBlock) k_courant(DevMesh M, const double* __restrict__ u,
                                                    const uint8_t* __restrict__ ekey, double dt,
                                                    double dt_fine,
                                                    unsigned long long* __restrict__ out) {
  const int32_t e = blockIdx.x * kBlock + threadIdx.x;
  double cf = 0.0, cc = 0.0;
  if (e < M.nE) {
    const int g = ekey ? ekey[e] : 0;
    if (g <= 4) {
      const bool fine = ekey && g <= 1;
      const double c = (ekey ? (fine ? dt_fine : dt) : dt) * fabs(u[e]) / M.e_dual[e];
      if (c > 0.0) {
        if (fine || !ekey)
          cf = c;
        else
          cc = c;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    cf = fmax(cf, __shfl_xor_sync(0xffffffffu, cf, o));
    cc = fmax(cc, __shfl_xor_sync(0xffffffffu, cc, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (cf > 0.0) atomicMax(out, __double_as_longlong(cf));
    if (cc > 0.0) atomicMax(out + 1, __double_as_longlong(cc));
  }
}

// pack a 0/1 byte array into a bitmask
__global__ void k_pack_bits(int32_t n, const uint8_t* __restrict__ a, uint32_t* __restrict__ bits) {
  const int32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 32 >= n) return;
  uint32_t x = 0;
  for (int b = 0; b < 32; ++b) {
    const int32_t i = w * 32 + b;
    if (i < n && a[i]) x |= 1u << b;
  }
  bits[w] = x;
}

__global__ void k_flag_key(int32_t n, const uint8_t* __restrict__ a, uint8_t* __restrict__ key) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = a[i] ? 0 : 0xFF;
}

// ---------------------------------------------------------------------------
// Order-preserving multi-group stream compaction with warp ballots.
// key[i] in [0, G) selects the group of element i (0xFF: none).  Output:
// group g's elements in ascending index order at out[g_base[g] + ...].
constexpr int kCompactItems = 8;  // items per thread
constexpr int kCompactTile = kBlock * kCompactItems;
constexpr int kMaxGroups = 12;

__global__ void __launch_bounds__(kBlock) k_compact_count(const uint8_t* __restrict__ key, int32_t n,
                                                          int G, int32_t* __restrict__ counts,
                                                          int32_t nblocks) {
  __shared__ int32_t s_cnt[kMaxGroups];
  if (threadIdx.x < kMaxGroups) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t base = int64_t(blockIdx.x) * kCompactTile;
  int32_t local[kMaxGroups];
  for (int g = 0; g < G; ++g) local[g] = 0;
  for (int it = 0; it < kCompactItems; ++it) {
    const int64_t idx = base + int64_t(it) * kBlock + threadIdx.x;
    const uint8_t k = idx < n ? key[idx] : 0xFF;
    for (int g = 0; g < G; ++g) local[g] += __popc(__ballot_sync(0xffffffffu, k == g));
  }
  if (lane == 0)
    for (int g = 0; g < G; ++g) atomicAdd(&s_cnt[g], local[g]);
  __syncthreads();
  if (threadIdx.x < G) counts[threadIdx.x * nblocks + blockIdx.x] = s_cnt[threadIdx.x];
}

// Exclusive scan of counts[G][nblocks] (row-major) in place; totals[g] =
// group size.  One block; sequential over chunks of kBlock.
__global__ void __launch_bounds__(kBlock) k_compact_scan(int32_t* counts, int32_t nblocks, int G,
                                                         int64_t* totals) {
  __shared__ int32_t s[kBlock];
  for (int g = 0; g < G; ++g) {
    int32_t carry = 0;
    int32_t* row = counts + int64_t(g) * nblocks;
    for (int32_t start = 0; start < nblocks; start += kBlock) {
      const int32_t i = start + threadIdx.x;
      const int32_t v = i < nblocks ? row[i] : 0;
      s[threadIdx.x] = v;
      __syncthreads();
      for (int off = 1; off < kBlock; off <<= 1) {
        const int32_t add = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
        __syncthreads();
        s[threadIdx.x] += add;
        __syncthreads();
      }
      if (i < nblocks) row[i] = carry + s[threadIdx.x] - v;
      const int32_t tot = s[kBlock - 1];
      __syncthreads();
      carry += tot;
    }
    if (threadIdx.x == 0) totals[g] = carry;
    __syncthreads();
  }
}

// Scatter: within a tile, item-major then warp-major then lane order is
// ascending index order, so ballot prefixes give ascending output.
__global__ void __launch_bounds__(kBlock) k_compact_scatter(const uint8_t* __restrict__ key, int32_t n,
                                                            int G, const int32_t* __restrict__ offs,
                                                            int32_t nblocks,
                                                            const int64_t* __restrict__ gbase,
                                                            int32_t* __restrict__ out) {
  __shared__ int32_t s_warp[kMaxGroups][kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = int64_t(blockIdx.x) * kCompactTile;
  int32_t run[kMaxGroups];
  for (int g = 0; g < G; ++g) run[g] = offs[g * nblocks + blockIdx.x];
  for (int it = 0; it < kCompactItems; ++it) {
    const int64_t idx = base + int64_t(it) * kBlock + threadIdx.x;
    const uint8_t k = idx < n ? key[idx] : 0xFF;
    unsigned mine = 0;
    for (int g = 0; g < G; ++g) {
      const unsigned bal = __ballot_sync(0xffffffffu, k == g);
      if (lane == 0) s_warp[g][warp] = __popc(bal);
      if (k == g) mine = bal;
    }
    __syncthreads();
    if (k < G) {
      int32_t pos = run[k] + __popc(mine & ((1u << lane) - 1u));
      for (int w = 0; w < warp; ++w) pos += s_warp[k][w];
      out[gbase[k] + pos] = int32_t(idx);
    }
    for (int g = 0; g < G; ++g) {
      int32_t tot = 0;
      for (int w = 0; w < kBlock / 32; ++w) tot += s_warp[g][w];
      run[g] += tot;
    }
    __syncthreads();
  }
}


// Move the parked coarse values of the concurrent LTS3 coarse step into the
// state (see Op::alt): dst[i] = src[i] on the band lists.
__global__ void k_copy_band(const int32_t* __restrict__ cl, int32_t nc,
                            const double* __restrict__ hsrc, double* __restrict__ hdst,
                            const int32_t* __restrict__ el, int32_t ne,
                            const double* __restrict__ usrc, double* __restrict__ udst) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nc) {
    const int32_t i = cl[t];
    hdst[i] = hsrc[i];
  } else if (t - nc < ne) {
    const int32_t e = el[t - nc];
    udst[e] = usrc[e];
  }
}

}  // namespace mswm_dev
