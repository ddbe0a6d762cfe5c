/*
 * mswm_cuda.h — C ABI of the B200-native LTS3 / TRiSK shallow-water path.
 *
 * This is the drop-in boundary for the reference (`mswm`, arXiv:2106.07154
 * re-creation under /root/reference/proj).  Every entry point below replaces
 * one reference interface; the citation after each declaration names it.
 * Plain pointers and sizes only: no C++ or torch types cross this boundary,
 * no exceptions escape it.  Every call returns an mswm_status; the message of
 * the last failure on a context is available from mswm_cuda_last_error().
 *
 * Ids at this boundary are always the caller's ("original") ids.  The
 * library may renumber entities internally for locality; it translates at
 * the boundary.  All calls are synchronous with respect to the host unless
 * they say otherwise.
 */
#ifndef MSWM_CUDA_H
#define MSWM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  Map 1:1 onto the reference exception hierarchy
 * (proj/include/mswm/errors.hpp:9-49). */
typedef enum {
  MSWM_OK = 0,
  MSWM_E_CONFIG = 1,     /* ConfigError   (errors.hpp:17-19) */
  MSWM_E_USAGE = 2,      /* UsageError    (errors.hpp:40-43) */
  MSWM_E_TOPOLOGY = 3,   /* TopologyError (errors.hpp:22-24) */
  MSWM_E_DRY_VERTEX = 4, /* DryVertexError{vertex} (errors.hpp:45-49) */
  MSWM_E_CUDA = 5,       /* CUDA runtime failure (no reference analogue) */
  MSWM_E_NCCL = 6,       /* NCCL failure (no reference analogue) */
  MSWM_E_NOMEM = 7       /* allocation failure */
} mswm_status;

/* Element-group bits (proj/include/mswm/integrators.hpp:43-61). */
enum {
  MSWM_CELLS_FINE_PLAIN = 1u << 0,
  MSWM_CELLS_UF1 = 1u << 1,
  MSWM_CELLS_UF2 = 1u << 2,
  MSWM_CELLS_IF1 = 1u << 3,
  MSWM_CELLS_IF2 = 1u << 4,
  MSWM_CELLS_COARSE = 1u << 5,
  MSWM_EDGES_FINE_PLAIN = 1u << 6,
  MSWM_EDGES_UFINE = 1u << 7,
  MSWM_EDGES_IF1 = 1u << 8,
  MSWM_EDGES_IF2 = 1u << 9,
  MSWM_EDGES_COARSE = 1u << 10,
  MSWM_CELLS_ALL = 0x3Fu,
  MSWM_EDGES_ALL = 0x7C0u,
  MSWM_MASK_ALL = 0x7FFu
};

/* Time-stepping schemes (proj/include/mswm/integrators.hpp:26). */
typedef enum {
  MSWM_SSPRK2 = 0,
  MSWM_SSPRK3 = 1,
  MSWM_RK4 = 2,
  MSWM_LTS2 = 3,
  MSWM_LTS3 = 4
} mswm_scheme;

/* Closure kinds of one masked evaluation: the dependency sets the reference
 * marks in shallow_water_tendencies (proj/src/operators.cpp:35-58) and keeps
 * in TendencyScratch::{flux,qt,cell,vertex}_ids (operators.hpp:32). */
typedef enum {
  MSWM_CLOSURE_FLUX = 0,
  MSWM_CLOSURE_QT = 1,
  MSWM_CLOSURE_K = 2,
  MSWM_CLOSURE_PV = 3
} mswm_closure_kind;

/* SoA views of the VoronoiMesh tables (proj/include/mswm/mesh.hpp:31-68).
 * The caller owns the memory; mswm_cuda_create copies what it needs.
 * Ring convention, ascending edge_cells/edge_vertices and sign rules are
 * the reference's (mesh.hpp:26-30). */
typedef struct mswm_mesh_desc {
  int32_t n_cells, n_edges, n_vertices;
  const int32_t* cell_offset;      /* [n_cells+1]  mesh.hpp:44 */
  const int32_t* cell_edges;       /* [cell_offset[n_cells]] mesh.hpp:45 */
  const int32_t* cell_vertices;    /* [cell_offset[n_cells]] mesh.hpp:46 */
  const int32_t* cell_cells;       /* [cell_offset[n_cells]] mesh.hpp:47 */
  const int32_t* edge_cells;       /* [n_edges][2] ascending, mesh.hpp:49 */
  const int32_t* edge_vertices;    /* [n_edges][2] ascending, mesh.hpp:50 */
  const int32_t* vertex_cells;     /* [n_vertices][3] mesh.hpp:51 */
  const int32_t* vertex_edges;     /* [n_vertices][3] mesh.hpp:52 */
  const int32_t* edge_edge_offset; /* [n_edges+1] mesh.hpp:56 */
  const int32_t* edge_edges;       /* [edge_edge_offset[n_edges]] mesh.hpp:57 */
  const int8_t* edge_cell_sign;    /* [n_edges][2] mesh.hpp:68 */
  const int8_t* edge_vertex_sign;  /* [n_edges][2] mesh.hpp:69 */
  const double* edge_len;          /* [n_edges] l_e  mesh.hpp:60 */
  const double* edge_dual_len;     /* [n_edges] d_e  mesh.hpp:61 */
  const double* cell_area;         /* [n_cells] A_i  mesh.hpp:62 */
  const double* vertex_area;       /* [n_vertices] A_v mesh.hpp:63 */
  const double* vertex_kite;       /* [n_vertices][3] mesh.hpp:65 */
  const double* edge_weight;       /* aligned with edge_edges, mesh.hpp:70 */
} mswm_mesh_desc;

typedef struct mswm_cuda_ctx mswm_cuda_ctx;

/* Create a context on CUDA device `device`: validates and uploads the mesh,
 * builds the device tables.  Replaces constructing SerialEvaluator
 * (proj/src/integrators.cpp:297-314, minus b/f which come from
 * mswm_cuda_set_fields).  cell_order (may be NULL = input order) is a
 * permutation of the cells for the internal memory layout, normally a
 * space-filling curve (mswm_mesh_locality_order); edges and vertices follow
 * it.  Results are bitwise independent of cell_order.
 * On failure *out is NULL and the message is available from
 * mswm_cuda_last_error(NULL). */
int mswm_cuda_create(const mswm_mesh_desc* mesh, int device,
                     const int32_t* cell_order, mswm_cuda_ctx** out);
void mswm_cuda_destroy(mswm_cuda_ctx* ctx);
/* Last error message of ctx, or of the last failed create when ctx is NULL. */
const char* mswm_cuda_last_error(const mswm_cuda_ctx* ctx);

/* Bottom topography b[n_cells], Coriolis f[n_vertices], gravity — the
 * evaluator's constant inputs (SerialEvaluator ctor, integrators.hpp:79-81). */
int mswm_cuda_set_fields(mswm_cuda_ctx* ctx, const double* b,
                         const double* f_vertex, double gravity);

/* Region classification on device from a host-evaluated fine predicate
 * (fine_mask[n_cells] != 0 means fine).  Replaces make_regions
 * (proj/src/regions.cpp:164-171 = label_cells :69-105 + label_underline_fine
 * :107-139 + label_edges :141-162 + rebuild_groups :35-67).  Outputs (any may
 * be NULL): labels with the reference's enum values (regions.hpp:12-21) and
 * the 11 group sizes in GroupBit order.  Warnings of label_underline_fine
 * are returned as bits in *warnings (1: uf1 empty, 2: uf2 empty,
 * 4: no plain fine cells), may be NULL. */
int mswm_cuda_set_regions(mswm_cuda_ctx* ctx, const uint8_t* fine_mask,
                          int interface_width, uint8_t* cell_label,
                          uint8_t* cell_sublabel, uint8_t* edge_label,
                          int64_t group_size[11], int* warnings);

/* Check label arrays the caller supplies (caller ids; does not change the
 * context's own region map) on the device.  Replaces the label checks of
 * validate_regions (proj/src/regions.cpp:173-288): band distances from the
 * label-0 set (:213-244), underline sublabels (:247-262; cell_sublabel NULL =
 * not assigned) and the fine-side-wins edge rule (:265-286; edge_label NULL =
 * not assigned).  Per check kind k -- 0 value out of range, 1 Interface1
 * outside 1..w, 2 Interface2 outside w+1..2w, 3 coarse within 2w, 4 wrong
 * underline sublabel, 5 wrong edge label -- counts[k] = offending elements and
 * first[k] = the lowest offending id (the one the reference names first), -1
 * if none.  The group lists of this library are compactions of the labels,
 * so validate_regions' list-cover checks have no counterpart. */
int mswm_cuda_validate_labels(mswm_cuda_ctx* ctx, const uint8_t* cell_label,
                              const uint8_t* cell_sublabel, const uint8_t* edge_label,
                              int interface_width, int64_t counts[6], int32_t first[6]);

/* Ascending original ids of group g (GroupBit index 0..10), the
 * RegionMap::cells_* / edges_* lists (regions.hpp:35-42). */
int mswm_cuda_get_group(mswm_cuda_ctx* ctx, int group, int32_t* ids);

/* Closure set of a masked evaluation (operators.cpp:35-58), ascending
 * original ids.  ids may be NULL to query the size only. */
int mswm_cuda_get_closure(mswm_cuda_ctx* ctx, unsigned mask, int kind,
                          int32_t* ids, int64_t* n);

/* TendencyEvaluator::eval (proj/include/mswm/integrators.hpp:68-73):
 * h[n_cells], u[n_edges] full host arrays; writes dh/du only on the masked
 * groups, leaves every other entry untouched.  Without regions only
 * MSWM_MASK_ALL is legal (UsageError, integrators.cpp:139-142).  Returns
 * MSWM_E_DRY_VERTEX (see mswm_cuda_dry_vertex) like the reference throws
 * DryVertexError (operators.cpp:82-84). */
int mswm_cuda_eval(mswm_cuda_ctx* ctx, const double* h, const double* u,
                   unsigned mask, double* dh, double* du);

/* Device-resident prognostic state (State, integrators.hpp:18-24). */
int mswm_cuda_state_upload(mswm_cuda_ctx* ctx, const double* h,
                           const double* u, double time);
int mswm_cuda_state_download(mswm_cuda_ctx* ctx, double* h, double* u,
                             double* time);

/* n_steps of Stepper::step (integrators.cpp:577-596) on the device state:
 * scheme in mswm_scheme, dt the coarse step for LTS and the global step
 * otherwise, M the substep count (LTS only).  LTS3 / LTS2 = lts_step(3 / 2)
 * (:412-575), RK4 = rk4_step (:370-410), SSPRK3 / SSPRK2 = ssprk_step(3 / 2)
 * (:337-368).
 * Steps are replayed from a captured CUDA graph.  Asynchronous when
 * `sync` is 0 (errors then surface at the next synchronous call).  n_steps
 * == 0 prepares only: plans built and the graph captured, nothing launched. */
int mswm_cuda_step(mswm_cuda_ctx* ctx, int scheme, double dt, int M,
                   int64_t n_steps, int sync);

/* WorkLedger counters (proj/include/mswm/ledger.hpp:25-60): cell_evals and
 * edge_evals are [4 regions][4 stages] row-major; steps may be NULL. */
int mswm_cuda_ledger(mswm_cuda_ctx* ctx, int64_t cell_evals[16],
                     int64_t edge_evals[16], int64_t* steps);
int mswm_cuda_ledger_reset(mswm_cuda_ctx* ctx);

/* Original id of the vertex of the last DryVertexError, -1 if none; *step =
 * the 1-based step of the mswm_cuda_step batch it happened in (the
 * reference's "during step k of n", harness.cpp:183-190), 0 for an eval
 * call.  Kernel A records (step, vertex) on the device; an asynchronous batch
 * reports it at the next synchronous call (step with sync=1, eval, sync,
 * state_download -- which still writes the state), and the earliest step
 * wins.  The flag is cleared only once reported. */
int mswm_cuda_dry_vertex(const mswm_cuda_ctx* ctx, int64_t* step);

/* Synchronise the context's stream; returns any pending error
 * (MSWM_E_DRY_VERTEX from an asynchronous step batch). */
int mswm_cuda_sync(mswm_cuda_ctx* ctx);
/* The cudaStream_t every kernel of ctx is launched on (for event timing). */
void* mswm_cuda_stream(mswm_cuda_ctx* ctx);

/* Per-evaluation device timing of the most recent step (profiling aid for
 * the roofline).  Enable before mswm_cuda_step; the captured step then
 * brackets every tendency evaluation (enable = 1), or only the first one
 * whose outputs cover at least half the mesh (enable = 2: two event nodes
 * per step instead of two per evaluation), with CUDA events.  After a step,
 * mswm_cuda_eval_profile fills up to `cap` entries: eval_ms[k] the device
 * time of evaluation k of the last replayed step, out_cells/out_edges its
 * output set sizes; returns the count in *n. */
int mswm_cuda_set_profiling(mswm_cuda_ctx* ctx, int enable);
int mswm_cuda_eval_profile(mswm_cuda_ctx* ctx, float* eval_ms,
                           int64_t* out_cells, int64_t* out_edges, int cap,
                           int* n);

/* Output kernel: kernel_path 0 = k_out over the explicit stencil tables
 * (the only output kernel; profiles/r2_phaseC_experiments.json records the
 * variants measured slower and removed).
 * identity_order = 1 when the internal numbering equals the caller's. */
int mswm_cuda_layout_info(const mswm_cuda_ctx* ctx, int* kernel_path,
                          int* identity_order);

/* Explicit stencil tables: offsets16 = 1 when the stencil ids are stored as
 * 16-bit offsets e' - e (20 B/edge; MSWM_ST16=0 at create disables them);
 * n_wide = edges with an offset outside int16, whose warps read the int32
 * table instead (edges_on_edge, mesh.hpp:60-61). */
int mswm_cuda_stencil_info(const mswm_cuda_ctx* ctx, int* offsets16, int64_t* n_wide);

/* 16-bit index records of the evaluation kernels (kernels.cuh DevMesh
 * v_rec / c_rec / e_cv16 / e_c16): packed16 bit 0 = in use (MSWM_PACK16 != 0),
 * bit 1 = the cell records too (ring size <= 6 meshes); the counts are the
 * vertices, cells and edges with an id offset outside int16, which their
 * warps read from the int32 tables instead. */
int mswm_cuda_index_info(const mswm_cuda_ctx* ctx, int* packed16, int64_t* n_wide_vertices,
                         int64_t* n_wide_cells, int64_t* n_wide_edges);

/* Number of this library's kernels one replay of the most recently used
 * step graph launches (the bench's gpu_launches evidence). */
int mswm_cuda_kernels_per_step(mswm_cuda_ctx* ctx, int64_t* n);

/* Cost replication (SchemeConfig::replication, integrators.hpp:33-39;
 * SerialEvaluator's `replication`, integrators.cpp:117-129): every
 * evaluation repeats the tendency arithmetic `replication` times
 * (operators.cpp:60) -- results unchanged, ledger counts scaled by it
 * (integrators.cpp:302-335).  MSWM_E_CONFIG when < 1. */
int mswm_cuda_set_replication(mswm_cuda_ctx* ctx, int replication);

/* LTS3 schedule of the most recent step graph: concurrent_coarse = 1 when
 * the coarse stage (integrators.cpp:557-563) ran on its own stream
 * concurrently with the substeps (with ranks: its halo exchange too, on a
 * second communicator), 0 in sequence, -1 not yet captured. */
int mswm_cuda_schedule_info(const mswm_cuda_ctx* ctx, int* concurrent_coarse);

/* Device diagnostics: total_mass (proj/src/harness.cpp:99-105) of the
 * device state, summed in ascending original cell id order (bitwise equal
 * to the reference). */
int mswm_cuda_total_mass(mswm_cuda_ctx* ctx, double* mass);

/* total_mass and total_energy (harness.cpp:99-123) of the device state from
 * per-cell terms computed on the device in the reference's operation order.
 * exact = 1: summed sequentially in ascending caller cell id (bitwise the
 * reference); exact = 0: a fixed-shape device tree sum (deterministic, not
 * the sequential rounding).  A rank context sums its owned cells. */
int mswm_cuda_diagnostics(mswm_cuda_ctx* ctx, int exact, double* mass,
                          double* energy);

/* courant_numbers (integrators.cpp:632-659) of the device velocity: max of
 * step |u_e| / d_e over fine + underline-fine edges (step dt / M) and over
 * interface + coarse edges (step dt); without a region map every edge at dt
 * and coarse = fine. */
int mswm_cuda_courant(mswm_cuda_ctx* ctx, double dt, int M, double* fine,
                      double* coarse);

/* ---- multi-rank (one process per GPU, or an in-process group) ----------
 * A rank context holds one rank's piece of the mesh (owned elements plus a
 * two-hop halo, the reference's block plan, partition.cpp:307-403) in local
 * numbering; outputs are the owned elements only and halo copies are
 * refreshed before every evaluation (the device form of ThreadedEvaluator's
 * per-eval copy-in, rank_pool.cpp:133-135). */

/* Partition of the mesh for n_parts ranks on the device (replaces
 * partition_multiconstraint's per-class split, partition.cpp:219-231, and
 * make_block_plan's edge ownership, partition.cpp:338-353): every region class
 * (fine incl. underline, coarse, interface) is cut into n_parts near-equal
 * consecutive runs of `sweep_order` (a permutation of the caller's cell ids,
 * e.g. a space-filling curve); an edge goes to the rank of its first cell
 * (edge_cells order) of the edge's own class.  Needs the region map of
 * mswm_cuda_set_regions.  Outputs in caller ids (either may be null);
 * MSWM_E_USAGE for a bad order / n_parts, MSWM_E_TOPOLOGY for an edge with no
 * cell of its class. */
int mswm_cuda_partition(mswm_cuda_ctx* ctx, const int32_t* sweep_order, int n_parts,
                        int32_t* rank_of_cell, int32_t* edge_owner);

/* Halo plan of a partition on the device (make_block_plan's 2-hop halo,
 * partition.cpp:355-392, for every rank at once): for each cell / edge /
 * vertex (caller ids) the bit set of the ranks whose local mesh -- owned
 * cells plus the cells within two hops, their ring edges and vertices --
 * holds it.  rank_of_cell[nC] in [0, n_ranks), n_ranks <= 64; null outputs
 * are skipped. */
int mswm_cuda_halo_reach(mswm_cuda_ctx* ctx, const int32_t* rank_of_cell, int n_ranks,
                         uint64_t* cell_reach, uint64_t* edge_reach, uint64_t* vertex_reach);

/* Region labels from the global RegionMap (regions.hpp:27-29 values),
 * indexed by local ids; outputs restricted to cell_owned / edge_owned
 * (NULL = all).  Replaces mswm_cuda_set_regions on a rank context. */
int mswm_cuda_set_labels(mswm_cuda_ctx* ctx, const uint8_t* cell_label,
                         const uint8_t* cell_sublabel, const uint8_t* edge_label,
                         const uint8_t* cell_owned, const uint8_t* edge_owned,
                         int interface_width);

/* Halo plan of rank `rank` of `n_ranks`: for each of n_peers peers,
 * counts[4*j..4*j+3] = (#cells sent, #edges sent, #cells received,
 * #edges received) and `ids` holds, peer after peer, those local ids in that
 * order.  Both sides must list shared elements in the same order. */
int mswm_cuda_set_halo(mswm_cuda_ctx* ctx, int rank, int n_ranks, int n_peers,
                       const int32_t* peers, const int64_t* counts,
                       const int32_t* ids);

/* Halo restriction per mask: the halo entries the
 * evaluation with `mask` reads, as positions within each peer's receive list
 * of mswm_cuda_set_halo (cells then edges), peers in set_halo order:
 * counts[j] entries for peer j, concatenated in pos (NULL: counts only).
 * Builds the mask's closure (as mswm_cuda_eval would). */
int mswm_cuda_halo_needs(mswm_cuda_ctx* ctx, unsigned mask, int64_t* counts,
                         int32_t* pos);

/* Install the restriction for `mask`: send_pos = positions within each
 * peer's send list that the peer needs (that peer's halo_needs for this
 * rank), recv_pos = this rank's own halo_needs.  The step graph then
 * exchanges only these entries before evaluations with `mask`, plus one
 * coarse-mask refresh before the coarse-only stage. */
int mswm_cuda_set_halo_mask(mswm_cuda_ctx* ctx, unsigned mask,
                            const int64_t* send_counts, const int32_t* send_pos,
                            const int64_t* recv_counts, const int32_t* recv_pos);

/* NCCL transport (one process per GPU): rank 0 creates a 128-byte unique id,
 * the caller broadcasts it, every rank calls mswm_cuda_comm_init.  The
 * exchange is NCCL point-to-point on the context's stream, captured in the
 * step graph.  NCCL is resolved at run time (libnccl.so.2). */
int mswm_cuda_nccl_unique_id(void* id_out /* 128 bytes */);
int mswm_cuda_comm_init(mswm_cuda_ctx* ctx, const void* unique_id, int rank,
                        int n_ranks);

/* In-process group: n rank contexts on one device stepped in lockstep on
 * one stream, halos exchanged by device copies (no kernel waits on another).
 * members[r] must be rank r of n. */
typedef struct mswm_cuda_group mswm_cuda_group;
int mswm_cuda_group_create(mswm_cuda_ctx* const* members, int n,
                           mswm_cuda_group** out);
void mswm_cuda_group_destroy(mswm_cuda_group* group);
int mswm_cuda_group_step(mswm_cuda_group* group, int scheme, double dt, int M,
                         int64_t n_steps);
/* Group halo copies through NCCL instead of device copies: a one-rank
 * communicator (two: the concurrent coarse step has its own) on the group's
 * device, every copy an ncclSend to self matched by the ncclRecv issued
 * after it -- the NCCL transport's calls, buffers and graph capture,
 * exercised on one GPU without kernels that wait on one another. */
int mswm_cuda_group_nccl_loopback(mswm_cuda_group* g);

/* ---- peer-store halo transport --------------------------------------------
 * Halo exchanges without a communication library: the pack kernel stores
 * into the neighbours' receive buffers through peer-mapped pointers (CUDA IPC
 * between the processes of one box, NVLink / NVSwitch peer access) and raises
 * a device flag at every neighbour; the unpack kernel waits for its
 * neighbours' flags (bounded polling: a silent neighbour is reported as
 * MSWM_E_NCCL by the next synchronous call).  Two launches per exchange inside
 * the step graph.  Replaces the copy-in of ThreadedEvaluator's ranks
 * (rank_pool.cpp:127-176) like the NCCL transport does.  Setup, after the
 * halo plans (mswm_cuda_set_halo, mswm_cuda_set_halo_mask) are final: every rank exports, imports each neighbour's
 * export (moved by the host, e.g. torch.distributed all_gather_object) and
 * enables.  A later change of the halo plans drops the transport. */

/* This rank's arena as a 64-byte cudaIpcMemHandle_t (NULL: skip) and the rows
 * (mask or -1 for the full halo, sending rank, byte offset, bytes between the
 * two halves, count) of where each neighbour's values land in it.  rows NULL:
 * query *n_rows. */
int mswm_cuda_peer_export(mswm_cuda_ctx* ctx, void* ipc_handle, int64_t* rows,
                          int64_t cap_rows, int64_t* n_rows);
int mswm_cuda_peer_import(mswm_cuda_ctx* ctx, int peer_rank, const void* ipc_handle,
                          const int64_t* rows, int64_t n_rows);
int mswm_cuda_peer_enable(mswm_cuda_ctx* ctx, int on);
/* One full-halo exchange of the state arrays in two host-ordered halves
 * (phase 0: pack + store + signal; phase 1: wait + unpack), synchronous;
 * phase 2 enqueues the wait + unpack and returns (mswm_cuda_sync awaits it). */
int mswm_cuda_peer_exchange(mswm_cuda_ctx* ctx, int phase);
/* The same transport between the members of an in-process group (plain
 * device pointers instead of IPC mappings). */
int mswm_cuda_group_peer(mswm_cuda_group* group, int on);

const char* mswm_cuda_group_last_error(const mswm_cuda_group* group);

#ifdef __cplusplus
}
#endif

#endif /* MSWM_CUDA_H */
