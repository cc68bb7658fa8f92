/*
 * libgis — B200 (sm_100a) implementation of the GIS graph-construction and
 * graph-pruning hot path (arxiv 2202.06111; reference package `cisgraph`
 * 0.1.0 at /root/reference/pkg/src/cisgraph, abbreviated cg/ below).
 *
 * Plain C ABI: device pointers are raw CUDA device addresses, host pointers
 * are plain host memory, sizes are int64_t.  Every entry point returns a
 * gis_status (0 = ok); on error gis_last_error() returns a thread-local
 * message.  All work is enqueued on the context's stream (gis_ctx_set_stream).
 *
 * Layouts:
 *   covering : depths int32[V], bits int64[V] (split path, first split MSB),
 *              lo/hi float64 SoA [n][V] (lo[d*V + i]); canonical CellId order.
 *   graph    : CSR, indptr int64[rows+1], indices int32[E], rows ascending,
 *              targets ascending and unique per row.
 *   masks    : uint8[V] (0/1);  bitmaps: uint32 words, bit i%32 of word i/32.
 */
#ifndef GIS_H_
#define GIS_H_

#ifndef __CUDACC_RTC__  /* NVRTC (user models, gis_jit.cu) brings its own */
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GIS_ABI_VERSION 1
#define GIS_MAX_DIM 4
#define GIS_MAX_PARAMS 64

typedef enum {
  GIS_OK = 0,
  GIS_E_INVALID = 1,   /* bad argument / unsupported configuration (ValueError) */
  GIS_E_CUDA = 2,      /* CUDA runtime error */
  GIS_E_OVERLAP = 3,   /* index boxes overlap (not a covering) */
  GIS_E_CAPACITY = 4,  /* size limit exceeded (slot table too large, ...) */
  GIS_E_STATE = 5      /* call sequence error (finish without begin, ...) */
} gis_status;

/* model kinds (paper_2202_06111_b200/system.py KIND_IDS) */
enum { GIS_IDENTITY = 0, GIS_SHIFT = 1, GIS_LINEAR = 2, GIS_AFFINE = 3, GIS_CSTR = 4,
       GIS_PENDULUM = 5, GIS_CSTR_DIMLESS = 6, GIS_LORENZ = 7, GIS_CARTPOLE = 8,
       GIS_JIT = 9 /* user-defined (gis_jit_register), model.jit = its id */ };
/* integrators: direct map, forward Euler, classical RK4 (cg/system.py:34-49),
 * or a single vector-field evaluation */
enum { GIS_MAP = 0, GIS_EULER = 1, GIS_RK4 = 2, GIS_RHS = 3 };

/* A device model: replaces the reference's SystemModel.step callable
 * (cg/system.py:52-75).  h = dt / substeps, computed by the caller. */
typedef struct gis_model {
  int32_t kind;
  int32_t integrator;
  int32_t substeps;
  int32_t n;
  int32_t m;
  int32_t jit;  /* GIS_JIT: the id gis_jit_register returned; else 0 */
  double h;
  double params[GIS_MAX_PARAMS];
} gis_model;

typedef struct gis_ctx gis_ctx;
typedef struct gis_index gis_index;

/* ---- user-defined models (the SystemModel plugin API, cg/system.py:52-75) -
 * CUDA C++ source for the model, compiled once by NVRTC into the same K1
 * kernels the built-in kinds use (sm_100a, reference operation order, CUDA
 * libm).  form 0: an ODE, `body` sets f[0..n-1] from x[0..n-1], u[0..m-1]
 * and the parameters p[] (model.params), integrated by `integrator` (GIS_EULER
 * or GIS_RK4, model.substeps steps of model.h); form 1: a direct map, `body`
 * sets y[0..n-1] (integrator GIS_MAP).  *id is then used as model.jit with
 * model.kind = GIS_JIT.  Identical registrations return the same id.
 * GIS_E_INVALID with the compiler log if the source does not compile. */
int gis_jit_register(gis_ctx* ctx, const char* body, int32_t form, int32_t n, int32_t m,
                     int32_t integrator, int32_t* id);
/* compile only (no device needed): GIS_OK and the cubin size, or
 * GIS_E_INVALID with the compiler log in gis_last_error() */
int gis_jit_compile_check(const char* body, int32_t form, int32_t n, int32_t m,
                          int32_t integrator, int64_t* cubin_bytes);

/* ---- context ------------------------------------------------------------ */
int gis_abi_version(void);
const char* gis_last_error(void);
int gis_ctx_create(gis_ctx** out, int device);
int gis_ctx_destroy(gis_ctx* ctx);
int gis_ctx_set_stream(gis_ctx* ctx, void* cuda_stream);
/* Cell bounds still arriving: the caller copies a covering's lo / hi to the
 * device in cell-range chunks on another stream and records events[c] once
 * the cells below ends[c] (ascending; the last = V) are in place.  The next
 * graph build (gis_build_graph_begin, whole covering, dense index) starts
 * integrating each chunk as its event completes, overlapping the copy of
 * the rest (a corner shared across a chunk boundary is integrated on both
 * sides); a build that cannot split (row range, box reuse, sparse index)
 * waits for all of them first.  The list is consumed by that build; n = 0
 * clears it (after waiting).  No other call reads the list: the caller
 * waits on the events itself before passing lo / hi anywhere else
 * (Covering does).  events: cudaEvent_t, alive until the build returns. */
int gis_ctx_input_chunks(gis_ctx* ctx, int32_t n, const int64_t* ends, void* const* events);
/* Return every device buffer the context holds (grow-only scratch, cached
 * index/CSR blocks) to its private memory pool and trim the pool to zero;
 * *released (may be NULL) receives the bytes given back to the device.  The
 * device's default memory pool is never modified by libgis. */
int gis_ctx_trim(gis_ctx* ctx, uint64_t* released);
/* bytes the context's private pool currently reserves from the device */
int gis_ctx_pool_reserved(gis_ctx* ctx, uint64_t* bytes);
/* number of libgis kernels launched through this context so far */
int64_t gis_ctx_launch_count(const gis_ctx* ctx);
/* per-phase CUDA-event timing: phases are 0 enclose (K1), 1 CSR rows (K2),
 * 2 CSR scans/compaction, 3 prune (K3), 4 index build, 5 covering updates */
#define GIS_NPHASE 6
int gis_ctx_enable_timing(gis_ctx* ctx, int on);
/* synchronises, returns accumulated ms and event counts per phase, resets */
int gis_ctx_phase_times(gis_ctx* ctx, double* ms, int64_t* counts);
/* K1 work since the last call (then reset; synchronises): `images` =
 * (cell, input, sample) images produced -- the reference's integrations,
 * cg/image.py:65-85 -- and `integrations` = the one-step integrations K1
 * actually ran.  They differ on graph builds over a dense index, where a
 * grid vertex shared by several cells' corner samples is integrated once. */
int gis_ctx_integrations(gis_ctx* ctx, int64_t* images, int64_t* integrations);
/* measured dense fp64 FMA throughput of this device (TFLOP/s) */
int gis_fp64_peak(gis_ctx* ctx, double* tflops);

/* ---- dynamics + enclosures ---------------------------------------------- */
/* SystemModel.map_points / step(x, u) (cg/system.py:71-75).
 * x, out: device float64 [N][n] row-major; u: host float64[m]. */
int gis_map_points(gis_ctx* ctx, const gis_model* model, const double* x, int64_t N,
                   const double* u, double* out);

/* batch_enclosures for U inputs at once (cg/image.py:65-85).
 * lo, hi: device SoA [n][B]; u: host [U][m]; frac: host [S][n] sample
 * fractions (cg/image.py:43-62); enc_lo/enc_hi: device [U][B][n];
 * valid: device uint8 [U][B]. */
int gis_batch_enclosures(gis_ctx* ctx, const gis_model* model, const double* lo,
                         const double* hi, int64_t B, const double* u, int32_t U,
                         const double* frac, int32_t S, double bloat, double* enc_lo,
                         double* enc_hi, uint8_t* valid);

/* ---- spatial index (replaces SpatialIndex, cg/geometry.py:416-505) ------- */
/* Index over a dyadic covering of the root box [root_lo, root_hi] (host
 * arrays).  depths/bits: device arrays in canonical order. */
int gis_index_build_dyadic(gis_ctx* ctx, int32_t n, const double* root_lo,
                           const double* root_hi, const int32_t* depths,
                           const int64_t* bits, int64_t V, gis_index** out);
/* Index over arbitrary pairwise-disjoint closed boxes (device SoA [n][V]). */
int gis_index_build_boxes(gis_ctx* ctx, int32_t n, const double* lo, const double* hi,
                          int64_t V, gis_index** out);
/* the same with the index kind chosen: mode 0 = automatic (dense slot table
 * when it fits -- <= 30 splits per axis, < 2^31 slots, and <= 2^24 or <= 1024
 * per cell -- else sparse), 1 = dense (GIS_E_CAPACITY if it does not fit),
 * 2 = sparse (sorted cell start codes, any depth up to 62: coverings the
 * reference's MAX_DEPTH allows, cg/geometry.py:34).  Every query of this
 * header works on both kinds with identical results. */
int gis_index_build_dyadic_mode(gis_ctx* ctx, int32_t n, const double* root_lo,
                                const double* root_hi, const int32_t* depths,
                                const int64_t* bits, int64_t V, int32_t mode, gis_index** out);
/* 1 if the index is sparse */
int gis_index_is_sparse(const gis_index* idx);
int gis_index_free(gis_index* idx);
/* slots per axis (out[n]) and total slot-table entries (-1: sparse index,
 * slots per axis then count the finest dyadic level) */
int gis_index_shape(const gis_index* idx, int64_t* slots_per_axis, int64_t* total);

/* query_boxes (cg/geometry.py:471-505) as CSR: for each of Q query boxes
 * (device SoA [n][Q]) the ascending indices of intersecting boxes (closed
 * semantics).  Two phases: begin fills qptr (device int64[Q+1]) and returns
 * the pair count; finish writes cells (device int32[pairs]). */
int gis_query_boxes_begin(gis_ctx* ctx, const gis_index* idx, const double* qlo,
                          const double* qhi, int64_t Q, int64_t* qptr, int64_t* n_pairs);
int gis_csr_finish(gis_ctx* ctx, int32_t* indices);

/* ---- graph build (build_graph_serial/parallel, cg/graph.py:181-351) ----- */
/* Symbolic image rows [row_begin, row_end) of the covering (lo/hi device SoA
 * [n][V]) against index idx: for each source cell and input, the sampled
 * enclosure (K1) is turned into a slot rectangle and the intersecting cells
 * are deduplicated across inputs into an ascending CSR row (K2).
 * indptr: device int64[rows+1]; *n_edges (host) receives E.  Then call
 * gis_csr_finish(ctx, indices) with a device int32[E] buffer. */
int gis_build_graph_begin(gis_ctx* ctx, const gis_index* idx, const gis_model* model,
                          const double* lo, const double* hi, int64_t V,
                          int64_t row_begin, int64_t row_end, const double* u,
                          int32_t U, const double* frac, int32_t S, double bloat,
                          int64_t* indptr, int64_t* n_edges);
/* gis_build_graph_begin for the coverings of an adaptive run (the same
 * graph).  memo_out (device float64 [rows][U][2n], may be NULL) receives
 * every pair's padded enclosure box (lo n, hi n; NaN lo[0]: no finite
 * sample).  origin (device int64 [V], may be NULL) gives each cell's index
 * in the previous covering, or -1 (gis_covering_origin); pairs of cells
 * whose origin lies in [memo_begin, memo_begin + memo_rows) take their box
 * from memo_in (that build's memo_out) instead of integrating: a cell's
 * box depends only on the cell, the input, the samples and the model.
 * With the previous build's rows (prev_indptr [memo_rows + 1] relative,
 * prev_indices: its global targets) and fwd (device int64 [previous V],
 * gis_covering_forward), those cells' rows are the previous rows mapped
 * forward -- unchanged targets kept, removed ones dropped, split ones
 * replaced by the children meeting one of the row's boxes -- instead of
 * being enumerated again (U <= 32).  Dense indices only. */
int gis_build_graph_memo_begin(gis_ctx* ctx, const gis_index* ix, const gis_model* model,
                               const double* lo, const double* hi, int64_t V,
                               int64_t row_begin, int64_t row_end, const double* u, int32_t U,
                               const double* frac, int32_t S, double bloat,
                               const int64_t* origin, const double* memo_in,
                               int64_t memo_begin, int64_t memo_rows,
                               const int64_t* prev_indptr, const int32_t* prev_indices,
                               const int64_t* fwd, double* memo_out, int64_t* indptr,
                               int64_t* n_edges);

/* _csr_from_pairs (cg/graph.py:181-193): CSR of the distinct (src, dst)
 * pairs, rows ascending and targets ascending per row.  src, dst: device
 * int64[n] in [0, V); indptr: device int64[V+1]; indices: device int32[>= n]
 * (the first *n_edges entries are written).  Used by merge_subgraphs. */
int gis_csr_from_pairs(gis_ctx* ctx, const int64_t* src, const int64_t* dst, int64_t n,
                       int64_t V, int64_t* indptr, int32_t* indices, int64_t* n_edges);
/* SymbolicImage.edge_pairs sources: src device int64[indptr[V]] */
int gis_csr_sources(gis_ctx* ctx, const int64_t* indptr, int64_t V, int64_t* src);

/* ---- pruning (non_leaving_mask, cg/analysis.py:120-161) ------------------ */
/* Keep mask of vertices that reach a cycle (zero-out-degree peeling fixed
 * point, tests/conftest.py:75-89) on one GPU. keep: device uint8[V]. */
int gis_prune(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
              uint8_t* keep, int32_t* rounds);
/* Sharded peeling: rows [v_begin, v_end) owned by this rank; alive: device
 * bitmap over all V vertices (replicated, exchanged by allgather between
 * sweeps); ptr: device int64[v_end - v_begin] opaque per-row scan state
 * (current target and row offset). */
int gis_peel_init(gis_ctx* ctx, const int64_t* indptr_local, int64_t V, int64_t v_begin,
                  int64_t v_end, uint32_t* alive, int64_t* ptr);
/* one sweep; *deaths (host) receives the number of owned vertices removed */
int gis_peel_sweep(gis_ctx* ctx, const int64_t* indptr_local, const int32_t* indices,
                   int64_t v_begin, int64_t v_end, uint32_t* alive, int64_t* ptr,
                   int64_t* deaths);
/* the same sweep without a host read: the owned deletions are added to the
 * device counter *deaths_dev (int64), so several sweeps and their all-gathers
 * can run before one all-reduce + read decides termination */
int gis_peel_sweep_acc(gis_ctx* ctx, const int64_t* indptr_local, const int32_t* indices,
                       int64_t v_begin, int64_t v_end, uint32_t* alive, int64_t* ptr,
                       int64_t* deaths_dev);
/* the owned rows' LOCAL fixed point: sweeps (one cooperative launch, block-
 * local sweeps between grid barriers) until a sweep of the owned range with
 * the bitmap as it stands deletes nothing; remote words are read, never
 * written.  Owned deletions are added to *deaths_dev (device int64).  The
 * multi-GPU loop is: local fixed point, all-gather of the owned words,
 * all-reduce of the deletions, until a round deletes nothing anywhere
 * (distributed.sharded_peel): one exchange per round instead of per sweep. */
int gis_peel_local(gis_ctx* ctx, const int64_t* indptr_local, const int32_t* indices,
                   int64_t v_begin, int64_t v_end, uint32_t* alive, int64_t* ptr,
                   int64_t* deaths_dev);
/* Multi-GPU pruning with the bitmap exchange fused into the sweep kernel
 * (replaces the per-sweep all-gather of gis_peel_sweep_acc + NCCL; same
 * result as gis_prune).  One cooperative launch per rank runs every sweep:
 * owned words are swept, then stored into every peer's bitmap replica over
 * peer memory (NVLink), then a flag barrier in peer memory sums the deletions.
 * indptr: rows [vbase, vbase + rows) (the rank's owned range,
 * distributed.owned_range); replica_addrs / flag_addrs: host arrays of R
 * device addresses, as mapped in this process (gis_ipc_open), of each rank's
 * bitmap replica (uint32[ceil(V/32)]) and flag area (uint64[2*R], zeroed at
 * allocation).  seq0: nonzero, advanced by *rounds + 1 after each call, the
 * same on every rank.  rank = -1 emulates all R ranks in one launch on this
 * GPU (replicas / flag areas all local; indptr then covers all V rows).
 * The replicas hold the surviving vertices on return. */
int gis_peel_p2p(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                 int64_t vbase, int64_t rows, const uint64_t* replica_addrs,
                 const uint64_t* flag_addrs, int32_t rank, int32_t R, uint32_t seq0,
                 int32_t* rounds);
/* CUDA IPC buffers for the replicas / flag areas: zero-filled cudaMalloc,
 * handle = 64 bytes (cudaIpcMemHandle_t) for the peers' gis_ipc_open */
int gis_ipc_alloc(gis_ctx* ctx, int64_t bytes, void** ptr, void* handle);
int gis_ipc_open(gis_ctx* ctx, const void* handle, void** ptr);
int gis_ipc_close(void* ptr);
int gis_ipc_free(void* ptr);
int gis_bitmap_to_mask(gis_ctx* ctx, const uint32_t* words, int64_t V, uint8_t* mask);
int gis_mask_to_bitmap(gis_ctx* ctx, const uint8_t* mask, int64_t V, uint32_t* words);

/* ---- SCC analysis (cg/analysis.py:51-161, cg/graph.py:125-139) ---------- */
/* Strongly connected components (replaces _tarjan_components +
 * strongly_connected_components).  comp: device int64[V], component id per
 * vertex, ids numbered by each component's smallest vertex (Tarjan's ids are
 * DFS pop order; the partition is identical).  sizes: device int64[V] and
 * nontrivial: device uint8[V] (size >= 2 or a self-loop), first *n_comp
 * entries valid.  stats (host int32[2], optional): outer iterations, grid
 * rounds. */
int gis_scc(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
            int64_t* comp, int64_t* sizes, uint8_t* nontrivial, int64_t* n_comp,
            int32_t* stats);
/* non_leaving_mask computed literally as the reference does
 * (cg/analysis.py:120-161): SCCs, seeds = every nontrivial component
 * (strict_largest = 0) or the largest one (ties: the component with the
 * smallest vertex), then the reverse-reachability closure of the seeds; all
 * zero when no component is nontrivial.  The default mode of the package
 * uses gis_prune (same set, cheaper); this is the strict mode and a
 * cross-check.  keep: device uint8[V]. */
int gis_non_leaving_scc(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                        int32_t strict_largest, uint8_t* keep, int32_t* rounds);
/* SymbolicImage.reverse_csr: rptr device int64[V+1], rind device int32[E];
 * sorted != 0 orders each row ascending (the reference's lexsort order). */
int gis_reverse_csr(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                    int64_t* rptr, int32_t* rind, int32_t sorted);
/* SymbolicImage.self_loop_mask: out device uint8[V] */
int gis_self_loops(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                   uint8_t* out);

/* ---- coverings (Covering.subdivide / retain, cg/geometry.py:343-385) ----- */
/* number of nonzero bytes of mask */
/* A uniform dyadic grid of `depth` cycled splits of the root [root_lo,
 * root_hi] (host double[n]), generated in canonical order without the
 * intermediate levels (replaces `depth` rounds of cg/geometry.py:343-372
 * subdivide on a one-cell covering; with limits, also the grid_mask
 * restriction of a non-dyadic initial grid).  Bounds are the per-axis faces
 * computed by repeated midpoints 0.5*(lo+hi), as the splits compute them.
 * limits: host int64[n] cells kept per axis (NULL = all).  depths == NULL:
 * size query into *V_out; else *V_out must hold that size and
 * depths/bits/lo/hi (SoA [n][V]) receive the cells. */
int gis_uniform_grid(gis_ctx* ctx, int32_t n, int32_t depth, const double* root_lo,
                     const double* root_hi, const int64_t* limits, int64_t* V_out,
                     int32_t* depths, int64_t* bits, double* lo, double* hi);
int gis_count_mask(gis_ctx* ctx, const uint8_t* mask, int64_t V, int64_t* count);
/* children of selected cells replace their parent in place (canonical order
 * is preserved); outputs sized V + count(sel).  sel == NULL selects all. */
int gis_subdivide(gis_ctx* ctx, int32_t n, int64_t V, const int32_t* depths,
                  const int64_t* bits, const double* lo, const double* hi,
                  const uint8_t* sel, int32_t* depths_out, int64_t* bits_out,
                  double* lo_out, double* hi_out);
/* mask of the cells of a uniform dyadic grid whose per-axis index is below
 * limits[d] (host int64[n]): a G_0 x .. x G_{n-1} grid embedded in the
 * power-of-two grid of an extended root box (non-dyadic initial grids) */
int gis_grid_mask(gis_ctx* ctx, int32_t n, int64_t V, const int32_t* depths,
                  const int64_t* bits, const int64_t* limits, uint8_t* out);
/* stable compaction of kept cells; outputs sized count(keep) */
int gis_retain(gis_ctx* ctx, int32_t n, int64_t V, const int32_t* depths,
               const int64_t* bits, const double* lo, const double* hi,
               const uint8_t* keep, int32_t* depths_out, int64_t* bits_out,
               double* lo_out, double* hi_out);
/* origin (device int64 [V_new]) of the covering subdivide(retain(c, keep),
 * sel) -- one adaptive step from c (V_old cells; keep NULL = all kept, then
 * V_mid = V_old) -- in c: each unchanged cell's index in c, -1 for the
 * children of selected cells (sel NULL = all selected).  For
 * gis_build_graph_memo_begin. */
int gis_covering_origin(gis_ctx* ctx, int64_t V_old, const uint8_t* keep, int64_t V_mid,
                        const uint8_t* sel, int64_t V_new, int64_t* origin);
/* the other direction (device int64 [V_old]): a cell's index in
 * subdivide(retain(c, keep), sel) if carried over unchanged, -2 - (index of
 * its first child) if selected (children are consecutive), -1 if removed */
int gis_covering_forward(gis_ctx* ctx, int64_t V_old, const uint8_t* keep, int64_t V_mid,
                         const uint8_t* sel, int64_t* fwd);

/* ---- adaptive selection (cg/adaptive.py:61-170) -------------------------- */
/* boundary mask: some enlarged-box probe lies in no closed cell of idx */
int gis_select_boundary(gis_ctx* ctx, const gis_index* idx, const double* lo,
                        const double* hi, int64_t V, double delta, int32_t face_points,
                        uint8_t* out);
/* exact k nearest centres (distance, index) of Q query points (device
 * [Q][n]) among the V cells (centres 0.5*(lo+hi)); excluded: a centre equal
 * to the query.  out_idx: device int64[Q][k] (-1 padded); out_cnt: int32[Q]. */
int gis_knn(gis_ctx* ctx, const gis_index* idx, const double* lo, const double* hi,
            int64_t V, const double* points, int64_t Q, int32_t k, int32_t exclude_point,
            int64_t* out_idx, int32_t* out_cnt);
/* select_neighborhood_mask: union of k-NN of boundary centres minus boundary */
int gis_select_neighborhood(gis_ctx* ctx, const gis_index* idx, const double* lo,
                            const double* hi, int64_t V, const uint8_t* boundary,
                            int32_t k, uint8_t* out);

/* Range forms for the multi-GPU engine (each rank takes its owned cells
 * [begin, end); masks stay indexed over all V cells):
 *  - boundary: writes out[begin..end) only;
 *  - neighbourhood: out (zeroed first) marks the k-NN of the boundary cells
 *    in [begin, end); exclude_boundary != 0 clears boundary cells afterwards
 *    (the single-GPU call), 0 leaves that to the caller after the ranks'
 *    masks are OR-reduced;
 *  - containment: the defect over new cells [begin, end). */
int gis_select_boundary_range(gis_ctx* ctx, const gis_index* idx, const double* lo,
                              const double* hi, int64_t V, int64_t begin, int64_t end,
                              double delta, int32_t face_points, uint8_t* out);
int gis_select_neighborhood_range(gis_ctx* ctx, const gis_index* idx, const double* lo,
                                  const double* hi, int64_t V, const uint8_t* boundary,
                                  int64_t begin, int64_t end, int32_t k,
                                  int32_t exclude_boundary, uint8_t* out);
/* a[i] = a[i] && !b[i] (device uint8[V]) */
int gis_mask_andnot(gis_ctx* ctx, uint8_t* a, const uint8_t* b, int64_t V);

/* ---- engine helpers (cg/engine.py:114-130, geometry.py:319-325) ---------- */
/* max over new cells of 1 - covered/volume against the previous index */
int gis_containment_defect(gis_ctx* ctx, const gis_index* prev, const double* prev_lo,
                           const double* prev_hi, int64_t prev_V, const double* lo,
                           const double* hi, int64_t V, double* defect);
/* largest cell diameter sqrt(sum_d (hi-lo)^2) (0 for V == 0) */
int gis_containment_defect_range(gis_ctx* ctx, const gis_index* prev, const double* prev_lo,
                                 const double* prev_hi, int64_t prev_V, const double* lo,
                                 const double* hi, int64_t V, int64_t begin, int64_t end,
                                 double* defect);
int gis_diameter(gis_ctx* ctx, int32_t n, const double* lo, const double* hi, int64_t V,
                 double* diameter);

/* ---- text formats (cg/graph.py:147-161, cg/geometry.py:588-620) --------- */
/* Edge list ("src_path dst_path\n" per edge, CSR order): row_off device
 * int64[V+1] receives the byte offset of each row's first line (row_off[V] =
 * total bytes); then gis_format_edges writes rows [row_begin, row_end) into
 * out (device, row_off[row_end] - row_off[row_begin] bytes). */
int gis_edge_list_offsets(gis_ctx* ctx, const int32_t* depths, const int64_t* indptr,
                          const int32_t* indices, int64_t V, int64_t* row_off);
int gis_format_edges(gis_ctx* ctx, const int32_t* depths, const int64_t* bits,
                     const int64_t* indptr, const int32_t* indices, int64_t V,
                     const int64_t* row_off, int64_t row_begin, int64_t row_end, char* out);
/* Cells-file rows ("path depth lo.. hi.. status\n", floats "%.17g") from
 * HOST arrays: depths int32[V], bits int64[V], lo/hi SoA [n][V], status
 * uint8[V] (0 retained, 1 boundary, 2 interior; NULL = retained).  *out is
 * malloc'ed (release with gis_free_host); threads <= 0 uses all cores. */
int gis_format_cells(const int32_t* depths, const int64_t* bits, const double* lo,
                     const double* hi, int32_t n, int64_t V, const uint8_t* status,
                     int32_t threads, char** out, int64_t* nbytes);
void gis_free_host(void* p);

#ifdef __cplusplus
}
#endif
#endif /* GIS_H_ */
