// Internal helpers shared by the libgis translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gis.h"

namespace gis {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);

struct Error {
  int code;
  std::string msg;
};

#define GIS_CUDA(expr)                                                          \
  do {                                                                          \
    cudaError_t e_ = (expr);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      throw ::gis::Error{GIS_E_CUDA, std::string(#expr) + ": " +                \
                                         cudaGetErrorString(e_)};               \
    }                                                                           \
  } while (0)

#define GIS_REQUIRE(cond, code, msg)                                            \
  do {                                                                          \
    if (!(cond)) throw ::gis::Error{(code), (msg)};                             \
  } while (0)

// Wrap an API body: converts exceptions into status + thread-local message.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return GIS_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GIS_E_INVALID;
  }
}

// -------------------------------------------------------------- tracing ----
// GIS_TRACE=1: host-side durations of allocation / synchronisation points
// longer than 1 ms go to stderr (diagnostics for host stalls).
bool trace_enabled();
double now_us();
void trace_slow(const char* what, double t0_us, size_t bytes = 0);

// ------------------------------------------------------------ scratch ------
enum ScratchSlot {
  SC_RECT = 0, SC_CNT, SC_TOFF, SC_TEMP, SC_ROWCNT, SC_BIG, SC_BITMAP, SC_CUB,
  SC_CUB2, SC_PARAMS, SC_MISC, SC_MISC2, SC_MISC3, SC_WIDE, SC_REPLAY, SC_COUNT_
};

enum Phase { PH_ENCLOSE = 0, PH_ROWS, PH_CSR_AUX, PH_PRUNE, PH_INDEX, PH_COVER, PH_COUNT_ };

struct PhaseEvt {
  int phase;
  cudaEvent_t a, b;
};

struct PendingCsr {
  bool active = false;
  int64_t rows = 0;
  int64_t edges = 0;
  const int64_t* indptr = nullptr;  // caller's device indptr
};

}  // namespace gis

struct gis_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  void* buf[gis::SC_COUNT_] = {};
  size_t cap[gis::SC_COUNT_] = {};
  void* pinned = nullptr;  // small pinned host staging for scalars
  // pinned upload ring: kRingSlots slots of kRingSlotBytes, each reusable once
  // its event (recorded after the copy that read it) has completed
  char* ring = nullptr;
  cudaEvent_t ring_evt[16] = {};
  int ring_next = 0;
  gis::PendingCsr pending;
  int64_t launches = 0;
  int num_sms = 148;
  bool timing = false;
  std::vector<gis::PhaseEvt> evts;
  std::vector<cudaEvent_t> free_evts;
  // private stream-ordered pool: every libgis device allocation comes from
  // it (release threshold unlimited, so steady-state reuse never maps new
  // memory), and gis_ctx_trim returns it to the device.  The device's
  // default pool -- used by other cudaMallocAsync users -- is left alone.
  cudaMemPool_t pool = nullptr;
};

namespace gis {

// grow-only scratch buffer bound to a slot of the context
void* scratch(gis_ctx* ctx, ScratchSlot s, size_t bytes);
// stream-ordered allocation from the context's private pool (free with
// cudaFreeAsync on any stream)
void* pool_alloc(gis_ctx* ctx, size_t bytes);
// synchronous copy of a few scalars device->host through pinned staging
void read_back(gis_ctx* ctx, void* host, const void* dev, size_t bytes);
// upload a small host array into a scratch slot (ordered on the stream)
void* upload(gis_ctx* ctx, ScratchSlot s, const void* host, size_t bytes);
// Process-wide cache of released device blocks (per device).  Reuse waits on
// an event recorded at release, so a block is handed out only after the work
// queued before its release.  Avoids cudaMallocAsync in steady state, which
// can stall the host for milliseconds while the pool maps memory.
void* cached_alloc(gis_ctx* ctx, size_t bytes);
void cached_free(void* p, size_t bytes, int device, cudaStream_t stream);
// host -> device copy of a host array through pinned staging: the host never
// waits for queued device work (a pageable cudaMemcpyAsync can)
void upload_to(gis_ctx* ctx, void* dev, const void* host, size_t bytes);

inline void count_launch(gis_ctx* ctx) {
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error{GIS_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Per-phase CUDA-event timing (enabled by gis_ctx_enable_timing): a scoped
// marker records an event pair on the context stream around a phase.
cudaEvent_t take_event(gis_ctx* ctx);
struct PhaseScope {
  gis_ctx* ctx;
  int phase;
  cudaEvent_t a = nullptr;
  PhaseScope(gis_ctx* c, int p) : ctx(c), phase(p) {
    if (ctx->timing) {
      a = take_event(ctx);
      cudaEventRecord(a, ctx->stream);
    }
  }
  ~PhaseScope() {
    if (a) {
      cudaEvent_t b = take_event(ctx);
      cudaEventRecord(b, ctx->stream);
      ctx->evts.push_back(PhaseEvt{phase, a, b});
    }
  }
};

// exclusive scans / reductions (CUB, compiled into libgis)
void exclusive_scan_i64(gis_ctx* ctx, const int64_t* in, int64_t* out, int64_t n);
void exclusive_scan_u8_to_i64(gis_ctx* ctx, const uint8_t* in, int64_t* out, int64_t n);
void sum_i64(gis_ctx* ctx, const int64_t* in, int64_t n, int64_t* dev_out);
void max_i32(gis_ctx* ctx, const int32_t* in, int64_t n, int* dev_out);

// First position in [p, e) whose target is set in the `alive` bitmap (e if
// none).  Dead targets come in long runs (rows ascend in CellId order and the
// dead set grows as regions), so 8 entries are probed per step as
// independent loads rather than one dependent load at a time.
__device__ __forceinline__ int64_t first_live(const int32_t* __restrict__ idx, int64_t p,
                                              int64_t e, const uint32_t* alive) {
  constexpr int kW = 8;
  auto bit = [&](int32_t t) { return (__ldcg(alive + (t >> 5)) >> (t & 31)) & 1u; };
  while (p + kW <= e) {
    int32_t c[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) c[j] = idx[p + j];
    unsigned live = 0;
#pragma unroll
    for (int j = 0; j < kW; ++j) live |= bit(c[j]) << j;
    if (live) return p + __ffs(live) - 1;
    p += kW;
  }
  while (p < e && !bit(idx[p])) ++p;
  return p;
}

// A grid-wide counter read after grid.sync(): one thread per block loads it
// and broadcasts through shared memory (every thread loading the same word
// serialises hundreds of thousands of requests on one L2 line).
__device__ __forceinline__ unsigned long long block_broadcast_load(
    const unsigned long long* p) {
  __shared__ unsigned long long v;
  __syncthreads();
  if (threadIdx.x == 0) v = *((volatile const unsigned long long*)p);
  __syncthreads();
  return v;
}

// ----------------------------------------------------------- grid index ---
// Rectilinear slot grid: per axis the sorted face coordinates F[0..ns] and a
// dense slot table mapping each grid slot to the covering cell that contains
// it (or -1).  Row-major, last axis fastest.
//
// Sparse dyadic index (coverings too deep, or too sparse, for a dense slot
// table: the reference's MAX_DEPTH = 62, cg/geometry.py:34): the cells'
// path-aligned start codes key[i] = bits << (62 - depth), ascending in
// canonical order (cg/geometry.py:200-203), and their depths.  A box query
// descends the implicit binary tree of the root's dyadic splits (axis =
// level mod n, midpoints 0.5*(lo+hi) exactly as Covering.subdivide computes
// them, cg/geometry.py:358), pruned by closed box intersection and by binary
// searches for the cells inside each node's code range; it visits the
// intersecting cells in ascending index order.  O(V) memory at any depth.
struct SparseDev {
  const uint64_t* key;   // [V] ascending
  const uint8_t* dep;    // [V]
  double rlo[GIS_MAX_DIM], rhi[GIS_MAX_DIM];
};

struct GridDev {
  int n;
  int64_t ns[GIS_MAX_DIM];       // slots per axis
  int64_t stride[GIS_MAX_DIM];   // slot-table strides
  const double* face[GIS_MAX_DIM];
  const int32_t* slot;
  const int32_t* cell_slo;       // per cell, per axis first slot  [n][V]
  const int32_t* cell_shi;       // per cell, per axis last slot   [n][V]
  int64_t V;
  int sparse;                    // 1: no slot table, query through `sp`
  SparseDev sp;
};

static constexpr int kSparseKeyBits = 62;  // = MAX_DEPTH

// Query boxes of K2-general (gis_cand.cu): box of pair p on axis d at
// lo[p * ps + d * ds] (AoS: ps = n, ds = 1; SoA query arrays: ps = 1,
// ds = Q); valid == nullptr: every pair valid.
struct PairBoxes {
  const double* lo;
  const double* hi;
  const uint8_t* valid;
  int64_t ps, ds;
};
void csr_from_candidates(gis_ctx* ctx, const GridDev& g, const PairBoxes* boxes,
                         const int32_t* rect, const int32_t* cnt, int64_t rows, int U,
                         int64_t* indptr, int64_t* n_edges);

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* __restrict__ k, int64_t a,
                                                   int64_t b, uint64_t x) {
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (__ldg(k + m) < x) a = m + 1; else b = m;
  }
  return a;
}

// Visit every cell whose closed box meets the closed box [ql, qh] (cg/
// geometry.py:497-501: lo <= cell_hi and cell_lo <= hi on every axis), in
// ascending cell index.  f(cell) returns false to stop early.  NaN bounds
// meet nothing.
template <int N, class F>
__device__ __forceinline__ void sparse_visit(const SparseDev& s, int64_t V,
                                             const double (&ql)[N], const double (&qh)[N],
                                             F&& f) {
  double lo[N], hi[N];
  bool meets = V > 0;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    lo[d] = s.rlo[d];
    hi[d] = s.rhi[d];
    meets = meets && ql[d] <= hi[d] && lo[d] <= qh[d];
  }
  if (!meets) return;
  // frame j = the node at level j on the current path: its cell interval
  // [a, b), which child is being visited (0 none yet, 1 left, 2 right) and
  // the box coordinate the child replaced
  int64_t fa[kSparseKeyBits + 1], fb[kSparseKeyBits + 1];
  uint8_t side[kSparseKeyBits + 1];
  double saved[kSparseKeyBits + 1];
  int j = 0;
  uint64_t path = 0;
  fa[0] = 0;
  fb[0] = V;
  side[0] = 0;
  bool fresh = true;  // the node at level j was just entered
  while (j >= 0) {
    if (fresh) {
      fresh = false;
      const int sh = kSparseKeyBits - j;
      const uint64_t start = path << sh;
      const uint64_t end = start + ((uint64_t)1 << sh);  // exclusive
      const int64_t a = lower_bound_u64(s.key, fa[j], fb[j], start);
      const int64_t b = lower_bound_u64(s.key, a, fb[j], end);
      if (a == b) {
        side[j] = 2;  // no cell inside: done with this node
      } else if (s.dep[a] == j) {  // the node is a cell of the covering
        if (!f(a)) return;
        side[j] = 2;
      } else {
        fa[j] = a;
        fb[j] = b;
        side[j] = 0;
      }
    }
    if (side[j] == 2 || j == kSparseKeyBits) {  // pop: restore the parent's box
      if (j == 0) return;
      const int ax = (j - 1) % N;
      if (path & 1u) lo[ax] = saved[j]; else hi[ax] = saved[j];
      path >>= 1;
      --j;
      continue;
    }
    // next child of node j: split axis j mod N at the midpoint
    const int ax = j % N;
    const double mid = __dmul_rn(0.5, __dadd_rn(lo[ax], hi[ax]));
    const int c = side[j]++;  // 0 -> left, 1 -> right
    double nlo = lo[ax], nhi = hi[ax];
    if (c == 0) nhi = mid; else nlo = mid;
    if (!(qh[ax] >= nlo && ql[ax] <= nhi)) continue;  // the child misses the query
    saved[j + 1] = (c == 0) ? hi[ax] : lo[ax];
    lo[ax] = nlo;
    hi[ax] = nhi;
    path = (path << 1) | (uint64_t)c;
    fa[j + 1] = fa[j];
    fb[j + 1] = fb[j];
    ++j;
    fresh = true;
  }
}

// Closed-interval slot range of [qlo, qhi] on one axis:
//   a = first j with F[j+1] >= qlo, b = last j with F[j] <= qhi.
// NaN bounds give an empty range (cg/geometry.py:497-501 semantics).
__device__ __forceinline__ void axis_range(const double* __restrict__ F, int64_t ns,
                                           double qlo, double qhi, int64_t& a,
                                           int64_t& b) {
  // a: first k in [1, ns] with F[k] >= qlo, minus 1 (ns if none)
  int64_t lo = 1, hi = ns + 1;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (F[mid] >= qlo) hi = mid; else lo = mid + 1;
  }
  a = lo - 1;
  // b: last k in [0, ns-1] with F[k] <= qhi (-1 if none)
  lo = 0; hi = ns;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (F[mid] <= qhi) lo = mid + 1; else hi = mid;
  }
  b = lo - 1;
}

}  // namespace gis

struct gis_index {
  cudaStream_t stream = nullptr;  // stream the index was built (and is released) on
  bool sparse = false;            // dyadic index without a slot table (SparseDev)
  uint64_t* skey = nullptr;       // sparse: [V] start codes
  uint8_t* sdep = nullptr;        // sparse: [V] depths
  size_t skey_bytes = 0, sdep_bytes = 0;
  double root_lo[GIS_MAX_DIM] = {}, root_hi[GIS_MAX_DIM] = {};
  int device = 0;
  size_t faces_bytes = 0, slot_bytes = 0, range_bytes = 0;
  int n = 0;
  int64_t V = 0;
  int64_t ns[GIS_MAX_DIM] = {};
  int64_t total = 0;
  double* faces = nullptr;      // concatenated per-axis face arrays (device)
  int64_t face_off[GIS_MAX_DIM] = {};
  int32_t* slot = nullptr;      // slot table (device)
  int32_t* cell_range = nullptr;  // [2][n][V] first/last slot per cell (device)
  gis::GridDev dev() const {
    gis::GridDev g{};
    g.n = n;
    g.V = V;
    int64_t s = 1;
    for (int d = n - 1; d >= 0; --d) {
      g.ns[d] = ns[d];
      g.stride[d] = s;
      s *= ns[d];
      g.face[d] = faces + face_off[d];
    }
    g.slot = slot;
    g.cell_slo = cell_range;
    g.cell_shi = cell_range + (size_t)n * V;
    g.sparse = sparse ? 1 : 0;
    g.sp.key = skey;
    g.sp.dep = sdep;
    for (int d = 0; d < GIS_MAX_DIM; ++d) {
      g.sp.rlo[d] = root_lo[d];
      g.sp.rhi[d] = root_hi[d];
    }
    return g;
  }
};

#define GIS_API extern "C" __attribute__((visibility("default")))
