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
struct GridDev {
  int n;
  int64_t ns[GIS_MAX_DIM];       // slots per axis
  int64_t stride[GIS_MAX_DIM];   // slot-table strides
  const double* face[GIS_MAX_DIM];
  const int32_t* slot;
  const int32_t* cell_slo;       // per cell, per axis first slot  [n][V]
  const int32_t* cell_shi;       // per cell, per axis last slot   [n][V]
  int64_t V;
};

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
    return g;
  }
};

#define GIS_API extern "C" __attribute__((visibility("default")))
