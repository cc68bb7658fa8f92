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

#include "gis.h"
#include "gis_device.cuh"

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
  SC_CUB2, SC_PARAMS, SC_MISC, SC_MISC2, SC_MISC3, SC_WIDE, SC_REPLAY, SC_TCAND, SC_CORNER,
  SC_OWNER, SC_COUNT_
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
  // K1 work counters since the last gis_ctx_integrations: (cell, input,
  // sample) images produced, and integrations planned on the host (per-pair
  // samples + shared lower corners); k1_self (device) adds the corners
  // without an owner that enclose_kernel integrated itself
  int64_t k1_logical = 0, k1_planned = 0;
  unsigned long long* k1_self = nullptr;
  // cell bounds still arriving (gis_ctx_input_chunks): chunk c's cells lie
  // below in_ends[c] and are in place once in_evts[c] has completed
  std::vector<int64_t> in_ends;
  std::vector<cudaEvent_t> in_evts;
};

namespace gis {

// the stream waits for every pending input chunk (gis_ctx_input_chunks)
void inputs_wait_all(gis_ctx* ctx);

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


// Graph builds that keep / reuse padded enclosure boxes across the
// coverings of an adaptive run (gis_build_graph_memo_begin).
struct EncList {
  const int64_t* cells = nullptr;   // the row range's cells to integrate, ascending
  const int32_t* inv = nullptr;     // [rows] position in `cells`, or -1
  int64_t nlist = 0;
  const int64_t* origin = nullptr;  // [V] cell's index in the previous covering, or -1
  const double* memo_in = nullptr;  // boxes of the previous covering's cells
  int64_t memo_begin = 0, memo_rows = 0;  //   [memo_begin, memo_begin + memo_rows)
  double* memo_out = nullptr;       // [rows][U][2n] this build's boxes, or NULL
  bool incr = false;                // unchanged rows come from the previous graph
};

// K2: CSR of the rows' slot rectangles (gis_graph.cu); `incr`: rows of
// unchanged cells forward-mapped from the previous graph instead
struct IncrRows;
void csr_from_rects(gis_ctx* ctx, const GridDev& g, const int32_t* rect, const int32_t* cnt,
                    int64_t rows, int U, int64_t* indptr, int64_t* n_edges,
                    const IncrRows* incr = nullptr);

void csr_from_candidates(gis_ctx* ctx, const GridDev& g, const PairBoxes* boxes,
                         const int32_t* rect, const int32_t* cnt, int64_t rows, int U,
                         int64_t* indptr, int64_t* n_edges);

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
  double g0[GIS_MAX_DIM] = {}, gs[GIS_MAX_DIM] = {};  // GridDev slot guesses
  gis::GridDev dev() const {
    gis::GridDev g{};
    g.n = n;
    g.V = V;
    int64_t s = 1;
    for (int d = n - 1; d >= 0; --d) {
      // sparse: one slot spanning the root (faces = root lo / hi), so a
      // dense-only computation can never index past the placeholder arrays
      g.ns[d] = sparse ? 1 : ns[d];
      g.stride[d] = s;
      s *= ns[d];
      g.face[d] = faces + face_off[d];
    }
    for (int d = 0; d < GIS_MAX_DIM; ++d) {
      g.g0[d] = g0[d];
      g.gs[d] = gs[d];
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
