// Context, scratch memory, error reporting and scan/reduce plumbing.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <cstdlib>
#include <mutex>

#include "gis_internal.cuh"

namespace gis {

static thread_local std::string g_last_error;

bool trace_enabled() {
  static const bool on = getenv("GIS_TRACE") != nullptr;
  return on;
}

double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

void trace_slow(const char* what, double t0_us, size_t bytes) {
  if (!trace_enabled()) return;
  const double dt = now_us() - t0_us;
  if (dt > 1000.0) fprintf(stderr, "[gis trace] %s %.1f ms (%zu bytes)\n", what, dt / 1e3, bytes);
}

void set_error(const std::string& msg) { g_last_error = msg; }

cudaEvent_t take_event(gis_ctx* ctx) {
  if (!ctx->free_evts.empty()) {
    cudaEvent_t e = ctx->free_evts.back();
    ctx->free_evts.pop_back();
    return e;
  }
  cudaEvent_t e;
  GIS_CUDA(cudaEventCreate(&e));
  return e;
}

// DFMA throughput probe: independent fma chains per thread
__global__ void dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

void* pool_alloc(gis_ctx* ctx, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  const double t0 = now_us();
  if (ctx->pool)
    GIS_CUDA(cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream));
  else
    GIS_CUDA(cudaMallocAsync(&p, bytes, ctx->stream));
  trace_slow("pool_alloc", t0, bytes);
  return p;
}

void* scratch(gis_ctx* ctx, ScratchSlot s, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (ctx->cap[s] >= bytes) return ctx->buf[s];
  if (ctx->buf[s]) GIS_CUDA(cudaFreeAsync(ctx->buf[s], ctx->stream));
  ctx->buf[s] = nullptr;
  ctx->cap[s] = 0;
  const size_t want = bytes + bytes / 4 + 256;
  ctx->buf[s] = pool_alloc(ctx, want);
  ctx->cap[s] = want;
  return ctx->buf[s];
}

void read_back(gis_ctx* ctx, void* host, const void* dev, size_t bytes) {
  GIS_REQUIRE(bytes <= 4096, GIS_E_INVALID, "read_back too large");
  const double t0 = now_us();
  GIS_CUDA(cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  GIS_CUDA(cudaStreamSynchronize(ctx->stream));
  trace_slow("read_back sync", t0, bytes);
  memcpy(host, ctx->pinned, bytes);
}

struct CachedBlock {
  void* p;
  size_t bytes;
  int device;
  cudaEvent_t ready;
};
static std::mutex g_cache_mu;
static std::vector<CachedBlock> g_cache;
static size_t g_cache_bytes = 0;
static constexpr size_t kCacheMaxBlocks = 32;
// bound on idle device memory the cache holds (outside torch's allocator)
static constexpr size_t kCacheMaxBytes = size_t(8) << 30;

void* cached_alloc(gis_ctx* ctx, size_t bytes) {
  if (bytes == 0) bytes = 16;
  CachedBlock hit{nullptr, 0, 0, nullptr};
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int best = -1;
    for (int i = 0; i < (int)g_cache.size(); ++i) {
      const CachedBlock& b = g_cache[i];
      if (b.device == ctx->device && b.bytes >= bytes && b.bytes <= 2 * bytes + (1 << 20) &&
          (best < 0 || b.bytes < g_cache[best].bytes))
        best = i;
    }
    if (best >= 0) {
      hit = g_cache[best];
      g_cache_bytes -= hit.bytes;
      g_cache.erase(g_cache.begin() + best);
    }
  }
  if (hit.p) {
    GIS_CUDA(cudaStreamWaitEvent(ctx->stream, hit.ready, 0));
    cudaEventDestroy(hit.ready);
    return hit.p;
  }
  return pool_alloc(ctx, bytes);
}

// release every cached block of `device` (stream-ordered after its last use)
static void cache_flush(int device, cudaStream_t stream) {
  std::vector<CachedBlock> evict;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t i = 0; i < g_cache.size();) {
      if (g_cache[i].device == device) {
        evict.push_back(g_cache[i]);
        g_cache_bytes -= g_cache[i].bytes;
        g_cache.erase(g_cache.begin() + i);
      } else {
        ++i;
      }
    }
  }
  for (const CachedBlock& b : evict) {
    cudaStreamWaitEvent(stream, b.ready, 0);
    cudaEventDestroy(b.ready);
    cudaFreeAsync(b.p, stream);
  }
}

void cached_free(void* p, size_t bytes, int device, cudaStream_t stream) {
  if (!p) return;
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(e, stream) != cudaSuccess) {
    if (e) cudaEventDestroy(e);
    cudaFreeAsync(p, stream);
    return;
  }
  std::vector<CachedBlock> evict;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.push_back(CachedBlock{p, bytes ? bytes : 16, device, e});
    g_cache_bytes += g_cache.back().bytes;
    while (g_cache.size() > kCacheMaxBlocks ||
           (g_cache_bytes > kCacheMaxBytes && g_cache.size() > 1)) {
      evict.push_back(g_cache.front());
      g_cache_bytes -= g_cache.front().bytes;
      g_cache.erase(g_cache.begin());
    }
  }
  for (const CachedBlock& b : evict) {
    cudaStreamWaitEvent(stream, b.ready, 0);
    cudaEventDestroy(b.ready);
    cudaFreeAsync(b.p, stream);
  }
}

static constexpr int kRingSlots = 16;
static constexpr size_t kRingSlotBytes = 256 << 10;

void upload_to(gis_ctx* ctx, void* dev, const void* host, size_t bytes) {
  if (bytes == 0) return;
  if (bytes > kRingSlotBytes || !ctx->ring) {
    // large (rare): pageable copy, then wait so the host buffer may be freed
    GIS_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    GIS_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  const int slot = ctx->ring_next;
  ctx->ring_next = (slot + 1) % kRingSlots;
  GIS_CUDA(cudaEventSynchronize(ctx->ring_evt[slot]));  // slot's previous copy done
  char* stage = ctx->ring + (size_t)slot * kRingSlotBytes;
  memcpy(stage, host, bytes);
  GIS_CUDA(cudaMemcpyAsync(dev, stage, bytes, cudaMemcpyHostToDevice, ctx->stream));
  GIS_CUDA(cudaEventRecord(ctx->ring_evt[slot], ctx->stream));
}

void* upload(gis_ctx* ctx, ScratchSlot s, const void* host, size_t bytes) {
  void* d = scratch(ctx, s, bytes);
  upload_to(ctx, d, host, bytes);
  return d;
}

void exclusive_scan_i64(gis_ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  if (n <= 0) return;
  size_t tb = 0;
  GIS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, ctx->stream));
  void* t = scratch(ctx, SC_CUB, tb);
  GIS_CUDA(cub::DeviceScan::ExclusiveSum(t, tb, in, out, n, ctx->stream));
  count_launch(ctx);
}

__global__ void u8_to_i64_kernel(const uint8_t* __restrict__ in, int64_t n, int64_t add,
                                 int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (in ? (int64_t)(in[i] != 0) : 1) + add;
  else if (i == n) out[i] = 0;
}

void exclusive_scan_u8_to_i64(gis_ctx* ctx, const uint8_t* in, int64_t* out, int64_t n) {
  int64_t* tmp = (int64_t*)scratch(ctx, SC_CUB2, (n + 1) * 8);
  u8_to_i64_kernel<<<(unsigned)ceil_div(n + 1, 256), 256, 0, ctx->stream>>>(in, n, 0, tmp);
  count_launch(ctx);
  exclusive_scan_i64(ctx, tmp, out, n + 1);
}

void sum_i64(gis_ctx* ctx, const int64_t* in, int64_t n, int64_t* dev_out) {
  size_t tb = 0;
  GIS_CUDA(cub::DeviceReduce::Sum(nullptr, tb, in, dev_out, n, ctx->stream));
  void* t = scratch(ctx, SC_CUB, tb);
  GIS_CUDA(cub::DeviceReduce::Sum(t, tb, in, dev_out, n, ctx->stream));
  count_launch(ctx);
}

void max_i32(gis_ctx* ctx, const int32_t* in, int64_t n, int* dev_out) {
  size_t tb = 0;
  GIS_CUDA(cub::DeviceReduce::Max(nullptr, tb, in, dev_out, n, ctx->stream));
  void* t = scratch(ctx, SC_CUB, tb);
  GIS_CUDA(cub::DeviceReduce::Max(t, tb, in, dev_out, n, ctx->stream));
  count_launch(ctx);
}

}  // namespace gis

using namespace gis;

GIS_API int gis_abi_version(void) { return GIS_ABI_VERSION; }

GIS_API const char* gis_last_error(void) { return g_last_error.c_str(); }

GIS_API int gis_ctx_create(gis_ctx** out, int device) {
  return guarded([&] {
    GIS_REQUIRE(out != nullptr, GIS_E_INVALID, "out is NULL");
    int ndev = 0;
    GIS_CUDA(cudaGetDeviceCount(&ndev));
    GIS_REQUIRE(device >= 0 && device < ndev, GIS_E_INVALID, "no such CUDA device");
    GIS_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    GIS_CUDA(cudaGetDeviceProperties(&prop, device));
    GIS_REQUIRE(prop.major >= 10, GIS_E_INVALID,
                "libgis is built for sm_100a (B200); device is sm_" +
                    std::to_string(prop.major * 10 + prop.minor));
    gis_ctx* c = new gis_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    if (cudaMallocHost(&c->pinned, 4096) != cudaSuccess) {
      delete c;
      throw Error{GIS_E_CUDA, "cudaMallocHost failed"};
    }
    if (cudaMallocHost((void**)&c->ring, (size_t)kRingSlots * kRingSlotBytes) != cudaSuccess)
      c->ring = nullptr;  // uploads fall back to synchronous pageable copies
    for (int i = 0; i < kRingSlots; ++i)
      GIS_CUDA(cudaEventCreateWithFlags(&c->ring_evt[i], cudaEventDisableTiming));
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&c->pool, &props) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;  // keep freed scratch cached in OUR pool
      cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    } else {
      cudaGetLastError();
      c->pool = nullptr;  // allocations fall back to the default pool, untouched
    }
    *out = c;
  });
}

namespace gis {
void inputs_wait_all(gis_ctx* ctx) {
  for (cudaEvent_t e : ctx->in_evts) GIS_CUDA(cudaStreamWaitEvent(ctx->stream, e, 0));
  ctx->in_evts.clear();
  ctx->in_ends.clear();
}
}  // namespace gis

GIS_API int gis_ctx_input_chunks(gis_ctx* ctx, int32_t n, const int64_t* ends,
                                 void* const* events) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(n >= 0 && (n == 0 || (ends && events)), GIS_E_INVALID, "bad chunk list");
    gis::inputs_wait_all(ctx);  // an earlier list not consumed: waited for, dropped
    for (int i = 0; i < n; ++i) {
      GIS_REQUIRE(ends[i] > (i ? ends[i - 1] : 0) && events[i], GIS_E_INVALID,
                  "chunk ends must ascend, events non-null");
      ctx->in_ends.push_back(ends[i]);
      ctx->in_evts.push_back((cudaEvent_t)events[i]);
    }
  });
}

GIS_API int gis_ctx_trim(gis_ctx* ctx, uint64_t* released) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    uint64_t before = 0, after = 0;
    if (ctx->pool)
      cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &before);
    for (int s = 0; s < SC_COUNT_; ++s) {
      if (ctx->buf[s]) GIS_CUDA(cudaFreeAsync(ctx->buf[s], ctx->stream));
      ctx->buf[s] = nullptr;
      ctx->cap[s] = 0;
    }
    cache_flush(ctx->device, ctx->stream);
    GIS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->pool) {
      GIS_CUDA(cudaMemPoolTrimTo(ctx->pool, 0));
      cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &after);
    }
    if (released) *released = before > after ? before - after : 0;
  });
}

GIS_API int gis_ctx_pool_reserved(gis_ctx* ctx, uint64_t* bytes) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(bytes, GIS_E_INVALID, "null argument");
    *bytes = 0;
    if (ctx->pool)
      GIS_CUDA(cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, bytes));
  });
}

GIS_API int gis_ctx_destroy(gis_ctx* ctx) {
  if (!ctx) return GIS_OK;
  cudaStreamSynchronize(ctx->stream);
  for (int s = 0; s < SC_COUNT_; ++s)
    if (ctx->buf[s]) cudaFreeAsync(ctx->buf[s], ctx->stream);
  cache_flush(ctx->device, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  if (ctx->k1_self) cudaFree(ctx->k1_self);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->ring) cudaFreeHost(ctx->ring);
  for (cudaEvent_t e : ctx->ring_evt)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return GIS_OK;
}

GIS_API int gis_ctx_set_stream(gis_ctx* ctx, void* stream) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(ctx != nullptr, GIS_E_INVALID, "ctx is NULL");
    ctx->stream = (cudaStream_t)stream;
  });
}

GIS_API int64_t gis_ctx_launch_count(const gis_ctx* ctx) { return ctx ? ctx->launches : 0; }

GIS_API int gis_ctx_enable_timing(gis_ctx* ctx, int on) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    ctx->timing = on != 0;
  });
}

GIS_API int gis_ctx_phase_times(gis_ctx* ctx, double* ms, int64_t* counts) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int p = 0; p < PH_COUNT_; ++p) { ms[p] = 0.0; counts[p] = 0; }
    for (const PhaseEvt& e : ctx->evts) {
      float t = 0.f;
      GIS_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
      ms[e.phase] += t;
      counts[e.phase] += 1;
      ctx->free_evts.push_back(e.a);
      ctx->free_evts.push_back(e.b);
    }
    ctx->evts.clear();
  });
}

GIS_API int gis_ctx_integrations(gis_ctx* ctx, int64_t* images, int64_t* integrations) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(images && integrations, GIS_E_INVALID, "null argument");
    unsigned long long self = 0;
    if (ctx->k1_self) {
      read_back(ctx, &self, ctx->k1_self, sizeof(self));
      GIS_CUDA(cudaMemsetAsync(ctx->k1_self, 0, sizeof(self), ctx->stream));
    }
    *images = ctx->k1_logical;
    *integrations = ctx->k1_planned + (int64_t)self;
    ctx->k1_logical = ctx->k1_planned = 0;
  });
}

GIS_API int gis_fp64_peak(gis_ctx* ctx, double* tflops) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    double* out = (double*)scratch(ctx, SC_MISC, 8);
    const int iters = 4096, threads = 256;
    const int blocks = ctx->num_sms * 8;
    dfma_probe_kernel<<<blocks, threads, 0, ctx->stream>>>(out, 64, 1.0000001, 1e-12);  // warm
    count_launch(ctx);
    cudaEvent_t a = take_event(ctx), b = take_event(ctx);
    GIS_CUDA(cudaEventRecord(a, ctx->stream));
    for (int r = 0; r < 5; ++r)
      dfma_probe_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters, 1.0000001, 1e-12);
    GIS_CUDA(cudaEventRecord(b, ctx->stream));
    GIS_CUDA(cudaEventSynchronize(b));
    float t = 0.f;
    GIS_CUDA(cudaEventElapsedTime(&t, a, b));
    ctx->free_evts.push_back(a);
    ctx->free_evts.push_back(b);
    const double flops = 5.0 * blocks * threads * (double)iters * 8.0 * 2.0;
    *tflops = flops / (t * 1e-3) / 1e12;
  });
}
