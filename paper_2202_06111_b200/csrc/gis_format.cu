// On-disk text formats of the reference:
//
//   edge list  (SymbolicImage.write_edge_list, cg/graph.py:147-161): one
//              "src_path dst_path\n" line per edge in CSR order; a path is
//              the cell's split bits, first split first, "-" for the root.
//              Integer/byte work: formatted on the GPU, warp per row, into a
//              device byte buffer the caller copies out in chunks.
//   cells file (write_cells_file, cg/geometry.py:588-620): one row per cell,
//              "path depth lo.. hi.. status\n" with floats in "%.17g".
//              Correctly rounded 17-digit decimal conversion is host work:
//              a multi-threaded C++ formatter over the host copies of the
//              covering arrays (glibc printf rounds correctly, as CPython's
//              format(x, ".17g") does).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <thread>

#include "gis_internal.cuh"

namespace gis {

__device__ __forceinline__ int path_len(int32_t depth) { return depth > 0 ? depth : 1; }

__device__ __forceinline__ void put_path(char* p, int32_t depth, int64_t bits) {
  if (depth <= 0) {
    p[0] = '-';
    return;
  }
  for (int j = 0; j < depth; ++j) p[j] = (char)('0' + ((bits >> (depth - 1 - j)) & 1));
}

// bytes of each row's lines: deg * (len(src) + 2) + sum len(dst)
__global__ void edge_row_bytes_kernel(const int32_t* __restrict__ depths,
                                      const int64_t* __restrict__ indptr,
                                      const int32_t* __restrict__ indices, int64_t V,
                                      int64_t* __restrict__ bytes) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r <= V; r += nw) {
    if (r == V) {
      if (lane == 0) bytes[V] = 0;
      continue;
    }
    const int64_t a = indptr[r], e = indptr[r + 1];
    int64_t s = 0;
    for (int64_t i = a + lane; i < e; i += 32) s += path_len(depths[indices[i]]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) bytes[r] = (e - a) * (path_len(depths[r]) + 2) + s;
  }
}

// lines of rows [r0, r1); row_off: exclusive scan of row bytes (global),
// written relative to row_off[r0]
__global__ void edge_write_kernel(const int32_t* __restrict__ depths,
                                  const int64_t* __restrict__ bits,
                                  const int64_t* __restrict__ indptr,
                                  const int32_t* __restrict__ indices,
                                  const int64_t* __restrict__ row_off, int64_t r0, int64_t r1,
                                  char* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t base0 = row_off[r0];
  for (int64_t r = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < r1;
       r += nw) {
    const int32_t sd = depths[r];
    const int64_t sb = bits[r];
    const int sl = path_len(sd);
    const int64_t a = indptr[r], e = indptr[r + 1];
    int64_t pos = row_off[r] - base0;
    for (int64_t i0 = a; i0 < e; i0 += 32) {
      const int64_t i = i0 + lane;
      int32_t td = 0;
      int64_t tb = 0;
      int len = 0;
      if (i < e) {
        const int32_t t = indices[i];
        td = depths[t];
        tb = bits[t];
        len = sl + path_len(td) + 2;
      }
      int incl = len;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (i < e) {
        char* p = out + pos + (incl - len);
        put_path(p, sd, sb);
        p[sl] = ' ';
        put_path(p + sl + 1, td, tb);
        p[len - 1] = '\n';
      }
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// -------------------------------------------------------- cells file ------
static void append_g17(std::string& s, double x) {
  char buf[40];
  if (x != x) {
    s += "nan";  // CPython prints every NaN as "nan"
    return;
  }
  const int k = snprintf(buf, sizeof(buf), "%.17g", x);
  s.append(buf, (size_t)k);
}

static void format_cells_range(const int32_t* depths, const int64_t* bits, const double* lo,
                               const double* hi, int n, int64_t V, const uint8_t* status,
                               int64_t a, int64_t b, std::string& s) {
  static const char* kStatus[3] = {"retained", "boundary", "interior"};
  s.reserve((size_t)(b - a) * (size_t)(48 + 50 * n));
  char num[24];
  for (int64_t i = a; i < b; ++i) {
    const int32_t d = depths[i];
    if (d <= 0) {
      s += '-';
    } else {
      for (int j = 0; j < d; ++j) s += (char)('0' + ((bits[i] >> (d - 1 - j)) & 1));
    }
    s += ' ';
    const int k = snprintf(num, sizeof(num), "%d", (int)d);
    s.append(num, (size_t)k);
    for (int q = 0; q < n; ++q) {
      s += ' ';
      append_g17(s, lo[(int64_t)q * V + i]);
    }
    for (int q = 0; q < n; ++q) {
      s += ' ';
      append_g17(s, hi[(int64_t)q * V + i]);
    }
    s += ' ';
    s += kStatus[status ? std::min<int>(status[i], 2) : 0];
    s += '\n';
  }
}

}  // namespace gis

using namespace gis;

GIS_API int gis_edge_list_offsets(gis_ctx* ctx, const int32_t* depths, const int64_t* indptr,
                                  const int32_t* indices, int64_t V, int64_t* row_off) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0, GIS_E_INVALID, "V out of range");
    int64_t* bytes = (int64_t*)scratch(ctx, SC_MISC2, (V + 1) * 8);
    const int64_t blocks = std::min<int64_t>(ceil_div((V + 1) * 32, 256), ctx->num_sms * 32);
    edge_row_bytes_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(depths, indptr, indices, V,
                                                                      bytes);
    count_launch(ctx);
    exclusive_scan_i64(ctx, bytes, row_off, V + 1);
  });
}

GIS_API int gis_format_edges(gis_ctx* ctx, const int32_t* depths, const int64_t* bits,
                             const int64_t* indptr, const int32_t* indices, int64_t V,
                             const int64_t* row_off, int64_t row_begin, int64_t row_end,
                             char* out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= V, GIS_E_INVALID,
                "row range out of bounds");
    if (row_end == row_begin) return;
    const int64_t blocks =
        std::min<int64_t>(ceil_div((row_end - row_begin) * 32, 256), ctx->num_sms * 32);
    edge_write_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(
        depths, bits, indptr, indices, row_off, row_begin, row_end, out);
    count_launch(ctx);
  });
}

GIS_API int gis_format_cells(const int32_t* depths, const int64_t* bits, const double* lo,
                             const double* hi, int32_t n, int64_t V, const uint8_t* status,
                             int32_t threads, char** out, int64_t* nbytes) {
  return guarded([&] {
    GIS_REQUIRE(n >= 1 && n <= GIS_MAX_DIM && V >= 0, GIS_E_INVALID, "bad covering shape");
    GIS_REQUIRE(out != nullptr && nbytes != nullptr, GIS_E_INVALID, "out is NULL");
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    T = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)T, 64, V / 4096 + 1}));
    std::vector<std::string> parts((size_t)T);
    std::vector<std::thread> pool;
    const int64_t step = ceil_div(std::max<int64_t>(V, 1), T);
    for (int t = 0; t < T; ++t) {
      const int64_t a = std::min<int64_t>(V, t * step), b = std::min<int64_t>(V, a + step);
      pool.emplace_back([&, t, a, b] {
        format_cells_range(depths, bits, lo, hi, n, V, status, a, b, parts[(size_t)t]);
      });
    }
    for (auto& th : pool) th.join();
    size_t total = 0;
    for (const auto& p : parts) total += p.size();
    char* buf = (char*)malloc(total ? total : 1);
    GIS_REQUIRE(buf != nullptr, GIS_E_CAPACITY, "out of host memory");
    size_t o = 0;
    for (const auto& p : parts) {
      memcpy(buf + o, p.data(), p.size());
      o += p.size();
    }
    *out = buf;
    *nbytes = (int64_t)total;
  });
}

GIS_API void gis_free_host(void* p) { free(p); }
