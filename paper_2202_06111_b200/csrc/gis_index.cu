// Grid index: the B200 replacement of the reference's blocked box tree
// (SpatialIndex, cg/geometry.py:416-505).
//
// A covering's cells are disjoint boxes whose faces lie on a rectilinear
// grid (for dyadic coverings: the recursive midpoints of the root box,
// cg/geometry.py:358; for arbitrary disjoint boxes: the sorted distinct
// face coordinates).  The index stores, per axis, the face coordinates and a
// dense slot table mapping every grid slot to the cell containing it (-1 if
// none).  A closed box query becomes one slot rectangle (binary search on
// each axis with the reference's closed comparisons) and the cells in it are
// table lookups; coarse cells occupy several slots and are deduplicated by
// the consumers.
#include <algorithm>
#include <cmath>

#include "gis_internal.cuh"

namespace gis {

__global__ void dyadic_ranges_kernel(const int32_t* __restrict__ depths,
                                     const int64_t* __restrict__ bits, int64_t V, GridDev g,
                                     int4 R, int32_t* __restrict__ cell_range,
                                     int32_t* __restrict__ slot, int* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int n = g.n;
  const int dep = depths[i];
  const int64_t b = bits[i];
  int64_t idx[GIS_MAX_DIM] = {0, 0, 0, 0};
  int cnt[GIS_MAX_DIM] = {0, 0, 0, 0};
  for (int l = 0; l < dep; ++l) {  // path bit l splits axis l mod n
    const int ax = l % n;
    idx[ax] = (idx[ax] << 1) | ((b >> (dep - 1 - l)) & 1);
    cnt[ax]++;
  }
  const int Rv[4] = {R.x, R.y, R.z, R.w};
  int64_t s0[GIS_MAX_DIM], s1[GIS_MAX_DIM];
  for (int d = 0; d < n; ++d) {
    const int sh = Rv[d] - cnt[d];
    if (sh < 0) { atomicOr(flag, 2); return; }
    s0[d] = idx[d] << sh;
    s1[d] = ((idx[d] + 1) << sh) - 1;
    cell_range[(int64_t)d * V + i] = (int32_t)s0[d];
    cell_range[(int64_t)(n + d) * V + i] = (int32_t)s1[d];
  }
  // scatter the cell index over its slot block
  int64_t c[GIS_MAX_DIM];
  for (int d = 0; d < n; ++d) c[d] = s0[d];
  while (true) {
    int64_t off = 0;
    for (int d = 0; d < n; ++d) off += c[d] * g.stride[d];
    if (atomicCAS(slot + off, -1, (int32_t)i) != -1) atomicOr(flag, 1);
    int d = n - 1;
    while (d >= 0 && c[d] == s1[d]) { c[d] = s0[d]; --d; }
    if (d < 0) break;
    c[d]++;
  }
}

// min and max depth in one pass (out[0] = min, out[1] = max; preset)
__global__ void depth_minmax_kernel(const int32_t* __restrict__ depths, int64_t V,
                                    int* __restrict__ out) {
  int mn = INT_MAX, mx = INT_MIN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = depths[i];
    mn = min(mn, d);
    mx = max(mx, d);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

// Sparse dyadic index: start codes and depths; flags a cell that is not
// strictly after its predecessor's code range (unsorted or overlapping).
__global__ void sparse_keys_kernel(const int32_t* __restrict__ depths,
                                   const int64_t* __restrict__ bits, int64_t V,
                                   uint64_t* __restrict__ key, uint8_t* __restrict__ dep,
                                   int* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int d = depths[i];
  const uint64_t k = (uint64_t)bits[i] << (kSparseKeyBits - d);
  key[i] = k;
  dep[i] = (uint8_t)d;
  if (i > 0) {
    const int dp = depths[i - 1];
    const uint64_t kp = (uint64_t)bits[i - 1] << (kSparseKeyBits - dp);
    const uint64_t endp = kp + ((uint64_t)1 << (kSparseKeyBits - dp));
    if (k < kp) atomicOr(flag, 8);
    else if (k < endp) atomicOr(flag, 1);
  }
}

__global__ void box_ranges_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                  int64_t V, GridDev g, int32_t* __restrict__ cell_range,
                                  int32_t* __restrict__ slot, int* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int n = g.n;
  int64_t s0[GIS_MAX_DIM], s1[GIS_MAX_DIM];
  for (int d = 0; d < n; ++d) {
    const double* F = g.face[d];
    const double l = lo[(int64_t)d * V + i], h = hi[(int64_t)d * V + i];
    // exact positions of the box faces in the face table
    int64_t a = 0, b = g.ns[d] + 1;
    while (a < b) { int64_t mid = (a + b) >> 1; if (F[mid] < l) a = mid + 1; else b = mid; }
    int64_t p = 0, q = g.ns[d] + 1;
    while (p < q) { int64_t mid = (p + q) >> 1; if (F[mid] < h) p = mid + 1; else q = mid; }
    s0[d] = a;
    s1[d] = p - 1;
    if (s1[d] < s0[d]) { atomicOr(flag, 4); return; }  // degenerate box
    cell_range[(int64_t)d * V + i] = (int32_t)s0[d];
    cell_range[(int64_t)(n + d) * V + i] = (int32_t)s1[d];
  }
  int64_t c[GIS_MAX_DIM];
  for (int d = 0; d < n; ++d) c[d] = s0[d];
  while (true) {
    int64_t off = 0;
    for (int d = 0; d < n; ++d) off += c[d] * g.stride[d];
    if (atomicCAS(slot + off, -1, (int32_t)i) != -1) atomicOr(flag, 1);
    int d = n - 1;
    while (d >= 0 && c[d] == s1[d]) { c[d] = s0[d]; --d; }
    if (d < 0) break;
    c[d]++;
  }
}

// Query boxes (SoA [n][Q]) -> slot rectangles [Q][2n] + counts (U = 1)
__global__ void rects_from_boxes_kernel(const double* __restrict__ qlo,
                                        const double* __restrict__ qhi, int64_t Q, GridDev g,
                                        int32_t* __restrict__ rect, int32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Q) return;
  const int n = g.n;
  int64_t count = 1;
  for (int d = 0; d < n; ++d) {
    int64_t a = 1, b = 0;
    if (count) {
      axis_range(g, d, qlo[(int64_t)d * Q + i], qhi[(int64_t)d * Q + i], a, b);
      if (a > b) count = 0; else count *= (b - a + 1);
    }
    rect[i * 2 * n + d] = (int32_t)a;
    rect[i * 2 * n + n + d] = (int32_t)b;
  }
  cnt[i] = (int32_t)count;
}

static const int64_t kMaxSlots = (int64_t)1 << 31;

static gis_index* alloc_index(gis_ctx* ctx, int n, int64_t V, const int64_t* ns,
                              const std::vector<std::vector<double>>& faces) {
  gis_index* ix = new gis_index();
  ix->stream = ctx->stream;
  ix->device = ctx->device;
  ix->n = n;
  ix->V = V;
  int64_t total = 1, nf = 0;
  for (int d = 0; d < n; ++d) {
    ix->ns[d] = ns[d];
    total *= ns[d];
    GIS_REQUIRE(total < kMaxSlots, GIS_E_CAPACITY,
                "grid index slot table exceeds 2^31 entries (covering too deep for a "
                "dense index)");
    ix->face_off[d] = nf;
    nf += ns[d] + 1;
    const double w = faces[d][ns[d]] - faces[d][0];
    ix->g0[d] = faces[d][0];
    ix->gs[d] = (std::isfinite(w) && w > 0) ? (double)ns[d] / w : 0.0;
  }
  ix->total = total;
  try {
    ix->faces_bytes = nf * sizeof(double);
    ix->slot_bytes = std::max<int64_t>(total, 1) * sizeof(int32_t);
    ix->range_bytes = std::max<int64_t>(2 * n * V, 1) * sizeof(int32_t);
    ix->faces = (double*)cached_alloc(ctx, ix->faces_bytes);
    ix->slot = (int32_t*)cached_alloc(ctx, ix->slot_bytes);
    ix->cell_range = (int32_t*)cached_alloc(ctx, ix->range_bytes);
    std::vector<double> flat;
    flat.reserve(nf);
    for (int d = 0; d < n; ++d) flat.insert(flat.end(), faces[d].begin(), faces[d].end());
    upload_to(ctx, ix->faces, flat.data(), nf * sizeof(double));
    GIS_CUDA(cudaMemsetAsync(ix->slot, 0xff, total * sizeof(int32_t), ctx->stream));
  } catch (...) {
    gis_index_free(ix);
    throw;
  }
  return ix;
}

static void check_flag(gis_ctx* ctx, int* dflag, gis_index* ix) {
  int flag = 0;
  read_back(ctx, &flag, dflag, sizeof(int));
  if (flag) {
    gis_index_free(ix);
    if (flag & 2) throw Error{GIS_E_INVALID, "cell deeper than the index resolution"};
    if (flag & 4) throw Error{GIS_E_INVALID, "degenerate (zero-width) box in index"};
    if (flag & 8) throw Error{GIS_E_INVALID, "cells are not in canonical order"};
    throw Error{GIS_E_OVERLAP, "index boxes overlap: not a covering of disjoint cells"};
  }
}

}  // namespace gis

using namespace gis;

// Dense slot tables above this many entries -- or above kSparseRatio slots
// per cell once past kSparseMin -- give way to the sparse index.
static constexpr int64_t kSparseMin = (int64_t)1 << 24;
static constexpr int64_t kSparseRatio = 1024;

GIS_API int gis_index_build_dyadic_mode(gis_ctx* ctx, int32_t n, const double* root_lo,
                                        const double* root_hi, const int32_t* depths,
                                        const int64_t* bits, int64_t V, int32_t mode,
                                        gis_index** out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(n >= 1 && n <= GIS_MAX_DIM, GIS_E_INVALID, "n out of range");
    GIS_REQUIRE(V >= 0, GIS_E_INVALID, "V must be >= 0");
    GIS_REQUIRE(V < INT_MAX, GIS_E_CAPACITY, "covering too large for int32 cell ids");
    GIS_REQUIRE(mode >= 0 && mode <= 2, GIS_E_INVALID, "mode must be 0 (auto), 1 (dense), "
                                                       "2 (sparse)");
    PhaseScope ps(ctx, PH_INDEX);
    int dmax = 0;
    if (V > 0) {
      // min / max depth (one read back per index build; min validates)
      int* dd = (int*)scratch(ctx, SC_MISC, 2 * sizeof(int));
      const int init[2] = {INT_MAX, INT_MIN};
      upload_to(ctx, dd, init, sizeof(init));
      depth_minmax_kernel<<<(unsigned)std::min<int64_t>(ceil_div(V, 256), ctx->num_sms * 8),
                            256, 0, ctx->stream>>>(depths, V, dd);
      count_launch(ctx);
      int mm[2];
      read_back(ctx, mm, dd, sizeof(mm));
      dmax = mm[1];
      GIS_REQUIRE(mm[0] >= 0, GIS_E_INVALID, "negative depth");
    }
    GIS_REQUIRE(dmax >= 0 && dmax <= 62, GIS_E_INVALID, "depth out of range");
    int R[GIS_MAX_DIM] = {0, 0, 0, 0};
    bool fits = true;
    double total_d = 1.0;
    for (int d = 0; d < n; ++d) {
      R[d] = (dmax + n - 1 - d) / n;  // splits of axis d at depth dmax
      fits = fits && R[d] <= 30;
      total_d *= std::ldexp(1.0, R[d]);
    }
    fits = fits && total_d < (double)kMaxSlots;
    const bool roomy = total_d <= (double)kSparseMin || total_d <= (double)kSparseRatio * V;
    GIS_REQUIRE(mode != 1 || fits, GIS_E_CAPACITY,
                "covering too deep for a dense grid index (use the sparse index)");
    const bool sparse = mode == 2 || (mode == 0 && !(fits && roomy));
    if (sparse) {
      gis_index* ix = new gis_index();
      ix->stream = ctx->stream;
      ix->device = ctx->device;
      ix->n = n;
      ix->V = V;
      ix->sparse = true;
      for (int d = 0; d < n; ++d) {
        ix->root_lo[d] = root_lo[d];
        ix->root_hi[d] = root_hi[d];
        ix->ns[d] = (int64_t)1 << std::min(R[d], 62);
        ix->face_off[d] = 0;
      }
      ix->total = -1;
      try {
        ix->skey_bytes = std::max<int64_t>(V, 1) * 8;
        ix->sdep_bytes = std::max<int64_t>(V, 1);
        ix->skey = (uint64_t*)cached_alloc(ctx, ix->skey_bytes);
        ix->sdep = (uint8_t*)cached_alloc(ctx, ix->sdep_bytes);
        // placeholders: sparse kernels never read faces / slots / ranges
        ix->faces_bytes = 2 * n * sizeof(double);
        ix->slot_bytes = ix->range_bytes = 16;
        ix->faces = (double*)cached_alloc(ctx, ix->faces_bytes);
        ix->slot = (int32_t*)cached_alloc(ctx, ix->slot_bytes);
        ix->cell_range = (int32_t*)cached_alloc(ctx, ix->range_bytes);
        std::vector<double> f;
        for (int d = 0; d < n; ++d) { f.push_back(root_lo[d]); f.push_back(root_hi[d]); }
        upload_to(ctx, ix->faces, f.data(), f.size() * sizeof(double));
        for (int d = 0; d < n; ++d) ix->face_off[d] = 2 * d;
      } catch (...) {
        gis_index_free(ix);
        throw;
      }
      if (V > 0) {
        int* flag = (int*)scratch(ctx, SC_MISC2, sizeof(int));
        GIS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
        sparse_keys_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
            depths, bits, V, ix->skey, ix->sdep, flag);
        count_launch(ctx);
        check_flag(ctx, flag, ix);
      }
      *out = ix;
      return;
    }
    int64_t ns[GIS_MAX_DIM] = {1, 1, 1, 1};
    std::vector<std::vector<double>> faces(n);
    for (int d = 0; d < n; ++d) {
      ns[d] = (int64_t)1 << R[d];
      // recursive midpoints 0.5*(lo+hi) exactly as the splits compute them
      std::vector<double>& F = faces[d];
      F.assign(ns[d] + 1, 0.0);
      F[0] = root_lo[d];
      F[ns[d]] = root_hi[d];
      for (int64_t len = ns[d]; len > 1; len >>= 1)
        for (int64_t i = 0; i < ns[d]; i += len) F[i + len / 2] = 0.5 * (F[i] + F[i + len]);
    }
    gis_index* ix = alloc_index(ctx, n, V, ns, faces);
    for (int d = 0; d < n; ++d) {
      ix->root_lo[d] = root_lo[d];
      ix->root_hi[d] = root_hi[d];
    }
    if (V > 0) {
      int* flag = (int*)scratch(ctx, SC_MISC2, sizeof(int));
      GIS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
      int4 Rv = make_int4(R[0], R[1], R[2], R[3]);
      dyadic_ranges_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
          depths, bits, V, ix->dev(), Rv, ix->cell_range, ix->slot, flag);
      count_launch(ctx);
      check_flag(ctx, flag, ix);
    }
    *out = ix;
  });
}

GIS_API int gis_index_build_dyadic(gis_ctx* ctx, int32_t n, const double* root_lo,
                                   const double* root_hi, const int32_t* depths,
                                   const int64_t* bits, int64_t V, gis_index** out) {
  return gis_index_build_dyadic_mode(ctx, n, root_lo, root_hi, depths, bits, V, 0, out);
}

GIS_API int gis_index_is_sparse(const gis_index* ix) { return ix && ix->sparse ? 1 : 0; }

GIS_API int gis_index_build_boxes(gis_ctx* ctx, int32_t n, const double* lo, const double* hi,
                                  int64_t V, gis_index** out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(n >= 1 && n <= GIS_MAX_DIM, GIS_E_INVALID, "n out of range");
    GIS_REQUIRE(V >= 0, GIS_E_INVALID, "V must be >= 0");
    std::vector<double> hl((size_t)n * V), hh((size_t)n * V);
    if (V > 0) {
      GIS_CUDA(cudaMemcpyAsync(hl.data(), lo, hl.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->stream));
      GIS_CUDA(cudaMemcpyAsync(hh.data(), hi, hh.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->stream));
      GIS_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    std::vector<std::vector<double>> faces(n);
    int64_t ns[GIS_MAX_DIM] = {1, 1, 1, 1};
    for (int d = 0; d < n; ++d) {
      std::vector<double>& F = faces[d];
      F.reserve(2 * V);
      for (int64_t i = 0; i < V; ++i) {
        const double a = hl[(size_t)d * V + i], b = hh[(size_t)d * V + i];
        GIS_REQUIRE(std::isfinite(a) && std::isfinite(b) && a <= b, GIS_E_INVALID,
                    "index boxes must be finite with lo <= hi");
        F.push_back(a);
        F.push_back(b);
      }
      std::sort(F.begin(), F.end());
      F.erase(std::unique(F.begin(), F.end()), F.end());
      if (F.size() < 2) F = {0.0, 1.0};  // empty index: one dummy slot
      ns[d] = (int64_t)F.size() - 1;
    }
    gis_index* ix = alloc_index(ctx, n, V, ns, faces);
    if (V > 0) {
      int* flag = (int*)scratch(ctx, SC_MISC2, sizeof(int));
      GIS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
      box_ranges_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
          lo, hi, V, ix->dev(), ix->cell_range, ix->slot, flag);
      count_launch(ctx);
      check_flag(ctx, flag, ix);
    }
    *out = ix;
  });
}

GIS_API int gis_index_free(gis_index* ix) {
  if (!ix) return GIS_OK;
  // back to the block cache, ordered after the work queued on the index's
  // stream (a plain cudaFree would synchronise the whole device)
  cached_free(ix->faces, ix->faces_bytes, ix->device, ix->stream);
  cached_free(ix->slot, ix->slot_bytes, ix->device, ix->stream);
  cached_free(ix->cell_range, ix->range_bytes, ix->device, ix->stream);
  if (ix->skey) cached_free(ix->skey, ix->skey_bytes, ix->device, ix->stream);
  if (ix->sdep) cached_free(ix->sdep, ix->sdep_bytes, ix->device, ix->stream);
  delete ix;
  return GIS_OK;
}

GIS_API int gis_index_shape(const gis_index* ix, int64_t* slots_per_axis, int64_t* total) {
  return guarded([&] {
    GIS_REQUIRE(ix != nullptr, GIS_E_INVALID, "index is NULL");
    for (int d = 0; d < ix->n; ++d) slots_per_axis[d] = ix->ns[d];
    *total = ix->total;
  });
}


GIS_API int gis_query_boxes_begin(gis_ctx* ctx, const gis_index* ix, const double* qlo,
                                  const double* qhi, int64_t Q, int64_t* qptr,
                                  int64_t* n_pairs) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(ix != nullptr, GIS_E_INVALID, "index is NULL");
    GridDev g = ix->dev();
    const int n = ix->n;
    if (ix->sparse) {  // the query boxes themselves (SoA [n][Q]) drive the visits
      PairBoxes pb{qlo, qhi, nullptr, 1, Q};
      csr_from_candidates(ctx, g, &pb, nullptr, nullptr, Q, 1, qptr, n_pairs);
      return;
    }
    int32_t* rect = (int32_t*)scratch(ctx, SC_RECT, std::max<int64_t>(Q, 1) * 2 * n * 4);
    int32_t* cnt = (int32_t*)scratch(ctx, SC_CNT, std::max<int64_t>(Q, 1) * 4);
    if (Q > 0) {
      rects_from_boxes_kernel<<<(unsigned)ceil_div(Q, 256), 256, 0, ctx->stream>>>(
          qlo, qhi, Q, g, rect, cnt);
      count_launch(ctx);
    }
    if (ix->V == 0 && Q > 0) {
      // empty index: nothing intersects
      GIS_CUDA(cudaMemsetAsync(cnt, 0, Q * 4, ctx->stream));
    }
    csr_from_rects(ctx, g, rect, cnt, Q, 1, qptr, n_pairs);
  });
}
