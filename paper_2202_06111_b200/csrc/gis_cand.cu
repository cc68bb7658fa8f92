// K2-general: CSR rows from explicit candidate lists.
//
// The warp-per-row kernels of gis_graph.cu read each (row, input) pair's
// candidates off a dense slot table and stage the U rectangles of a row in
// shared memory (U <= 128).  Two cases fall outside that and take this
// pipeline instead, with the same output (per source the ascending unique
// targets, cg/graph.py:181-193 `_csr_from_pairs`):
//
//   * a sparse dyadic index (coverings deeper than a dense slot table can
//     hold, up to the reference's MAX_DEPTH = 62, cg/geometry.py:34): the
//     pairs' candidates come from sparse_visit over the enclosure boxes;
//   * more than 128 inputs (e.g. m = 2 at 21 x 21 = 441 grid points,
//     cg/system.py:78-116): the candidates are the slots of the rectangles.
//
//   count  per pair (thread): candidates (sparse: a visit that only counts;
//          dense: the rectangle's slot count)
//   scan   pair offsets; row offsets = the offsets of each row's first pair
//   fill   per pair (thread): cell ids at the pair's offset (INT_MAX for
//          empty slots)
//   sort   cub segmented sort, one segment per row
//   unique warp per row: in-place compaction of the distinct ids, counts
//   scan   counts -> indptr; gis_csr_finish compacts as for K2
#include <cub/device/device_segmented_sort.cuh>

#include "gis_internal.cuh"

namespace gis {


template <int N>
__device__ __forceinline__ bool load_box(const PairBoxes& b, int64_t p, double (&l)[N],
                                         double (&h)[N]) {
  if (b.valid && b.valid[p] == 0) return false;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    l[d] = b.lo[p * b.ps + d * b.ds];
    h[d] = b.hi[p * b.ps + d * b.ds];
  }
  return true;
}

template <int N>
__global__ void sparse_count_kernel(GridDev g, PairBoxes b, int64_t P,
                                    int64_t* __restrict__ pc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > P) return;
  int64_t c = 0;
  double l[N], h[N];
  if (p < P && load_box<N>(b, p, l, h))
    sparse_visit<N>(g.sp, g.V, l, h, [&](int64_t) { ++c; return true; });
  pc[p] = c;  // pc[P] = 0: the exclusive scan yields the total
}

template <int N>
__global__ void sparse_fill_kernel(GridDev g, PairBoxes b, int64_t P,
                                   const int64_t* __restrict__ poff, int32_t* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double l[N], h[N];
  if (!load_box<N>(b, p, l, h)) return;
  int32_t* o = out + poff[p];
  sparse_visit<N>(g.sp, g.V, l, h, [&](int64_t c) { *o++ = (int32_t)c; return true; });
}

__global__ void rect_count_kernel(const int32_t* __restrict__ cnt, int64_t P,
                                  int64_t* __restrict__ pc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p <= P) pc[p] = p < P ? cnt[p] : 0;
}

// the slots of pair p's rectangle (row-major, last axis fastest) -> cells
template <int N>
__global__ void rect_fill_kernel(GridDev g, const int32_t* __restrict__ rect,
                                 const int32_t* __restrict__ cnt, int64_t P,
                                 const int64_t* __restrict__ poff, int32_t* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P || cnt[p] == 0) return;
  const int32_t* R = rect + p * 2 * N;
  int64_t c[N];
#pragma unroll
  for (int d = 0; d < N; ++d) c[d] = R[d];
  int32_t* o = out + poff[p];
  while (true) {
    int64_t s = 0;
#pragma unroll
    for (int d = 0; d < N; ++d) s += c[d] * g.stride[d];
    const int32_t cell = __ldg(g.slot + s);
    *o++ = cell < 0 ? INT_MAX : cell;
    int d = N - 1;
    while (d >= 0 && c[d] == R[N + d]) { c[d] = R[d]; --d; }
    if (d < 0) break;
    c[d]++;
  }
}

__global__ void row_offsets_kernel(const int64_t* __restrict__ poff, int64_t rows, int U,
                                   int64_t* __restrict__ roff) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= rows) roff[r] = poff[r * U];
}

// warp per row: the sorted segment's distinct ids (INT_MAX dropped) moved to
// the segment's start, in place (a write never passes the warp's reads)
__global__ void segment_unique_kernel(const int64_t* __restrict__ roff, int64_t rows,
                                      int32_t* __restrict__ keys, int64_t* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    const int64_t a = roff[r], e = roff[r + 1];
    int64_t w = a;
    int32_t prev = INT_MIN;
    for (int64_t base = a; base < e; base += 32) {
      const int64_t i = base + lane;
      const int32_t v = i < e ? keys[i] : INT_MAX;
      int32_t left = __shfl_up_sync(0xffffffffu, v, 1);
      if (lane == 0) left = prev;
      const bool keep = v != INT_MAX && v != left;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      prev = __shfl_sync(0xffffffffu, v, 31);
      __syncwarp();
      if (keep) keys[w + __popc(m & ((1u << lane) - 1u))] = v;
      w += __popc(m);
      __syncwarp();
    }
    if (lane == 0) rowcnt[r] = w - a;
  }
}

template <int N>
static void launch_count_fill(gis_ctx* ctx, const GridDev& g, const PairBoxes* boxes,
                              const int32_t* rect, const int32_t* cnt, int64_t P, int64_t* pc,
                              int64_t* poff, int32_t* out, int phase) {
  const unsigned nb = (unsigned)ceil_div(P + 1, 256);
  if (phase == 0) {
    if (boxes) sparse_count_kernel<N><<<nb, 256, 0, ctx->stream>>>(g, *boxes, P, pc);
    else rect_count_kernel<<<nb, 256, 0, ctx->stream>>>(cnt, P, pc);
  } else {
    if (boxes) sparse_fill_kernel<N><<<nb, 256, 0, ctx->stream>>>(g, *boxes, P, poff, out);
    else rect_fill_kernel<N><<<nb, 256, 0, ctx->stream>>>(g, rect, cnt, P, poff, out);
  }
  count_launch(ctx);
}

// Rows of `rows` x U pairs; boxes != nullptr: sparse candidates of the
// pairs' boxes, else the dense rectangles (rect, cnt).  Leaves the CSR
// pending for gis_csr_finish, like csr_from_rects.
void csr_from_candidates(gis_ctx* ctx, const GridDev& g, const PairBoxes* boxes,
                         const int32_t* rect, const int32_t* cnt, int64_t rows, int U,
                         int64_t* indptr, int64_t* n_edges) {
  GIS_REQUIRE(g.V < INT_MAX, GIS_E_CAPACITY, "covering too large for int32 targets");
  ctx->pending = PendingCsr{};
  const int64_t P = rows * U;
  int64_t* pc = (int64_t*)scratch(ctx, SC_ROWCNT, (P + 1) * 8);
  int64_t* poff = (int64_t*)scratch(ctx, SC_BIG, (P + 1) * 8);
  int64_t total = 0;
  auto count_fill = [&](int phase, int32_t* out) {
    switch (g.n) {
      case 1: launch_count_fill<1>(ctx, g, boxes, rect, cnt, P, pc, poff, out, phase); break;
      case 2: launch_count_fill<2>(ctx, g, boxes, rect, cnt, P, pc, poff, out, phase); break;
      case 3: launch_count_fill<3>(ctx, g, boxes, rect, cnt, P, pc, poff, out, phase); break;
      case 4: launch_count_fill<4>(ctx, g, boxes, rect, cnt, P, pc, poff, out, phase); break;
      default: throw Error{GIS_E_INVALID, "dimension out of range"};
    }
  };
  int64_t* roff = (int64_t*)scratch(ctx, SC_TOFF, (rows + 1) * 8);
  {
    PhaseScope ps(ctx, PH_CSR_AUX);
    count_fill(0, nullptr);
    exclusive_scan_i64(ctx, pc, poff, P + 1);
    row_offsets_kernel<<<(unsigned)ceil_div(rows + 1, 256), 256, 0, ctx->stream>>>(poff, rows, U,
                                                                                    roff);
    count_launch(ctx);
  }
  read_back(ctx, &total, poff + P, 8);
  GIS_REQUIRE(total < INT_MAX, GIS_E_CAPACITY,
              "more than 2^31 candidate edges in one build (split the rows)");
  int32_t* raw = (int32_t*)scratch(ctx, SC_WIDE, std::max<int64_t>(total, 1) * 4);
  int32_t* sorted = (int32_t*)scratch(ctx, SC_TEMP, std::max<int64_t>(total, 1) * 4);
  int64_t* rowcnt = (int64_t*)scratch(ctx, SC_ROWCNT, (rows + 1) * 8);  // pc is dead now
  {
    PhaseScope ps(ctx, PH_ROWS);
    if (total > 0) {
      count_fill(1, raw);
      size_t tb = 0;
      GIS_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, raw, sorted, (int)total,
                                                  (int)rows, roff, roff + 1, ctx->stream));
      void* tmp = scratch(ctx, SC_CUB, tb);
      GIS_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, tb, raw, sorted, (int)total, (int)rows,
                                                  roff, roff + 1, ctx->stream));
      count_launch(ctx);
      const int64_t blocks = std::min<int64_t>(ceil_div(rows * 32, 256), ctx->num_sms * 16);
      segment_unique_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, ctx->stream>>>(
          roff, rows, sorted, rowcnt);
      count_launch(ctx);
    } else if (rows > 0) {
      GIS_CUDA(cudaMemsetAsync(rowcnt, 0, rows * 8, ctx->stream));
    }
    GIS_CUDA(cudaMemsetAsync(rowcnt + rows, 0, 8, ctx->stream));
  }
  {
    PhaseScope ps(ctx, PH_CSR_AUX);
    exclusive_scan_i64(ctx, rowcnt, indptr, rows + 1);
  }
  int64_t E = 0;
  read_back(ctx, &E, indptr + rows, 8);
  ctx->pending.active = true;
  ctx->pending.rows = rows;
  ctx->pending.edges = E;
  ctx->pending.indptr = indptr;
  *n_edges = E;
}

}  // namespace gis
