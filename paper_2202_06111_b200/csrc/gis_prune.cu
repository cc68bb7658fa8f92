// K3: non-leaving pruning (replaces non_leaving_mask, cg/analysis.py:120-161).
//
// The reference computes the reverse-reachability closure of the nontrivial
// SCCs (Tarjan, a pure-Python loop).  That set equals the fixed point of
// deleting vertices with no surviving successor (tests/conftest.py:75-89,
// asserted by tests/test_analysis.py:74-82 and tests/test_acceptance.py:
// 252-272).  We compute that fixed point directly on the forward CSR, with
// no transpose:
//
//   alive    : bitmap over vertices (1 = not yet deleted)
//   state[v] : (current target << 32) | offset in v's row; every target
//              before the offset is known deleted.  Target -2 = not started.
//
// A sweep probes each alive vertex's current target (one coalesced 8-byte
// state read + a bitmap bit, usually L2-resident); only when that target
// has died does it read the row, advancing past deleted targets.  A vertex
// whose row is exhausted is deleted (bits only go 1 -> 0, so concurrent
// readers at worst see a deletion one sweep late).  Offsets only move
// forward, so all sweeps together read each edge at most once plus one state
// probe per alive vertex per sweep.  The loop ends after a sweep that
// deletes nothing.  Deletions are published with warp ballots + atomicAnd on
// the bitmap word.
#include <cooperative_groups.h>

#include "gis_internal.cuh"

namespace cg = cooperative_groups;

namespace gis {

__device__ __forceinline__ bool alive_bit(const uint32_t* alive, int32_t t) {
  return (__ldcg(alive + (t >> 5)) >> (t & 31)) & 1u;
}

static constexpr int64_t kNotStarted = (int64_t)(-2) * ((int64_t)1 << 32);

// One sweep over words [w0, w1) of vertices (warp per bitmap word).
// Rows are addressed through indptr (local rows: vertex v -> row v - vbase).
__device__ __forceinline__ unsigned long long sweep_words(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t vbase,
    int64_t vend, uint32_t* alive, int64_t* __restrict__ state, int64_t w0, int64_t w1,
    int64_t wstep) {
  const int lane = threadIdx.x & 31;
  unsigned long long deaths = 0;
  for (int64_t w = w0; w < w1; w += wstep) {
    const uint32_t word = __ldcg(alive + w);
    if (word == 0u) continue;
    const int64_t v = w * 32 + lane;
    bool dead = false;
    if (v < vend && ((word >> lane) & 1u)) {
      const int64_t row = v - vbase;
      const int64_t st = state[row];
      const int32_t t = (int32_t)(st >> 32);
      if (t < 0 || !alive_bit(alive, t)) {
        const int64_t a = indptr[row];
        const int64_t e = indptr[row + 1];
        int64_t p = a + (t == -2 ? 0 : (int64_t)(uint32_t)st + 1);
        p = first_live(indices, p, e, alive);
        dead = (p == e);
        state[row] = dead ? ((int64_t)(-1) << 32)
                          : (((int64_t)indices[p] << 32) | (int64_t)(uint32_t)(p - a));
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, dead);
    if (m && lane == 0) {
      atomicAnd(alive + w, ~m);
      deaths += __popc(m);
    }
  }
  return deaths;
}

__global__ void peel_init_kernel(int64_t nrows, int64_t* __restrict__ ptr,
                                 uint32_t* __restrict__ alive, int64_t V, int64_t words) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) ptr[i] = kNotStarted;
  if (i < words) {
    const int64_t rem = V - i * 32;
    alive[i] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  }
}

__global__ void __launch_bounds__(256)
    peel_coop_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                     int64_t V, uint32_t* alive, int64_t* __restrict__ ptr,
                     unsigned long long* counters, int* rounds_out) {
  cg::grid_group grid = cg::this_grid();
  const int64_t words = (V + 31) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  __shared__ unsigned long long bsum;
  int round = 0;
  while (true) {
    if (threadIdx.x == 0) bsum = 0;
    __syncthreads();
    const unsigned long long d = sweep_words(indptr, indices, 0, V, alive, ptr, gw, words, nw);
    if (d) atomicAdd(&bsum, d);
    __syncthreads();
    if (threadIdx.x == 0 && bsum) atomicAdd(counters + (round % 3), bsum);
    grid.sync();
    const unsigned long long total = block_broadcast_load(counters + (round % 3));
    if (grid.thread_rank() == 0) counters[(round + 2) % 3] = 0ull;  // used again in round+2
    ++round;
    if (total == 0) break;
  }
  if (grid.thread_rank() == 0) *rounds_out = round;
}

__global__ void peel_sweep_kernel(const int64_t* __restrict__ indptr,
                                  const int32_t* __restrict__ indices, int64_t vbase,
                                  int64_t vend, uint32_t* alive, int64_t* __restrict__ ptr,
                                  unsigned long long* counter) {
  const int64_t w0 = (vbase >> 5) + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int64_t w1 = (vend + 31) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  __shared__ unsigned long long bsum;
  if (threadIdx.x == 0) bsum = 0;
  __syncthreads();
  const unsigned long long d = sweep_words(indptr, indices, vbase, vend, alive, ptr, w0, w1, nw);
  if (d) atomicAdd(&bsum, d);
  __syncthreads();
  if (threadIdx.x == 0 && bsum) atomicAdd(counter, bsum);
}

__global__ void bitmap_to_mask_kernel(const uint32_t* __restrict__ words, int64_t V,
                                      uint8_t* __restrict__ mask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < V) mask[i] = (uint8_t)((words[i >> 5] >> (i & 31)) & 1u);
}

__global__ void mask_to_bitmap_kernel(const uint8_t* __restrict__ mask, int64_t V,
                                      uint32_t* __restrict__ words) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nwords = (V + 31) >> 5;
  const bool b = (i < V) && mask[i];
  const unsigned m = __ballot_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && (i >> 5) < nwords) words[i >> 5] = m;
}

}  // namespace gis

using namespace gis;

GIS_API int gis_bitmap_to_mask(gis_ctx* ctx, const uint32_t* words, int64_t V, uint8_t* mask) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (V <= 0) return;
    bitmap_to_mask_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(words, V, mask);
    count_launch(ctx);
  });
}

GIS_API int gis_mask_to_bitmap(gis_ctx* ctx, const uint8_t* mask, int64_t V, uint32_t* words) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (V <= 0) return;
    mask_to_bitmap_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(mask, V, words);
    count_launch(ctx);
  });
}

GIS_API int gis_prune(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                      uint8_t* keep, int32_t* rounds) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX, GIS_E_INVALID, "V out of range");
    if (V == 0) { if (rounds) *rounds = 0; return; }
    PhaseScope ps(ctx, PH_PRUNE);
    const int64_t words = (V + 31) >> 5;
    uint32_t* alive = (uint32_t*)scratch(ctx, SC_BITMAP, words * 4);
    int64_t* ptr = (int64_t*)scratch(ctx, SC_TOFF, V * 8);
    struct Ctr { unsigned long long c[3]; int rounds; };
    Ctr* ctr = (Ctr*)scratch(ctx, SC_MISC3, sizeof(Ctr));
    GIS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Ctr), ctx->stream));
    const int64_t nt = std::max(V, words);
    peel_init_kernel<<<(unsigned)ceil_div(nt, 256), 256, 0, ctx->stream>>>(V, ptr, alive, V,
                                                                           words);
    count_launch(ctx);
    int per_sm = 0;
    GIS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peel_coop_kernel, 256, 0));
    GIS_REQUIRE(per_sm >= 1, GIS_E_CUDA, "peel kernel cannot be resident");
    int64_t blocks = (int64_t)per_sm * ctx->num_sms;
    blocks = std::min<int64_t>(blocks, std::max<int64_t>(ceil_div(words * 32, 256), 1));
    unsigned long long* counters = ctr->c;
    int* rounds_d = &ctr->rounds;
    void* args[] = {(void*)&indptr, (void*)&indices, (void*)&V, (void*)&alive,
                    (void*)&ptr,    (void*)&counters, (void*)&rounds_d};
    GIS_CUDA(cudaLaunchCooperativeKernel((const void*)peel_coop_kernel, dim3((unsigned)blocks),
                                         dim3(256), args, 0, ctx->stream));
    count_launch(ctx);
    bitmap_to_mask_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(alive, V, keep);
    count_launch(ctx);
    if (rounds) {
      int r = 0;
      read_back(ctx, &r, rounds_d, sizeof(int));
      *rounds = r;
    }
  });
}

GIS_API int gis_peel_init(gis_ctx* ctx, const int64_t* indptr_local, int64_t V, int64_t v_begin,
                          int64_t v_end, uint32_t* alive, int64_t* ptr) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(0 <= v_begin && v_begin <= v_end && v_end <= V, GIS_E_INVALID,
                "bad owned range");
    const int64_t words = (V + 31) >> 5;
    const int64_t nrows = v_end - v_begin;
    const int64_t nt = std::max<int64_t>(std::max(nrows, words), 1);
    peel_init_kernel<<<(unsigned)ceil_div(nt, 256), 256, 0, ctx->stream>>>(nrows, ptr, alive, V,
                                                                           words);
    count_launch(ctx);
  });
}

GIS_API int gis_peel_sweep_acc(gis_ctx* ctx, const int64_t* indptr_local,
                               const int32_t* indices, int64_t v_begin, int64_t v_end,
                               uint32_t* alive, int64_t* ptr, int64_t* deaths_dev) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (v_end <= v_begin) return;  // empty shard
    GIS_REQUIRE(v_begin % 32 == 0, GIS_E_INVALID, "owned range must start on a bitmap word");
    const int64_t words = ((v_end + 31) >> 5) - (v_begin >> 5);
    if (words > 0) {
      const int64_t blocks = std::min<int64_t>(ceil_div(words * 32, 256), ctx->num_sms * 8);
      peel_sweep_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(
          indptr_local, indices, v_begin, v_end, alive, ptr, (unsigned long long*)deaths_dev);
      count_launch(ctx);
    }
  });
}

GIS_API int gis_peel_sweep(gis_ctx* ctx, const int64_t* indptr_local, const int32_t* indices,
                           int64_t v_begin, int64_t v_end, uint32_t* alive, int64_t* ptr,
                           int64_t* deaths) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    *deaths = 0;
    if (v_end <= v_begin) return;  // empty shard
    GIS_REQUIRE(v_begin % 32 == 0, GIS_E_INVALID, "owned range must start on a bitmap word");
    unsigned long long* ctr = (unsigned long long*)scratch(ctx, SC_MISC3, 8);
    GIS_CUDA(cudaMemsetAsync(ctr, 0, 8, ctx->stream));
    const int64_t words = ((v_end + 31) >> 5) - (v_begin >> 5);
    if (words > 0) {
      const int64_t blocks = std::min<int64_t>(ceil_div(words * 32, 256), ctx->num_sms * 8);
      peel_sweep_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(indptr_local, indices, v_begin,
                                                                   v_end, alive, ptr, ctr);
      count_launch(ctx);
    }
    unsigned long long d = 0;
    read_back(ctx, &d, ctr, 8);
    *deaths = (int64_t)d;
  });
}
