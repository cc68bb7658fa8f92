// K6: strongly connected components, reverse CSR, self loops and the
// strict-largest non-leaving mode (replaces cg/analysis.py:51-161 Tarjan +
// strongly_connected_components + non_leaving_mask(strict_largest=True), and
// SymbolicImage.reverse_csr / self_loop_mask, cg/graph.py:125-139).
//
// Tarjan is a sequential DFS.  The same partition is computed here by
// trim + colour propagation, all in one cooperative kernel:
//
//   trim     : delete vertices with no surviving successor or no surviving
//              predecessor (each is a trivial singleton component).  Scan
//              pointers into the forward and the reverse row only move
//              forward (as in K3), so all trim sweeps together read each
//              edge at most twice.
//   colour   : colour(v) = min vertex that reaches v among survivors,
//              pushed along forward edges with atomicMin; a vertex pushes
//              only in the round after its colour dropped.
//   mark     : every root r = colour(r) seeds a backward BFS over reverse
//              edges restricted to colour r; the marked set is exactly the
//              component of r, whose smallest vertex is r.  Marked vertices
//              are deleted and the loop repeats (trim first).
//
// Component ids are assigned afterwards in order of each component's
// smallest vertex (Tarjan's ids are DFS pop order; the reference's tests pin
// the partition, not the numbering: tests/test_analysis.py:21-63).
#include <cooperative_groups.h>

#include <cub/device/device_segmented_sort.cuh>

#include "gis_internal.cuh"

namespace cg = cooperative_groups;

namespace gis {

__device__ __forceinline__ bool live(const uint32_t* alive, int32_t t) {
  return (__ldcg(alive + (t >> 5)) >> (t & 31)) & 1u;
}

struct SccArgs {
  const int64_t* fro;   // forward row pointers [V+1]
  const int32_t* fidx;  // forward targets
  const int64_t* rro;   // reverse row pointers [V+1]
  const int32_t* ridx;  // reverse sources
  int64_t V;
  uint32_t* alive;      // bitmap of unassigned vertices
  int64_t* fp;          // forward trim pointers
  int64_t* bp;          // backward trim pointers
  int32_t* color;
  int32_t* stamp;       // colour frontier: round in which the colour dropped
  int32_t* mark;        // backward BFS: round of marking, -1 = unmarked
  int32_t* rep;         // smallest vertex of the assigned component
  unsigned long long* ctr;  // [3] rotating grid-wide counters
  int32_t* stats;       // [0] outer iterations, [1] grid rounds
  int32_t* qa;          // frontier queues (ping-pong), V entries each
  int32_t* qb;
  unsigned long long* qn;   // [3] rotating queue lengths
};

// Append v to queue q (length counter *n) with one atomic per warp.
__device__ __forceinline__ void warp_append(bool want, int32_t v, int32_t* q,
                                            unsigned long long* n) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(n, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (want) q[base + __popc(m & ((1u << lane) - 1u))] = v;
}

// Grid-wide sum of one value per thread; every thread gets the total.
struct GridSum {
  cg::grid_group grid;
  unsigned long long* ctr;
  int round = 0;
  __device__ unsigned long long operator()(unsigned long long v) {
    __shared__ unsigned long long bsum;
    if (threadIdx.x == 0) bsum = 0;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&bsum, v);
    __syncthreads();
    if (threadIdx.x == 0 && bsum) atomicAdd(ctr + (round % 3), bsum);
    grid.sync();
    const unsigned long long total = block_broadcast_load(ctr + (round % 3));
    if (grid.thread_rank() == 0) ctr[(round + 2) % 3] = 0ull;  // reused two rounds on
    ++round;
    return total;
  }
};

__global__ void __launch_bounds__(256) scc_coop_kernel(SccArgs a) {
  cg::grid_group grid = cg::this_grid();
  GridSum gsum{grid, a.ctr};
  const int lane = threadIdx.x & 31;
  const int64_t V = a.V;
  const int64_t words = (V + 31) >> 5;
  const int64_t gw = (int64_t)(grid.thread_rank() >> 5);
  const int64_t nw = (int64_t)(grid.size() >> 5);
  int outer = 0;
  int qrounds = 0;  // frontier rounds (colour + mark)
  while (true) {
    // ---- trim to a fixed point ------------------------------------------
    while (true) {
      unsigned long long deaths = 0;
      for (int64_t w = gw; w < words; w += nw) {
        const uint32_t word = __ldcg(a.alive + w);
        if (word == 0u) continue;
        const int64_t v = w * 32 + lane;
        bool dead = false;
        if (v < V && ((word >> lane) & 1u)) {
          int64_t p = a.fp[v];
          const int64_t e = a.fro[v + 1];
          p = first_live(a.fidx, p, e, a.alive);
          a.fp[v] = p;
          dead = (p == e);
          if (!dead) {
            int64_t q = a.bp[v];
            const int64_t e2 = a.rro[v + 1];
            q = first_live(a.ridx, q, e2, a.alive);
            a.bp[v] = q;
            dead = (q == e2);
          }
          if (dead) a.rep[v] = (int32_t)v;
        }
        const unsigned m = __ballot_sync(0xffffffffu, dead);
        if (m && lane == 0) {
          atomicAnd(a.alive + w, ~m);
          deaths += __popc(m);
        }
      }
      if (gsum(deaths) == 0) break;
    }
    // ---- survivors? ------------------------------------------------------
    unsigned long long cnt = 0;
    for (int64_t w = gw * 32 + lane; w < words; w += nw * 32) cnt += __popc(__ldcg(a.alive + w));
    if (gsum(cnt) == 0) break;
    ++outer;
    // Colour propagation and the backward marking run on frontier queues:
    // a warp per queued vertex, lanes over its row, so a round costs its
    // frontier rather than a scan of all V vertices.  Queue lengths rotate
    // over three counters (round k reads qn[k%3], appends to qn[(k+1)%3],
    // clears qn[(k+2)%3]), so no extra barrier is needed per round.
    if (grid.thread_rank() == 0) { a.qn[0] = 0; a.qn[1] = 0; a.qn[2] = 0; }
    grid.sync();
    for (int64_t vb = (int64_t)gw * 32; vb < V; vb += (int64_t)nw * 32) {
      const int64_t v = vb + lane;
      const bool on = v < V && live(a.alive, (int32_t)v);
      if (on) {
        a.color[v] = (int32_t)v;
        a.stamp[v] = 0;
        a.mark[v] = -1;
      }
      warp_append(on, (int32_t)v, a.qa, a.qn + 0);
    }
    grid.sync();
    // ---- colour propagation ----------------------------------------------
    {
      int32_t* cur = a.qa;
      int32_t* nxt = a.qb;
      for (int k = 0;; ++k) {
        const unsigned long long n = block_broadcast_load(a.qn + (k % 3));
        if (n == 0) break;
        if (grid.thread_rank() == 0) a.qn[(k + 2) % 3] = 0ull;
        for (int64_t i = gw; i < (int64_t)n; i += nw) {
          const int32_t v = cur[i];
          const int32_t c = __ldcg(a.color + v);
          const int64_t e = a.fro[v + 1];
          for (int64_t i0 = a.fro[v]; i0 < e; i0 += 32) {
            const int64_t j = i0 + lane;
            bool add = false;
            int32_t t = -1;
            if (j < e) {
              t = a.fidx[j];
              if (c < __ldcg(a.color + t) && live(a.alive, t) && atomicMin(a.color + t, c) > c)
                add = atomicExch(a.stamp + t, k + 1) != k + 1;  // once per round
            }
            warp_append(add, t, nxt, a.qn + ((k + 1) % 3));
          }
        }
        ++qrounds;
        grid.sync();
        int32_t* tq = cur;
        cur = nxt;
        nxt = tq;
      }
    }
    // ---- roots, then backward BFS within each colour ----------------------
    if (grid.thread_rank() == 0) { a.qn[0] = 0; a.qn[1] = 0; a.qn[2] = 0; }
    grid.sync();
    for (int64_t vb = (int64_t)gw * 32; vb < V; vb += (int64_t)nw * 32) {
      const int64_t v = vb + lane;
      const bool root = v < V && live(a.alive, (int32_t)v) && __ldcg(a.color + v) == (int32_t)v;
      if (root) a.mark[v] = 0;
      warp_append(root, (int32_t)v, a.qa, a.qn + 0);
    }
    grid.sync();
    {
      int32_t* cur = a.qa;
      int32_t* nxt = a.qb;
      for (int k = 0;; ++k) {
        const unsigned long long n = block_broadcast_load(a.qn + (k % 3));
        if (n == 0) break;
        if (grid.thread_rank() == 0) a.qn[(k + 2) % 3] = 0ull;
        for (int64_t i = gw; i < (int64_t)n; i += nw) {
          const int32_t v = cur[i];
          const int32_t c = __ldcg(a.color + v);
          const int64_t e = a.rro[v + 1];
          for (int64_t i0 = a.rro[v]; i0 < e; i0 += 32) {
            const int64_t j = i0 + lane;
            bool add = false;
            int32_t s = -1;
            if (j < e) {
              s = a.ridx[j];
              add = __ldcg(a.mark + s) == -1 && __ldcg(a.color + s) == c && live(a.alive, s) &&
                    atomicCAS(a.mark + s, -1, k + 1) == -1;
            }
            warp_append(add, s, nxt, a.qn + ((k + 1) % 3));
          }
        }
        ++qrounds;
        grid.sync();
        int32_t* tq = cur;
        cur = nxt;
        nxt = tq;
      }
    }
    // ---- assign the marked components -------------------------------------
    for (int64_t w = gw; w < words; w += nw) {
      const uint32_t word = __ldcg(a.alive + w);
      if (word == 0u) continue;
      const int64_t v = w * 32 + lane;
      bool done = false;
      if (v < V && ((word >> lane) & 1u) && __ldcg(a.mark + v) >= 0) {
        a.rep[v] = __ldcg(a.color + v);
        done = true;
      }
      const unsigned m = __ballot_sync(0xffffffffu, done);
      if (m && lane == 0) atomicAnd(a.alive + w, ~m);
    }
    grid.sync();
  }
  if (grid.thread_rank() == 0) {
    a.stats[0] = outer;
    a.stats[1] = gsum.round + qrounds;
  }
}

__global__ void scc_init_kernel(const int64_t* __restrict__ fro, const int64_t* __restrict__ rro,
                                int64_t V, int64_t* __restrict__ fp, int64_t* __restrict__ bp,
                                uint32_t* __restrict__ alive, int32_t* __restrict__ rep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < V) {
    fp[i] = fro[i];
    bp[i] = rro[i];
    rep[i] = -1;
  }
  const int64_t words = (V + 31) >> 5;
  if (i < words) {
    const int64_t rem = V - i * 32;
    alive[i] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  }
}

// ---------------------------------------------------------- reverse CSR ---
// in-degree count and scatter: warp per source row (coalesced row reads)
__global__ void indeg_kernel(const int64_t* __restrict__ fro, const int32_t* __restrict__ fidx,
                             int64_t V, unsigned long long* __restrict__ cnt) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w; s < V; s += nw)
    for (int64_t i = fro[s] + lane; i < fro[s + 1]; i += 32) atomicAdd(cnt + fidx[i], 1ull);
}

__global__ void scatter_kernel(const int64_t* __restrict__ fro, const int32_t* __restrict__ fidx,
                               int64_t V, unsigned long long* __restrict__ cursor,
                               int32_t* __restrict__ ridx) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w; s < V; s += nw)
    for (int64_t i = fro[s] + lane; i < fro[s + 1]; i += 32)
      ridx[atomicAdd(cursor + fidx[i], 1ull)] = (int32_t)s;
}

__global__ void self_loop_kernel(const int64_t* __restrict__ fro, const int32_t* __restrict__ fidx,
                                 int64_t V, uint8_t* __restrict__ out) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  uint8_t f = 0;
  for (int64_t i = fro[v]; i < fro[v + 1]; ++i)
    if (fidx[i] == (int32_t)v) { f = 1; break; }
  out[v] = f;
}

// ---------------------------------------------------------- numbering -----
__global__ void is_rep_kernel(const int32_t* __restrict__ rep, int64_t V, uint8_t* __restrict__ f) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V) f[v] = rep[v] == (int32_t)v;
}

__global__ void comp_id_kernel(const int32_t* __restrict__ rep, const int64_t* __restrict__ off,
                               int64_t V, int64_t* __restrict__ comp,
                               unsigned long long* __restrict__ sizes) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int64_t c = off[rep[v]];
  comp[v] = c;
  atomicAdd(sizes + c, 1ull);
}

__global__ void nontrivial_kernel(const int32_t* __restrict__ rep,
                                  const int64_t* __restrict__ off,
                                  const unsigned long long* __restrict__ sizes,
                                  const uint8_t* __restrict__ loops, int64_t V,
                                  uint8_t* __restrict__ nontriv) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V || rep[v] != (int32_t)v) return;
  const int64_t c = off[v];
  nontriv[c] = (sizes[c] >= 2 || loops[v]) ? 1 : 0;
}

// strict-largest seed: max over nontrivial components of (size, -id)
__global__ void best_comp_kernel(const unsigned long long* __restrict__ sizes,
                                 const uint8_t* __restrict__ nontriv, int64_t C,
                                 unsigned long long* __restrict__ best) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C || !nontriv[c]) return;
  atomicMax(best, (sizes[c] << 32) | (0xffffffffull - (unsigned long long)c));
}

__global__ void seed_kernel(const int64_t* __restrict__ comp, int64_t V,
                            const unsigned long long* __restrict__ best,
                            int32_t* __restrict__ mark) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const unsigned long long b = *best;
  const int64_t c = b ? (int64_t)(0xffffffffull - (b & 0xffffffffull)) : -1;
  mark[v] = comp[v] == c ? 0 : -1;
}

// default mode: every vertex of a nontrivial component seeds the closure
__global__ void seed_all_kernel(const int64_t* __restrict__ comp,
                                const uint8_t* __restrict__ nontriv, int64_t V,
                                int32_t* __restrict__ mark) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V) mark[v] = nontriv[comp[v]] ? 0 : -1;
}

// reverse-reachability closure of the vertices with mark == 0
__global__ void __launch_bounds__(256) closure_coop_kernel(const int64_t* __restrict__ rro,
                                                           const int32_t* __restrict__ ridx,
                                                           int64_t V, int32_t* mark,
                                                           int32_t* qa, int32_t* qb,
                                                           unsigned long long* qn,
                                                           int32_t* rounds) {
  // frontier queues as in scc_coop_kernel: qn[k % 3] holds round k's length
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)(grid.thread_rank() >> 5);
  const int64_t nw = (int64_t)(grid.size() >> 5);
  for (int64_t vb = gw * 32; vb < V; vb += nw * 32) {
    const int64_t v = vb + lane;
    warp_append(v < V && mark[v] == 0, (int32_t)v, qa, qn + 0);
  }
  grid.sync();
  int32_t* cur = qa;
  int32_t* nxt = qb;
  int k = 0;
  for (;; ++k) {
    const unsigned long long n = block_broadcast_load(qn + (k % 3));
    if (n == 0) break;
    if (grid.thread_rank() == 0) qn[(k + 2) % 3] = 0ull;
    for (int64_t i = gw; i < (int64_t)n; i += nw) {
      const int32_t v = cur[i];
      const int64_t e = rro[v + 1];
      for (int64_t i0 = rro[v]; i0 < e; i0 += 32) {
        const int64_t j = i0 + lane;
        int32_t s = -1;
        bool add = false;
        if (j < e) {
          s = ridx[j];
          add = __ldcg(mark + s) == -1 && atomicCAS(mark + s, -1, k + 1) == -1;
        }
        warp_append(add, s, nxt, qn + ((k + 1) % 3));
      }
    }
    grid.sync();
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
  if (grid.thread_rank() == 0) *rounds = k;
}

__global__ void mark_to_mask_kernel(const int32_t* __restrict__ mark, int64_t V,
                                    uint8_t* __restrict__ keep) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V) keep[v] = mark[v] >= 0;
}

// ------------------------------------------------------------ host side ---
// Device allocation released at scope exit (stream-ordered pool).
struct DevBuf {
  gis_ctx* ctx;
  void* p = nullptr;
  DevBuf(gis_ctx* c, size_t bytes) : ctx(c) {
    p = pool_alloc(ctx, bytes ? bytes : 16);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
  template <class T> T* as() const { return (T*)p; }
};

static int64_t edges_of(gis_ctx* ctx, const int64_t* indptr, int64_t V) {
  int64_t E = 0;
  read_back(ctx, &E, indptr + V, 8);
  GIS_REQUIRE(E >= 0 && E < ((int64_t)1 << 40), GIS_E_INVALID, "bad indptr");
  return E;
}

static void reverse_csr(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                        int64_t E, int64_t* rptr, int32_t* rind, bool sorted) {
  DevBuf cnt(ctx, (V + 1) * 8);
  GIS_CUDA(cudaMemsetAsync(cnt.p, 0, (V + 1) * 8, ctx->stream));
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(V * 32, 256), ctx->num_sms * 16);
  indeg_kernel<<<blocks, 256, 0, ctx->stream>>>(indptr, indices, V, cnt.as<unsigned long long>());
  count_launch(ctx);
  exclusive_scan_i64(ctx, cnt.as<int64_t>(), rptr, V + 1);
  if (E == 0) return;
  GIS_CUDA(cudaMemcpyAsync(cnt.p, rptr, V * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  scatter_kernel<<<blocks, 256, 0, ctx->stream>>>(indptr, indices, V,
                                                  cnt.as<unsigned long long>(), rind);
  count_launch(ctx);
  if (!sorted) return;
  // rows ascending, as the reference's lexsort((src, dst)) leaves them
  DevBuf alt(ctx, E * 4);
  cub::DoubleBuffer<int32_t> keys(rind, alt.as<int32_t>());
  size_t tb = 0;
  GIS_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys, E, V, rptr, rptr + 1,
                                              ctx->stream));
  DevBuf tmp(ctx, tb);
  GIS_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, keys, E, V, rptr, rptr + 1,
                                              ctx->stream));
  count_launch(ctx);
  if (keys.Current() != rind)
    GIS_CUDA(cudaMemcpyAsync(rind, keys.Current(), E * 4, cudaMemcpyDeviceToDevice, ctx->stream));
}

template <class K>
static int64_t coop_blocks(gis_ctx* ctx, K kernel, int64_t work_threads) {
  int per_sm = 0;
  GIS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
  GIS_REQUIRE(per_sm >= 1, GIS_E_CUDA, "cooperative kernel cannot be resident");
  int64_t blocks = (int64_t)per_sm * ctx->num_sms;
  return std::max<int64_t>(std::min<int64_t>(blocks, ceil_div(work_threads, 256)), 1);
}

// SCC partition of the graph whose reverse CSR is (rptr, rind): comp[v]
// (device int64[V]) numbered by smallest member, sizes (device int64[V],
// first n_comp used) and nontrivial (device uint8[V], first n_comp used).
// Returns n_comp; stats_host (optional) receives {outer iterations, grid rounds}.
static int64_t scc(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                   const int64_t* rptr, const int32_t* rind, int64_t* comp, int64_t* sizes,
                   uint8_t* nontriv, int32_t* stats_host) {
  const int64_t words = (V + 31) >> 5;
  DevBuf alive(ctx, words * 4), fp(ctx, V * 8), bp(ctx, V * 8), color(ctx, V * 4),
      stamp(ctx, V * 4), mark(ctx, V * 4), rep(ctx, V * 4), qa(ctx, V * 4), qb(ctx, V * 4),
      misc(ctx, 128);
  // misc: [0, 24) rotating counters, [32, 40) stats, [40, 48) component count,
  // [64, 88) rotating queue lengths
  GIS_CUDA(cudaMemsetAsync(misc.p, 0, 128, ctx->stream));
  int32_t* stats = (int32_t*)(misc.as<char>() + 32);
  scc_init_kernel<<<(unsigned)ceil_div(std::max(V, words), 256), 256, 0, ctx->stream>>>(
      indptr, rptr, V, fp.as<int64_t>(), bp.as<int64_t>(), alive.as<uint32_t>(),
      rep.as<int32_t>());
  count_launch(ctx);
  SccArgs a{indptr, indices, rptr, rind, V, alive.as<uint32_t>(), fp.as<int64_t>(),
            bp.as<int64_t>(), color.as<int32_t>(), stamp.as<int32_t>(), mark.as<int32_t>(),
            rep.as<int32_t>(), misc.as<unsigned long long>(), stats, qa.as<int32_t>(),
            qb.as<int32_t>(), misc.as<unsigned long long>() + 8};
  const int64_t blocks = coop_blocks(ctx, scc_coop_kernel, words * 32);
  void* args[] = {(void*)&a};
  GIS_CUDA(cudaLaunchCooperativeKernel((const void*)scc_coop_kernel, dim3((unsigned)blocks),
                                       dim3(256), args, 0, ctx->stream));
  count_launch(ctx);

  // number components by smallest member
  DevBuf flag(ctx, V), off(ctx, (V + 1) * 8), loops(ctx, V);
  is_rep_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(rep.as<int32_t>(), V,
                                                                     flag.as<uint8_t>());
  count_launch(ctx);
  exclusive_scan_u8_to_i64(ctx, flag.as<uint8_t>(), off.as<int64_t>(), V);
  GIS_CUDA(cudaMemsetAsync(sizes, 0, V * 8, ctx->stream));
  comp_id_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
      rep.as<int32_t>(), off.as<int64_t>(), V, comp, (unsigned long long*)sizes);
  count_launch(ctx);
  self_loop_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(indptr, indices, V,
                                                                        loops.as<uint8_t>());
  count_launch(ctx);
  nontrivial_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
      rep.as<int32_t>(), off.as<int64_t>(), (const unsigned long long*)sizes,
      loops.as<uint8_t>(), V, nontriv);
  count_launch(ctx);
  GIS_CUDA(cudaMemcpyAsync(misc.as<char>() + 40, off.as<int64_t>() + V, 8,
                           cudaMemcpyDeviceToDevice, ctx->stream));
  struct { int32_t st[2]; int64_t n; } out{};
  read_back(ctx, &out, misc.as<char>() + 32, 16);
  if (stats_host) {
    stats_host[0] = out.st[0];
    stats_host[1] = out.st[1];
  }
  return out.n;
}

}  // namespace gis

using namespace gis;

GIS_API int gis_reverse_csr(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                            int64_t V, int64_t* rptr, int32_t* rind, int32_t sorted) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX, GIS_E_INVALID, "V out of range");
    if (V == 0) {
      GIS_CUDA(cudaMemsetAsync(rptr, 0, 8, ctx->stream));
      return;
    }
    reverse_csr(ctx, indptr, indices, V, edges_of(ctx, indptr, V), rptr, rind, sorted != 0);
  });
}

GIS_API int gis_self_loops(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                           int64_t V, uint8_t* out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX, GIS_E_INVALID, "V out of range");
    if (V == 0) return;
    self_loop_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(indptr, indices, V,
                                                                          out);
    count_launch(ctx);
  });
}

GIS_API int gis_scc(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                    int64_t* comp, int64_t* sizes, uint8_t* nontrivial, int64_t* n_comp,
                    int32_t* stats) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX, GIS_E_INVALID, "V out of range");
    *n_comp = 0;
    if (stats) stats[0] = stats[1] = 0;
    if (V == 0) return;
    PhaseScope ps(ctx, PH_PRUNE);
    const int64_t E = edges_of(ctx, indptr, V);
    DevBuf rptr(ctx, (V + 1) * 8), rind(ctx, E * 4);
    reverse_csr(ctx, indptr, indices, V, E, rptr.as<int64_t>(), rind.as<int32_t>(), false);
    *n_comp = scc(ctx, indptr, indices, V, rptr.as<int64_t>(), rind.as<int32_t>(), comp, sizes,
                  nontrivial, stats);
  });
}

GIS_API int gis_non_leaving_scc(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                                int64_t V, int32_t strict_largest, uint8_t* keep,
                                int32_t* rounds) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX, GIS_E_INVALID, "V out of range");
    if (rounds) *rounds = 0;
    if (V == 0) return;
    PhaseScope ps(ctx, PH_PRUNE);
    const int64_t E = edges_of(ctx, indptr, V);
    DevBuf rptr(ctx, (V + 1) * 8), rind(ctx, E * 4), comp(ctx, V * 8), sizes(ctx, V * 8),
        nontriv(ctx, V), mark(ctx, V * 4), misc(ctx, 128);
    reverse_csr(ctx, indptr, indices, V, E, rptr.as<int64_t>(), rind.as<int32_t>(), false);
    const int64_t C = scc(ctx, indptr, indices, V, rptr.as<int64_t>(), rind.as<int32_t>(),
                          comp.as<int64_t>(), sizes.as<int64_t>(), nontriv.as<uint8_t>(),
                          nullptr);
    // misc: [0, 24) rotating counters, [32, 40) best key, [40, 44) closure rounds
    GIS_CUDA(cudaMemsetAsync(misc.p, 0, 128, ctx->stream));
    unsigned long long* ctr = misc.as<unsigned long long>();
    unsigned long long* best = ctr + 4;
    int32_t* rd = (int32_t*)(ctr + 5);
    if (C > 0 && strict_largest) {
      best_comp_kernel<<<(unsigned)ceil_div(C, 256), 256, 0, ctx->stream>>>(
          (const unsigned long long*)sizes.as<int64_t>(), nontriv.as<uint8_t>(), C, best);
      count_launch(ctx);
    }
    int32_t* markp = mark.as<int32_t>();
    if (strict_largest) {
      seed_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(comp.as<int64_t>(), V,
                                                                       best, markp);
    } else {
      seed_all_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
          comp.as<int64_t>(), nontriv.as<uint8_t>(), V, markp);
    }
    count_launch(ctx);
    const int64_t* rp = rptr.as<int64_t>();
    const int32_t* ri = rind.as<int32_t>();
    DevBuf cqa(ctx, V * 4), cqb(ctx, V * 4);
    unsigned long long* cqn = ctr + 8;  // misc [64, 88), zeroed above
    int32_t* qa_p = cqa.as<int32_t>();
    int32_t* qb_p = cqb.as<int32_t>();
    const int64_t blocks = coop_blocks(ctx, closure_coop_kernel, ((V + 31) >> 5) * 32);
    void* args[] = {(void*)&rp, (void*)&ri, (void*)&V, (void*)&markp, (void*)&qa_p,
                    (void*)&qb_p, (void*)&cqn, (void*)&rd};
    GIS_CUDA(cudaLaunchCooperativeKernel((const void*)closure_coop_kernel, dim3((unsigned)blocks),
                                         dim3(256), args, 0, ctx->stream));
    count_launch(ctx);
    mark_to_mask_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(markp, V, keep);
    count_launch(ctx);
    int32_t r = 0;
    read_back(ctx, &r, rd, 4);
    if (rounds) *rounds = r;
  });
}
