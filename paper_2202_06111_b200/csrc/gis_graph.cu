// K2: symbolic-image CSR build (replaces _edges_for_range + query_boxes +
// _csr_from_pairs + merge_subgraphs, cg/graph.py:181-270 and
// cg/geometry.py:471-505).
//
// Input: per (row, input) the closed slot rectangle of its enclosure (K1
// epilogue) and the rectangle's slot count.  Per row the candidate targets
// are the slot-table entries of the U rectangles (duplicates across inputs
// and across the slots of coarse cells).  The row is produced sorted and
// unique, which is exactly the reference's lexsort + dedupe per source.
//
//   step 1  row totals T_r = sum_u cnt, exclusive scan -> candidate offsets
//   step 2  one warp per row (rows_kernel, software-pipelined row loads):
//           when the rectangles' bounding box holds <= 2048 slots, mark them
//           in a shared slot bitmap and sort only the unique slots' cells;
//           otherwise sort all T_r candidates.  Register sorts of <= 256
//           keys run in a lean high-occupancy pass; wider rows are listed
//           and redone by passes with 512- and 1024-key sorts; rows with
//           T_r > 1024 go to a block-per-row bitmap over all cells
//   step 3  exclusive scan of unique counts -> indptr
//   step 4  (gis_csr_finish) compaction into the caller's indices buffer
//
// Also here: gis_csr_from_pairs (radix sort of (src, dst) keys, dedupe, CSR)
// for merge_subgraphs, and gis_csr_sources.
#include <cub/device/device_radix_sort.cuh>

#include "gis_internal.cuh"

namespace gis {

static constexpr int kWarpsPerBlock = 8;
static constexpr int kMaxU = 128;       // inputs staged per warp in shared memory
static constexpr int kWarpCap = 1024;   // candidates sorted in registers per warp


// Per row: its candidate count T (slots of its U rectangles, duplicates
// included) and the room its deduplicated row needs in `temp`.  The room is
// T, or -- when `tcand` is given (3-D / 4-D, where the U rectangles overlap
// heavily: config 5's rows have T ~ 900 candidates in a ~400-slot box) --
// min(T, slots of the rectangles' bounding box), which bounds the unique
// targets too; T then goes to tcand (config 5's scratch: 30 -> 21 GB).
template <int N>
__global__ void row_total_kernel(const int32_t* __restrict__ cnt,
                                 const int32_t* __restrict__ rect, int64_t rows, int U,
                                 int64_t* __restrict__ tot, int64_t* __restrict__ tcand) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > rows) return;
  int64_t s = 0, room = 0;
  if (r < rows) {
    int32_t bl[N], bh[N];
#pragma unroll
    for (int d = 0; d < N; ++d) { bl[d] = INT_MAX; bh[d] = INT_MIN; }
    for (int u = 0; u < U; ++u) {
      const int32_t c = cnt[r * U + u];
      s += c;
      if (tcand && c > 0) {
        const int32_t* R = rect + (r * U + u) * 2 * N;
#pragma unroll
        for (int d = 0; d < N; ++d) { bl[d] = min(bl[d], R[d]); bh[d] = max(bh[d], R[N + d]); }
      }
    }
    room = s;
    if (tcand) {
      tcand[r] = s;
      int64_t vol = s > 0 ? 1 : 0;
#pragma unroll
      for (int d = 0; d < N; ++d) vol *= s > 0 ? (int64_t)(bh[d] - bl[d] + 1) : 1;
      room = min(s, vol);
    }
  }
  tot[r] = room;  // tot[rows] = 0 so the exclusive scan yields the grand total
}

static constexpr int kBmBits = 2048;  // slot bitmap over a row's bounding box
static constexpr int64_t kRoomBytes = (int64_t)8 << 30;
// Rows with at most this many candidates sort them directly.  The bitmap
// pass's fixed cost (bitmap clear, marking, extraction, slot decode) beats
// sorting a few keys per lane only in 2-D, where candidates are enumerated
// incrementally; in 3-D / 4-D the bitmap pass wins even for short rows
// (K2).
template <int N>
constexpr int kDirectMax = (N <= 2) ? 128 : 0;
static constexpr int kBmWords = kBmBits / 32;

template <int N>
struct RowStage {
  union {
    struct {
      int32_t pre[kMaxU + 1];   // prefix of candidate counts over inputs
      int32_t rpre[kMaxU + 1];  // prefix of rectangle rows (all axes but the last)
      int32_t lo[kMaxU][N];     // rectangle origin
      int32_t ext[kMaxU][N];    // rectangle extents
    };
    int32_t keys[kWarpCap];     // unique slots' cells (after the bitmap pass)
  };
  uint32_t bm[kBmWords];
};

template <int N>
__device__ __forceinline__ int32_t candidate(const RowStage<N>& st, int U, int32_t e,
                                             const GridDev& g) {
  // input whose rectangle holds candidate e
  int a = 0, b = U;  // pre[a] <= e < pre[b]
  while (b - a > 1) {
    const int mid = (a + b) >> 1;
    if (st.pre[mid] <= e) a = mid; else b = mid;
  }
  int32_t off = e - st.pre[a];
  int64_t s = 0;
#pragma unroll
  for (int d = N - 1; d > 0; --d) {
    int32_t rr;
    const int32_t q = div_small(off, st.ext[a][d], rr);
    s += (int64_t)(st.lo[a][d] + rr) * g.stride[d];
    off = q;
  }
  s += (int64_t)(st.lo[a][0] + off) * g.stride[0];  // off < ext[a][0]
  const int32_t c = __ldg(g.slot + s);
  return c < 0 ? INT_MAX : c;
}

// Bitonic sort of W*K keys, K per lane (lane-major) over the first W lanes
// (W = 8, 16 or 32; lanes past W hold INT_MAX and pair only among
// themselves, since every shuffle partner differs in bits below W).
// Strides >= K pair keys across lanes (shuffles; rolled for K >= 16 to bound
// code size), strides < K pair keys inside a lane (unrolled: static register
// indices).
template <int K, int W = 32>
__device__ __forceinline__ void warp_bitonic(int32_t (&key)[K], int lane) {
#pragma unroll
  for (int size = 2; size <= W * K; size <<= 1) {
    const bool asc_lane = ((lane * K) & size) == 0;
    auto cross = [&](int stride) {
      const int lm = stride / K;
      const bool keep_min = ((lane & lm) == 0) == asc_lane;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t o = __shfl_xor_sync(0xffffffffu, key[k], lm);
        key[k] = keep_min ? min(key[k], o) : max(key[k], o);
      }
    };
    if constexpr (K >= 16) {  // wide (rare) rows: rolled, to bound code size
#pragma unroll 1
      for (int stride = size >> 1; stride >= K; stride >>= 1) cross(stride);
    } else {
#pragma unroll
      for (int stride = size >> 1; stride >= K; stride >>= 1) cross(stride);
    }
#pragma unroll
    for (int stride = (size >> 1) < K ? (size >> 1) : K >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if ((k & stride) == 0) {
          const bool asc = (((lane * K) + k) & size) == 0;
          const int32_t x = key[k], y = key[k | stride];
          if ((x > y) == asc) { key[k] = y; key[k | stride] = x; }
        }
      }
    }
  }
}

// Sort the per-lane keys (K per lane over the first W lanes, INT_MAX =
// none), drop duplicates and INT_MAX, write ascending to out; returns the
// number written.
template <int K, int W = 32>
__device__ __forceinline__ int32_t sort_unique_write_keys(int32_t (&key)[K], int lane,
                                                          int32_t* __restrict__ out) {
  warp_bitonic<K, W>(key, lane);
  int32_t prev = __shfl_up_sync(0xffffffffu, key[K - 1], 1);
  if (lane == 0) prev = INT_MIN;
  unsigned keep = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = (k == 0) ? prev : key[k - 1];
    if (key[k] != INT_MAX && key[k] != p) keep |= 1u << k;
  }
  const int mine = __popc(keep);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < W; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, W - 1);
  int pos = incl - mine;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (keep & (1u << k)) out[pos++] = key[k];
  return total;
}

// Sort the T keys produced by load(e), drop duplicates and INT_MAX, write
// ascending to out; returns the number written.
template <int K, class Load, int W = 32>
__device__ __forceinline__ int32_t sort_unique_write(int32_t T, int lane, Load load,
                                                     int32_t* __restrict__ out) {
  int32_t key[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t e = lane * K + k;
    key[k] = (e < T && lane < W) ? load(e) : INT_MAX;
  }
  return sort_unique_write_keys<K, W>(key, lane, out);
}

// Sort-unique-write with the register width chosen from the key count; KMAX
// (keys per lane) bounds the widest instantiation, and so the kernel's
// register footprint.
template <int KMAX, class Load>
__device__ __forceinline__ int32_t sort_dispatch(int32_t T, int lane, Load load,
                                                 int32_t* __restrict__ out) {
  // short rows sort over the first 8 / 16 lanes: fewer bitonic stages
  if (T <= 8) return sort_unique_write<1, Load, 8>(T, lane, load, out);
  if (T <= 16) return sort_unique_write<1, Load, 16>(T, lane, load, out);
  if (T <= 32) return sort_unique_write<1>(T, lane, load, out);
  if (T <= 64) return sort_unique_write<2>(T, lane, load, out);
  if (T <= 128) return sort_unique_write<4>(T, lane, load, out);
  if constexpr (KMAX >= 8) if (T <= 256) return sort_unique_write<8>(T, lane, load, out);
  if constexpr (KMAX >= 16) if (T <= 512) return sort_unique_write<16>(T, lane, load, out);
  if constexpr (KMAX >= 32) return sort_unique_write<32>(T, lane, load, out);
  return -1;
}

// Candidates e0 .. e0+K-1 of a row into key[] (INT_MAX past T): one binary
// search and one decode for e0, then an odometer over the rectangle's slots
// (last axis fastest), moving on to the next non-empty rectangle at its end.
template <int N, int K>
__device__ __forceinline__ void candidate_run(const RowStage<N>& st, int U, int32_t e0,
                                              int32_t T, const GridDev& g,
                                              int32_t (&key)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) key[k] = INT_MAX;
  if (e0 >= T) return;
  int a = 0, b = U;  // pre[a] <= e0 < pre[b]
  while (b - a > 1) {
    const int mid = (a + b) >> 1;
    if (st.pre[mid] <= e0) a = mid; else b = mid;
  }
  int32_t c[N];
  int32_t off = e0 - st.pre[a];
#pragma unroll
  for (int d = N - 1; d > 0; --d) {
    int32_t rr;
    off = div_small(off, st.ext[a][d], rr);
    c[d] = rr;
  }
  c[0] = off;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (e0 + k >= T) break;
    int64_t s = 0;
#pragma unroll
    for (int d = 0; d < N; ++d) s += (int64_t)(st.lo[a][d] + c[d]) * g.stride[d];
    const int32_t cell = __ldg(g.slot + s);
    key[k] = cell < 0 ? INT_MAX : cell;
    // next slot of this rectangle, or the first slot of the next one
    int d = N - 1;
    while (d >= 0 && ++c[d] == st.ext[a][d]) { c[d] = 0; --d; }
    if (d < 0) {
      ++a;
      while (a + 1 < U && st.pre[a + 1] <= e0 + k + 1) ++a;  // skip empty rectangles
    }
  }
}

template <int N, int K>
__device__ __forceinline__ int32_t direct_sort(const RowStage<N>& st, int U, int32_t T,
                                               const GridDev& g, int lane,
                                               int32_t* __restrict__ out) {
  int32_t key[K];
  candidate_run<N, K>(st, U, lane * K, T, g, key);
  return sort_unique_write_keys<K>(key, lane, out);
}

template <int N, int KMAX>
__device__ __forceinline__ int32_t direct_dispatch(const RowStage<N>& st, int U, int32_t T,
                                                   const GridDev& g, int lane,
                                                   int32_t* __restrict__ out) {
  if (T <= 32) return direct_sort<N, 1>(st, U, T, g, lane, out);
  if (T <= 64) return direct_sort<N, 2>(st, U, T, g, lane, out);
  if (T <= 128) return direct_sort<N, 4>(st, U, T, g, lane, out);
  if constexpr (KMAX >= 8) if (T <= 256) return direct_sort<N, 8>(st, U, T, g, lane, out);
  if constexpr (KMAX >= 16) if (T <= 512) return direct_sort<N, 16>(st, U, T, g, lane, out);
  if constexpr (KMAX >= 32) return direct_sort<N, 32>(st, U, T, g, lane, out);
  return -1;
}

// Deduplicate a row's candidate slots in a shared bitmap over the bounding
// box of its rectangles (one contiguous bit run per rectangle row along axis
// 0, set with word-masked atomicOr), then sort only the unique slots' cells.
// The bitmap is laid out with axis 0 fastest, then axis 1, ...: the cyclic
// splits refine axis 0 first and axis 1 next, so on a mixed-depth grid a
// coarse cell spans neighbouring slots along those axes, and a slot whose
// left (axis 0) or lower (axis 1) neighbour in the same bitmap word holds the
// same cell is not emitted (the cell's first occurrence is).  Coarse-cell
// duplicates then rarely push a row past this pass's sort; the sort's unique
// removes any that remain.  Returns the row's edge count; -1 (stage
// untouched) when more than kWarpCap slots are set; -2 (stage consumed: to
// the next pass) when more than 32 KMAX cells remain.
template <int N, int KMAX>
__device__ __forceinline__ int32_t bitmap_row(RowStage<N>& st, int U, const GridDev& g,
                                              const int32_t (&bl)[N], const int32_t (&bext)[N],
                                              int lane, int32_t* __restrict__ out) {
  uint32_t* bm = st.bm;
#pragma unroll
  for (int i = lane; i < kBmWords; i += 32) bm[i] = 0u;
  __syncwarp();
  const int32_t RR = st.rpre[U];  // rectangle rows along axis 0, over all inputs
  for (int32_t q = lane; q < RR; q += 32) {
    int a = 0, b = U;  // rpre[a] <= q < rpre[b]
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (st.rpre[mid] <= q) a = mid; else b = mid;
    }
    int32_t off = q - st.rpre[a];
    int32_t c[N];
#pragma unroll
    for (int d = N - 1; d > 1; --d) {
      int32_t rr;
      off = div_small(off, st.ext[a][d], rr);
      c[d] = rr;
    }
    if (N > 1) c[1] = off;  // off < ext[a][1]
    int32_t base = 0;
#pragma unroll
    for (int d = N - 1; d > 0; --d) base = base * bext[d] + (st.lo[a][d] + c[d] - bl[d]);
    base = base * bext[0] + (st.lo[a][0] - bl[0]);
    const int32_t b0 = base, b1 = base + st.ext[a][0];
    for (int32_t wi = b0 >> 5; wi <= (b1 - 1) >> 5; ++wi) {
      const int32_t lo = max(b0 - wi * 32, 0), hi = min(b1 - wi * 32, 32);
      const uint32_t m = (hi - lo == 32) ? 0xffffffffu : (((1u << (hi - lo)) - 1u) << lo);
      atomicOr(bm + wi, m);
    }
  }
  __syncwarp();
  int cnt = 0;
#pragma unroll
  for (int i = lane; i < kBmWords; i += 32) cnt += __popc(bm[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  const int Us = cnt;
  if (Us > kWarpCap) return -1;
  __syncwarp();  // rectangle stage is dead from here on: keys alias it
  // one bitmap word per step, one bit per lane: slot -> cell, placed in bit
  // order (axis 0 fastest)
  int32_t vol = 1, sbase = 0, str[N];
  float rinv[N];
#pragma unroll
  for (int d = 0; d < N; ++d) {
    vol *= bext[d];
    str[d] = (int32_t)g.stride[d];  // slot tables hold < 2^31 entries
    sbase += bl[d] * str[d];
    rinv[d] = 1.0f / (float)bext[d];
  }
  const int nwords = (vol + 31) >> 5;
  const int b0x = bext[0];
  int base = 0;
  for (int wi = 0; wi < nwords; ++wi) {
    const uint32_t word = bm[wi];
    const bool set = (word >> lane) & 1u;
    int32_t cell = INT_MIN, c0 = 0, c1 = 0;
    if (set) {
      int32_t bi = wi * 32 + lane;  // < 2^11: the float quotient is off by at most one
      int32_t s = sbase;
#pragma unroll
      for (int d = 0; d < N - 1; ++d) {
        int32_t qq = (int32_t)((float)bi * rinv[d]);
        int32_t rr = bi - qq * bext[d];
        if (rr < 0) { --qq; rr += bext[d]; } else if (rr >= bext[d]) { ++qq; rr -= bext[d]; }
        s += rr * str[d];
        if (d == 0) c0 = rr;
        if (d == 1) c1 = rr;
        bi = qq;
      }
      s += bi * str[N - 1];
      if (N == 1) c0 = bi;
      if (N == 2) c1 = bi;
      cell = __ldg(g.slot + s);
    }
    // the same cell at the axis-0 or axis-1 neighbour of this word: not emitted
    const int32_t left = __shfl_up_sync(0xffffffffu, cell, 1);
    const int src = lane >= b0x ? lane - b0x : lane;
    const int32_t down = __shfl_sync(0xffffffffu, cell, src);
    bool emit = set && cell >= 0;
    if (emit && c0 > 0 && lane > 0 && left == cell) emit = false;
    if (emit && N > 1 && c1 > 0 && lane >= b0x && down == cell) emit = false;
    const unsigned em = __ballot_sync(0xffffffffu, emit);
    if (emit) st.keys[base + __popc(em & ((1u << lane) - 1u))] = cell;
    base += __popc(em);
  }
  __syncwarp();
  if (base > 32 * KMAX) return -2;  // stage consumed: the row goes to the next pass
  const int32_t* keys = st.keys;
  auto load = [&](int32_t e) { return keys[e]; };
  return sort_dispatch<KMAX>(base, lane, load, out);
}

// One warp per row.  Pass 1 (KMAX = 8, lean registers for occupancy) takes
// rows whose sort fits 256 keys and appends the others to `wide`; pass 2
// (KMAX = 16) and pass 3 (KMAX = 32) run over the lists the previous pass
// left (rows_list).  Rows with more than kWarpCap candidates go to
// big_rows_kernel.
template <int N, int KMAX>
#ifndef GIS_K2_WIDE_BLOCKS  // pass-2 blocks per SM: 4 (64 registers, a few spills) beat 3 (80): config 5 15.1 vs 16.2 ms
#define GIS_K2_WIDE_BLOCKS 4
#endif
__global__ void __launch_bounds__(32 * kWarpsPerBlock,
                                  KMAX <= 8 ? 5 : (KMAX <= 16 ? GIS_K2_WIDE_BLOCKS : 2))
    rows_kernel(GridDev g, const int32_t* __restrict__ rect, const int32_t* __restrict__ cnt,
                int64_t rows, int U, const int64_t* __restrict__ toff,
                const int64_t* __restrict__ tcand,
                int32_t* __restrict__ temp, int64_t* __restrict__ rowcnt,
                int64_t* __restrict__ big, int64_t* __restrict__ nbig,
                int64_t* __restrict__ wide, int64_t* __restrict__ nwide,
                const int64_t* __restrict__ rows_list, const int64_t* __restrict__ nlist) {
  __shared__ RowStage<N> stage[kWarpsPerBlock];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  RowStage<N>& st = stage[w];
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  // Software pipelining: the next row's offsets, counts and rectangles (lane
  // u holds input u when U <= 32) are loaded before the current row is
  // processed, hiding their HBM latency behind the dedupe work.
  struct RowIn {
    int64_t t0, T;  // output offset, candidate count
    int32_t c;
    int32_t R[2 * N];
  };
  const bool pre = U <= 32;
  if (rows_list) rows = *nlist;
  auto row_of = [&](int64_t i) { return rows_list ? rows_list[i] : i; };
  auto fetch = [&](int64_t i, RowIn& in) {
    const int64_t r = row_of(i);
    in.t0 = toff[r];
    in.T = tcand ? tcand[r] : toff[r + 1] - in.t0;
    in.c = 0;
    if (pre && lane < U) {
      in.c = cnt[r * U + lane];
      const int32_t* R = rect + (r * U + lane) * 2 * N;
#pragma unroll
      for (int d = 0; d < 2 * N; ++d) in.R[d] = R[d];
    }
  };
  RowIn cur, nxt;
  int64_t i = (int64_t)blockIdx.x * kWarpsPerBlock + w;
  if (i < rows) fetch(i, cur);
  for (; i < rows; i += nwarps) {
    if (i + nwarps < rows) fetch(i + nwarps, nxt);
    const int64_t r = row_of(i);
    const int64_t T = cur.T;
    if (T == 0 || T > kWarpCap) {
      if (lane == 0) {
        if (T == 0) rowcnt[r] = 0;
        else big[atomicAdd((unsigned long long*)nbig, 1ull)] = r;
      }
      cur = nxt;
      continue;
    }
    // stage the U rectangles: prefix of counts and of rectangle rows, origin
    // and extents; bounding box of the non-empty ones
    int32_t carry = 0, rcarry = 0;
    int32_t bl[N], bh[N];
#pragma unroll
    for (int d = 0; d < N; ++d) { bl[d] = INT_MAX; bh[d] = INT_MIN; }
    for (int u0 = 0; u0 < U; u0 += 32) {
      const int u = u0 + lane;
      int32_t c = 0, rr = 0;
      if (u < U) {
        int32_t Rl[2 * N];
        if (pre) {
          c = cur.c;
#pragma unroll
          for (int d = 0; d < 2 * N; ++d) Rl[d] = cur.R[d];
        } else {
          c = cnt[r * U + u];
          const int32_t* R = rect + (r * U + u) * 2 * N;
#pragma unroll
          for (int d = 0; d < 2 * N; ++d) Rl[d] = R[d];
        }
        rr = c > 0 ? 1 : 0;
#pragma unroll
        for (int d = 0; d < N; ++d) {
          const int32_t lo = Rl[d], hi = Rl[N + d];
          st.lo[u][d] = lo;
          st.ext[u][d] = hi - lo + 1;
          if (d > 0) rr *= hi - lo + 1;  // bitmap_row marks runs along axis 0
          if (c > 0) { bl[d] = min(bl[d], lo); bh[d] = max(bh[d], hi); }
        }
      }
      int32_t incl = c, rincl = rr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        const int32_t rv = __shfl_up_sync(0xffffffffu, rincl, o);
        if (lane >= o) { incl += v; rincl += rv; }
      }
      if (u < U) { st.pre[u] = carry + incl - c; st.rpre[u] = rcarry + rincl - rr; }
      carry += __shfl_sync(0xffffffffu, incl, 31);
      rcarry += __shfl_sync(0xffffffffu, rincl, 31);
    }
    if (lane == 0) { st.pre[U] = carry; st.rpre[U] = rcarry; }
    int64_t vol = 1;
    int32_t bext[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        bl[d] = min(bl[d], __shfl_xor_sync(0xffffffffu, bl[d], o));
        bh[d] = max(bh[d], __shfl_xor_sync(0xffffffffu, bh[d], o));
      }
      bext[d] = bh[d] - bl[d] + 1;
      vol *= bext[d];
    }
    __syncwarp();
    int32_t* out = temp + cur.t0;
    const int32_t t = (int32_t)T;
    int32_t total = -1;
    if (vol <= kBmBits && t > kDirectMax<N>) total = bitmap_row<N, KMAX>(st, U, g, bl, bext, lane, out);
    if (total == -1 && t <= 32 * KMAX)  // candidates straight from the rectangles
      total = direct_dispatch<N, KMAX>(st, U, t, g, lane, out);
    if (lane == 0) {
      if (total >= 0) rowcnt[r] = total;
      else if (wide) wide[atomicAdd((unsigned long long*)nwide, 1ull)] = r;  // to pass 2
    }
    __syncwarp();
    cur = nxt;
  }
}

// ---- short rows, two per warp (3-D / 4-D first pass) -----------------------
// Most of a short row's cost is per-row fixed work done warp-wide (staging
// and prefix of the rectangles, bounding-box reduction, bitmap clear and
// count, a 32-lane sort of ~14 keys).  Here a half-warp (16 lanes) takes a
// row: the same slot-bitmap dedupe as bitmap_row over a bounding box of <=
// kHalfBits slots, then a 16-lane sort of <= 32 unique cells.  Rows that do
// not fit (more than 16 inputs, a larger box, more unique slots, T >
// kWarpCap) go to `rest` for rows_kernel.  Every shuffle / ballot / sync
// names only the half-warp's lanes, so the two halves may diverge.
static constexpr int kHalfBits = 1024;
static constexpr int kHalfWords = kHalfBits / 32;
static constexpr int kHalfU = 16;
static constexpr int kHalfKeys = 32;

template <int N>
struct HalfStage {
  int32_t pre[kHalfU + 1];
  int32_t rpre[kHalfU + 1];
  int32_t lo[kHalfU][N];
  int32_t ext[kHalfU][N];
  int32_t keys[kHalfKeys];
  uint32_t bm[kHalfWords];
};

// bitonic sort of 16*K keys over the half-warp (lane-major), then unique +
// write; returns the number written
template <int K>
__device__ __forceinline__ int32_t half_sort_unique_write(int32_t (&key)[K], int hl,
                                                         unsigned hm,
                                                         int32_t* __restrict__ out) {
#pragma unroll
  for (int size = 2; size <= 16 * K; size <<= 1) {
    const bool asc_lane = ((hl * K) & size) == 0;
#pragma unroll
    for (int stride = size >> 1; stride >= K; stride >>= 1) {
      const int lm = stride / K;
      const bool keep_min = ((hl & lm) == 0) == asc_lane;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t o = __shfl_xor_sync(hm, key[k], lm, 16);
        key[k] = keep_min ? min(key[k], o) : max(key[k], o);
      }
    }
#pragma unroll
    for (int stride = (size >> 1) < K ? (size >> 1) : K >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if ((k & stride) == 0) {
          const bool asc = (((hl * K) + k) & size) == 0;
          const int32_t x = key[k], y = key[k | stride];
          if ((x > y) == asc) { key[k] = y; key[k | stride] = x; }
        }
      }
    }
  }
  int32_t prev = __shfl_up_sync(hm, key[K - 1], 1, 16);
  if (hl == 0) prev = INT_MIN;
  unsigned keep = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = (k == 0) ? prev : key[k - 1];
    if (key[k] != INT_MAX && key[k] != p) keep |= 1u << k;
  }
  const int mine = __popc(keep);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int v = __shfl_up_sync(hm, incl, o, 16);
    if (hl >= o) incl += v;
  }
  const int total = __shfl_sync(hm, incl, 15, 16);
  int pos = incl - mine;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (keep & (1u << k)) out[pos++] = key[k];
  return total;
}

template <int N>
__global__ void __launch_bounds__(256)
    rows_half_kernel(GridDev g, const int32_t* __restrict__ rect, const int32_t* __restrict__ cnt,
                     int64_t rows, int U, const int64_t* __restrict__ toff,
                     const int64_t* __restrict__ tcand, int32_t* __restrict__ temp, int64_t* __restrict__ rowcnt,
                     int64_t* __restrict__ rest, int64_t* __restrict__ nrest) {
  __shared__ HalfStage<N> stage[16];
  const int hl = threadIdx.x & 15;
  const int grp = threadIdx.x >> 4;
  const unsigned hm = 0xffffu << (threadIdx.x & 16);
  HalfStage<N>& st = stage[grp];
  const int64_t ngroups = (int64_t)gridDim.x * 16;
  for (int64_t r = (int64_t)blockIdx.x * 16 + grp; r < rows; r += ngroups) {
    const int64_t t0 = toff[r], T = tcand ? tcand[r] : toff[r + 1] - t0;
    if (T == 0) {
      if (hl == 0) rowcnt[r] = 0;
      continue;
    }
    bool fits = U <= kHalfU && T <= kWarpCap;
    int32_t bl[N], bh[N];
#pragma unroll
    for (int d = 0; d < N; ++d) { bl[d] = INT_MAX; bh[d] = INT_MIN; }
    if (fits) {  // stage the rectangles (lane u = input u)
      int32_t c = 0, rr = 0;
      if (hl < U) {
        c = cnt[r * U + hl];
        const int32_t* R = rect + (r * U + hl) * 2 * N;
        rr = c > 0 ? 1 : 0;
#pragma unroll
        for (int d = 0; d < N; ++d) {
          const int32_t lo = R[d], hi = R[N + d];
          st.lo[hl][d] = lo;
          st.ext[hl][d] = hi - lo + 1;
          if (d < N - 1) rr *= hi - lo + 1;
          if (c > 0) { bl[d] = lo; bh[d] = hi; }
        }
      }
      int32_t incl = c, rincl = rr;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const int32_t v = __shfl_up_sync(hm, incl, o, 16);
        const int32_t rv = __shfl_up_sync(hm, rincl, o, 16);
        if (hl >= o) { incl += v; rincl += rv; }
      }
      if (hl < U) { st.pre[hl] = incl - c; st.rpre[hl] = rincl - rr; }
      if (hl == 15) { st.pre[U] = incl; st.rpre[U] = rincl; }
    }
    int64_t vol = 1;
    int32_t bext[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        bl[d] = min(bl[d], __shfl_xor_sync(hm, bl[d], o, 16));
        bh[d] = max(bh[d], __shfl_xor_sync(hm, bh[d], o, 16));
      }
      bext[d] = bh[d] - bl[d] + 1;
      vol *= bext[d];
    }
    fits = fits && vol <= kHalfBits;
    int32_t Us = 0;
    if (fits) {
      uint32_t* bm = st.bm;
#pragma unroll
      for (int i = hl; i < kHalfWords; i += 16) bm[i] = 0u;
      __syncwarp(hm);
      const int32_t RR = st.rpre[U];
      for (int32_t q = hl; q < RR; q += 16) {
        int a = 0, b = U;  // rpre[a] <= q < rpre[b]
        while (b - a > 1) {
          const int mid = (a + b) >> 1;
          if (st.rpre[mid] <= q) a = mid; else b = mid;
        }
        int32_t off = q - st.rpre[a];
        int32_t base = st.lo[a][N - 1] - bl[N - 1];
        int32_t bstride = bext[N - 1];
#pragma unroll
        for (int d = N - 2; d > 0; --d) {
          int32_t rr;
          const int32_t qq = div_small(off, st.ext[a][d], rr);
          base += (st.lo[a][d] + rr - bl[d]) * bstride;
          bstride *= bext[d];
          off = qq;
        }
        if (N > 1) base += (st.lo[a][0] + off - bl[0]) * bstride;
        const int32_t b0 = base, b1 = base + st.ext[a][N - 1];
        for (int32_t wi = b0 >> 5; wi <= (b1 - 1) >> 5; ++wi) {
          const int32_t lo = max(b0 - wi * 32, 0), hi = min(b1 - wi * 32, 32);
          const uint32_t m = (hi - lo == 32) ? 0xffffffffu : (((1u << (hi - lo)) - 1u) << lo);
          atomicOr(bm + wi, m);
        }
      }
      __syncwarp(hm);
      const int nwords = (int)((vol + 31) >> 5);
      int c = 0;
      for (int i = hl; i < nwords; i += 16) c += __popc(bm[i]);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) c += __shfl_xor_sync(hm, c, o, 16);
      Us = c;
      fits = Us <= kHalfKeys;
    }
    if (!fits) {
      if (hl == 0) rest[atomicAdd((unsigned long long*)nrest, 1ull)] = r;
      __syncwarp(hm);
      continue;
    }
    // extraction, 16 bitmap bits per step (one per lane), in box row-major order
    int32_t sbase = 0, str[N];
    float rinv[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
      str[d] = (int32_t)g.stride[d];
      sbase += bl[d] * str[d];
      rinv[d] = 1.0f / (float)bext[d];
    }
    const int nsteps = (int)((vol + 15) >> 4);
    int base = 0;
    for (int hw = 0; hw < nsteps; ++hw) {
      const uint32_t bits = (st.bm[hw >> 1] >> ((hw & 1) * 16)) & 0xffffu;
      if ((bits >> hl) & 1u) {
        int32_t bi = hw * 16 + hl;  // < 2^10: the float quotient is off by at most one
        int32_t s = sbase;
#pragma unroll
        for (int d = N - 1; d > 0; --d) {
          int32_t qq = (int32_t)((float)bi * rinv[d]);
          int32_t rr = bi - qq * bext[d];
          if (rr < 0) { --qq; rr += bext[d]; } else if (rr >= bext[d]) { ++qq; rr -= bext[d]; }
          s += rr * str[d];
          bi = qq;
        }
        s += bi * str[0];
        const int32_t cell = __ldg(g.slot + s);
        st.keys[base + __popc(bits & ((1u << hl) - 1u))] = cell < 0 ? INT_MAX : cell;
      }
      base += __popc(bits);
    }
    __syncwarp(hm);
    int32_t key[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int e = hl * 2 + k;
      key[k] = e < Us ? st.keys[e] : INT_MAX;
    }
    const int32_t total = half_sort_unique_write<2>(key, hl, hm, temp + t0);
    if (hl == 0) rowcnt[r] = total;
    __syncwarp(hm);
  }
}

// Rows with more than kWarpCap candidates: one block per row marks a bitmap
// over all V target cells, then emits set bits in ascending order.
template <int N>
__global__ void __launch_bounds__(256)
    big_rows_kernel(GridDev g, const int32_t* __restrict__ rect, const int32_t* __restrict__ cnt,
                    int U, const int64_t* __restrict__ toff, int32_t* __restrict__ temp,
                    int64_t* __restrict__ rowcnt, const int64_t* __restrict__ big,
                    const int64_t* __restrict__ nbig, uint32_t* __restrict__ bitmaps,
                    int64_t words) {
  __shared__ int32_t scan[256];
  __shared__ int64_t base_s;
  uint32_t* bm = bitmaps + (int64_t)blockIdx.x * words;
  const int64_t nb = *nbig;
  for (int64_t bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const int64_t r = big[bi];
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0u;
    __syncthreads();
    for (int u = 0; u < U; ++u) {
      const int64_t c = cnt[r * U + u];
      if (c == 0) continue;
      const int32_t* R = rect + (r * U + u) * 2 * N;
      int64_t ext[N];
#pragma unroll
      for (int d = 0; d < N; ++d) ext[d] = (int64_t)R[N + d] - R[d] + 1;
      for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
        int64_t off = e, s = 0;
#pragma unroll
        for (int d = N - 1; d >= 0; --d) {
          const int64_t q = off / ext[d];
          s += (R[d] + (off - q * ext[d])) * g.stride[d];
          off = q;
        }
        const int32_t cell = g.slot[s];
        if (cell >= 0) atomicOr(bm + (cell >> 5), 1u << (cell & 31));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    int32_t* out = temp + toff[r];
    for (int64_t w0 = 0; w0 < words; w0 += blockDim.x) {
      const int64_t wi = w0 + threadIdx.x;
      const uint32_t word = (wi < words) ? bm[wi] : 0u;
      const int c = __popc(word);
      scan[threadIdx.x] = c;
      __syncthreads();
      for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // Hillis-Steele inclusive scan
        const int v = (threadIdx.x >= (unsigned)o) ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
      }
      int64_t pos = base_s + scan[threadIdx.x] - c;
      uint32_t x = word;
      while (x) {
        const int b = __ffs(x) - 1;
        out[pos++] = (int32_t)(wi * 32 + b);
        x &= x - 1;
      }
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) base_s += scan[threadIdx.x];
      __syncthreads();
    }
    if (threadIdx.x == 0) rowcnt[r] = base_s;
    __syncthreads();
  }
}

// Deduplicated rows (at their candidate offsets in temp) to the final CSR.
// G lanes per row: short rows (3-D / 4-D) take 8 lanes, so a warp has four
// rows' offset loads in flight instead of one.
template <int G>
__global__ void compact_kernel(const int64_t* __restrict__ toff, const int32_t* __restrict__ temp,
                               const int64_t* __restrict__ indptr, int64_t rows,
                               int32_t* __restrict__ indices) {
  const int lane = threadIdx.x & (G - 1);
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; r < rows;
       r += ngroups) {
    const int64_t a = indptr[r], n = indptr[r + 1] - a;
    const int32_t* src = temp + toff[r];
    for (int64_t k = lane; k < n; k += G) indices[a + k] = src[k];
  }
}

// ---- rows of unchanged cells from the previous graph ---------------------
// In an adaptive step c' = subdivide(retain(c, keep), sel) a cell carried
// over unchanged keeps its padded boxes, so its row in c' is the previous
// row mapped forward: a target still there unchanged stays (it met the same
// boxes), a removed one goes, and a split one gives those of its two
// children that meet one of the row's boxes -- no cell of c' can meet a box
// whose cell of c (itself or its parent) did not.  The test is the
// reference's closed-box one (cg/geometry.py:497-501), which is what the
// slot rectangles compute on a dense index.  Order: fwd preserves the
// canonical order and children are consecutive.
static constexpr int kIncrMaxU = 32;  // inputs of rows mapped forward

struct IncrRows {
  const int64_t* origin;       // [V] index in c, or -1
  int64_t memo_begin, memo_rows;
  const double* boxes;         // [memo_rows][U][2n] padded boxes of c's rows
  const int64_t* prev_indptr;  // [memo_rows + 1] c's rows (relative)
  const int32_t* prev_indices; //   targets: global cells of c
  const int64_t* fwd;          // [V of c] -> c' (see forward_kernel)
  const double* lo;            // c' SoA [n][V]
  const double* hi;
  int64_t row0;                // first row of this build
};

__global__ void incr_total_kernel(IncrRows a, int64_t rows, int64_t* __restrict__ tot) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t o = a.origin[a.row0 + r] - a.memo_begin;
  if (o >= 0 && o < a.memo_rows) tot[r] += 2 * (a.prev_indptr[o + 1] - a.prev_indptr[o]);
}

// One warp per row, 32 targets at a time (a lane per target); the next
// chunk's forward-map loads are issued before this one is processed.  A
// lane holding a split target tests both children against the row's U
// boxes (staged in shared memory) in one pass.  Latency bound: a chain of
// dependent loads per target (r02bb ncu: long-scoreboard stalls).
static constexpr int kIncrWarps = 8;

template <int N>
__global__ void __launch_bounds__(kIncrWarps * 32)
    incr_rows_kernel(IncrRows a, int64_t rows, int64_t V, int U, const int64_t* __restrict__ toff,
                     int32_t* __restrict__ temp, int64_t* __restrict__ rowcnt) {
  __shared__ double sbox[kIncrWarps][kIncrMaxU * 2 * N];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* bx = sbox[w];
  const int64_t nwarps = (int64_t)gridDim.x * kIncrWarps;
  for (int64_t r = (int64_t)blockIdx.x * kIncrWarps + w; r < rows; r += nwarps) {
    const int64_t o = a.origin[a.row0 + r] - a.memo_begin;
    if (o < 0 || o >= a.memo_rows) continue;  // a new cell: K2 built its row
    __syncwarp();
    for (int i = lane; i < U * 2 * N; i += 32) bx[i] = a.boxes[o * U * 2 * N + i];
    __syncwarp();
    const int64_t p0 = a.prev_indptr[o], p1 = a.prev_indptr[o + 1];
    int32_t* dst = temp + toff[r];
    int64_t out = 0;
    auto fetch = [&](int64_t i) { return i < p1 ? __ldg(a.fwd + __ldg(a.prev_indices + i)) : -1; };
    int64_t fn = fetch(p0 + lane);
    for (int64_t i0 = p0; i0 < p1; i0 += 32) {
      const int64_t f = fn;
      fn = fetch(i0 + 32 + lane);
      int take = f >= 0 ? 1 : 0;
      const int64_t c0 = f <= -2 ? -2 - f : f;
      if (f <= -2) {
        double lo0[N], hi0[N], lo1[N], hi1[N];
#pragma unroll
        for (int d = 0; d < N; ++d) {
          lo0[d] = __ldg(a.lo + d * V + c0);
          hi0[d] = __ldg(a.hi + d * V + c0);
          lo1[d] = __ldg(a.lo + d * V + c0 + 1);
          hi1[d] = __ldg(a.hi + d * V + c0 + 1);
        }
        for (int u = 0; u < U && take != 3; ++u) {
          const double* b = bx + u * 2 * N;
          bool m0 = true, m1 = true;
#pragma unroll
          for (int d = 0; d < N; ++d) {
            const double bl = b[d], bh = b[N + d];
            m0 = m0 && bl <= hi0[d] && lo0[d] <= bh;
            m1 = m1 && bl <= hi1[d] && lo1[d] <= bh;
          }
          take |= (m0 ? 1 : 0) | (m1 ? 2 : 0);
        }
      }
      const int k = __popc(take);
      int incl = k;  // warp inclusive scan of the counts
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      int64_t pos = out + incl - k;
      if (take & 1) dst[pos++] = (int32_t)c0;
      if (take & 2) dst[pos] = (int32_t)(c0 + 1);
      out += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) rowcnt[r] = out;
  }
}

template <int N>
static void launch_rows(gis_ctx* ctx, const GridDev& g, const int32_t* rect, const int32_t* cnt,
                        int64_t rows, int U, const int64_t* toff, const int64_t* tcand,
                        int32_t* temp, int64_t* rowcnt, int64_t* big, int64_t* nbig,
                        int64_t total) {
  // wide-row lists, each [count][rows entries], in one scratch slot
  int64_t* wl = (int64_t*)scratch(ctx, SC_WIDE, (3 * rows + 6) * 8);
  int64_t* wl2 = wl + rows + 2;
  int64_t* wl0 = wl2 + rows + 2;
  GIS_CUDA(cudaMemsetAsync(wl, 0, 8, ctx->stream));
  GIS_CUDA(cudaMemsetAsync(wl2, 0, 8, ctx->stream));
  int64_t blocks = ceil_div(rows, kWarpsPerBlock);
  blocks = std::min<int64_t>(blocks, (int64_t)ctx->num_sms * 64);
  if (blocks > 0) {
    // pass 0 (3-D / 4-D, few inputs, short rows on average): two rows per
    // warp; the rows it leaves go to list 0 for pass 1
    // (config 4: ~14 targets per row, 27.8 vs 45.2 ms over three passes;
    // config 5's rows, ~90 targets, stay on rows_kernel)
    const bool half = N >= 3 && U <= kHalfU && total <= 128 * rows;
    if (half) {
      GIS_CUDA(cudaMemsetAsync(wl0, 0, 8, ctx->stream));
      rows_half_kernel<N><<<(unsigned)std::min<int64_t>(ceil_div(rows, 16),
                                                        (int64_t)ctx->num_sms * 64),
                            256, 0, ctx->stream>>>(g, rect, cnt, rows, U, toff, tcand, temp,
                                                   rowcnt, wl0 + 1, wl0);
      count_launch(ctx);
    }
    // pass 1: sorts of <= 256 keys; wider rows to list 1
    rows_kernel<N, 8><<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, ctx->stream>>>(
        g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, wl + 1, wl,
        half ? wl0 + 1 : nullptr, half ? wl0 : nullptr);
    count_launch(ctx);
    // pass 2 over list 1 (<= 512 keys; wider rows to list 2), pass 3 over
    // list 2; grids sized for the worst case exit at once on empty lists
    const int64_t wb = std::min<int64_t>(blocks, (int64_t)ctx->num_sms * GIS_K2_WIDE_BLOCKS);
    rows_kernel<N, 16><<<(unsigned)wb, 32 * kWarpsPerBlock, 0, ctx->stream>>>(
        g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, wl2 + 1, wl2, wl + 1, wl);
    count_launch(ctx);
    rows_kernel<N, 32><<<(unsigned)std::min<int64_t>(wb, ctx->num_sms * 2),
                         32 * kWarpsPerBlock, 0, ctx->stream>>>(
        g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, nullptr, nullptr, wl2 + 1,
        wl2);
    count_launch(ctx);
  }
  const int64_t words = std::max<int64_t>(ceil_div(g.V, 32), 1);
  const int bb = ctx->num_sms;
  uint32_t* bitmaps = (uint32_t*)scratch(ctx, SC_BITMAP, (size_t)bb * words * 4);
  big_rows_kernel<N><<<bb, 256, 0, ctx->stream>>>(g, rect, cnt, U, toff, temp, rowcnt, big, nbig,
                                                  bitmaps, words);
  count_launch(ctx);
}

void csr_from_rects(gis_ctx* ctx, const GridDev& g, const int32_t* rect, const int32_t* cnt,
                    int64_t rows, int U, int64_t* indptr, int64_t* n_edges,
                    const IncrRows* incr) {
  GIS_REQUIRE(U >= 1, GIS_E_INVALID, "need at least one input");
  if (U > kMaxU) {  // rectangles do not fit the warp's shared staging: K2-general
    GIS_REQUIRE(!incr, GIS_E_INVALID, "incremental rows need U <= 32");
    csr_from_candidates(ctx, g, nullptr, rect, cnt, rows, U, indptr, n_edges);
    return;
  }
  GIS_REQUIRE(g.V < INT_MAX, GIS_E_CAPACITY, "covering too large for int32 targets");
  ctx->pending = PendingCsr{};
  int64_t* toff = (int64_t*)scratch(ctx, SC_TOFF, (rows + 1) * 8);
  int64_t total = 0;
  int64_t* tcand = nullptr;
  auto totals = [&](int64_t* tc) {
    PhaseScope ps_aux(ctx, PH_CSR_AUX);
    int64_t* tot = (int64_t*)scratch(ctx, SC_ROWCNT, (rows + 1) * 8);
    const unsigned nb = (unsigned)ceil_div(rows + 1, 256);
    switch (g.n) {
      case 1: row_total_kernel<1><<<nb, 256, 0, ctx->stream>>>(cnt, rect, rows, U, tot, tc); break;
      case 2: row_total_kernel<2><<<nb, 256, 0, ctx->stream>>>(cnt, rect, rows, U, tot, tc); break;
      case 3: row_total_kernel<3><<<nb, 256, 0, ctx->stream>>>(cnt, rect, rows, U, tot, tc); break;
      case 4: row_total_kernel<4><<<nb, 256, 0, ctx->stream>>>(cnt, rect, rows, U, tot, tc); break;
      default: throw Error{GIS_E_INVALID, "dimension out of range"};
    }
    count_launch(ctx);
    if (incr) {  // room for the forward-mapped rows of unchanged cells
      incr_total_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, ctx->stream>>>(*incr, rows, tot);
      count_launch(ctx);
    }
    exclusive_scan_i64(ctx, tot, toff, rows + 1);
    read_back(ctx, &total, toff + rows, 8);
  };
  if (incr) {
    // the rows K2 enumerates see their own candidate counts (tcand: 0 for
    // the unchanged cells' rows, whose room in temp is the forward map's)
    tcand = (int64_t*)scratch(ctx, SC_TCAND, (rows + 1) * 8);
    totals(tcand);
  } else {
    totals(nullptr);
    // A candidate buffer past kRoomBytes (config 5: 19 GB): size it by
    // min(T, bounding-box slots) per row instead (one more pass over the
    // rectangles, ~1 ms there), T kept in tcand.  Below that the extra pass
    // would cost more than the memory it saves.
    if (g.n >= 3 && total * 4 > kRoomBytes) {
      tcand = (int64_t*)scratch(ctx, SC_TCAND, (rows + 1) * 8);
      totals(tcand);
    }
  }
  int32_t* temp = (int32_t*)scratch(ctx, SC_TEMP, std::max<int64_t>(total, 1) * 4);
  int64_t* rowcnt = (int64_t*)scratch(ctx, SC_ROWCNT, (rows + 1) * 8);
  int64_t* big = (int64_t*)scratch(ctx, SC_BIG, (rows + 1) * 8);
  int64_t* nbig = (int64_t*)scratch(ctx, SC_MISC3, 8);
  GIS_CUDA(cudaMemsetAsync(nbig, 0, 8, ctx->stream));
  GIS_CUDA(cudaMemsetAsync(rowcnt + rows, 0, 8, ctx->stream));
  if (total > 0) {
    PhaseScope ps(ctx, PH_ROWS);
    switch (g.n) {
      case 1: launch_rows<1>(ctx, g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, total); break;
      case 2: launch_rows<2>(ctx, g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, total); break;
      case 3: launch_rows<3>(ctx, g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, total); break;
      case 4: launch_rows<4>(ctx, g, rect, cnt, rows, U, toff, tcand, temp, rowcnt, big, nbig, total); break;
      default: throw Error{GIS_E_INVALID, "dimension out of range"};
    }
  } else if (rows > 0) {
    GIS_CUDA(cudaMemsetAsync(rowcnt, 0, rows * 8, ctx->stream));
  }
  if (incr && rows > 0) {  // after K2: these rows' counts are overwritten
    PhaseScope ps(ctx, PH_ROWS);
    const unsigned blocks =
        (unsigned)std::min<int64_t>(ceil_div(rows, kIncrWarps), (int64_t)ctx->num_sms * 16);
    const int64_t Vn = g.V;
    auto go = [&](auto kernel) {
      kernel<<<blocks, kIncrWarps * 32, 0, ctx->stream>>>(*incr, rows, Vn, U, toff, temp, rowcnt);
    };
    switch (g.n) {
      case 1: go(incr_rows_kernel<1>); break;
      case 2: go(incr_rows_kernel<2>); break;
      case 3: go(incr_rows_kernel<3>); break;
      default: go(incr_rows_kernel<4>); break;
    }
    count_launch(ctx);
  }
  {
    PhaseScope ps_aux(ctx, PH_CSR_AUX);
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

// ---- CSR from edge pairs (_csr_from_pairs, cg/graph.py:181-193) -----------
__global__ void pair_keys_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                                 int64_t n, int64_t V, uint64_t* __restrict__ keys,
                                 int* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = src[i], d = dst[i];
  if (s < 0 || s >= V || d < 0 || d >= V) {
    *bad = 1;
    keys[i] = 0;
    return;
  }
  keys[i] = (uint64_t)s * (uint64_t)V + (uint64_t)d;
}

__global__ void unique_pairs_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t V,
                                    uint8_t* __restrict__ first,
                                    unsigned long long* __restrict__ rowcnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool f = (i == 0) || keys[i] != keys[i - 1];
  first[i] = f;
  if (f) atomicAdd(rowcnt + keys[i] / (uint64_t)V, 1ull);
}

__global__ void scatter_pairs_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t V,
                                     const uint8_t* __restrict__ first,
                                     const int64_t* __restrict__ pos,
                                     int32_t* __restrict__ indices) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && first[i]) indices[pos[i]] = (int32_t)(keys[i] % (uint64_t)V);
}

__global__ void csr_sources_kernel(const int64_t* __restrict__ indptr, int64_t V,
                                   int64_t* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < V; r += nw)
    for (int64_t i = indptr[r] + lane; i < indptr[r + 1]; i += 32) src[i] = r;
}

void enclose(gis_ctx* ctx, const gis_model* model, const double* lo, const double* hi,
             int64_t V, int64_t c0, int64_t ncells, const double* u, int U,
             const double* frac, int S, double bloat, int mode, double* enc_lo,
             double* enc_hi, uint8_t* valid, int32_t* rect, int32_t* cnt,
             const GridDev* grid, const EncList* list = nullptr);

}  // namespace gis

using namespace gis;

GIS_API int gis_csr_finish(gis_ctx* ctx, int32_t* indices) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(ctx->pending.active, GIS_E_STATE, "gis_csr_finish without a pending CSR");
    const PendingCsr p = ctx->pending;
    ctx->pending.active = false;
    if (p.rows > 0 && p.edges > 0) {
      PhaseScope ps(ctx, PH_CSR_AUX);
      const int64_t* toff = (const int64_t*)ctx->buf[SC_TOFF];
      const int32_t* temp = (const int32_t*)ctx->buf[SC_TEMP];
      if (p.edges < 16 * p.rows) {  // short rows: 8 lanes each
        const int64_t blocks = std::min<int64_t>(ceil_div(p.rows * 8, 256), ctx->num_sms * 32);
        compact_kernel<8><<<(unsigned)blocks, 256, 0, ctx->stream>>>(toff, temp, p.indptr,
                                                                     p.rows, indices);
      } else {
        const int64_t blocks = std::min<int64_t>(ceil_div(p.rows * 32, 256), ctx->num_sms * 32);
        compact_kernel<32><<<(unsigned)blocks, 256, 0, ctx->stream>>>(toff, temp, p.indptr,
                                                                      p.rows, indices);
      }
      count_launch(ctx);
    }
  });
}

namespace gis {

// cells of rows [row0, row0 + rows) without a reusable box
__global__ void memo_new_kernel(const int64_t* __restrict__ origin, int64_t row0, int64_t rows,
                                int64_t memo_begin, int64_t memo_rows, uint8_t* __restrict__ isnew) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t o = origin[row0 + r] - memo_begin;
  isnew[r] = (o >= 0 && o < memo_rows) ? 0 : 1;
}

__global__ void memo_list_kernel(const uint8_t* __restrict__ isnew,
                                 const int64_t* __restrict__ pos, int64_t row0, int64_t rows,
                                 int64_t* __restrict__ cells, int32_t* __restrict__ inv) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (isnew[r]) cells[pos[r]] = row0 + r;
  inv[r] = isnew[r] ? (int32_t)pos[r] : -1;
}

struct MemoIn {
  const int64_t* origin;
  const double* memo_in;
  int64_t memo_begin, memo_rows;
  double* memo_out;
  const int64_t* prev_indptr;   // previous graph's rows [memo_begin, +memo_rows), or NULL
  const int32_t* prev_indices;
  const int64_t* fwd;
};

static void build_graph(gis_ctx* ctx, const gis_index* ix, const gis_model* model,
                        const double* lo, const double* hi, int64_t V, int64_t row_begin,
                        int64_t row_end, const double* u, int32_t U, const double* frac,
                        int32_t S, double bloat, const MemoIn* memo, int64_t* indptr,
                        int64_t* n_edges);

}  // namespace gis

GIS_API int gis_build_graph_begin(gis_ctx* ctx, const gis_index* ix, const gis_model* model,
                                  const double* lo, const double* hi, int64_t V,
                                  int64_t row_begin, int64_t row_end, const double* u,
                                  int32_t U, const double* frac, int32_t S, double bloat,
                                  int64_t* indptr, int64_t* n_edges) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    gis::build_graph(ctx, ix, model, lo, hi, V, row_begin, row_end, u, U, frac, S, bloat,
                     nullptr, indptr, n_edges);
  });
}

GIS_API int gis_build_graph_memo_begin(gis_ctx* ctx, const gis_index* ix,
                                       const gis_model* model, const double* lo,
                                       const double* hi, int64_t V, int64_t row_begin,
                                       int64_t row_end, const double* u, int32_t U,
                                       const double* frac, int32_t S, double bloat,
                                       const int64_t* origin, const double* memo_in,
                                       int64_t memo_begin, int64_t memo_rows,
                                       const int64_t* prev_indptr, const int32_t* prev_indices,
                                       const int64_t* fwd, double* memo_out, int64_t* indptr,
                                       int64_t* n_edges) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(!origin || (memo_in && memo_begin >= 0 && memo_rows >= 0), GIS_E_INVALID,
                "origin given without the previous boxes");
    GIS_REQUIRE(ix == nullptr || !ix->sparse || (!origin && !memo_out), GIS_E_INVALID,
                "box reuse needs a dense index");
    GIS_REQUIRE(!prev_indptr || (origin && prev_indices && fwd), GIS_E_INVALID,
                "the previous rows need origin, indices and fwd");
    const gis::MemoIn m{origin, memo_in, memo_begin, memo_rows, memo_out,
                        prev_indptr, prev_indices, fwd};
    gis::build_graph(ctx, ix, model, lo, hi, V, row_begin, row_end, u, U, frac, S, bloat,
                     (origin || memo_out) ? &m : nullptr, indptr, n_edges);
  });
}

namespace gis {

static void build_graph(gis_ctx* ctx, const gis_index* ix, const gis_model* model,
                        const double* lo, const double* hi, int64_t V, int64_t row_begin,
                        int64_t row_end, const double* u, int32_t U, const double* frac,
                        int32_t S, double bloat, const MemoIn* memo, int64_t* indptr,
                        int64_t* n_edges) {
  {
    GIS_REQUIRE(ix != nullptr, GIS_E_INVALID, "index is NULL");
    GIS_REQUIRE(model != nullptr && model->n == ix->n, GIS_E_INVALID,
                "model dimension does not match the index");
    GIS_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= V, GIS_E_INVALID,
                "row range out of bounds");
    const int64_t rows = row_end - row_begin;
    const int n = ix->n;
    GridDev g = ix->dev();
    if (ix->sparse) {  // enclosure boxes, then candidates from the sparse index
      const int64_t P = std::max<int64_t>(rows * U, 1);
      double* box = (double*)scratch(ctx, SC_RECT, P * 2 * n * 8);
      uint8_t* valid = (uint8_t*)scratch(ctx, SC_CNT, P);
      if (rows > 0) {
        PhaseScope ps(ctx, PH_ENCLOSE);
        gis::enclose(ctx, model, lo, hi, V, row_begin, rows, u, U, frac, S, bloat, 2, box,
                     box + P * n, valid, nullptr, nullptr, &g);
      }
      PairBoxes pb{box, box + P * n, valid, n, 1};
      csr_from_candidates(ctx, g, &pb, nullptr, nullptr, rows, U, indptr, n_edges);
      return;
    }
    int32_t* rect = (int32_t*)scratch(ctx, SC_RECT, std::max<int64_t>(rows * U, 1) * 2 * n * 4);
    int32_t* cnt = (int32_t*)scratch(ctx, SC_CNT, std::max<int64_t>(rows * U, 1) * 4);
    // unchanged cells' rows forward-mapped from the previous graph (K2 skips them)
    const bool incr_ok = memo && memo->origin && memo->prev_indptr && U <= kIncrMaxU;
    if (rows > 0) {
      PhaseScope ps(ctx, PH_ENCLOSE);
      EncList list;
      if (memo) {
        list.memo_out = memo->memo_out;
        if (memo->origin) {  // integrate only the cells without a kept box
          list.origin = memo->origin;
          list.memo_in = memo->memo_in;
          list.memo_begin = memo->memo_begin;
          list.memo_rows = memo->memo_rows;
          uint8_t* isnew = (uint8_t*)scratch(ctx, SC_MISC3, rows);
          int64_t* pos = (int64_t*)scratch(ctx, SC_MISC2, (rows + 1) * 8);
          int64_t* cells = (int64_t*)scratch(ctx, SC_TEMP, std::max<int64_t>(rows, 1) * 8);
          int32_t* inv = (int32_t*)scratch(ctx, SC_ROWCNT, std::max<int64_t>(rows, 1) * 4);
          const unsigned nb = (unsigned)ceil_div(rows, 256);
          memo_new_kernel<<<nb, 256, 0, ctx->stream>>>(memo->origin, row_begin, rows,
                                                       memo->memo_begin, memo->memo_rows, isnew);
          count_launch(ctx);
          exclusive_scan_u8_to_i64(ctx, isnew, pos, rows);
          memo_list_kernel<<<nb, 256, 0, ctx->stream>>>(isnew, pos, row_begin, rows, cells, inv);
          count_launch(ctx);
          read_back(ctx, &list.nlist, pos + rows, sizeof(int64_t));
          list.cells = cells;
          list.inv = inv;
        }
      }
      list.incr = incr_ok;
      gis::enclose(ctx, model, lo, hi, V, row_begin, rows, u, U, frac, S, bloat, 1, nullptr,
                   nullptr, nullptr, rect, cnt, &g, memo ? &list : nullptr);
    }
    if (incr_ok) {
      const IncrRows ir{memo->origin,      memo->memo_begin,   memo->memo_rows, memo->memo_in,
                        memo->prev_indptr, memo->prev_indices, memo->fwd,       lo,
                        hi,                row_begin};
      csr_from_rects(ctx, g, rect, cnt, rows, U, indptr, n_edges, &ir);
    } else {
      csr_from_rects(ctx, g, rect, cnt, rows, U, indptr, n_edges);
    }
  }
}

}  // namespace gis

GIS_API int gis_csr_sources(gis_ctx* ctx, const int64_t* indptr, int64_t V, int64_t* src) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0, GIS_E_INVALID, "V out of range");
    if (V == 0) return;
    const int64_t blocks = std::min<int64_t>(ceil_div(V * 32, 256), ctx->num_sms * 32);
    csr_sources_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(indptr, V, src);
    count_launch(ctx);
  });
}

GIS_API int gis_csr_from_pairs(gis_ctx* ctx, const int64_t* src, const int64_t* dst, int64_t n,
                               int64_t V, int64_t* indptr, int32_t* indices, int64_t* n_edges) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX && n >= 0, GIS_E_INVALID, "sizes out of range");
    *n_edges = 0;
    GIS_CUDA(cudaMemsetAsync(indptr, 0, (V + 1) * 8, ctx->stream));
    if (n == 0 || V == 0) {
      GIS_REQUIRE(n == 0, GIS_E_INVALID, "edge endpoint out of range");
      return;
    }
    const unsigned nb = (unsigned)ceil_div(n, 256);
    void* buf = cached_alloc(ctx, (size_t)n * 8 * 2 + (size_t)n + 64);
    uint64_t* keys = (uint64_t*)buf;
    uint64_t* sorted = keys + n;
    uint8_t* first = (uint8_t*)(sorted + n);
    int* bad = (int*)(((uintptr_t)(first + n) + 15) & ~(uintptr_t)15);
    GIS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    pair_keys_kernel<<<nb, 256, 0, ctx->stream>>>(src, dst, n, V, keys, bad);
    count_launch(ctx);
    int hbad = 0;
    read_back(ctx, &hbad, bad, sizeof(int));
    if (hbad) {
      cached_free(buf, (size_t)n * 8 * 2 + (size_t)n + 64, ctx->device, ctx->stream);
      throw Error{GIS_E_INVALID, "edge endpoint out of range"};
    }
    int end_bit = 1;
    while (end_bit < 64 && ((uint64_t)1 << end_bit) < (uint64_t)V * (uint64_t)V) ++end_bit;
    size_t tb = 0;
    GIS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, n, 0, end_bit,
                                            ctx->stream));
    void* tmp = scratch(ctx, SC_CUB, tb);
    GIS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, n, 0, end_bit, ctx->stream));
    count_launch(ctx);
    int64_t* rowcnt = (int64_t*)scratch(ctx, SC_ROWCNT, (V + 1) * 8);
    GIS_CUDA(cudaMemsetAsync(rowcnt, 0, (V + 1) * 8, ctx->stream));
    unique_pairs_kernel<<<nb, 256, 0, ctx->stream>>>(sorted, n, V, first,
                                                     (unsigned long long*)rowcnt);
    count_launch(ctx);
    // own buffer for the positions: SC_TOFF / SC_TEMP may hold a pending CSR
    int64_t* pos = (int64_t*)cached_alloc(ctx, (size_t)(n + 1) * 8);
    exclusive_scan_u8_to_i64(ctx, first, pos, n);
    scatter_pairs_kernel<<<nb, 256, 0, ctx->stream>>>(sorted, n, V, first, pos, indices);
    count_launch(ctx);
    exclusive_scan_i64(ctx, rowcnt, indptr, V + 1);
    read_back(ctx, n_edges, indptr + V, 8);
    cached_free(pos, (size_t)(n + 1) * 8, ctx->device, ctx->stream);
    cached_free(buf, (size_t)n * 8 * 2 + (size_t)n + 64, ctx->device, ctx->stream);
  });
}
