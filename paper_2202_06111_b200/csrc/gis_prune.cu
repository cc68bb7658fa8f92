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

#include <type_traits>

#include "gis_internal.cuh"

namespace cg = cooperative_groups;

namespace gis {

__device__ __forceinline__ bool alive_bit(const uint32_t* alive, int32_t t) {
  return (__ldcg(alive + (t >> 5)) >> (t & 31)) & 1u;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef GIS_PEEL_TRACE  // diagnostics build (tools/peel_trace.py): per sweep, the
// time block b finished its words ([r][1 + b]) and the grid barrier's exit
// ([r][0]); the kernel's start in g_peel_t0
__device__ unsigned long long g_peel_trace[64][1024];
__device__ unsigned long long g_peel_start[64][1024];  // block b's sweep start
__device__ unsigned long long g_peel_t0;
}  // namespace gis
GIS_API int gis_debug_peel_trace(unsigned long long* out, unsigned long long* t0) {
  cudaMemcpyFromSymbol(out, gis::g_peel_trace, sizeof(gis::g_peel_trace));
  cudaMemcpyFromSymbol(out + 64 * 1024, gis::g_peel_start, sizeof(gis::g_peel_start));
  return (int)cudaMemcpyFromSymbol(t0, gis::g_peel_t0, 8);
}
namespace gis {
#endif

static constexpr int64_t kNotStarted = (int64_t)(-2) * ((int64_t)1 << 32);

// One sweep over words [w0, w1) of vertices (warp per bitmap word).
// Rows are addressed through indptr (local rows: vertex v -> row v - vbase).
// Peers whose replicas receive each changed word (fused multi-GPU prune).
struct PushTo {
  uint32_t* const* rep = nullptr;
  int R = 0, me = 0;
};

// Per-vertex scan state.  Wide (int64): (current target << 32) | offset in
// the row.  Compact (int32, gis_prune on graphs whose wide state would not
// stay L2-resident): the current target alone; when it has died, its offset
// is found again by binary search (rows are ascending and unique).  Both: -2
// = not started, -1 = row exhausted (vertex deleted).
template <bool COMPACT>
struct ScanState;

template <>
struct ScanState<false> {
  int64_t* s;
  __device__ __forceinline__ int32_t target(int64_t row) const {
    return (int32_t)(s[row] >> 32);
  }
  // first row position to probe once the current target is known dead
  __device__ __forceinline__ int64_t resume(int64_t row, int32_t t, int64_t a, int64_t,
                                            const int32_t*) const {
    return a + (t == -2 ? 0 : (int64_t)(uint32_t)s[row] + 1);
  }
  __device__ __forceinline__ void store(int64_t row, bool dead, int32_t tgt, int64_t off) {
    s[row] = dead ? ((int64_t)(-1) << 32) : (((int64_t)tgt << 32) | (int64_t)(uint32_t)off);
  }
};

template <>
struct ScanState<true> {
  int32_t* s;
  __device__ __forceinline__ int32_t target(int64_t row) const { return s[row]; }
  __device__ __forceinline__ int64_t resume(int64_t, int32_t t, int64_t a, int64_t e,
                                            const int32_t* __restrict__ idx) const {
    if (t == -2) return a;
    int64_t lo = a, hi = e;  // the dead target's position: first entry >= t
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(idx + mid) < t) lo = mid + 1; else hi = mid;
    }
    return lo + 1;
  }
  __device__ __forceinline__ void store(int64_t row, bool dead, int32_t tgt, int64_t) {
    s[row] = dead ? -1 : tgt;
  }
};

// One sweep over the words a source hands out (warp per bitmap word; each
// word goes to one warp per sweep).  next() returns the warp's next word,
// or -1.  Rows are addressed through indptr (local rows: vertex v -> row
// v - vbase).
template <bool COMPACT, class Next>
__device__ __forceinline__ unsigned long long sweep_loop(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t vbase,
    int64_t vend, uint32_t* alive, ScanState<COMPACT> state, Next next,
    PushTo push = PushTo()) {
  const int lane = threadIdx.x & 31;
  unsigned long long deaths = 0;
  // The word and the lane's scan state of the next word are loaded while
  // the current one is processed (a word has one warp per sweep, so neither
  // changes in between): per word, only the probe of the current target's
  // bit is left on the critical path.
  auto load = [&](int64_t w, uint32_t& word, int32_t& t) {
    const int64_t v = w * 32 + lane;
    word = __ldcg(alive + w);
    t = v < vend ? state.target(v - vbase) : -1;
  };
  uint32_t word_n = 0u;
  int32_t t_n = -1;
  int64_t w = next();
  if (w >= 0) load(w, word_n, t_n);
  while (w >= 0) {
    const uint32_t word = word_n;
    const int32_t t = t_n;
    const int64_t wn = next();
    if (wn >= 0) load(wn, word_n, t_n);
    if (word != 0u) {
      const int64_t v = w * 32 + lane;
      bool dead = false;
      if (v < vend && ((word >> lane) & 1u)) {
        const int64_t row = v - vbase;
        if (t < 0 || !alive_bit(alive, t)) {
          const int64_t a = indptr[row];
          const int64_t e = indptr[row + 1];
          int64_t p = state.resume(row, t, a, e, indices);
          // each lane walks its own dead run, software-pipelined probes.
          // Measured and dropped: a warp-cooperative walk (32 entries per
          // step) of all rows (config 2 prune 0.52 -> 1.03 ms) or of the
          // last <= 4 walkers of a word (no gain), and an L2 bulk prefetch
          // of the rest of the row at the walk's start (slower)
          p = first_live(indices, p, e, alive);
          dead = (p == e);
          state.store(row, dead, dead ? -1 : indices[p], p - a);
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, dead);
      if (m && lane == 0) {
        // the warp owns word w for this sweep: the new value is final for it
        const uint32_t now = atomicAnd(alive + w, ~m) & ~m;
        deaths += __popc(m);
        for (int q = 0; q < push.R; ++q)
          if (q != push.me) __stcg(push.rep[q] + w, now);
      }
    }
    w = wn;
  }
  return deaths;
}

// Four words per warp step (K3 peel_coop_kernel): lane l owns vertices
// 4(l%8) ... 4(l%8)+3 of word l/8 of a 128-vertex group, so a lane keeps
// four target probes in flight and a warp step covers four bitmap words; the
// eight lanes of a word combine their death masks by shuffles.
template <bool COMPACT>
__device__ __forceinline__ void load_targets4(const ScanState<COMPACT>& st, int64_t row,
                                              int64_t nvalid, int32_t (&t)[4]);
template <>
__device__ __forceinline__ void load_targets4(const ScanState<false>& st, int64_t row,
                                              int64_t nvalid, int32_t (&t)[4]) {
  if (nvalid >= 4) {
    const longlong2 a = __ldcg((const longlong2*)(st.s + row));
    const longlong2 b = __ldcg((const longlong2*)(st.s + row) + 1);
    t[0] = (int32_t)(a.x >> 32); t[1] = (int32_t)(a.y >> 32);
    t[2] = (int32_t)(b.x >> 32); t[3] = (int32_t)(b.y >> 32);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = q < nvalid ? (int32_t)(st.s[row + q] >> 32) : -1;
  }
}
template <>
__device__ __forceinline__ void load_targets4(const ScanState<true>& st, int64_t row,
                                              int64_t nvalid, int32_t (&t)[4]) {
  if (nvalid >= 4) {
    const int4 a = __ldcg((const int4*)(st.s + row));
    t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = q < nvalid ? st.s[row + q] : -1;
  }
}

template <bool COMPACT, class Next>
__device__ __forceinline__ unsigned long long sweep_loop4(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t vbase,
    int64_t vend, uint32_t* alive, ScanState<COMPACT> state, Next next) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & 7;
  const int64_t W1 = (vend + 31) >> 5;
  unsigned long long deaths = 0;
  auto load = [&](int64_t g, uint32_t& bits, int32_t (&t)[4]) {
    const int64_t w = g + (lane >> 3);
    const int64_t v0 = w * 32 + 4 * sub;
    bits = w < W1 ? (__ldcg(alive + w) >> (4 * sub)) & 0xFu : 0u;
    const int64_t nvalid = vend - v0;
    if (nvalid < 4) bits &= nvalid <= 0 ? 0u : ((1u << nvalid) - 1u);
    if (bits) load_targets4(state, v0 - vbase, nvalid, t);
  };
  uint32_t bits_n = 0u;
  int32_t t_n[4] = {-1, -1, -1, -1};
  int64_t g = next();
  if (g >= 0) load(g, bits_n, t_n);
  while (g >= 0) {
    const uint32_t bits = bits_n;
    int32_t t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = t_n[q];
    const int64_t gn = next();
    if (gn >= 0) load(gn, bits_n, t_n);
    uint32_t dead = 0u;
    if (bits) {
      uint32_t tw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // four probes in flight
        const bool probe = ((bits >> q) & 1u) && t[q] >= 0;
        tw[q] = probe ? (__ldcg(alive + (t[q] >> 5)) >> (t[q] & 31)) & 1u : 0u;
      }
      const int64_t v0 = (g + (lane >> 3)) * 32 + 4 * sub;
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        if (!((bits >> q) & 1u) || tw[q]) continue;
        const int64_t row = v0 + q - vbase;
        const int64_t a = indptr[row];
        const int64_t e = indptr[row + 1];
        int64_t p = state.resume(row, t[q], a, e, indices);
        p = first_live(indices, p, e, alive);
        const bool d = (p == e);
        state.store(row, d, d ? -1 : indices[p], p - a);
        dead |= (uint32_t)d << q;
      }
    }
    if (__any_sync(0xffffffffu, dead != 0u)) {
      uint32_t m = dead << (4 * sub);
      m |= __shfl_xor_sync(0xffffffffu, m, 1);
      m |= __shfl_xor_sync(0xffffffffu, m, 2);
      m |= __shfl_xor_sync(0xffffffffu, m, 4);
      if (sub == 0 && m) {
        atomicAnd(alive + g + (lane >> 3), ~m);
        deaths += __popc(m);
      }
    }
    g = gn;
  }
  return deaths;
}

// Static assignment: words w0, w0 + wstep, ... below w1.
template <bool COMPACT = false>
__device__ __forceinline__ unsigned long long sweep_words(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t vbase,
    int64_t vend, uint32_t* alive, ScanState<COMPACT> state, int64_t w0, int64_t w1,
    int64_t wstep, PushTo push = PushTo()) {
  int64_t w = w0 - wstep;
  auto next = [&]() -> int64_t {
    w += wstep;
    return w < w1 ? w : -1;
  };
  return sweep_loop<COMPACT>(indptr, indices, vbase, vend, alive, state, next, push);
}

template <class T>
__global__ void peel_init_kernel(int64_t nrows, T* __restrict__ ptr,
                                 uint32_t* __restrict__ alive, int64_t V, int64_t words) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) ptr[i] = sizeof(T) == 8 ? (T)kNotStarted : (T)-2;
  if (i < words) {
    const int64_t rem = V - i * 32;
    alive[i] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  }
}

// Fixed point over rows [vbase, vend): one cooperative kernel, one sweep
// over the range per grid barrier, until a sweep deletes nothing (remote
// words, if any, are read as they stand).  Block-local repeated sweeps
// between grid barriers were measured and dropped: deletion chains follow
// the dynamics' images across the domain, so the phase count equalled the
// sweep count (config 2: 15) and the local sweeps only added time (DESIGN.md
// section 1).
// 4 resident blocks per SM (<= 64 registers): with the look-ahead loads the
// kernel holds 70 registers unconstrained (3 blocks: config 2 0.47 ms);
// 5-8 blocks spill (0.37-0.47 ms); 4: 0.35 ms (tools/ab_peel.py, r02ag).
// VEC4 (graphs with >= 16 four-word groups per resident warp, e.g. config 4):
// once a sweep deleted fewer than 1/256 of the vertices, later sweeps take
// four words per warp step (sweep_loop4), which cuts the per-word issue cost
// of the long tail of sparse sweeps (config 4 4.28 -> 3.71 ms).  On smaller
// graphs the four-fold fewer work items leave warps idle (config 2 0.35 ->
// 1.2 ms with VEC4 throughout), and in dense sweeps a lane's four serial row
// walks cost more than they save (profiles/r02bj_ab_peel_vec4.jsonl).
template <bool COMPACT, bool VEC4>
__global__ void __launch_bounds__(256, 4)
    peel_coop_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                     int64_t vbase, int64_t vend, uint32_t* alive, void* ptr,
                     unsigned long long* counters, int* rounds_out,
                     unsigned long long* deaths_out) {
  using Elem = typename std::conditional<COMPACT, int32_t, int64_t>::type;
  const ScanState<COMPACT> state{(Elem*)ptr};
  cg::grid_group grid = cg::this_grid();
  // Words: block b takes words W0 + b, W0 + b + B, ... (B blocks; dying
  // regions are contiguous, so interleaving spreads their row walks over
  // all blocks -- contiguous chunks per block were 2x slower), and its
  // warps take them one at a time from a shared counter: a warp held up by
  // long row walks does not hold up words the block's other warps can take.
  const int64_t W0 = vbase >> 5, W1 = (vend + 31) >> 5;
  __shared__ unsigned long long bsum;
  __shared__ int wnext;
  const int lane = threadIdx.x & 31;
  unsigned long long all = 0;
  unsigned long long prev = ~0ull >> 16;  // deaths in the previous sweep
  int round = 0;
#ifdef GIS_PEEL_TRACE
  if (grid.thread_rank() == 0) g_peel_t0 = globaltimer_ns();
#endif
  while (true) {
    if (threadIdx.x == 0) { bsum = 0; wnext = 0; }
    __syncthreads();
#ifdef GIS_PEEL_TRACE
    if (threadIdx.x == 0 && round < 64 && blockIdx.x < 1023)
      g_peel_start[round][1 + blockIdx.x] = globaltimer_ns();
#endif
    unsigned long long d;
    if (VEC4 && 256ull * prev < (unsigned long long)(vend - vbase)) {
      auto next4 = [&]() -> int64_t {
        int i = 0;
        if (lane == 0) i = atomicAdd(&wnext, 1);
        const int64_t g =
            W0 + 4 * (blockIdx.x + (int64_t)__shfl_sync(0xffffffffu, i, 0) * gridDim.x);
        return g < W1 ? g : -1;
      };
      d = sweep_loop4<COMPACT>(indptr, indices, vbase, vend, alive, state, next4);
    } else {
      auto next = [&]() -> int64_t {
        int i = 0;
        if (lane == 0) i = atomicAdd(&wnext, 1);
        const int64_t w = W0 + blockIdx.x + (int64_t)__shfl_sync(0xffffffffu, i, 0) * gridDim.x;
        return w < W1 ? w : -1;
      };
      d = sweep_loop<COMPACT>(indptr, indices, vbase, vend, alive, state, next);
    }
    if (d) atomicAdd(&bsum, d);
    __syncthreads();
    if (threadIdx.x == 0 && bsum) atomicAdd(counters + (round % 3), bsum);
#ifdef GIS_PEEL_TRACE
    if (threadIdx.x == 0 && round < 64 && blockIdx.x < 1023)
      g_peel_trace[round][1 + blockIdx.x] = globaltimer_ns();
#endif
    grid.sync();
#ifdef GIS_PEEL_TRACE
    if (grid.thread_rank() == 0 && round < 64) g_peel_trace[round][0] = globaltimer_ns();
#endif
    const unsigned long long total = block_broadcast_load(counters + (round % 3));
    if (grid.thread_rank() == 0) counters[(round + 2) % 3] = 0ull;  // used again in round+2
    all += total;
    prev = total;
    ++round;
    if (total == 0) break;
  }
  if (grid.thread_rank() == 0) {
    *rounds_out = round;
    if (deaths_out) atomicAdd(deaths_out, all);
  }
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
  const unsigned long long d =
      sweep_words<false>(indptr, indices, vbase, vend, alive, ScanState<false>{ptr}, w0, w1, nw);
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


// ---- multi-GPU pruning fused with the bitmap exchange over peer memory ----
//
// One cooperative kernel per rank runs every sweep of the multi-GPU prune;
// the per-sweep NCCL all-gather of the host-driven path (distributed.py) is
// replaced by stores into the peers' bitmap replicas over NVLink plus a
// flag barrier in peer memory:
//
//   sweep   : the owned words of the local replica (sweep_words); a warp
//             that deletes vertices of a word stores the word's new value
//             into every peer's replica right away (a word has one writer,
//             its owner, and one warp per sweep; peers only read it), so
//             only changed words cross NVLink, overlapped with the sweep;
//   signal  : after a system-scope fence, the leader thread writes
//             (seq << 32 | owned deletions) into slot [seq & 1][rank] of every
//             rank's flag area (relaxed system-scope stores), then polls its
//             own area until all R ranks posted seq, fences again (acquire),
//             and sums the deletions; the sweep loop ends on a global sum of
//             zero, which every rank computes identically.
//
// A rank is at most one flag ahead of any other (it posts sweep r+1 only
// after reading everyone's sweep r), so two parity slots suffice.  An entry
// handshake (seq0) keeps peers from pushing into a replica before its owner
// has initialised it.  Pushes from a faster rank's next sweep may land
// during this rank's sweep: bits only go 1 -> 0 and the fixed point does not
// depend on when a deletion is seen.
//
// rank < 0 emulates all R ranks in one launch on one GPU (blocks split into
// R groups, replicas and flag areas on this GPU): the same protocol, with
// grid-wide barriers, so that its logic is testable without R GPUs.
struct P2PPeel {
  const int64_t* indptr;   // rows of this rank's owned range (or all V if emulated)
  const int32_t* indices;
  int64_t V, vbase;        // row r of indptr is vertex vbase + r
  uint32_t* const* rep;    // [R] replica address per rank, as mapped here
  unsigned long long* const* flag;  // [R] flag area per rank ([2][R] u64 each)
  int64_t* state;
  unsigned long long* counters;  // [R][3]
  unsigned long long* gtotal;    // [R]
  int rank, R;
  uint32_t seq0;
  int* rounds_out;
  int* err;
};

// One system-scope fence, then relaxed system-scope flag stores / polls: the
// release / acquire pattern with one MEMBAR.SYS per barrier side instead of
// one per peer.
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}


// Post (seq, value) to every rank and wait for every rank's post of seq;
// returns the sum of the posted values, or sets *err on a timeout.
__device__ unsigned long long flag_barrier(const P2PPeel& a, int me, uint32_t seq,
                                           unsigned long long value) {
  const int slot = seq & 1u;
  const unsigned long long word = ((unsigned long long)seq << 32) | (value & 0xffffffffull);
  // release: every store this rank made (pushes by all its blocks happen
  // before via grid.sync + their own system fences) before the posts
  fence_acq_rel_sys();
  for (int q = 0; q < a.R; ++q) st_relaxed_sys(a.flag[q] + slot * a.R + me, word);
  unsigned long long sum = 0;
  const unsigned long long* mine = a.flag[me] + slot * a.R;
  const unsigned long long t0 = globaltimer_ns();
  for (int q = 0; q < a.R; ++q) {
    unsigned long long v;
    while (((v = ld_relaxed_sys(mine + q)) >> 32) != seq) {
      // ranks enter after their own graph builds, so a wait can be long;
      // a minute without a post means a peer is gone
      if (globaltimer_ns() - t0 > 60ull * 1000000000ull) {
        atomicExch(a.err, 1);
        return 0;
      }
      __nanosleep(64);
    }
    sum += v & 0xffffffffull;
  }
  fence_acq_rel_sys();  // acquire: the peers' pushes are visible from here on
  return sum;
}

__global__ void __launch_bounds__(256) peel_p2p_kernel(P2PPeel a) {
  cg::grid_group grid = cg::this_grid();
  const bool emulate = a.rank < 0;
  const int bpr = emulate ? (int)gridDim.x / a.R : (int)gridDim.x;  // host: R | gridDim.x
  const int me = emulate ? (int)blockIdx.x / bpr : a.rank;
  const int lb = (int)blockIdx.x - (emulate ? me * bpr : 0);
  const int64_t words = (a.V + 31) >> 5;
  const int64_t W = std::max<int64_t>(1, (words + a.R - 1) / a.R);  // word_partition
  const int64_t w0 = std::min<int64_t>(words, (int64_t)me * W);
  const int64_t w1 = std::min<int64_t>(words, w0 + W);
  const int64_t vend = std::min<int64_t>(a.V, w1 * 32);
  const int64_t gw = w0 + (((int64_t)lb * blockDim.x + threadIdx.x) >> 5);
  const int64_t nw = ((int64_t)bpr * blockDim.x) >> 5;
  uint32_t* alive = a.rep[me];
  const bool leader = lb == 0 && threadIdx.x == 0;
  __shared__ unsigned long long bsum;

  if (leader) flag_barrier(a, me, a.seq0, 0);  // every replica is initialised
  grid.sync();
  int round = 0;
  while (true) {
    if (threadIdx.x == 0) bsum = 0;
    __syncthreads();
    PushTo push;
    push.rep = a.rep;
    push.R = a.R;
    push.me = me;
    const unsigned long long d = sweep_words<false>(a.indptr, a.indices, a.vbase, vend, alive,
                                                    ScanState<false>{a.state}, gw, w1, nw, push);
    if (d) atomicAdd(&bsum, d);
    if (a.R > 1) __threadfence_system();  // this thread's pushes before the flag
    __syncthreads();
    if (threadIdx.x == 0 && bsum) atomicAdd(a.counters + me * 3 + round % 3, bsum);
    grid.sync();
    if (leader) {
      const unsigned long long mine = a.counters[me * 3 + round % 3];
      a.gtotal[me] = a.R > 1 ? flag_barrier(a, me, a.seq0 + 1 + round, mine) : mine;
      a.counters[me * 3 + (round + 2) % 3] = 0ull;  // used again in round + 2
    }
    grid.sync();
    // the global sum is the same on every rank (and every emulated rank)
    const unsigned long long total = block_broadcast_load(a.gtotal + me);
    ++round;
    if (total == 0 || *(volatile int*)a.err) break;
  }
  if (leader && me == (emulate ? 0 : a.rank)) *a.rounds_out = round;
}
}  // namespace gis

using namespace gis;

template <bool COMPACT>
static void launch_peel_coop(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                             int64_t vbase, int64_t vend, uint32_t* alive, void* ptr,
                             unsigned long long* counters, int* rounds_d,
                             unsigned long long* deaths_d) {
  int per_sm = 0, per_sm4 = 0;  // both forms must be co-resident grids
  GIS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm,
                                                         peel_coop_kernel<COMPACT, false>, 256, 0));
  GIS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm4,
                                                         peel_coop_kernel<COMPACT, true>, 256, 0));
  per_sm = std::min(per_sm, per_sm4);
  GIS_REQUIRE(per_sm >= 1, GIS_E_CUDA, "peel kernel cannot be resident");
  const int64_t words = ((vend + 31) >> 5) - (vbase >> 5);
  int64_t blocks = (int64_t)per_sm * ctx->num_sms;
  blocks = std::min<int64_t>(blocks, std::max<int64_t>(ceil_div(words * 32, 256), 1));
  // four-word steps only when they still give every warp >= 16 groups a sweep
  const bool vec4 = words / 4 >= 16 * blocks * 8;
  void* args[] = {(void*)&indptr, (void*)&indices, (void*)&vbase, (void*)&vend, (void*)&alive,
                  (void*)&ptr,    (void*)&counters, (void*)&rounds_d, (void*)&deaths_d};
  GIS_CUDA(cudaLaunchCooperativeKernel(
      vec4 ? (const void*)peel_coop_kernel<COMPACT, true> : (const void*)peel_coop_kernel<COMPACT, false>,
      dim3((unsigned)blocks), dim3(256), args, 0, ctx->stream));
  count_launch(ctx);
}

// The wide scan state (8 bytes per vertex) is kept while it stays well inside
// L2; past that the compact one (4 bytes, target only) halves what every
// sweep streams (config 4: 134 MB of state per sweep otherwise, > the 126 MB
// L2).
static constexpr int64_t kWideStateMaxBytes = (int64_t)48 << 20;

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
    const bool compact = V * 8 > kWideStateMaxBytes;
    void* ptr = scratch(ctx, SC_TOFF, V * (compact ? 4 : 8));
    struct Ctr { unsigned long long c[3]; int rounds; };
    Ctr* ctr = (Ctr*)scratch(ctx, SC_MISC3, sizeof(Ctr));
    GIS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Ctr), ctx->stream));
    const int64_t nt = std::max(V, words);
    if (compact)
      peel_init_kernel<int32_t><<<(unsigned)ceil_div(nt, 256), 256, 0, ctx->stream>>>(
          V, (int32_t*)ptr, alive, V, words);
    else
      peel_init_kernel<int64_t><<<(unsigned)ceil_div(nt, 256), 256, 0, ctx->stream>>>(
          V, (int64_t*)ptr, alive, V, words);
    count_launch(ctx);
    if (compact)
      launch_peel_coop<true>(ctx, indptr, indices, 0, V, alive, ptr, ctr->c, &ctr->rounds,
                             nullptr);
    else
      launch_peel_coop<false>(ctx, indptr, indices, 0, V, alive, ptr, ctr->c, &ctr->rounds,
                              nullptr);
    int* rounds_d = &ctr->rounds;
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
    peel_init_kernel<int64_t><<<(unsigned)ceil_div(nt, 256), 256, 0, ctx->stream>>>(nrows, ptr, alive, V,
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

GIS_API int gis_peel_local(gis_ctx* ctx, const int64_t* indptr_local, const int32_t* indices,
                           int64_t v_begin, int64_t v_end, uint32_t* alive, int64_t* ptr,
                           int64_t* deaths_dev) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (v_end <= v_begin) return;  // empty shard
    GIS_REQUIRE(v_begin % 32 == 0, GIS_E_INVALID, "owned range must start on a bitmap word");
    PhaseScope ps(ctx, PH_PRUNE);
    struct Ctr { unsigned long long c[3]; int rounds; };
    Ctr* ctr = (Ctr*)scratch(ctx, SC_MISC2, sizeof(Ctr));
    GIS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Ctr), ctx->stream));
    launch_peel_coop<false>(ctx, indptr_local, indices, v_begin, v_end, alive, ptr, ctr->c,
                     &ctr->rounds, (unsigned long long*)deaths_dev);
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

GIS_API int gis_peel_p2p(gis_ctx* ctx, const int64_t* indptr, const int32_t* indices, int64_t V,
                         int64_t vbase, int64_t rows, const uint64_t* replica_addrs,
                         const uint64_t* flag_addrs, int32_t rank, int32_t R, uint32_t seq0,
                         int32_t* rounds) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V >= 0 && V < INT_MAX && rows >= 0 && vbase >= 0, GIS_E_INVALID,
                "V / rows out of range");
    GIS_REQUIRE(R >= 1 && R <= 64 && rank < R && replica_addrs && flag_addrs, GIS_E_INVALID,
                "bad rank / world size / address tables");
    GIS_REQUIRE(seq0 != 0, GIS_E_INVALID, "seq0 must be nonzero (flag areas start zeroed)");
    if (V == 0) { if (rounds) *rounds = 0; return; }
    PhaseScope ps(ctx, PH_PRUNE);
    const int64_t words = (V + 31) >> 5;
    // device copies of the address tables, then counters / totals / flags
    struct Tail { int err; int rounds; };
    const size_t tab = (size_t)R * 8, ctr = (size_t)R * 3 * 8, tot = (size_t)R * 8;
    char* misc = (char*)scratch(ctx, SC_MISC3, 2 * tab + ctr + tot + sizeof(Tail));
    upload_to(ctx, misc, replica_addrs, tab);
    upload_to(ctx, misc + tab, flag_addrs, tab);
    GIS_CUDA(cudaMemsetAsync(misc + 2 * tab, 0, ctr + tot + sizeof(Tail), ctx->stream));
    int64_t* state = (int64_t*)scratch(ctx, SC_TOFF, std::max<int64_t>(rows, 1) * 8);
    // the replica(s) of this process start all-alive (every word, not only
    // the owned ones); the scan state of the rows starts "not started"
    const int q0 = rank < 0 ? 0 : rank, q1 = rank < 0 ? R : rank + 1;
    for (int q = q0; q < q1; ++q) {
      const int64_t nrows = q == q0 ? rows : 0;
      peel_init_kernel<int64_t><<<(unsigned)ceil_div(std::max(nrows, words), 256), 256, 0,
                         ctx->stream>>>(nrows, state, (uint32_t*)(uintptr_t)replica_addrs[q], V,
                                        words);
      count_launch(ctx);
    }
    int per_sm = 0;
    GIS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peel_p2p_kernel, 256, 0));
    GIS_REQUIRE(per_sm >= 1, GIS_E_CUDA, "peel kernel cannot be resident");
    int64_t blocks = (int64_t)per_sm * ctx->num_sms;
    const int64_t want = std::max<int64_t>(ceil_div(ceil_div(words, R) * 32, 256), 1);
    if (rank < 0) {  // emulation: R equal block groups, all resident
      const int64_t bpr = std::min<int64_t>(blocks / R, want);
      GIS_REQUIRE(bpr >= 1, GIS_E_INVALID, "too many emulated ranks for one GPU");
      blocks = bpr * R;
    } else {
      blocks = std::min(blocks, want);
    }
    P2PPeel a;
    a.indptr = indptr;
    a.indices = indices;
    a.V = V;
    a.vbase = vbase;
    a.rep = (uint32_t* const*)misc;
    a.flag = (unsigned long long* const*)(misc + tab);
    a.state = state;
    a.counters = (unsigned long long*)(misc + 2 * tab);
    a.gtotal = (unsigned long long*)(misc + 2 * tab + ctr);
    Tail* tail = (Tail*)(misc + 2 * tab + ctr + tot);
    a.rank = rank;
    a.R = R;
    a.seq0 = seq0;
    a.err = &tail->err;
    a.rounds_out = &tail->rounds;
    void* args[] = {(void*)&a};
    GIS_CUDA(cudaLaunchCooperativeKernel((const void*)peel_p2p_kernel, dim3((unsigned)blocks),
                                         dim3(256), args, 0, ctx->stream));
    count_launch(ctx);
    Tail t{0, 0};
    read_back(ctx, &t, tail, sizeof(Tail));
    GIS_REQUIRE(t.err == 0, GIS_E_STATE, "peer rank did not answer the sweep barrier");
    if (rounds) *rounds = t.rounds;
  });
}

// Device buffers shared with peer processes (CUDA IPC): allocated whole with
// cudaMalloc (an IPC handle names an allocation base), zero-filled.
GIS_API int gis_ipc_alloc(gis_ctx* ctx, int64_t bytes, void** ptr, void* handle) {
  return guarded([&] {
    GIS_REQUIRE(ctx && ptr && handle && bytes > 0, GIS_E_INVALID, "null context or argument");
    void* p = nullptr;
    GIS_CUDA(cudaMalloc(&p, (size_t)bytes));
    GIS_CUDA(cudaMemset(p, 0, (size_t)bytes));
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      GIS_CUDA(e);
    }
    memcpy(handle, &h, sizeof(h));
    *ptr = p;
  });
}

GIS_API int gis_ipc_open(gis_ctx* ctx, const void* handle, void** ptr) {
  return guarded([&] {
    GIS_REQUIRE(ctx && ptr && handle, GIS_E_INVALID, "null context or argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    GIS_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

GIS_API int gis_ipc_close(void* ptr) {
  return guarded([&] { if (ptr) GIS_CUDA(cudaIpcCloseMemHandle(ptr)); });
}

GIS_API int gis_ipc_free(void* ptr) {
  return guarded([&] { if (ptr) GIS_CUDA(cudaFree(ptr)); });
}
