// Device-only helpers shared by the libgis kernels and by the kernels NVRTC
// compiles for user-defined models (gis_jit.cu): no host headers here, so
// the same source compiles under nvcc and NVRTC (__CUDACC_RTC__).
#pragma once

#ifdef __CUDACC_RTC__
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef unsigned char uint8_t;
#ifndef INFINITY
#define INFINITY __longlong_as_double(0x7ff0000000000000LL)
#endif
#ifndef INT_MAX
#define INT_MAX 2147483647
#define INT_MIN (-INT_MAX - 1)
#endif
#else
#include <climits>
#include <cmath>
#include <cstdint>
#endif

#include "gis.h"

namespace gis {

// q = x / d, r = x % d for 0 <= x < 2^22, d >= 1: float reciprocal (one
// MUFU.RCP) and a one-step correction instead of an integer division
__device__ __forceinline__ int32_t div_small(int32_t x, int32_t d, int32_t& r) {
  int32_t q = (int32_t)((float)x * __frcp_rn((float)d));
  r = x - q * d;
  if (r < 0) { --q; r += d; } else if (r >= d) { ++q; r -= d; }
  return q;
}

// First position in [p, e) whose target is set in the `alive` bitmap (e if
// none).  Dead targets come in long runs (rows ascend in CellId order and the
// dead set grows as regions), so 8 entries are probed per step as
// independent loads rather than one dependent load at a time, and the next
// 8 targets are loaded during the probe (config 2 prune 0.41 -> 0.40 ms,
// config 4 4.3 -> 4.0 ms; 16 per step: slower, registers).
__device__ __forceinline__ int64_t first_live(const int32_t* __restrict__ idx, int64_t p,
                                              int64_t e, const uint32_t* alive) {
#ifndef GIS_PEEL_PROBES  // experiments (build.py --variant)
#define GIS_PEEL_PROBES 8
#endif
  constexpr int kW = GIS_PEEL_PROBES;
  auto bit = [&](int32_t t) { return (__ldcg(alive + (t >> 5)) >> (t & 31)) & 1u; };
  // Software-pipelined: the next kW targets are loaded while the current
  // kW bits are probed, so a long dead run costs one memory round trip per
  // kW entries instead of two (index load, then bitmap load).
  if (p >= e) return e;
  int32_t c[kW];
#pragma unroll
  for (int j = 0; j < kW; ++j) c[j] = (p + j < e) ? idx[p + j] : 0;
  while (true) {
    const int64_t q = p + kW;
    int32_t nx[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) nx[j] = (q + j < e) ? idx[q + j] : 0;
    unsigned live = 0;
#pragma unroll
    for (int j = 0; j < kW; ++j) live |= ((p + j < e) ? bit(c[j]) : 0u) << j;
    if (live) return p + __ffs(live) - 1;
    if (q >= e) return e;
    p = q;
#pragma unroll
    for (int j = 0; j < kW; ++j) c[j] = nx[j];
  }
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
//
// Sparse dyadic index (coverings too deep, or too sparse, for a dense slot
// table: the reference's MAX_DEPTH = 62, cg/geometry.py:34): the cells'
// path-aligned start codes key[i] = bits << (62 - depth), ascending in
// canonical order (cg/geometry.py:200-203), and their depths.  A box query
// descends the implicit binary tree of the root's dyadic splits (axis =
// level mod n, midpoints 0.5*(lo+hi) exactly as Covering.subdivide computes
// them, cg/geometry.py:358), pruned by closed box intersection and by binary
// searches for the cells inside each node's code range; it visits the
// intersecting cells in ascending index order.  O(V) memory at any depth.
struct SparseDev {
  const uint64_t* key;   // [V] ascending
  const uint8_t* dep;    // [V]
  double rlo[GIS_MAX_DIM], rhi[GIS_MAX_DIM];
};

struct GridDev {
  int n;
  int64_t ns[GIS_MAX_DIM];       // slots per axis
  int64_t stride[GIS_MAX_DIM];   // slot-table strides
  const double* face[GIS_MAX_DIM];
  const int32_t* slot;
  const int32_t* cell_slo;       // per cell, per axis first slot  [n][V]
  const int32_t* cell_shi;       // per cell, per axis last slot   [n][V]
  int64_t V;
  int sparse;                    // 1: no slot table, query through `sp`
  // 1: 2-D dense index of a dyadic covering, so the slot (i0, i1) at the
  // finest depth D has the D-bit split path whose bits alternate between
  // the axes; cells are contiguous, ascending ranges of those codes (K2's
  // Morton-tile rows, gis_graph.cu)
  int morton;
  SparseDev sp;
  // per axis F[0] and ns / (F[ns] - F[0]): the slot a coordinate falls in
  // if the faces were uniform (exactly so up to rounding on dyadic grids) --
  // the starting guess of the axis_range searches
  double g0[GIS_MAX_DIM], gs[GIS_MAX_DIM];
};

static constexpr int kSparseKeyBits = 62;  // = MAX_DEPTH

// Query boxes of K2-general (gis_cand.cu): box of pair p on axis d at
// lo[p * ps + d * ds] (AoS: ps = n, ds = 1; SoA query arrays: ps = 1,
// ds = Q); valid == nullptr: every pair valid.
struct PairBoxes {
  const double* lo;
  const double* hi;
  const uint8_t* valid;
  int64_t ps, ds;
};


__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* __restrict__ k, int64_t a,
                                                   int64_t b, uint64_t x) {
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (__ldg(k + m) < x) a = m + 1; else b = m;
  }
  return a;
}

// Visit every cell whose closed box meets the closed box [ql, qh] (cg/
// geometry.py:497-501: lo <= cell_hi and cell_lo <= hi on every axis), in
// ascending cell index.  f(cell) returns false to stop early.  NaN bounds
// meet nothing.
template <int N, class F>
__device__ __forceinline__ void sparse_visit(const SparseDev& s, int64_t V,
                                             const double (&ql)[N], const double (&qh)[N],
                                             F&& f) {
  double lo[N], hi[N];
  bool meets = V > 0;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    lo[d] = s.rlo[d];
    hi[d] = s.rhi[d];
    meets = meets && ql[d] <= hi[d] && lo[d] <= qh[d];
  }
  if (!meets) return;
  // frame j = the node at level j on the current path: its cell interval
  // [a, b), which child is being visited (0 none yet, 1 left, 2 right) and
  // the box coordinate the child replaced
  int64_t fa[kSparseKeyBits + 1], fb[kSparseKeyBits + 1];
  uint8_t side[kSparseKeyBits + 1];
  double saved[kSparseKeyBits + 1];
  int j = 0;
  uint64_t path = 0;
  fa[0] = 0;
  fb[0] = V;
  side[0] = 0;
  bool fresh = true;  // the node at level j was just entered
  while (j >= 0) {
    if (fresh) {
      fresh = false;
      const int sh = kSparseKeyBits - j;
      const uint64_t start = path << sh;
      const uint64_t end = start + ((uint64_t)1 << sh);  // exclusive
      const int64_t a = lower_bound_u64(s.key, fa[j], fb[j], start);
      const int64_t b = lower_bound_u64(s.key, a, fb[j], end);
      if (a == b) {
        side[j] = 2;  // no cell inside: done with this node
      } else if (s.dep[a] == j) {  // the node is a cell of the covering
        if (!f(a)) return;
        side[j] = 2;
      } else {
        fa[j] = a;
        fb[j] = b;
        side[j] = 0;
      }
    }
    if (side[j] == 2 || j == kSparseKeyBits) {  // pop: restore the parent's box
      if (j == 0) return;
      const int ax = (j - 1) % N;
      if (path & 1u) lo[ax] = saved[j]; else hi[ax] = saved[j];
      path >>= 1;
      --j;
      continue;
    }
    // next child of node j: split axis j mod N at the midpoint
    const int ax = j % N;
    const double mid = __dmul_rn(0.5, __dadd_rn(lo[ax], hi[ax]));
    const int c = side[j]++;  // 0 -> left, 1 -> right
    double nlo = lo[ax], nhi = hi[ax];
    if (c == 0) nhi = mid; else nlo = mid;
    if (!(qh[ax] >= nlo && ql[ax] <= nhi)) continue;  // the child misses the query
    saved[j + 1] = (c == 0) ? hi[ax] : lo[ax];
    lo[ax] = nlo;
    hi[ax] = nhi;
    path = (path << 1) | (uint64_t)c;
    fa[j + 1] = fa[j];
    fb[j + 1] = fb[j];
    ++j;
    fresh = true;
  }
}

// Slot ranges of a coordinate interval on one axis of the grid index.  The
// answers are monotone searches over the sorted faces F[0..ns]; each starts
// at the slot the coordinate would fall in if the faces were uniform (they
// are, up to rounding, on dyadic grids: GridDev::g0 / gs) and walks to the
// exact answer with the searches' own comparisons -- two face loads per
// bound instead of a log2(ns)-deep chain of dependent loads -- finishing
// with a binary search after a few steps (non-uniform faces).  NaN bounds
// give empty ranges (cg/geometry.py:497-501 semantics).
__device__ __forceinline__ int64_t guess_face(double q, int64_t ns, double g0, double gs) {
  double t = (q - g0) * gs;
  t = t >= 0.0 ? t : 0.0;  // NaN -> 0
  t = t <= (double)(ns - 1) ? t : (double)(ns - 1);
  return (int64_t)t;
}

// smallest k in [lo, hi] with pred(F[k]) (hi + 1 if none), pred monotone
// (false ... false true ... true); k: the starting guess in [lo, hi]
template <class P>
__device__ __forceinline__ int64_t first_true(const double* __restrict__ F, int64_t lo,
                                              int64_t hi, int64_t k, P pred) {
  constexpr int kWalk = 3;
  int w = 0;
  if (pred(__ldg(F + k))) {  // the answer is <= k: walk down
    while (k > lo && w < kWalk && pred(__ldg(F + k - 1))) { --k; ++w; }
    if (w < kWalk || k == lo) return k;
    hi = k;  // in [lo, k]
  } else {  // the answer is > k: walk up
    ++k;
    while (k <= hi && w < kWalk && !pred(__ldg(F + k))) { ++k; ++w; }
    if (w < kWalk || k > hi) return k;
    lo = k;  // in [k, hi + 1]
    ++hi;
  }
  while (lo < hi) {  // first true in [lo, hi), else hi
    const int64_t mid = (lo + hi) >> 1;
    if (pred(__ldg(F + mid))) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Closed interval: a = first j with F[j+1] >= qlo, b = last j with
// F[j] <= qhi (the slots the closed box meets on this axis).
__device__ __forceinline__ void axis_range(const GridDev& g, int d, double qlo, double qhi,
                                           int64_t& a, int64_t& b) {
  const double* F = g.face[d];
  const int64_t ns = g.ns[d];
  a = qlo != qlo ? ns
                 : first_true(F, 1, ns, guess_face(qlo, ns, g.g0[d], g.gs[d]) + 1,
                              [&](double f) { return f >= qlo; }) - 1;
  b = qhi != qhi ? -1
                 : first_true(F, 0, ns - 1, guess_face(qhi, ns, g.g0[d], g.gs[d]),
                              [&](double f) { return !(f <= qhi); }) - 1;
}

// Open interval: the slots a box overlaps with positive length on this axis
// (F[j+1] > qlo and F[j] < qhi).  Used where only positive-volume overlaps
// contribute (containment: a merely touching cell adds +0.0).
__device__ __forceinline__ void axis_range_open(const GridDev& g, int d, double qlo,
                                                double qhi, int64_t& a, int64_t& b) {
  const double* F = g.face[d];
  const int64_t ns = g.ns[d];
  a = qlo != qlo ? ns
                 : first_true(F, 1, ns, guess_face(qlo, ns, g.g0[d], g.gs[d]) + 1,
                              [&](double f) { return f > qlo; }) - 1;
  b = qhi != qhi ? -1
                 : first_true(F, 0, ns - 1, guess_face(qhi, ns, g.g0[d], g.gs[d]),
                              [&](double f) { return !(f < qhi); }) - 1;
}

}  // namespace gis
