// K4: covering updates and adaptive selection on the device.
//
//  * subdivide  (Covering.subdivide, cg/geometry.py:343-372): a selected
//    cell's two children take its place in canonical order (they are the
//    only cells whose path extends the parent's), so the update is an
//    exclusive scan of (1 + sel) and a scatter -- no sort.
//  * retain     (cg/geometry.py:374-385): stable compaction.
//  * boundary   (select_boundary_mask, cg/adaptive.py:61-123): point location
//    of the 2^n enlarged-box corners (+ face midpoints) in the slot table.
//  * k-NN       (knn_indices_many, cg/geometry.py:529-555, and
//    select_neighborhood_mask, cg/adaptive.py:136-150): exact top-k by
//    (distance, index) with an expanding slot window and a proven bound.
//  * containment defect (cg/engine.py:114-130) and diameter.
#include <cub/device/device_radix_sort.cuh>

#include <vector>

#include "gis_internal.cuh"

namespace gis {

// ----------------------------------------------------------- subdivide ---
template <int N>
__global__ void subdivide_kernel(int64_t V, const int32_t* __restrict__ depths,
                                 const int64_t* __restrict__ bits, const double* __restrict__ lo,
                                 const double* __restrict__ hi, const uint8_t* __restrict__ sel,
                                 const int64_t* __restrict__ pos,
                                 int32_t* __restrict__ depths_out, int64_t* __restrict__ bits_out,
                                 double* __restrict__ lo_out, double* __restrict__ hi_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int64_t V2 = pos[V];  // output cells
  const int64_t o = pos[i];
  const int32_t dep = depths[i];
  const int64_t b = bits[i];
  const bool s = sel ? sel[i] != 0 : true;
  if (!s) {
    depths_out[o] = dep;
    bits_out[o] = b;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      lo_out[d * V2 + o] = lo[d * V + i];
      hi_out[d * V2 + o] = hi[d * V + i];
    }
    return;
  }
  const int ax = dep % N;
  depths_out[o] = dep + 1;
  depths_out[o + 1] = dep + 1;
  bits_out[o] = b << 1;
  bits_out[o + 1] = (b << 1) | 1;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    const double l = lo[d * V + i], h = hi[d * V + i];
    if (d == ax) {
      const double mid = __dmul_rn(0.5, __dadd_rn(l, h));  // cg/geometry.py:358
      lo_out[d * V2 + o] = l;
      hi_out[d * V2 + o] = mid;
      lo_out[d * V2 + o + 1] = mid;
      hi_out[d * V2 + o + 1] = h;
    } else {
      lo_out[d * V2 + o] = l;
      hi_out[d * V2 + o] = h;
      lo_out[d * V2 + o + 1] = l;
      hi_out[d * V2 + o + 1] = h;
    }
  }
}

template <int N>
__global__ void retain_kernel(int64_t V, const int32_t* __restrict__ depths,
                              const int64_t* __restrict__ bits, const double* __restrict__ lo,
                              const double* __restrict__ hi, const uint8_t* __restrict__ keep,
                              const int64_t* __restrict__ pos,
                              int32_t* __restrict__ depths_out, int64_t* __restrict__ bits_out,
                              double* __restrict__ lo_out, double* __restrict__ hi_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V || !keep[i]) return;
  const int64_t V2 = pos[V];  // kept cells
  const int64_t o = pos[i];
  depths_out[o] = depths[i];
  bits_out[o] = bits[i];
#pragma unroll
  for (int d = 0; d < N; ++d) {
    lo_out[d * V2 + o] = lo[d * V + i];
    hi_out[d * V2 + o] = hi[d * V + i];
  }
}

// origin[c'] of a covering c' = subdivide(retain(c, keep), sel): the index
// in c of every cell carried over unchanged (kept and not selected); the
// children of selected cells stay -1.  posk / pos: exclusive scans of keep
// (NULL: all kept) and sel.
__global__ void origin_kernel(int64_t V, const uint8_t* __restrict__ keep,
                              const int64_t* __restrict__ posk, const uint8_t* __restrict__ sel,
                              const int64_t* __restrict__ pos, int64_t V_new,
                              int64_t* __restrict__ origin) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V || (keep && !keep[i])) return;
  const int64_t j = keep ? posk[i] : i;
  if (sel[j]) return;
  const int64_t o = j + pos[j];  // subdivide: cell j moves past one extra cell per split before it
  if (o < V_new) origin[o] = i;
}

// fwd[i] for the cells i of c in c' = subdivide(retain(c, keep), sel): the
// index in c' of a cell carried over unchanged, -2 - (index of its first
// child) for a selected cell (children are consecutive), -1 if not kept.
__global__ void forward_kernel(int64_t V, const uint8_t* __restrict__ keep,
                               const int64_t* __restrict__ posk, const uint8_t* __restrict__ sel,
                               const int64_t* __restrict__ pos, int64_t* __restrict__ fwd) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  if (keep && !keep[i]) {
    fwd[i] = -1;
    return;
  }
  const int64_t j = keep ? posk[i] : i;
  const bool split = sel ? sel[j] != 0 : true;
  const int64_t o = j + (sel ? pos[j] : j);
  fwd[i] = split ? -2 - o : o;
}

__global__ void add_index_kernel(const int64_t* __restrict__ p, int64_t V,
                                 int64_t* __restrict__ o) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= V) o[i] = p[i] + i;
}

// Keep the cells of a uniform dyadic grid whose per-axis index is below
// limit[d] (a G_0 x ... x G_{n-1} grid embedded in the power-of-two grid of
// an extended root box; RunConfig.initial_grid).
__global__ void grid_mask_kernel(const int32_t* __restrict__ depths,
                                 const int64_t* __restrict__ bits, int64_t V, int n,
                                 longlong4 limit, uint8_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int dep = depths[i];
  const int64_t b = bits[i];
  int64_t idx[GIS_MAX_DIM] = {0, 0, 0, 0};
  for (int l = 0; l < dep; ++l) {
    const int ax = l % n;
    idx[ax] = (idx[ax] << 1) | ((b >> (dep - 1 - l)) & 1);
  }
  const int64_t lim[4] = {limit.x, limit.y, limit.z, limit.w};
  bool keep = true;
  for (int d = 0; d < n; ++d) keep = keep && idx[d] < lim[d];
  out[i] = keep ? 1 : 0;
}

// Uniform grid of `depth` cycled splits, generated directly: cell code c in
// [0, 2^depth) has bits = c (canonical order of equal-depth cells is bits
// order) and per-axis coordinates from de-interleaving c (axis = level mod
// n); its bounds are the host face arrays' entries coord, coord + 1 -- the
// values repeated midpoint splits produce.  keep[c] = every coordinate
// below its limit (all ones without limits).
__global__ void uniform_keep_kernel(int64_t ncodes, int depth, int n, longlong4 limit,
                                    uint8_t* __restrict__ keep) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncodes) return;
  int64_t idx[GIS_MAX_DIM] = {0, 0, 0, 0};
  for (int l = 0; l < depth; ++l) {
    const int ax = l % n;
    idx[ax] = (idx[ax] << 1) | ((c >> (depth - 1 - l)) & 1);
  }
  const int64_t lim[4] = {limit.x, limit.y, limit.z, limit.w};
  bool k = true;
  for (int d = 0; d < n; ++d) k = k && idx[d] < lim[d];
  keep[c] = k ? 1 : 0;
}

__global__ void uniform_write_kernel(int64_t ncodes, int depth, int n,
                                     const uint8_t* __restrict__ keep,
                                     const int64_t* __restrict__ pos,
                                     const double* __restrict__ faces, longlong4 foff,
                                     int64_t V, int32_t* __restrict__ depths,
                                     int64_t* __restrict__ bits, double* __restrict__ lo,
                                     double* __restrict__ hi) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncodes || (keep && !keep[c])) return;
  const int64_t o = pos ? pos[c] : c;
  int64_t idx[GIS_MAX_DIM] = {0, 0, 0, 0};
  for (int l = 0; l < depth; ++l) {
    const int ax = l % n;
    idx[ax] = (idx[ax] << 1) | ((c >> (depth - 1 - l)) & 1);
  }
  const int64_t fo[4] = {foff.x, foff.y, foff.z, foff.w};
  depths[o] = depth;
  bits[o] = c;
  for (int d = 0; d < n; ++d) {  // SoA [n][V]
    lo[d * V + o] = faces[fo[d] + idx[d]];
    hi[d * V + o] = faces[fo[d] + idx[d] + 1];
  }
}

__global__ void count_mask_kernel(const uint8_t* __restrict__ m, int64_t V,
                                  unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x)
    c += m[i] != 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ------------------------------------------------------ boundary select ---
template <int N>
__global__ void boundary_kernel(GridDev g, const double* __restrict__ lo,
                                const double* __restrict__ hi, int64_t V, int64_t begin,
                                int64_t end, double delta, int face_points,
                                uint8_t* __restrict__ out) {
  const int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= end) return;
  double src[3][N];  // enlarged lo, enlarged hi, centre (cg/adaptive.py:69-72)
#pragma unroll
  for (int d = 0; d < N; ++d) {
    const double l = lo[d * V + i], h = hi[d * V + i];
    const double hw = __dmul_rn(0.5, __dsub_rn(h, l));
    const double pad = __dmul_rn(delta, hw);
    src[0][d] = __dsub_rn(l, pad);
    src[1][d] = __dadd_rn(h, pad);
    src[2][d] = __dmul_rn(0.5, __dadd_rn(l, h));
  }
  const int ncorner = 1 << N;
  const int nface = face_points ? N * (1 << (N - 1)) : 0;
  // the slot range of each of the 3 probe coordinates per axis, searched
  // once (3N binary searches instead of one per probe and axis: 64 -> 12 in
  // 4-D); a probe's range is the per-axis pick by its choice
  int64_t ra[3][N], rb[3][N];
  if (!g.sparse) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (c == 2 && !face_points) break;
#pragma unroll
      for (int d = 0; d < N; ++d)
        axis_range(g, d, src[c][d], src[c][d], ra[c][d], rb[c][d]);
    }
  }
  bool boundary = false;
  for (int pr = 0; pr < ncorner + nface && !boundary; ++pr) {
    int choice[N];
    if (pr < ncorner) {
#pragma unroll
      for (int d = 0; d < N; ++d) choice[d] = (pr >> (N - 1 - d)) & 1;
    } else {
      const int q = pr - ncorner;
      const int free_ax = q >> (N - 1);
      const int code = q & ((1 << (N - 1)) - 1);
      int k = 0;
#pragma unroll
      for (int d = 0; d < N; ++d) {
        if (d == free_ax) choice[d] = 2;
        else { choice[d] = (code >> (N - 2 - k)) & 1; ++k; }
      }
    }
    if (g.sparse) {  // some closed cell contains the probe point
      double pq[N];
#pragma unroll
      for (int d = 0; d < N; ++d) pq[d] = src[choice[d]][d];
      bool hit = false;
      sparse_visit<N>(g.sp, g.V, pq, pq, [&](int64_t) { hit = true; return false; });
      if (!hit) boundary = true;
      continue;
    }
    // slots containing the probe on each axis (1 or 2 when on a face)
    int64_t a[N], b[N];
    bool empty = false;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      const int c = choice[d];  // selects, not a dynamic index (registers)
      a[d] = c == 0 ? ra[0][d] : (c == 1 ? ra[1][d] : ra[2][d]);
      b[d] = c == 0 ? rb[0][d] : (c == 1 ? rb[1][d] : rb[2][d]);
      if (a[d] > b[d]) empty = true;
    }
    bool covered = false;
    if (!empty) {
      int64_t c[N];
#pragma unroll
      for (int d = 0; d < N; ++d) c[d] = a[d];
      while (true) {
        int64_t off = 0;
#pragma unroll
        for (int d = 0; d < N; ++d) off += c[d] * g.stride[d];
        if (__ldg(g.slot + off) >= 0) { covered = true; break; }
        int d = N - 1;
        while (d >= 0 && c[d] == b[d]) { c[d] = a[d]; --d; }
        if (d < 0) break;
        c[d]++;
      }
    }
    if (!covered) boundary = true;
  }
  out[i] = boundary ? 1 : 0;
}

// ---------------------------------------------------------------- k-NN ---
// Warp per query.  The current top-k (k <= 32 * KPL) lives across lanes,
// KPL entries per lane (entry j in lane j / KPL, slot j % KPL), sorted by
// (distance, index).  Candidates are the distinct cells meeting a window of
// slots around the query; a cell outside the window has its centre strictly
// farther than the window's inner margin, so the result is final once the
// k-th distance is below that margin (or the window spans the grid).
// Larger k: every centre's distance, then a stable radix sort (knn_all).
template <int N>
__device__ __forceinline__ double centre_dist(const double* __restrict__ lo,
                                              const double* __restrict__ hi, int64_t V,
                                              int64_t c, const double (&q)[N], bool& same) {
  double s = 0.0;
  same = true;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    const double cc = __dmul_rn(0.5, __dadd_rn(lo[d * V + c], hi[d * V + c]));
    same = same && (cc == q[d]);
    const double df = __dsub_rn(cc, q[d]);
    s = (d == 0) ? __dmul_rn(df, df) : __dadd_rn(s, __dmul_rn(df, df));
  }
  return __dsqrt_rn(s);
}

__device__ __forceinline__ bool entry_less(double d1, int64_t i1, double d2, int64_t i2) {
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

template <int KPL>
struct TopK {
  double d[KPL];
  int64_t i[KPL];
  int cnt;
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int s = 0; s < KPL; ++s) { d[s] = INFINITY; i[s] = INT64_MAX; }
    cnt = 0;
  }
  // entry j (warp-uniform j) broadcast to all lanes
  __device__ __forceinline__ void get(int j, double& dd, int64_t& ii) const {
    double sd = d[0];
    int64_t si = i[0];
#pragma unroll
    for (int s = 1; s < KPL; ++s)
      if ((j % KPL) == s) { sd = d[s]; si = i[s]; }
    dd = __shfl_sync(0xffffffffu, sd, j / KPL);
    ii = __shfl_sync(0xffffffffu, si, j / KPL);
  }
  __device__ __forceinline__ void insert(double nd, int64_t ni, int k, int lane) {
    if (cnt == k) {
      double kd;
      int64_t ki;
      get(k - 1, kd, ki);
      if (!entry_less(nd, ni, kd, ki)) return;
    }
    int c = 0;
#pragma unroll
    for (int s = 0; s < KPL; ++s)
      c += (lane * KPL + s < cnt && entry_less(d[s], i[s], nd, ni)) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    const int posn = c;
    const double cd = __shfl_up_sync(0xffffffffu, d[KPL - 1], 1);
    const int64_t ci = __shfl_up_sync(0xffffffffu, i[KPL - 1], 1);
#pragma unroll
    for (int s = KPL - 1; s >= 0; --s) {
      const int j = lane * KPL + s;
      const double pd = (s == 0) ? cd : d[s > 0 ? s - 1 : 0];
      const int64_t pi = (s == 0) ? ci : i[s > 0 ? s - 1 : 0];
      if (j == posn) { d[s] = nd; i[s] = ni; }
      else if (j > posn && j < k) { d[s] = pd; i[s] = pi; }
    }
    cnt = min(cnt + 1, k);
  }
};

// Sparse index: windows are closed coordinate boxes [q - R, q + R], R
// doubling from the smallest width of the cell at q.  All lanes run the same
// (warp-uniform) visit of the window's cells in index order and insert each
// candidate together.  A cell outside the window lies farther than R on some
// axis, so the result is final once the k-th distance is below R (or the
// window holds the whole root box).
template <int N, int KPL>
__device__ void knn_warp_sparse(const GridDev& g, const double* __restrict__ lo,
                                const double* __restrict__ hi, int64_t V, const double (&q)[N],
                                int k, bool exclude, TopK<KPL>& top) {
  const int lane = threadIdx.x & 31;
  double R = INFINITY;
  sparse_visit<N>(g.sp, g.V, q, q, [&](int64_t c) {
#pragma unroll
    for (int d = 0; d < N; ++d) R = fmin(R, hi[d * V + c] - lo[d * V + c]);
    return false;
  });
  if (!(R > 0.0) || isinf(R)) {  // q outside every cell: a fraction of the root
    R = INFINITY;
#pragma unroll
    for (int d = 0; d < N; ++d) R = fmin(R, (g.sp.rhi[d] - g.sp.rlo[d]) * (1.0 / 1024.0));
    if (!(R > 0.0)) R = 1.0;
  }
  for (;; R *= 2.0) {
    double wl[N], wh[N];
    bool whole = true;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      wl[d] = q[d] - R;
      wh[d] = q[d] + R;
      whole = whole && wl[d] <= g.sp.rlo[d] && wh[d] >= g.sp.rhi[d];
    }
    top.reset();
    sparse_visit<N>(g.sp, g.V, wl, wh, [&](int64_t c) {
      bool same;
      const double dd = centre_dist<N>(lo, hi, V, c, q, same);
      if (!(exclude && same)) top.insert(dd, c, k, lane);
      return true;
    });
    if (whole) return;
    if (top.cnt == k) {
      double kth;
      int64_t ki;
      top.get(k - 1, kth, ki);
      if (kth < R * (1.0 - 1e-12)) return;
    }
  }
}

template <int N, int KPL>
__device__ void knn_warp(const GridDev& g, const double* __restrict__ lo,
                         const double* __restrict__ hi, int64_t V, const double (&q)[N], int k,
                         bool exclude, TopK<KPL>& top, double r0 = 0.0) {
  const int lane = threadIdx.x & 31;
  if (g.sparse) {
    knn_warp_sparse<N, KPL>(g, lo, hi, V, q, k, exclude, top);
    return;
  }
  // Windows are closed boxes [q - R, q + R] in slot space, R doubling from
  // r0 (the query cell's smallest width: no other centre is nearer than
  // that along its narrowest axis) or else the smallest width of the
  // query's slot: anisotropic cells (cart-pole's theta slots are 14x
  // narrower than the others) get a window proportional to their own widths
  // rather than a cube of slots.  Any start gives the same answer.
  double R = r0;
  if (!(R > 0.0) || isinf(R)) {
    R = INFINITY;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      int64_t a, b;
      axis_range(g, d, q[d], q[d], a, b);
      if (a > b) a = (q[d] < g.face[d][0]) ? 0 : g.ns[d] - 1;  // outside the grid on this axis
      R = fmin(R, g.face[d][a + 1] - g.face[d][a]);
    }
  }
  if (!(R > 0.0)) R = 1.0;  // degenerate faces: any positive start works
  for (;; R *= 2.0) {
    int64_t wl[N], wh[N], wn[N];
    int64_t W = 1;
    bool whole = true;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      axis_range(g, d, q[d] - R, q[d] + R, wl[d], wh[d]);
      if (wl[d] > wh[d]) wl[d] = wh[d] = (q[d] < g.face[d][0]) ? 0 : g.ns[d] - 1;
      wn[d] = wh[d] - wl[d] + 1;
      W *= wn[d];
      whole = whole && wl[d] == 0 && wh[d] == g.ns[d] - 1;
    }
    top.reset();
    for (int64_t base = 0; base < W; base += 32) {
      const int64_t e = base + lane;
      double cd = INFINITY;
      int64_t ci = -1;
      if (e < W) {
        int64_t s = 0;
        int64_t co[N];
        if (W < (1 << 22)) {  // window offsets decoded with float reciprocals
          int32_t off = (int32_t)e;
#pragma unroll
          for (int d = N - 1; d >= 0; --d) {
            int32_t rr;
            off = div_small(off, (int32_t)wn[d], rr);
            co[d] = wl[d] + rr;
            s += co[d] * g.stride[d];
          }
        } else {
          int64_t off = e;
#pragma unroll
          for (int d = N - 1; d >= 0; --d) {
            co[d] = wl[d] + off % wn[d];
            off /= wn[d];
            s += co[d] * g.stride[d];
          }
        }
        const int32_t c = __ldg(g.slot + s);
        if (c >= 0) {
          bool first = true;  // count a coarse cell once: at its first slot in the window
#pragma unroll
          for (int d = 0; d < N; ++d)
            first = first && (co[d] == max(wl[d], (int64_t)g.cell_slo[d * g.V + c]));
          if (first) {
            bool same;
            const double dd = centre_dist<N>(lo, hi, V, c, q, same);
            if (!(exclude && same)) { cd = dd; ci = c; }
          }
        }
      }
      // insert this batch's candidates one at a time (warp-parallel shift);
      // once k are held, only those ahead of the current k-th can enter
      if (top.cnt == k) {
        double kd;
        int64_t kidx;
        top.get(k - 1, kd, kidx);
        if (ci >= 0 && !entry_less(cd, ci, kd, kidx)) ci = -1;
      }
      unsigned pend = __ballot_sync(0xffffffffu, ci >= 0);
      while (pend) {
        const int src = __ffs(pend) - 1;
        pend &= pend - 1;
        top.insert(__shfl_sync(0xffffffffu, cd, src), __shfl_sync(0xffffffffu, ci, src), k,
                   lane);
      }
    }
    if (whole) return;
    if (top.cnt == k) {
      double margin = INFINITY;
#pragma unroll
      for (int d = 0; d < N; ++d) {
        if (wl[d] > 0) margin = fmin(margin, q[d] - g.face[d][wl[d]]);
        if (wh[d] < g.ns[d] - 1) margin = fmin(margin, g.face[d][wh[d] + 1] - q[d]);
      }
      double kth;
      int64_t ki;
      top.get(k - 1, kth, ki);
      if (kth < margin * (1.0 - 1e-12)) return;
    }
  }
}

template <int N, int KPL>
__global__ void knn_kernel(GridDev g, const double* __restrict__ lo, const double* __restrict__ hi,
                           int64_t V, const double* __restrict__ pts, int64_t Q, int k,
                           int exclude, int64_t* __restrict__ out_idx, int32_t* __restrict__ out_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (qi >= Q) return;
  double q[N];
#pragma unroll
  for (int d = 0; d < N; ++d) q[d] = pts[qi * N + d];
  TopK<KPL> top;
  knn_warp<N, KPL>(g, lo, hi, V, q, k, exclude != 0, top);
#pragma unroll
  for (int s = 0; s < KPL; ++s) {
    const int j = lane * KPL + s;
    if (j < k) out_idx[qi * k + j] = (j < top.cnt) ? top.i[s] : -1;
  }
  if (lane == 0) out_cnt[qi] = top.cnt;
}

template <int N, int KPL>
__global__ void neighborhood_kernel(GridDev g, const double* __restrict__ lo,
                                    const double* __restrict__ hi, int64_t V,
                                    const int64_t* __restrict__ qcells, int64_t Q, int k,
                                    uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (qi >= Q) return;
  const int64_t c = qcells[qi];
  double q[N];
  double r0 = INFINITY;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    q[d] = __dmul_rn(0.5, __dadd_rn(lo[d * V + c], hi[d * V + c]));
    r0 = fmin(r0, hi[d * V + c] - lo[d * V + c]);
  }
  TopK<KPL> top;
  knn_warp<N, KPL>(g, lo, hi, V, q, k, true, top, r0);
#pragma unroll
  for (int s = 0; s < KPL; ++s)
    if (lane * KPL + s < top.cnt) out[top.i[s]] = 1;
}

// k > 32 * kMaxKpl: distance of every centre to one query as a sortable key
// (non-negative doubles order like their bit patterns; excluded = max)
template <int N>
__global__ void knn_all_keys_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                    int64_t V, const double* __restrict__ qp, int exclude,
                                    unsigned long long* __restrict__ keys,
                                    int64_t* __restrict__ vals) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= V) return;
  double q[N];
#pragma unroll
  for (int d = 0; d < N; ++d) q[d] = qp[d];
  bool same;
  const double dd = centre_dist<N>(lo, hi, V, c, q, same);
  keys[c] = (exclude && same) ? ~0ull : (unsigned long long)__double_as_longlong(dd);
  vals[c] = c;
}

template <int N>
__global__ void centre_of_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                 int64_t V, const int64_t* __restrict__ cell,
                                 double* __restrict__ q) {
  if (threadIdx.x < N) {
    const int64_t c = *cell;
    q[threadIdx.x] = __dmul_rn(0.5, __dadd_rn(lo[threadIdx.x * V + c], hi[threadIdx.x * V + c]));
  }
}

__global__ void knn_all_emit_kernel(const unsigned long long* __restrict__ keys,
                                    const int64_t* __restrict__ vals, int64_t V, int k,
                                    int64_t* __restrict__ out_idx, int32_t* __restrict__ out_cnt,
                                    uint8_t* __restrict__ mark) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const bool ok = j < V && keys[j] != ~0ull;
  if (out_idx) out_idx[j] = ok ? vals[j] : -1;
  if (mark && ok) mark[vals[j]] = 1;
  if (out_cnt && ok && (j + 1 == k || j + 1 == V || keys[j + 1] == ~0ull)) *out_cnt = (int32_t)(j + 1);
}

// list[pos[i]] = base + i for the set entries of m[0..V)
__global__ void gather_selected_kernel(const uint8_t* __restrict__ m, const int64_t* __restrict__ pos,
                                       int64_t V, int64_t base, int64_t* __restrict__ list) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < V && m[i]) list[pos[i]] = base + i;
}

__global__ void andnot_kernel(uint8_t* __restrict__ out, const uint8_t* __restrict__ b, int64_t V) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < V) out[i] = out[i] && !b[i];
}

// -------------------------------------------------- containment + diam ---
__device__ __forceinline__ void atomic_max_pos(unsigned long long* a, double v) {
  // nonnegative doubles order like their bit patterns
  atomicMax(a, (unsigned long long)__double_as_longlong(v));
}

template <int N>
__global__ void containment_kernel(GridDev g, const double* __restrict__ plo,
                                   const double* __restrict__ phi, int64_t PV,
                                   const double* __restrict__ lo, const double* __restrict__ hi,
                                   int64_t V, int64_t begin, int64_t end,
                                   unsigned long long* __restrict__ best,
                                   int* __restrict__ neg) {
  const int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= end) return;
  double l[N], h[N];
  int64_t a[N], b[N];
  bool empty = false;
  double vol = 1.0;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    l[d] = lo[d * V + i];
    h[d] = hi[d * V + i];
    vol = (d == 0) ? __dsub_rn(h[d], l[d]) : __dmul_rn(vol, __dsub_rn(h[d], l[d]));
    if (g.sparse) continue;
    // slots overlapping the cell with positive length only: a previous cell
    // that merely touches it adds max(0, ...) = +0.0 to the sum in the
    // reference (cg/engine.py:114-130), so skipping it changes no bit -- and
    // in 4-D a cell touches 3^4 slots of its own resolution (config 5
    // containment 17 -> <1 ms)
    axis_range_open(g, d, l[d], h[d], a[d], b[d]);
    if (a[d] > b[d]) empty = true;
  }
  double covered = 0.0;
  if (g.sparse) {  // the previous covering's cells meeting the new cell, ascending
    sparse_visit<N>(g.sp, g.V, l, h, [&](int64_t pc) {
      double inter = 1.0;
#pragma unroll
      for (int d = 0; d < N; ++d) {
        const double w = fmax(0.0, __dsub_rn(fmin(h[d], phi[d * PV + pc]),
                                             fmax(l[d], plo[d * PV + pc])));
        inter = (d == 0) ? w : __dmul_rn(inter, w);
      }
      covered = __dadd_rn(covered, inter);
      return true;
    });
    empty = true;  // the slot walk below is skipped
  }
  if (!empty) {
    int64_t c[N];
#pragma unroll
    for (int d = 0; d < N; ++d) c[d] = a[d];
    while (true) {
      int64_t off = 0;
#pragma unroll
      for (int d = 0; d < N; ++d) off += c[d] * g.stride[d];
      const int32_t pc = g.slot[off];
      if (pc >= 0) {
        bool first = true;
#pragma unroll
        for (int d = 0; d < N; ++d)
          first = first && (c[d] == max(a[d], (int64_t)g.cell_slo[d * g.V + pc]));
        if (first) {
          double inter = 1.0;
#pragma unroll
          for (int d = 0; d < N; ++d) {
            const double w = fmax(0.0, __dsub_rn(fmin(h[d], phi[d * PV + pc]),
                                                 fmax(l[d], plo[d * PV + pc])));
            inter = (d == 0) ? w : __dmul_rn(inter, w);
          }
          covered = __dadd_rn(covered, inter);
        }
      }
      int d = N - 1;
      while (d >= 0 && c[d] == b[d]) { c[d] = a[d]; --d; }
      if (d < 0) break;
      c[d]++;
    }
  }
  const double defect = __dsub_rn(1.0, __ddiv_rn(covered, vol));
  if (defect > 0) atomic_max_pos(best, defect);
  else if (!(defect <= 0)) atomicOr(neg, 1);  // NaN (zero volume)
}

template <int N>
__global__ void diameter_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                int64_t V, unsigned long long* __restrict__ best) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      const double w = __dsub_rn(hi[d * V + i], lo[d * V + i]);
      s = (d == 0) ? __dmul_rn(w, w) : __dadd_rn(s, __dmul_rn(w, w));
    }
    m = fmax(m, __dsqrt_rn(s));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_pos(best, m);
}

template <template <int> class F, class... A>
void by_dim(int n, A&&... args) {
  switch (n) {
    case 1: F<1>::go(args...); break;
    case 2: F<2>::go(args...); break;
    case 3: F<3>::go(args...); break;
    case 4: F<4>::go(args...); break;
    default: throw Error{GIS_E_INVALID, "dimension out of range"};
  }
}

static int64_t count_mask_dev(gis_ctx* ctx, const uint8_t* m, int64_t V) {
  unsigned long long* c = (unsigned long long*)scratch(ctx, SC_MISC, 8);
  GIS_CUDA(cudaMemsetAsync(c, 0, 8, ctx->stream));
  if (V > 0) {
    const int64_t blocks = std::min<int64_t>(ceil_div(V, 256), ctx->num_sms * 8);
    count_mask_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(m, V, c);
    count_launch(ctx);
  }
  unsigned long long h = 0;
  read_back(ctx, &h, c, 8);
  return (int64_t)h;
}

template <int N>
struct SubdivideL {
  static void go(gis_ctx* ctx, int64_t V, const int32_t* depths, const int64_t* bits,
                 const double* lo, const double* hi, const uint8_t* sel, const int64_t* pos,
                 int32_t* dout, int64_t* bout, double* lout, double* hout) {
    subdivide_kernel<N><<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
        V, depths, bits, lo, hi, sel, pos, dout, bout, lout, hout);
    count_launch(ctx);
  }
};

template <int N>
struct RetainL {
  static void go(gis_ctx* ctx, int64_t V, const int32_t* depths, const int64_t* bits,
                 const double* lo, const double* hi, const uint8_t* keep, const int64_t* pos,
                 int32_t* dout, int64_t* bout, double* lout, double* hout) {
    retain_kernel<N><<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
        V, depths, bits, lo, hi, keep, pos, dout, bout, lout, hout);
    count_launch(ctx);
  }
};

template <int N>
struct BoundaryL {
  static void go(gis_ctx* ctx, const GridDev& g, const double* lo, const double* hi, int64_t V,
                 int64_t begin, int64_t end, double delta, int fp, uint8_t* out) {
    boundary_kernel<N><<<(unsigned)ceil_div(end - begin, 128), 128, 0, ctx->stream>>>(
        g, lo, hi, V, begin, end, delta, fp, out);
    count_launch(ctx);
  }
};

static constexpr int kMaxKpl = 8;  // warp top-k up to 256 entries

template <int N>
struct KnnL {
  static void go(gis_ctx* ctx, const GridDev& g, const double* lo, const double* hi, int64_t V,
                 const double* pts, int64_t Q, int k, int ex, int64_t* oi, int32_t* oc) {
    const unsigned blocks = (unsigned)ceil_div(Q * 32, 128);
    if (k <= 32) knn_kernel<N, 1><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, pts, Q, k, ex, oi, oc);
    else if (k <= 64) knn_kernel<N, 2><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, pts, Q, k, ex, oi, oc);
    else if (k <= 128) knn_kernel<N, 4><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, pts, Q, k, ex, oi, oc);
    else knn_kernel<N, 8><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, pts, Q, k, ex, oi, oc);
    count_launch(ctx);
  }
};

template <int N>
struct NeighL {
  static void go(gis_ctx* ctx, const GridDev& g, const double* lo, const double* hi, int64_t V,
                 const int64_t* qc, int64_t Q, int k, uint8_t* out) {
    const unsigned blocks = (unsigned)ceil_div(Q * 32, 128);
    if (k <= 32) neighborhood_kernel<N, 1><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, qc, Q, k, out);
    else if (k <= 64) neighborhood_kernel<N, 2><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, qc, Q, k, out);
    else if (k <= 128) neighborhood_kernel<N, 4><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, qc, Q, k, out);
    else neighborhood_kernel<N, 8><<<blocks, 128, 0, ctx->stream>>>(g, lo, hi, V, qc, Q, k, out);
    count_launch(ctx);
  }
};

// k beyond the warp top-k: per query, all distances + stable radix sort
template <int N>
struct KnnAllL {
  static void go(gis_ctx* ctx, const double* lo, const double* hi, int64_t V, const double* pts,
                 const int64_t* qcells, int64_t Q, int k, int ex, int64_t* oi, int32_t* oc,
                 uint8_t* mark) {
    unsigned long long *keys, *keys2;
    int64_t *vals, *vals2;
    double* qbuf;
    keys = (unsigned long long*)pool_alloc(ctx, V * 8 * 4 + 64);
    keys2 = keys + V;
    vals = (int64_t*)(keys2 + V);
    vals2 = vals + V;
    qbuf = (double*)(vals2 + V);
    size_t tb = 0;
    GIS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, vals2, V, 0, 64,
                                             ctx->stream));
    void* tmp = nullptr;
    tmp = pool_alloc(ctx, tb ? tb : 16);
    for (int64_t q = 0; q < Q; ++q) {
      const double* qp = pts ? pts + q * N : qbuf;
      if (!pts) {
        centre_of_kernel<N><<<1, 32, 0, ctx->stream>>>(lo, hi, V, qcells + q, qbuf);
        count_launch(ctx);
      }
      knn_all_keys_kernel<N><<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(
          lo, hi, V, qp, ex, keys, vals);
      count_launch(ctx);
      GIS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, vals, vals2, V, 0, 64,
                                               ctx->stream));
      count_launch(ctx);
      if (oc) GIS_CUDA(cudaMemsetAsync(oc + q, 0, 4, ctx->stream));
      knn_all_emit_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, ctx->stream>>>(
          keys2, vals2, V, k, oi ? oi + q * k : nullptr, oc ? oc + q : nullptr, mark);
      count_launch(ctx);
    }
    GIS_CUDA(cudaFreeAsync(tmp, ctx->stream));
    GIS_CUDA(cudaFreeAsync(keys, ctx->stream));
  }
};

template <int N>
struct ContainL {
  static void go(gis_ctx* ctx, const GridDev& g, const double* plo, const double* phi, int64_t PV,
                 const double* lo, const double* hi, int64_t V, int64_t begin, int64_t end,
                 unsigned long long* best, int* neg) {
    containment_kernel<N><<<(unsigned)ceil_div(end - begin, 128), 128, 0, ctx->stream>>>(
        g, plo, phi, PV, lo, hi, V, begin, end, best, neg);
    count_launch(ctx);
  }
};

template <int N>
struct DiamL {
  static void go(gis_ctx* ctx, const double* lo, const double* hi, int64_t V,
                 unsigned long long* best) {
    const int64_t blocks = std::min<int64_t>(std::max<int64_t>(ceil_div(V, 256), 1),
                                             ctx->num_sms * 8);
    diameter_kernel<N><<<(unsigned)blocks, 256, 0, ctx->stream>>>(lo, hi, V, best);
    count_launch(ctx);
  }
};

}  // namespace gis

using namespace gis;

GIS_API int gis_grid_mask(gis_ctx* ctx, int32_t n, int64_t V, const int32_t* depths,
                          const int64_t* bits, const int64_t* limits, uint8_t* out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(n >= 1 && n <= GIS_MAX_DIM, GIS_E_INVALID, "n out of range");
    if (V <= 0) return;
    longlong4 lim = make_longlong4(limits[0], n > 1 ? limits[1] : 0, n > 2 ? limits[2] : 0,
                                   n > 3 ? limits[3] : 0);
    grid_mask_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(depths, bits, V, n, lim,
                                                                          out);
    count_launch(ctx);
  });
}

GIS_API int gis_uniform_grid(gis_ctx* ctx, int32_t n, int32_t depth, const double* root_lo,
                             const double* root_hi, const int64_t* limits, int64_t* V_out,
                             int32_t* depths, int64_t* bits, double* lo, double* hi) {
  return guarded([&] {
    GIS_REQUIRE(ctx && root_lo && root_hi && V_out, GIS_E_INVALID, "null context or argument");
    GIS_REQUIRE(n >= 1 && n <= GIS_MAX_DIM && depth >= 0 && depth <= 40, GIS_E_INVALID,
                "n or depth out of range");
    const int64_t ncodes = (int64_t)1 << depth;
    int64_t splits[GIS_MAX_DIM] = {0, 0, 0, 0}, foff[GIS_MAX_DIM] = {0, 0, 0, 0};
    int64_t nf = 0;
    for (int d = 0; d < n; ++d) {
      splits[d] = (depth + n - 1 - d) / n;  // geometry._axis_splits
      GIS_REQUIRE(splits[d] <= 24, GIS_E_CAPACITY, "grid too fine along one axis");
      foff[d] = nf;
      nf += ((int64_t)1 << splits[d]) + 1;
    }
    // per-axis faces: recursive midpoints 0.5*(lo+hi), exactly as the splits
    // compute them (cg/geometry.py:358; the same recursion as the index)
    std::vector<double> faces(nf);
    for (int d = 0; d < n; ++d) {
      double* F = faces.data() + foff[d];
      const int64_t ns = (int64_t)1 << splits[d];
      F[0] = root_lo[d];
      F[ns] = root_hi[d];
      for (int64_t len = ns; len > 1; len >>= 1)
        for (int64_t i = 0; i < ns; i += len) F[i + len / 2] = 0.5 * (F[i] + F[i + len]);
    }
    int64_t lim[GIS_MAX_DIM] = {0, 0, 0, 0};
    bool all = true;
    for (int d = 0; d < n; ++d) {
      lim[d] = limits ? std::min<int64_t>(limits[d], (int64_t)1 << splits[d])
                      : (int64_t)1 << splits[d];
      GIS_REQUIRE(lim[d] >= 1, GIS_E_INVALID, "grid limits must be positive");
      all = all && lim[d] == ((int64_t)1 << splits[d]);
    }
    int64_t V = 1;
    for (int d = 0; d < n; ++d) V *= lim[d];
    if (!depths) { *V_out = V; return; }  // size query
    GIS_REQUIRE(*V_out == V, GIS_E_INVALID, "output sized for a different grid");
    double* fdev = (double*)upload(ctx, SC_PARAMS, faces.data(), (size_t)nf * 8);
    const longlong4 L = make_longlong4(lim[0], lim[1], lim[2], lim[3]);
    const longlong4 F = make_longlong4(foff[0], foff[1], foff[2], foff[3]);
    const unsigned blocks = (unsigned)ceil_div(ncodes, 256);
    uint8_t* keep = nullptr;
    int64_t* pos = nullptr;
    if (!all) {
      keep = (uint8_t*)scratch(ctx, SC_BITMAP, ncodes);
      pos = (int64_t*)scratch(ctx, SC_TOFF, (ncodes + 1) * 8);
      uniform_keep_kernel<<<blocks, 256, 0, ctx->stream>>>(ncodes, depth, n, L, keep);
      count_launch(ctx);
      exclusive_scan_u8_to_i64(ctx, keep, pos, ncodes);
    }
    uniform_write_kernel<<<blocks, 256, 0, ctx->stream>>>(ncodes, depth, n, keep, pos, fdev, F, V,
                                                          depths, bits, lo, hi);
    count_launch(ctx);
  });
}

GIS_API int gis_count_mask(gis_ctx* ctx, const uint8_t* mask, int64_t V, int64_t* count) {
  return guarded([&] {
    GIS_REQUIRE(ctx && count, GIS_E_INVALID, "null context or output");
    *count = count_mask_dev(ctx, mask, V);
  });
}

GIS_API int gis_subdivide(gis_ctx* ctx, int32_t n, int64_t V, const int32_t* depths,
                          const int64_t* bits, const double* lo, const double* hi,
                          const uint8_t* sel, int32_t* depths_out, int64_t* bits_out,
                          double* lo_out, double* hi_out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (V <= 0) return;
    int64_t* pos = (int64_t*)scratch(ctx, SC_TOFF, (V + 1) * 8);
    int64_t* pos2 = (int64_t*)scratch(ctx, SC_ROWCNT, (V + 1) * 8);
    // output slot of cell i = i + (number of selected cells before i)
    exclusive_scan_u8_to_i64(ctx, sel, pos, V);
    add_index_kernel<<<(unsigned)ceil_div(V + 1, 256), 256, 0, ctx->stream>>>(pos, V, pos2);
    count_launch(ctx);
    by_dim<SubdivideL>(n, ctx, V, depths, bits, lo, hi, sel, (const int64_t*)pos2, depths_out,
                       bits_out, lo_out, hi_out);
  });
}

GIS_API int gis_covering_origin(gis_ctx* ctx, int64_t V_old, const uint8_t* keep,
                                int64_t V_mid, const uint8_t* sel, int64_t V_new,
                                int64_t* origin) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V_old >= 0 && V_mid >= 0 && V_new >= 0 && origin, GIS_E_INVALID,
                "sizes out of range");
    GIS_REQUIRE(keep || V_mid == V_old, GIS_E_INVALID, "V_mid != V_old without a keep mask");
    if (V_new == 0) return;
    GIS_CUDA(cudaMemsetAsync(origin, 0xff, V_new * 8, ctx->stream));
    if (!sel || V_old == 0 || V_mid == 0) return;  // full subdivision: every cell is new
    int64_t* posk = nullptr;
    if (keep) {
      posk = (int64_t*)scratch(ctx, SC_TOFF, (V_old + 1) * 8);
      exclusive_scan_u8_to_i64(ctx, keep, posk, V_old);
    }
    int64_t* pos = (int64_t*)scratch(ctx, SC_ROWCNT, (V_mid + 1) * 8);
    exclusive_scan_u8_to_i64(ctx, sel, pos, V_mid);
    origin_kernel<<<(unsigned)ceil_div(V_old, 256), 256, 0, ctx->stream>>>(
        V_old, keep, posk, sel, pos, V_new, origin);
    count_launch(ctx);
  });
}

GIS_API int gis_covering_forward(gis_ctx* ctx, int64_t V_old, const uint8_t* keep,
                                 int64_t V_mid, const uint8_t* sel, int64_t* fwd) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(V_old >= 0 && V_mid >= 0 && fwd, GIS_E_INVALID, "sizes out of range");
    GIS_REQUIRE(keep || V_mid == V_old, GIS_E_INVALID, "V_mid != V_old without a keep mask");
    if (V_old == 0) return;
    int64_t* posk = nullptr;
    if (keep) {
      posk = (int64_t*)scratch(ctx, SC_TOFF, (V_old + 1) * 8);
      exclusive_scan_u8_to_i64(ctx, keep, posk, V_old);
    }
    int64_t* pos = nullptr;
    if (sel && V_mid > 0) {
      pos = (int64_t*)scratch(ctx, SC_ROWCNT, (V_mid + 1) * 8);
      exclusive_scan_u8_to_i64(ctx, sel, pos, V_mid);
    }
    forward_kernel<<<(unsigned)ceil_div(V_old, 256), 256, 0, ctx->stream>>>(V_old, keep, posk,
                                                                              sel, pos, fwd);
    count_launch(ctx);
  });
}

GIS_API int gis_retain(gis_ctx* ctx, int32_t n, int64_t V, const int32_t* depths,
                       const int64_t* bits, const double* lo, const double* hi,
                       const uint8_t* keep, int32_t* depths_out, int64_t* bits_out,
                       double* lo_out, double* hi_out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (V <= 0) return;
    int64_t* pos = (int64_t*)scratch(ctx, SC_TOFF, (V + 1) * 8);
    exclusive_scan_u8_to_i64(ctx, keep, pos, V);
    by_dim<RetainL>(n, ctx, V, depths, bits, lo, hi, keep, (const int64_t*)pos, depths_out,
                    bits_out, lo_out, hi_out);
  });
}

GIS_API int gis_select_boundary_range(gis_ctx* ctx, const gis_index* ix, const double* lo,
                                      const double* hi, int64_t V, int64_t begin, int64_t end,
                                      double delta, int32_t face_points, uint8_t* out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(ix != nullptr, GIS_E_INVALID, "index is NULL");
    GIS_REQUIRE(0 <= begin && begin <= end && end <= V, GIS_E_INVALID, "cell range out of bounds");
    if (end <= begin) return;
    by_dim<BoundaryL>(ix->n, ctx, ix->dev(), lo, hi, V, begin, end, delta, (int)face_points,
                      out);
  });
}

GIS_API int gis_select_boundary(gis_ctx* ctx, const gis_index* ix, const double* lo,
                                const double* hi, int64_t V, double delta, int32_t face_points,
                                uint8_t* out) {
  return gis_select_boundary_range(ctx, ix, lo, hi, V, 0, std::max<int64_t>(V, 0), delta,
                                   face_points, out);
}

GIS_API int gis_knn(gis_ctx* ctx, const gis_index* ix, const double* lo, const double* hi,
                    int64_t V, const double* points, int64_t Q, int32_t k, int32_t exclude_point,
                    int64_t* out_idx, int32_t* out_cnt) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(ix != nullptr && ix->V == V, GIS_E_INVALID, "index does not match the cells");
    GIS_REQUIRE(k >= 1, GIS_E_INVALID, "k must be >= 1");
    if (Q <= 0) return;
    GIS_REQUIRE(V > 0, GIS_E_INVALID, "k-NN over an empty covering");
    if (k <= 32 * kMaxKpl)
      by_dim<KnnL>(ix->n, ctx, ix->dev(), lo, hi, V, points, Q, (int)k, (int)exclude_point,
                   out_idx, out_cnt);
    else
      by_dim<KnnAllL>(ix->n, ctx, lo, hi, V, points, (const int64_t*)nullptr, Q, (int)k,
                      (int)exclude_point, out_idx, out_cnt, (uint8_t*)nullptr);
  });
}

GIS_API int gis_select_neighborhood_range(gis_ctx* ctx, const gis_index* ix, const double* lo,
                                          const double* hi, int64_t V, const uint8_t* boundary,
                                          int64_t begin, int64_t end, int32_t k,
                                          int32_t exclude_boundary, uint8_t* out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(ix != nullptr && ix->V == V, GIS_E_INVALID, "index does not match the cells");
    GIS_REQUIRE(k >= 0, GIS_E_INVALID, "k must be >= 0");
    GIS_REQUIRE(0 <= begin && begin <= end && end <= V, GIS_E_INVALID, "cell range out of bounds");
    if (V <= 0) return;
    GIS_CUDA(cudaMemsetAsync(out, 0, V, ctx->stream));
    const int64_t R = end - begin;
    if (k == 0 || R == 0) return;
    int64_t* pos = (int64_t*)scratch(ctx, SC_TOFF, (R + 1) * 8);
    exclusive_scan_u8_to_i64(ctx, boundary + begin, pos, R);
    int64_t Q = 0;
    read_back(ctx, &Q, pos + R, 8);
    if (Q > 0) {
      if (k >= V - 1) {
        // every other cell is among the k nearest of any query (clamped)
        GIS_CUDA(cudaMemsetAsync(out, 1, V, ctx->stream));
      } else {
        int64_t* list = (int64_t*)scratch(ctx, SC_BIG, Q * 8);
        gather_selected_kernel<<<(unsigned)ceil_div(R, 256), 256, 0, ctx->stream>>>(
            boundary + begin, pos, R, begin, list);
        count_launch(ctx);
        if (k <= 32 * kMaxKpl)
          by_dim<NeighL>(ix->n, ctx, ix->dev(), lo, hi, V, (const int64_t*)list, Q, (int)k, out);
        else
          by_dim<KnnAllL>(ix->n, ctx, lo, hi, V, (const double*)nullptr, (const int64_t*)list, Q,
                          (int)k, 1, (int64_t*)nullptr, (int32_t*)nullptr, out);
      }
    }
    if (exclude_boundary) {
      andnot_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(out, boundary, V);
      count_launch(ctx);
    }
  });
}

GIS_API int gis_select_neighborhood(gis_ctx* ctx, const gis_index* ix, const double* lo,
                                    const double* hi, int64_t V, const uint8_t* boundary,
                                    int32_t k, uint8_t* out) {
  return gis_select_neighborhood_range(ctx, ix, lo, hi, V, boundary, 0, std::max<int64_t>(V, 0),
                                       k, 1, out);
}

GIS_API int gis_mask_andnot(gis_ctx* ctx, uint8_t* a, const uint8_t* b, int64_t V) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    if (V <= 0) return;
    andnot_kernel<<<(unsigned)ceil_div(V, 256), 256, 0, ctx->stream>>>(a, b, V);
    count_launch(ctx);
  });
}

GIS_API int gis_containment_defect_range(gis_ctx* ctx, const gis_index* prev,
                                         const double* prev_lo, const double* prev_hi,
                                         int64_t prev_V, const double* lo, const double* hi,
                                         int64_t V, int64_t begin, int64_t end, double* defect) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(prev != nullptr && prev->V == prev_V, GIS_E_INVALID,
                "index does not match the previous cells");
    GIS_REQUIRE(0 <= begin && begin <= end && end <= V, GIS_E_INVALID, "cell range out of bounds");
    *defect = 0.0;
    if (end <= begin) return;
    struct R { unsigned long long best; int neg; };
    R* r = (R*)scratch(ctx, SC_MISC2, sizeof(R));
    GIS_CUDA(cudaMemsetAsync(r, 0, sizeof(R), ctx->stream));
    by_dim<ContainL>(prev->n, ctx, prev->dev(), prev_lo, prev_hi, prev_V, lo, hi, V, begin, end,
                     &r->best, &r->neg);
    R h{};
    read_back(ctx, &h, r, sizeof(R));
    double d;
    memcpy(&d, &h.best, 8);
    *defect = h.neg ? NAN : d;
  });
}

GIS_API int gis_containment_defect(gis_ctx* ctx, const gis_index* prev, const double* prev_lo,
                                   const double* prev_hi, int64_t prev_V, const double* lo,
                                   const double* hi, int64_t V, double* defect) {
  return gis_containment_defect_range(ctx, prev, prev_lo, prev_hi, prev_V, lo, hi, V, 0,
                                      std::max<int64_t>(V, 0), defect);
}

GIS_API int gis_diameter(gis_ctx* ctx, int32_t n, const double* lo, const double* hi, int64_t V,
                         double* diameter) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    *diameter = 0.0;
    if (V <= 0) return;
    unsigned long long* b = (unsigned long long*)scratch(ctx, SC_MISC2, 8);
    GIS_CUDA(cudaMemsetAsync(b, 0, 8, ctx->stream));
    by_dim<DiamL>(n, ctx, lo, hi, V, b);
    unsigned long long h = 0;
    read_back(ctx, &h, b, 8);
    memcpy(diameter, &h, 8);
  });
}
