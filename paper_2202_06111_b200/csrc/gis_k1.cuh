// K1 kernels (sampled one-step image enclosures, cg/image.py:59-85, fused
// with the slot-rectangle epilogue that feeds K2) and the point map.  Device
// code only: gis_image.cu instantiates these for the built-in models, and
// gis_jit.cu has NVRTC instantiate them for user-defined models.
#pragma once

#include "gis_models.cuh"

namespace gis {

struct EncArgs {
  const double* lo;
  const double* hi;
  int64_t V;        // SoA stride
  int64_t c0;       // first cell
  int64_t ncells;   // cells in range (or in `cells`)
  // Graph builds with a cell list (cells reused from the previous covering
  // are not integrated, gis_build_graph_memo_begin): local cell lc is
  // cells[lc]; outputs go to pair (cells[lc] - row0) * U + ui of the row
  // range, and inv[cell - row0] is the cell's list position or -1.
  const int64_t* cells;
  const int32_t* inv;
  int64_t row0, nrows;
  double* memo;     // mode 1: padded boxes [out pair][lo n, hi n], or NULL
  int U;
  int m;
  int S;
  int L;
  const double* tables;  // device: u [U][m], frac [S][n], omf [S][n], params[64]
  double half_bloat;
  StepSizes st;
  int sub;
  int mode;  // 0 = boxes [input][cell], 1 = rects, 2 = boxes [cell][input]
  double* enc_lo;
  double* enc_hi;
  uint8_t* valid;
  int32_t* rect;  // [pair][2N]
  int32_t* cnt;   // [pair]
  GridDev grid;
  unsigned* replays;           // device counter of pairs left to the replay kernel
  double prm[GIS_MAX_PARAMS];  // model parameters (+ folds): constant-bank operands
  // Shared grid corners (graph build on a dense index, ODE models).  The
  // sample table is ordered so that samples [0, S1) are integrated per pair
  // and [S1, S) are cell corners (fractions all 0 / 1), the first of them the
  // cell's lower corner.  A corner of one cell is, bitwise, the lower corner
  // of the cell above it: corner_kernel integrates every pair's lower corner
  // once into corner0, corner_owner_kernel finds for each cell and corner the
  // cell whose lower corner it is (owner, -1: none in range, or the points
  // differ), and enclose_kernel reads those images instead of integrating
  // the corner again.  S1 == S: no sharing.
  int S1;
  double* corner0;              // [pair][N] images of the lower corners
  int32_t* owner;               // [k - 1][ncells], k = 1 .. S - S1 - 1
  unsigned long long* selfint;  // corner integrations left to enclose_kernel
  uint8_t cbits[16];            // corner bits of sample S1 + k (bit d: hi on axis d)
};

// Image of a lower corner whose integration tripped the speculative trig
// range check (a signalling NaN: arithmetic never produces one).
static constexpr unsigned long long kCornerBad = 0x7FF40BAD0BAD0BADull;

// Models whose vector field calls sin/cos take the speculative trig path.
template <int KIND>
constexpr bool kSpeculativeTrig = (KIND == GIS_PENDULUM || KIND == GIS_CARTPOLE);

// Sentinels of a pair K1 left to the replay kernel (its outputs unwritten).
static constexpr int32_t kReplayCnt = -1;    // graph build: cnt[p]
static constexpr uint8_t kReplayValid = 2;   // batch_enclosures: valid[o]

__device__ __forceinline__ int64_t cell_of(const EncArgs& a, int64_t lc) {
  return a.cells ? __ldg(a.cells + lc) : a.c0 + lc;
}
__device__ __forceinline__ int64_t out_pair(const EncArgs& a, int64_t p, int64_t cell, int ui) {
  return a.cells ? (cell - a.row0) * a.U + ui : p;
}

// Sample point lo*(1-f) + hi*f (cg/image.py:62).  The cell bounds are
// re-read (L1-resident) per sample instead of held in 2N registers.
template <int N>
__device__ __forceinline__ void sample_point(const EncArgs& a, int64_t cell, const double* sf,
                                             const double* so, int s, double (&x)[N]) {
#pragma unroll
  for (int d = 0; d < N; ++d)
    x[d] = __dadd_rn(__dmul_rn(__ldg(a.lo + d * a.V + cell), so[s * N + d]),
                     __dmul_rn(__ldg(a.hi + d * a.V + cell), sf[s * N + d]));
}

// Graph-build output of one pair's padded box: its closed slot rectangle
// and count (a NaN bound gives the empty rectangle, count 0), and the box
// itself into the memo when one is kept.
template <int N>
__device__ __forceinline__ void emit_rect(const EncArgs& a, int64_t p, const double (&elo)[N],
                                          const double (&ehi)[N]) {
  if (a.memo) {  // for the next covering's unchanged cells
    double* mo = a.memo + p * (2 * N);
#pragma unroll
    for (int d = 0; d < N; ++d) {
      mo[d] = elo[d];
      mo[N + d] = ehi[d];
    }
  }
  int32_t r[2 * N];
  int64_t count = 1;
#pragma unroll
  for (int d = 0; d < N; ++d) {
    int64_t lo_s = 1, hi_s = 0;
    if (count) {
      axis_range(a.grid, d, elo[d], ehi[d], lo_s, hi_s);
      if (lo_s > hi_s) count = 0; else count *= (hi_s - lo_s + 1);
    }
    r[d] = (int32_t)lo_s;
    r[N + d] = (int32_t)hi_s;
  }
  int32_t* dst = a.rect + p * (2 * N);
#pragma unroll
  for (int k = 0; k < 2 * N; ++k) dst[k] = r[k];
  a.cnt[p] = (int32_t)count;
}

// Padded box -> output: the enclosure (mode 0) or its closed slot rectangle
// on the grid index (mode 1, the graph build).
template <int N>
__device__ __forceinline__ void finish_pair(const EncArgs& a, int64_t p, int64_t lc, int ui,
                                            const double (&mn)[N], const double (&mx)[N],
                                            int ok_any) {
  double elo[N], ehi[N];
#pragma unroll
  for (int d = 0; d < N; ++d) {  // pad = (0.5*bloat)*(hi-lo)  (cg/image.py:82-84)
    const double pad = __dmul_rn(a.half_bloat, __dsub_rn(mx[d], mn[d]));
    elo[d] = __dsub_rn(mn[d], pad);
    ehi[d] = __dadd_rn(mx[d], pad);
  }
  if (a.mode != 1) {  // mode 0: [input][cell] (batch_enclosures); mode 2: [cell][input]
    const int64_t o = a.mode == 2 ? p : (int64_t)ui * a.ncells + lc;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      a.enc_lo[o * N + d] = elo[d];
      a.enc_hi[o * N + d] = ehi[d];
    }
    a.valid[o] = (uint8_t)ok_any;
    return;
  }
  if (!ok_any) elo[0] = __longlong_as_double(0x7ff8000000000000LL);  // NaN: meets nothing
  emit_rect<N>(a, p, elo, ehi);
}

// One sample of one pair integrated in registers (the sticky range flag of
// the speculative trig path in `bad`).
template <int KIND, int N, int INTEG>
__device__ __forceinline__ void integrate_sample(const EncArgs& a, const RegModel<KIND>& rm,
                                                 const StepSizes& st, int nsub, int64_t cell,
                                                 const double* sf, const double* so, int s,
                                                 double (&x)[N], unsigned& bad) {
  sample_point<N>(a, cell, sf, so, s, x);
  if constexpr (kSpeculativeTrig<KIND>) {
    TrigSpec spec;
    Integrator<KIND, N, INTEG>::run(x, rm, st, nsub, a.m, spec);
    bad |= spec.bad;
  } else {
    TrigExact ex;
    Integrator<KIND, N, INTEG>::run(x, rm, st, nsub, a.m, ex);
  }
}

template <int INTEG>
constexpr bool kSharesCorners = (INTEG == GIS_EULER || INTEG == GIS_RK4);

template <int N>
__device__ __forceinline__ void fold_sample(const double (&x)[N], double (&mn)[N],
                                            double (&mx)[N], int& ok_any) {
  bool fin = true;
#pragma unroll
  for (int d = 0; d < N; ++d) fin = fin && isfinite(x[d]);
  if (fin) {  // finite = all coordinates finite; valid = some finite sample
    ok_any = 1;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      // plain compare-selects: no operand is NaN here (fmin / fmax spend
      // ~8 instructions each on NaN quieting)
      mn[d] = x[d] < mn[d] ? x[d] : mn[d];
      mx[d] = x[d] > mx[d] ? x[d] : mx[d];
    }
  }
}

// Hot kernel.  Trig-field models integrate with TrigSpec: the polynomial
// sin/cos and the branch-free division unconditionally, a sticky flag for
// any operand outside their ranges.  A pair with a flagged sample is left to
// enclose_replay_kernel (sentinel output + counter) instead of replaying
// in-line, so the range-checked slow paths -- and the registers their calls
// need -- are not part of this kernel (cart-pole 124 -> 88 registers).
// Resident 256-thread blocks per SM the register budget is cut for (the
// occupancy of this latency-bound fp64 kernel): 4 (<= 64 registers) by
// default; 3 (<= 80) for the fields that spill at 64.  Cart-pole RK4 holds
// 94-127 registers unconstrained (2 blocks); with shared corners (fewer
// integrations per pair, more of the pair's fixed work) 4 blocks at 64 with
// spills beats 3 at 80 (config 5 enclose_kernel 67.1 -> 65.6 ms, 2 blocks
// 70.3; r02be), where before them 3 blocks won (243 -> 212 ms).
template <int KIND, int INTEG>
struct K1MinBlocks { static constexpr int value = 4; };
#ifndef GIS_CARTPOLE_MINBLOCKS
#define GIS_CARTPOLE_MINBLOCKS 4
#endif
template <int INTEG>
struct K1MinBlocks<GIS_CARTPOLE, INTEG> { static constexpr int value = GIS_CARTPOLE_MINBLOCKS; };
template <int INTEG>
struct K1MinBlocks<GIS_CSTR, INTEG> { static constexpr int value = 3; };
template <int INTEG>
struct K1MinBlocks<GIS_CSTR_DIMLESS, INTEG> { static constexpr int value = 3; };
template <int INTEG>
struct K1MinBlocks<GIS_AFFINE, INTEG> { static constexpr int value = 3; };
template <int INTEG>  // user fields (gis_jit.cu): room for arbitrary code
struct K1MinBlocks<GIS_JIT, INTEG> { static constexpr int value = 2; };
#ifdef GIS_PENDULUM_MINBLOCKS  // experiments (build.py --variant)
template <>
struct K1MinBlocks<GIS_PENDULUM, GIS_RK4> { static constexpr int value = GIS_PENDULUM_MINBLOCKS; };
#endif
#ifdef GIS_LORENZ_MINBLOCKS
template <>
struct K1MinBlocks<GIS_LORENZ, GIS_RK4> { static constexpr int value = GIS_LORENZ_MINBLOCKS; };
#endif

template <int KIND, int N, int INTEG>
__global__ void __launch_bounds__(256, K1MinBlocks<KIND, INTEG>::value)
    enclose_kernel(const __grid_constant__ EncArgs a) {
  extern __shared__ double sm[];
  const int nt = a.U * a.m + 2 * a.S * N;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) sm[i] = a.tables[i];
  __syncthreads();
  const double* su = sm;
  const double* sf = sm + a.U * a.m;
  const double* so = sf + a.S * N;

  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int L = a.L;
  const int64_t p = g / L;
  const int sub = (int)(g & (L - 1));
  const int64_t npairs = a.ncells * a.U;
  if (p >= npairs) return;  // whole L-lane groups exit together
  const int64_t lc = p / a.U;
  const int ui = (int)(p - lc * a.U);
  const int64_t cell = cell_of(a, lc);
  RegModel<KIND> rm;  // input in registers, parameters in the kernel's param space
  rm.load(a.prm, su + ui * a.m, a.m);
  const StepSizes st = a.st;
  const int nsub = a.sub;

  double mn[N], mx[N];
#pragma unroll
  for (int d = 0; d < N; ++d) {
    mn[d] = INFINITY;
    mx[d] = -INFINITY;
  }
  int ok_any = 0;
  unsigned bad = 0u;
  for (int s = sub; s < a.S1; s += L) {
    double x[N];
    integrate_sample<KIND, N, INTEG>(a, rm, st, nsub, cell, sf, so, s, x, bad);
    fold_sample<N>(x, mn, mx, ok_any);
  }
  if constexpr (kSharesCorners<INTEG>) {
    const int nc = a.S - a.S1;  // 0 unless sharing; at most 2^N
    if (nc > 0) {
      // unrolled over the 2^N possible corners so that the owner and image
      // loads of different corners are independent (issued back to back,
      // not one memory round trip after another)
      unsigned miss = 0u;
#pragma unroll
      for (int k = 0; k < (1 << N); ++k) {
        if (k < nc && (k & (L - 1)) == sub) {
          int64_t src = p;
          if (k > 0 && a.cbits[k] != 0u) {
            const int32_t o = __ldg(a.owner + (int64_t)(k - 1) * a.ncells + lc);
            src = (int64_t)o * a.U + ui;
            if (o < 0) {
              miss |= 1u << k;
              continue;
            }
          }
          double x[N];
#pragma unroll
          for (int d = 0; d < N; ++d) x[d] = __ldg(a.corner0 + src * N + d);
          if constexpr (kSpeculativeTrig<KIND>)
            bad |= (unsigned)((unsigned long long)__double_as_longlong(x[0]) == kCornerBad);
          fold_sample<N>(x, mn, mx, ok_any);
        }
      }
      while (miss) {  // no owner (root's upper faces, coarser neighbour, range edge)
        const int k = __ffs(miss) - 1;
        miss &= miss - 1u;
        double x[N];
        integrate_sample<KIND, N, INTEG>(a, rm, st, nsub, cell, sf, so, a.S1 + k, x, bad);
        fold_sample<N>(x, mn, mx, ok_any);
      }
    }
  }
  if (L > 1) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned gmask =
        (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(unsigned)(L - 1)));
    for (int off = L >> 1; off > 0; off >>= 1) {
#pragma unroll
      for (int d = 0; d < N; ++d) {
        const double omn = __shfl_xor_sync(gmask, mn[d], off, L);
        const double omx = __shfl_xor_sync(gmask, mx[d], off, L);
        mn[d] = omn < mn[d] ? omn : mn[d];
        mx[d] = omx > mx[d] ? omx : mx[d];
      }
      ok_any |= __shfl_xor_sync(gmask, ok_any, off, L);
      if constexpr (kSpeculativeTrig<KIND>) bad |= __shfl_xor_sync(gmask, bad, off, L);
    }
  }
  if (sub != 0) return;
  const int64_t po = out_pair(a, p, cell, ui);
  if (kSpeculativeTrig<KIND> && bad) {  // rare: far outside X
    if (a.mode == 0) a.valid[(int64_t)ui * a.ncells + lc] = kReplayValid;
    else if (a.mode == 2) a.valid[p] = kReplayValid;
    else a.cnt[po] = kReplayCnt;
    atomicAdd(a.replays, 1u);
    return;
  }
  finish_pair<N>(a, po, lc, ui, mn, mx, ok_any);
}

// Lower corner (sample S1) of every pair, integrated once: the images the
// pair and its grid neighbours below read (EncArgs::corner0).
template <int KIND, int N, int INTEG>
__global__ void __launch_bounds__(256, K1MinBlocks<KIND, INTEG>::value)
    corner_kernel(const __grid_constant__ EncArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.ncells * a.U) return;
  const int64_t lc = p / a.U;
  const int ui = (int)(p - lc * a.U);
  const double* sf = a.tables + a.U * a.m;
  const double* so = sf + a.S * N;
  RegModel<KIND> rm;
  rm.load(a.prm, a.tables + ui * a.m, a.m);
  double x[N];
  unsigned bad = 0u;
  integrate_sample<KIND, N, INTEG>(a, rm, a.st, a.sub, cell_of(a, lc), sf, so, a.S1, x, bad);
  if (kSpeculativeTrig<KIND> && bad) x[0] = __longlong_as_double((long long)kCornerBad);
#pragma unroll
  for (int d = 0; d < N; ++d) a.corner0[p * N + d] = x[d];
}

// For each cell in range and each corner sample k >= 1: the cell (local
// index) whose lower corner is that corner -- the slot above the corner
// along every axis, looked up in the slot table -- accepted only when its
// lower-corner sample point equals this cell's corner sample point bit for
// bit (so the two integrations are the same computation).  Counts the
// corners left without an owner (integrated by enclose_kernel).
template <int N>
__global__ void __launch_bounds__(256) corner_owner_kernel(const __grid_constant__ EncArgs a) {
  const int64_t lc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const GridDev& g = a.grid;
  unsigned misses = 0;
  if (lc < a.ncells) {
    const int64_t cell = cell_of(a, lc);
    const double* sf = a.tables + a.U * a.m;
    const double* so = sf + a.S * N;
    int64_t slo[N], shi[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
      slo[d] = __ldg(g.cell_slo + d * g.V + cell);
      shi[d] = __ldg(g.cell_shi + d * g.V + cell);
    }
    const int nc = a.S - a.S1;
#pragma unroll
    for (int k = 1; k < (1 << N); ++k) {
      if (k >= nc) break;
      const unsigned c = a.cbits[k];
      int32_t own = -1;
      if (c != 0u) {
        bool in = true;
        int64_t s = 0;
#pragma unroll
        for (int d = 0; d < N; ++d) {
          const int64_t sd = ((c >> d) & 1u) ? shi[d] + 1 : slo[d];
          in = in && sd < g.ns[d];
          s += sd * g.stride[d];
        }
        const int64_t q = in ? (int64_t)__ldg(g.slot + s) : -1;
        // q's position in this launch: its local index, or -1
        int64_t ql = -1;
        if (a.cells) {
          if (q >= a.row0 && q < a.row0 + a.nrows) ql = __ldg(a.inv + (q - a.row0));
        } else if (q >= a.c0 && q < a.c0 + a.ncells) {
          ql = q - a.c0;
        }
        if (ql >= 0) {
          double mine[N], theirs[N];
          sample_point<N>(a, cell, sf, so, a.S1 + k, mine);
          sample_point<N>(a, q, sf, so, a.S1, theirs);
          bool same = true;
#pragma unroll
          for (int d = 0; d < N; ++d)
            same = same && __double_as_longlong(mine[d]) == __double_as_longlong(theirs[d]);
          if (same) own = (int32_t)ql;
        }
        misses += own < 0;
      }
      a.owner[(int64_t)(k - 1) * a.ncells + lc] = own;
    }
  }
  // corner integrations enclose_kernel will do: misses x inputs
  for (int off = 16; off > 0; off >>= 1) misses += __shfl_xor_sync(0xffffffffu, misses, off);
  if ((threadIdx.x & 31) == 0 && misses) atomicAdd(a.selfint, (unsigned long long)misses * a.U);
}

// Pairs of cells unchanged since the previous covering of an adaptive run
// (origin[cell] = the cell's index there, inside the rows the previous
// build kept boxes for): the padded box that build kept becomes this
// build's slot rectangle -- on the new grid -- with no integration.  The
// box depends only on the cell, the input, the samples and the model, so
// it is the box this build would compute.
// With rects == 0 the rows of these cells come from the previous graph
// (incr_rows_kernel): the pairs only get count 0 here, and their boxes are
// copied on for the next covering.
template <int N>
__global__ void __launch_bounds__(256) memo_rect_kernel(const __grid_constant__ EncArgs a,
                                                        const int64_t* __restrict__ origin,
                                                        const double* __restrict__ memo_in,
                                                        int64_t memo_begin, int64_t memo_rows,
                                                        int rects) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.nrows * a.U) return;
  const int64_t r = t / a.U;
  const int ui = (int)(t - r * a.U);
  const int64_t o = __ldg(origin + a.row0 + r) - memo_begin;
  if (o < 0 || o >= memo_rows) return;  // a new cell: enclose_kernel integrates it
  const double* b = memo_in + (o * a.U + ui) * (2 * N);
  if (!rects) {
    a.cnt[t] = 0;
    if (a.memo) {
#pragma unroll
      for (int d = 0; d < 2 * N; ++d) a.memo[t * (2 * N) + d] = __ldg(b + d);
    }
    return;
  }
  double elo[N], ehi[N];
#pragma unroll
  for (int d = 0; d < N; ++d) {
    elo[d] = __ldg(b + d);
    ehi[d] = __ldg(b + N + d);
  }
  emit_rect<N>(a, t, elo, ehi);
}

// The pairs K1 left behind, recomputed whole with TrigExact (range-checked
// sin/cos, IEEE division outside div_newton's range; identical to TrigSpec
// on in-range operands).  Exits at once when K1 flagged nothing (the
// BASELINE configs); otherwise scans the sentinels.
template <int KIND, int N, int INTEG>
__global__ void __launch_bounds__(256) enclose_replay_kernel(const __grid_constant__ EncArgs a) {
  if (*(volatile const unsigned*)a.replays == 0u) return;
  const double* su = a.tables;
  const double* sf = su + a.U * a.m;
  const double* so = sf + a.S * N;
  const int64_t npairs = a.ncells * a.U;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lc = p / a.U;
    const int ui = (int)(p - lc * a.U);
    const int64_t cell = cell_of(a, lc);
    const int64_t po = out_pair(a, p, cell, ui);
    const bool flagged = a.mode == 0   ? a.valid[(int64_t)ui * a.ncells + lc] == kReplayValid
                         : a.mode == 2 ? a.valid[p] == kReplayValid
                                       : a.cnt[po] == kReplayCnt;
    if (!flagged) continue;
    RegModel<KIND> rm;
    rm.load(a.prm, su + ui * a.m, a.m);
    double mn[N], mx[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
      mn[d] = INFINITY;
      mx[d] = -INFINITY;
    }
    int ok_any = 0;
    for (int s = 0; s < a.S; ++s) {
      double x[N];
      sample_point<N>(a, cell, sf, so, s, x);
      TrigExact ex;
      Integrator<KIND, N, INTEG>::run(x, rm, a.st, a.sub, a.m, ex);
      fold_sample<N>(x, mn, mx, ok_any);
    }
    finish_pair<N>(a, po, lc, ui, mn, mx, ok_any);
  }
}

// ------------------------------------------------------------ map points ---
struct MapArgs {
  const double* x;
  double* out;
  int64_t N;
  const double* tables;  // u[m], params[64]
  int m;
  StepSizes st;
  int sub;
};

template <int KIND, int N, int INTEG>
__global__ void map_kernel(MapArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  double x[N];
#pragma unroll
  for (int d = 0; d < N; ++d) x[d] = a.x[i * N + d];
  TrigExact ex;
  Integrator<KIND, N, INTEG>::run(x, a.tables, a.tables + a.m, a.st, a.sub, a.m, ex);
#pragma unroll
  for (int d = 0; d < N; ++d) a.out[i * N + d] = x[d];
}

}  // namespace gis
