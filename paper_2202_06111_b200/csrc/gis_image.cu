// K1: sampled one-step image enclosures (cg/image.py:59-85) fused with the
// slot-rectangle computation that feeds the CSR build (K2).
//
// Work unit: one (cell, input) pair, processed by L lanes (L = 1..32, a power
// of two) that split the S samples; each lane integrates its samples in
// registers (fp64, exact reference operation order), keeps a masked min/max,
// and the L partial boxes are combined with xor-shuffles.  The pair's first
// lane pads the box by (0.5*bloat)*(hi-lo) and either stores the box
// (batch_enclosures) or converts it into the closed slot rectangle of the
// grid index (graph build).
#include "gis_k1.cuh"

#include <cmath>
#include <cstdlib>
#include <vector>

namespace gis {

template <int KIND, int N, int INTEG>
struct LaunchEnclose {
  // one cell range [a.c0, a.c0 + a.ncells): corner owners and lower corners
  // (owners are looked for inside the range only), then the pairs
  static void part(gis_ctx* ctx, const EncArgs& a) {
    const int64_t threads = a.ncells * a.U * a.L;
    if (threads == 0) return;
    const int bs = 256;
    if constexpr (kSharesCorners<INTEG>) {
      if (a.S1 < a.S) {  // owners of the shared corners, then the lower corners
        corner_owner_kernel<N><<<(unsigned)ceil_div(a.ncells, bs), bs, 0, ctx->stream>>>(a);
        count_launch(ctx);
        corner_kernel<KIND, N, INTEG>
            <<<(unsigned)ceil_div(a.ncells * a.U, bs), bs, 0, ctx->stream>>>(a);
        count_launch(ctx);
      }
    }
    const size_t smem = (size_t)(a.U * a.m + 2 * a.S * N) * sizeof(double);
    if (smem > 48 * 1024)
      GIS_CUDA(cudaFuncSetAttribute(enclose_kernel<KIND, N, INTEG>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    enclose_kernel<KIND, N, INTEG>
        <<<(unsigned)ceil_div(threads, bs), bs, smem, ctx->stream>>>(a);
    count_launch(ctx);
  }

  static void go(gis_ctx* ctx, EncArgs& a) {
    const int64_t threads = a.ncells * a.U * a.L;
    if (threads == 0) {
      inputs_wait_all(ctx);
      return;
    }
    if (ctx->in_evts.empty() || a.cells || a.memo || a.mode != 1) {
      inputs_wait_all(ctx);
      part(ctx, a);
    } else {
      // cell bounds arriving in chunks (gis_ctx_input_chunks): each chunk's
      // cells start as soon as its copy is in, overlapping the next copies
      const int n = N;
      const int nc = a.S - a.S1;
      int64_t s0 = a.c0;
      const int64_t end = a.c0 + a.ncells;
      for (size_t c = 0; c < ctx->in_evts.size() && s0 < end; ++c) {
        GIS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->in_evts[c], 0));
        const int64_t s1 = c + 1 == ctx->in_evts.size() ? end : std::min(ctx->in_ends[c], end);
        if (s1 <= s0) continue;
        EncArgs b = a;
        const int64_t off = s0 - a.c0;
        b.c0 = s0;
        b.ncells = s1 - s0;
        b.row0 = s0;
        b.nrows = s1 - s0;
        b.rect = a.rect + off * a.U * 2 * n;
        b.cnt = a.cnt + off * a.U;
        if (a.S1 < a.S) {
          b.corner0 = a.corner0 + off * a.U * n;
          b.owner = a.owner + (int64_t)(nc - 1) * off;
        }
        part(ctx, b);
        s0 = s1;
      }
      inputs_wait_all(ctx);
    }
    if constexpr (kSpeculativeTrig<KIND>) {
      const int64_t npairs = a.ncells * a.U;
      const int64_t blocks = std::min<int64_t>(ceil_div(npairs, 256), (int64_t)ctx->num_sms * 8);
      enclose_replay_kernel<KIND, N, INTEG><<<(unsigned)blocks, 256, 0, ctx->stream>>>(a);
      count_launch(ctx);
    }
  }
};

void jit_enclose(gis_ctx* ctx, const gis_model& m, EncArgs& a);  // gis_jit.cu
void jit_map(gis_ctx* ctx, const gis_model& m, MapArgs& a);

// lanes per pair: enough threads to fill the chip, samples split evenly
static int choose_lanes(int64_t pairs, int S, int num_sms) {
  const int64_t want = (int64_t)num_sms * 2048 * 2;
  int L = 1;
  while (L < 32 && pairs * L < want && L < S) L <<= 1;
  return L;
}

// Shared corners (EncArgs::S1): the sample order that puts the samples
// integrated per pair first, then the cell corners, the lower corner (all
// fractions 0) leading them.  Empty when the table has no lower corner, no
// other corner, or more corner samples than a cell has corners.
static std::vector<int> corner_order(const double* frac, int S, int n, int* S1, uint8_t* cbits) {
  std::vector<int> rest, corners, bits(S, -1);
  for (int s = 0; s < S; ++s) {
    int b = 0;
    for (int d = 0; d < n && b >= 0; ++d) {
      const double f = frac[(size_t)s * n + d];
      if (f == 1.0) b |= 1 << d;
      else if (!(f == 0.0 && !std::signbit(f))) b = -1;
    }
    bits[s] = b;
  }
  int lower = -1;
  for (int s = 0; s < S; ++s)
    if (bits[s] == 0) { lower = s; break; }
  for (int s = 0; s < S; ++s) {
    if (s == lower) continue;
    (bits[s] >= 0 ? corners : rest).push_back(s);
  }
  if (lower < 0 || corners.empty() || corners.size() + 1 > ((size_t)1 << n)) return {};
  std::vector<int> order(rest);
  order.push_back(lower);
  order.insert(order.end(), corners.begin(), corners.end());
  *S1 = (int)rest.size();
  for (size_t k = 0; k < corners.size() + 1; ++k) cbits[k] = (uint8_t)bits[order[*S1 + k]];
  return order;
}

static const double* upload_tables(gis_ctx* ctx, const gis_model* model, const double* u,
                                   int U, const double* frac, int S) {
  const int n = model->n, m = model->m;
  std::vector<double> t((size_t)U * m + 2 * (size_t)S * n);
  size_t o = 0;
  for (int i = 0; i < U * m; ++i) t[o++] = u[i];
  for (int i = 0; i < S * n; ++i) t[o++] = frac[i];
  for (int i = 0; i < S * n; ++i) t[o++] = 1.0 - frac[i];  // numpy's (1.0 - frac)
  return (const double*)upload(ctx, SC_PARAMS, t.data(), t.size() * sizeof(double));
}

static void check_model(const gis_model* model) {
  GIS_REQUIRE(model != nullptr, GIS_E_INVALID, "model is NULL");
  GIS_REQUIRE(model->n >= 1 && model->n <= GIS_MAX_DIM, GIS_E_INVALID, "model n out of range");
  GIS_REQUIRE(model->m >= 1 && model->m <= GIS_MAX_DIM, GIS_E_INVALID, "model m out of range");
  if (model->integrator == GIS_EULER || model->integrator == GIS_RK4) {
    GIS_REQUIRE(model->substeps >= 1, GIS_E_INVALID, "substeps must be >= 1");
    GIS_REQUIRE(model->h > 0, GIS_E_INVALID, "step size must be positive");
  }
}

// Enclosures of cells [c0, c0+ncells) for all U inputs; mode 1 emits slot
// rectangles against `grid` (used by the graph build).
void enclose(gis_ctx* ctx, const gis_model* model, const double* lo, const double* hi,
             int64_t V, int64_t c0, int64_t ncells, const double* u, int U,
             const double* frac, int S, double bloat, int mode, double* enc_lo,
             double* enc_hi, uint8_t* valid, int32_t* rect, int32_t* cnt,
             const GridDev* grid, const EncList* list) {
  check_model(model);
  GIS_REQUIRE(U >= 1 && S >= 1, GIS_E_INVALID, "need at least one input and one sample");
  GIS_REQUIRE((int64_t)U * model->m + 2 * (int64_t)S * model->n <= 12000, GIS_E_INVALID,
              "input/sample tables too large");
  GIS_REQUIRE(bloat >= 0, GIS_E_INVALID, "bloat must be nonnegative");
  // cell bounds arriving in chunks are only split over by a plain graph
  // build (LaunchEnclose::go); everything else waits for all of them
  if (!(mode == 1 && !list && model->kind != GIS_JIT)) inputs_wait_all(ctx);
  EncArgs a{};
  a.lo = lo;
  a.hi = hi;
  a.V = V;
  a.c0 = c0;
  a.ncells = ncells;
  a.row0 = c0;
  a.nrows = ncells;
  const int64_t rows = ncells;
  if (list) {  // graph build keeping boxes; with an origin, only new cells integrate
    a.memo = list->memo_out;
    if (list->origin) {
      a.cells = list->cells;
      a.inv = list->inv;
      a.ncells = ncells = list->nlist;
    }
  }
  a.U = U;
  a.m = model->m;
  a.S = S;
  a.S1 = S;
  // graph build on a dense index with an ODE model: cell corners are
  // integrated once per grid vertex instead of once per cell touching it
  // (GIS_K1_SHARE=0 turns it off, for A/B runs)
  std::vector<double> permuted;
  const char* share_env = getenv("GIS_K1_SHARE");
  const bool ode = model->integrator == GIS_EULER || model->integrator == GIS_RK4;
  if (mode == 1 && grid && !grid->sparse && ode && model->kind != GIS_JIT && ncells > 0 &&
      !(share_env && share_env[0] == '0') &&
      (double)ncells * U * model->n * 8 <= 16e9) {
    const std::vector<int> order = corner_order(frac, S, model->n, &a.S1, a.cbits);
    if (!order.empty()) {
      const int n = model->n;
      permuted.resize((size_t)S * n);
      for (int s = 0; s < S; ++s)
        for (int d = 0; d < n; ++d) permuted[(size_t)s * n + d] = frac[(size_t)order[s] * n + d];
      frac = permuted.data();
      const int nc = S - a.S1;
      a.corner0 = (double*)scratch(ctx, SC_CORNER, (size_t)ncells * U * n * 8);
      a.owner = (int32_t*)scratch(ctx, SC_OWNER, std::max<size_t>((size_t)(nc - 1) * ncells * 4, 4));
      if (!ctx->k1_self) {
        GIS_CUDA(cudaMalloc(&ctx->k1_self, sizeof(unsigned long long)));
        GIS_CUDA(cudaMemsetAsync(ctx->k1_self, 0, sizeof(unsigned long long), ctx->stream));
      }
      a.selfint = ctx->k1_self;
    }
  }
  ctx->k1_logical += rows * U * S;
  ctx->k1_planned += ncells * U * (a.S1 < S ? a.S1 + 1 : S);
  a.L = choose_lanes(ncells * U, a.S1, ctx->num_sms);
  a.tables = upload_tables(ctx, model, u, U, frac, S);
  model_params(*model, a.prm);
  a.replays = (unsigned*)scratch(ctx, SC_REPLAY, 16);
  GIS_CUDA(cudaMemsetAsync(a.replays, 0, sizeof(unsigned), ctx->stream));
  a.half_bloat = 0.5 * bloat;
  a.st = StepSizes::of(model->h);
  a.sub = model->substeps;
  a.mode = mode;
  a.enc_lo = enc_lo;
  a.enc_hi = enc_hi;
  a.valid = valid;
  a.rect = rect;
  a.cnt = cnt;
  if (grid) a.grid = *grid;
  if (list && list->origin && rows > 0) {  // reused boxes: no integration
    const unsigned blocks = (unsigned)ceil_div(rows * U, 256);
    auto go = [&](auto kernel) {
      kernel<<<blocks, 256, 0, ctx->stream>>>(a, list->origin, list->memo_in, list->memo_begin,
                                              list->memo_rows, list->incr ? 0 : 1);
    };
    switch (model->n) {
      case 1: go(memo_rect_kernel<1>); break;
      case 2: go(memo_rect_kernel<2>); break;
      case 3: go(memo_rect_kernel<3>); break;
      default: go(memo_rect_kernel<4>); break;
    }
    count_launch(ctx);
  }
  if (model->kind == GIS_JIT) jit_enclose(ctx, *model, a);
  else dispatch_model<LaunchEnclose>(*model, ctx, a);
}

template <int KIND, int N, int INTEG>
struct LaunchMap {
  static void go(gis_ctx* ctx, MapArgs& a) {
    if (a.N == 0) return;
    map_kernel<KIND, N, INTEG><<<(unsigned)ceil_div(a.N, 128), 128, 0, ctx->stream>>>(a);
    count_launch(ctx);
  }
};

}  // namespace gis

using namespace gis;

GIS_API int gis_map_points(gis_ctx* ctx, const gis_model* model, const double* x, int64_t N,
                           const double* u, double* out) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    check_model(model);
    GIS_REQUIRE(N >= 0, GIS_E_INVALID, "N must be >= 0");
    std::vector<double> t(model->m + GIS_MAX_PARAMS);
    for (int i = 0; i < model->m; ++i) t[i] = u[i];
    model_params(*model, t.data() + model->m);
    MapArgs a{};
    a.x = x;
    a.out = out;
    a.N = N;
    a.tables = (const double*)upload(ctx, SC_PARAMS, t.data(), t.size() * sizeof(double));
    a.m = model->m;
    a.st = StepSizes::of(model->h);
    a.sub = model->substeps;
    if (model->kind == GIS_JIT) jit_map(ctx, *model, a);
    else dispatch_model<LaunchMap>(*model, ctx, a);
  });
}

GIS_API int gis_batch_enclosures(gis_ctx* ctx, const gis_model* model, const double* lo,
                                 const double* hi, int64_t B, const double* u, int32_t U,
                                 const double* frac, int32_t S, double bloat, double* enc_lo,
                                 double* enc_hi, uint8_t* valid) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(B >= 0, GIS_E_INVALID, "B must be >= 0");
    gis::enclose(ctx, model, lo, hi, B, 0, B, u, U, frac, S, bloat, 0, enc_lo, enc_hi, valid,
                 nullptr, nullptr, nullptr, nullptr);
  });
}
