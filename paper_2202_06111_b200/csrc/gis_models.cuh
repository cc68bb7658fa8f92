// Device vector fields / maps and their discretisations.
//
// This translation-unit family is compiled with -fmad=false: every + - * /
// below is a separately rounded IEEE operation evaluated left to right, in
// the operation order of the model definitions in
// paper_2202_06111_b200/system.py (and of the numpy step functions the
// reference evaluates through its SystemModel plugin API,
// cg/system.py:52-75).  sin/cos/exp are CUDA's double-precision libm
// (<= 2 ulp) or the polynomial fast paths of gis_math.cuh (<= 2 ulp), the
// only source of difference from numpy.
#pragma once

#ifdef __CUDACC_RTC__
#include "gis_device.cuh"
#else
#include "gis_internal.cuh"
#endif
#include "gis_math.cuh"

namespace gis {

// Transcendental providers for the vector fields.
//   TrigExact : gis_math.cuh's range-checked fast paths (polynomial in range,
//               CUDA libm otherwise); a branch + reconvergence per call.
//   TrigSpec  : the polynomial unconditionally, no branch; a sticky flag
//               records any argument outside the polynomial's range.  The
//               caller replays a flagged sample with TrigExact, so results
//               are identical to TrigExact's.
// Both also provide the fused fields' division: div_newton (<= 1 ulp) on
// its range -- TrigSpec unconditionally with a range flag, TrigExact with
// IEEE `/` outside the range.
struct TrigExact {
  __device__ __forceinline__ double sin(double x) { return fast_sin(x); }
  // identical to TrigSpec's division on its range, IEEE `/` outside it
  __device__ __forceinline__ double div(double n, double d) {
    return div_in_range(n, d) ? div_newton(n, d) : n / d;
  }
  __device__ __forceinline__ void sincos(double x, double* s, double* c) {
    fast_sincos(x, s, c);
  }
  __device__ __forceinline__ void sincos_small(double x, double* s, double* c) {
    fast_sincos_small(x, s, c);
  }
};

struct TrigSpec {
  unsigned bad = 0u;
  __device__ __forceinline__ double sin(double x) {
    bad |= !abs_below(x, kSinLimitHi);
    return sin_poly(x);
  }
  __device__ __forceinline__ void sincos(double x, double* s, double* c) {
    bad |= !abs_below(x, kCosLimitHi);
    *s = sin_poly(x);
    *c = cos_poly(x);
  }
  __device__ __forceinline__ void sincos_small(double x, double* s, double* c) {
    bad |= !abs_below(x, kSmallLimitHi);
    sincos_small_poly(x, s, c);
  }
  __device__ __forceinline__ double div(double n, double d) {
    bad |= !div_in_range(n, d);
    return div_newton(n, d);
  }
};

template <int KIND, int N>
struct Field;  // ODE right-hand sides: f = F(x, u)

// pendulum (BASELINE configs 1-2): params a, b
template <>
struct Field<GIS_PENDULUM, 2> {
  template <class Tr, bool FUSED = true>
  static __device__ __forceinline__ void eval(const double (&x)[2], const double* u,
                                              const double* P, double (&f)[2], Tr& tr) {
    const double a = P[0], b = P[1];
    f[0] = x[1];
    if constexpr (FUSED) {
      // ((-a) sin x1 - b x2) + u with two roundings: the damping + input term
      // is formed off the sin's dependency chain and the sin enters last
      f[1] = fma(-a, tr.sin(x[0]), fma(-b, x[1], u[0]));
    } else {  // the reference order, one rounding per operation
      f[1] = ((-a) * tr.sin(x[0]) - b * x[1]) + u[0];
    }
  }
};

// CSTR Table 2 (cg/system.py:148-166): params qV, c_Af, T_f, -E/R, k0, c1, c2
template <>
struct Field<GIS_CSTR, 2> {
  template <class Tr, bool FUSED = true>
  static __device__ __forceinline__ void eval(const double (&x)[2], const double* u,
                                              const double* P, double (&f)[2], Tr& tr) {
    const double ca = x[0], temp = x[1];
    const double rate = P[4] * exp(P[3] / temp) * ca;
    f[0] = P[0] * (P[1] - ca) - rate;
    f[1] = P[0] * (P[2] - temp) + P[5] * rate + P[6] * (u[0] - temp);
  }
};

// dimensionless CSTR (BASELINE config 3): params Da, gamma, B, beta
template <>
struct Field<GIS_CSTR_DIMLESS, 2> {
  template <class Tr, bool FUSED = true>
  static __device__ __forceinline__ void eval(const double (&x)[2], const double* u,
                                              const double* P, double (&f)[2], Tr& tr) {
    const double t = (P[0] * (1.0 - x[0])) * exp(x[1] / (1.0 + x[1] / P[1]));
    f[0] = (-x[0]) + t;
    f[1] = ((-x[1]) + P[2] * t) - P[3] * (x[1] - u[0]);
  }
};

// controlled Lorenz (BASELINE config 4): params sigma, rho, beta
template <>
struct Field<GIS_LORENZ, 3> {
  template <class Tr, bool FUSED = true>
  static __device__ __forceinline__ void eval(const double (&x)[3], const double* u,
                                              const double* P, double (&f)[3], Tr& tr) {
    f[0] = P[0] * (x[1] - x[0]);
    if constexpr (FUSED) {
      f[1] = fma(x[0], P[1] - x[2], -x[1]) + u[0];
      f[2] = fma(x[0], x[1], -(P[2] * x[2]));
    } else {
      f[1] = (x[0] * (P[1] - x[2]) - x[1]) + u[0];
      f[2] = x[0] * x[1] - P[2] * x[2];
    }
  }
};

// cart-pole, gym form (BASELINE config 5): params g, mp, l, M, pml, 4/3, 1/M,
// and host-folded pml/M, l*4/3, l*mp/M (system.py CartPoleStep.param_vector)
template <>
struct Field<GIS_CARTPOLE, 4> {
  template <class Tr, bool FUSED = true>
  static __device__ __forceinline__ void eval(const double (&x)[4], const double* u,
                                              const double* P, double (&f)[4], Tr& tr) {
    double s, c;
    // theta stays within |theta| < 0.375 over a step from X (|theta| <= 0.21):
    // the small-angle pair, 4 fp64 instructions fewer per evaluation
    tr.sincos_small(x[2], &s, &c);
    const double om = x[3];
    double temp, thacc;
    f[0] = x[1];
    if constexpr (FUSED) {
      // temp = (F + pml w^2 sin th) / M; u/M is loop-invariant per thread
      temp = fma(P[7] * (om * om), s, u[0] * P[6]);
      // l (4/3 - mp cos^2 / M) = l*4/3 - (l mp/M) cos^2: one fma
      thacc = tr.div(fma(P[0], s, -(c * temp)), fma(-P[9], c * c, P[8]));
      f[1] = fma(-(P[7] * thacc), c, temp);
    } else {  // the reference order (oracle/gis_oracle.py _rhs_cartpole)
      temp = (u[0] + (P[4] * (om * om)) * s) / P[3];
      thacc = (P[0] * s - c * temp) / (P[2] * (P[5] - (P[1] * (c * c)) / P[3]));
      f[1] = temp - ((P[4] * thacc) * c) / P[3];
    }
    f[2] = om;
    f[3] = thacc;
  }
};

template <int KIND, int N>
struct Map;  // direct maps x+ = G(x, u)

template <int N>
struct Map<GIS_IDENTITY, N> {  // cg/system.py:233-235
  static __device__ __forceinline__ void eval(double (&x)[N], const double*, const double*,
                                              int) {}
};

template <int N>
struct Map<GIS_SHIFT, N> {  // cg/system.py:247-252
  static __device__ __forceinline__ void eval(double (&x)[N], const double*,
                                              const double* P, int) {
#pragma unroll
    for (int d = 0; d < N; ++d) x[d] = x[d] + P[0];
  }
};

template <int N>
struct Map<GIS_LINEAR, N> {  // cg/system.py:188-196: a*x + u0
  static __device__ __forceinline__ void eval(double (&x)[N], const double* u,
                                              const double* P, int) {
#pragma unroll
    for (int d = 0; d < N; ++d) x[d] = P[0] * x[d] + u[0];
  }
};

template <int N>
struct Map<GIS_AFFINE, N> {  // ((sum_k x_k A_jk) + (sum_l u_l B_jl)) + c_j
  static __device__ __forceinline__ void eval(double (&x)[N], const double* u,
                                              const double* P, int m) {
    const double* A = P;
    const double* B = P + N * N;
    const double* c = B + N * m;
    double y[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double ax = x[0] * A[j * N];
#pragma unroll
      for (int k = 1; k < N; ++k) ax = ax + x[k] * A[j * N + k];
      double bu = u[0] * B[j * m];
      for (int l = 1; l < m; ++l) bu = bu + u[l] * B[j * m + l];
      y[j] = ax + bu + c[j];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = y[j];
  }
};

// Model parameters + input of one thread.  The parameters live in the
// kernel's parameter space (``__grid_constant__`` argument): uniform across
// the grid, so ptxas reads them as constant-bank / uniform-register operands
// and they cost no per-thread registers (cart-pole's ten parameters used to
// take 20).  The input is per (cell, input) pair, in registers.
template <int KIND>
struct RegModel {
  double u[GIS_MAX_DIM];
  const double* P;
  __device__ __forceinline__ void load(const double* params, const double* uv, int m) {
#pragma unroll
    for (int j = 0; j < GIS_MAX_DIM; ++j) u[j] = (j < m) ? uv[j] : 0.0;
    P = params;
  }
  __device__ __forceinline__ const double* params() const { return P; }
};

// Host-folded products appended to a model's parameter vector (slots after
// the model's own, see model_params): Lorenz RK4 folds sigma into the step
// sizes (Integrator<GIS_LORENZ, 3, GIS_RK4>).
static constexpr int kLorenzFold = 3;  // (0.5h)sigma, h sigma, (h/6)sigma, (0.5h)beta, h beta

// Step sizes, folded on the host exactly as the reference's numpy does
// (cg/system.py:44-49 evaluates 0.5*h and h/6 once per call): passing them as
// kernel parameters keeps ptxas from re-deriving 0.5*h with a DMUL per stage.
struct StepSizes {
  double h, half, h6;
  static StepSizes of(double h) { return StepSizes{h, 0.5 * h, h / 6.0}; }
};

// A value the compiler must keep rather than recompute: ptxas otherwise
// rematerialises the RK4 stage points (DMUL + DADD each) in the final
// combination, spending fp64-pipe issue slots to save a register.
__device__ __forceinline__ double keep(double v) {
  double r;
  asm("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}

// Fused (one-rounding) updates x + a*k for the BASELINE fields whose states
// stay well-conditioned (pendulum, Lorenz, cart-pole): 62 instead of 74 DP
// instructions per pendulum RK4 substep, states within 1e-12 relative of the
// reference (tests/test_gpu_parity.py).  The CSTR fields keep the reference's
// two-rounding order: their exponential makes trajectories leaving X
// ill-conditioned, where a one-ulp change grows past 1e-10.
template <int KIND>
struct Fused {
  static constexpr bool value =
      KIND == GIS_PENDULUM || KIND == GIS_LORENZ || KIND == GIS_CARTPOLE;
};

template <bool F>
__device__ __forceinline__ double axpy(double a, double k, double x) {
  if constexpr (F) return fma(a, k, x);
  else return x + a * k;
}

// Advance one state by the model's discretisation.
//   EULER: x <- x + h f(x)                 (repeated sub times)
//   RK4  : cg/system.py:44-49, k2 = f(x + (0.5h) k1), ...,
//          x <- x + (h/6) (((k1 + 2 k2) + 2 k3) + k4)
template <int KIND, int N, int INTEG>
struct Integrator {
  template <class Tr>
  static __device__ __forceinline__ void run(double (&x)[N], const RegModel<KIND>& rm,
                                             const StepSizes& st, int sub, int m, Tr& tr) {
    run(x, rm.u, rm.params(), st, sub, m, tr);
  }
  template <class Tr>
  static __device__ __forceinline__ void run(double (&x)[N], const double* u,
                                             const double* P, const StepSizes& st, int sub,
                                             int m, Tr& tr) {
    if constexpr (INTEG == GIS_MAP) {
      Map<KIND, N>::eval(x, u, P, m);
    } else if constexpr (INTEG == GIS_RHS) {  // the field alone, reference order
      double f[N];
      Field<KIND, N>::template eval<Tr, false>(x, u, P, f, tr);
#pragma unroll
      for (int d = 0; d < N; ++d) x[d] = f[d];
    } else if constexpr (INTEG == GIS_EULER) {
      // Euler keeps the reference's operation order for every model: it is
      // cheap (no BASELINE throughput config uses it), and with its single
      // update per step one-ulp differences would land exactly-representable
      // images (bloat 0, dyadic grids) on the other side of a grid face
      constexpr bool F = false;
      const double h = st.h;
      for (int s = 0; s < sub; ++s) {
        double f[N];
        Field<KIND, N>::template eval<Tr, false>(x, u, P, f, tr);
#pragma unroll
        for (int d = 0; d < N; ++d) x[d] = axpy<F>(h, f[d], x[d]);
      }
    } else {
      constexpr bool F = Fused<KIND>::value;
      const double h = st.h, half = st.half, h6 = st.h6;
      for (int s = 0; s < sub; ++s) {
        // acc = ((k1 + 2 k2) + 2 k3) accumulated as each stage is produced:
        // the same roundings as the reference's combination (2.0*k is exact,
        // so fma(2, k, acc) rounds like acc + 2.0*k), with N live
        // accumulators instead of three stage vectors
        double acc[N], k[N], t[N];
        Field<KIND, N>::eval(x, u, P, acc, tr);
#pragma unroll
        for (int d = 0; d < N; ++d) t[d] = axpy<F>(half, acc[d], x[d]);
        Field<KIND, N>::eval(t, u, P, k, tr);
#pragma unroll
        for (int d = 0; d < N; ++d) {
          t[d] = axpy<F>(half, k[d], x[d]);
          acc[d] = fma(2.0, k[d], acc[d]);
        }
        Field<KIND, N>::eval(t, u, P, k, tr);
#pragma unroll
        for (int d = 0; d < N; ++d) {
          t[d] = axpy<F>(h, k[d], x[d]);
          acc[d] = fma(2.0, k[d], acc[d]);
        }
        Field<KIND, N>::eval(t, u, P, k, tr);
#pragma unroll
        for (int d = 0; d < N; ++d) x[d] = axpy<F>(h6, acc[d] + k[d], x[d]);
      }
    }
  }
};

// Lorenz RK4 with the linear terms folded into the step sizes.
//  * The first component of the field is sigma (y - x); it is only ever used
//    scaled by a step size (the stage points and the final combination), so
//    the stages carry a = y - x and the updates use the host-folded
//    (c sigma).
//  * The third state's stage value t2 = x2 + c k2' enters the field only as
//    rho - t2 and -beta t2, which are formed directly from x2 and the
//    previous stage's k2': (rho - x2) - c k2' and (-beta x2) - (beta c) k2',
//    with rho - x2 and -beta x2 once per substep; t2 itself is never formed.
// 40 instead of 49 fp64 instructions per substep.  A few roundings are
// folded away; states stay within the 1e-12 contract like the other fused
// updates (tests/test_gpu_parity.py) and the full-size graphs equal the
// reference's (tests/test_gpu_edges.py digests).
template <>
struct Integrator<GIS_LORENZ, 3, GIS_RK4> {
  template <class Tr>
  static __device__ __forceinline__ void run(double (&x)[3], const RegModel<GIS_LORENZ>& rm,
                                             const StepSizes& st, int sub, int m, Tr& tr) {
    run(x, rm.u, rm.params(), st, sub, m, tr);
  }
  template <class Tr>
  static __device__ __forceinline__ void run(double (&x)[3], const double* u, const double* P,
                                             const StepSizes& st, int sub, int, Tr&) {
    const double h = st.h, half = st.half, h6 = st.h6, uu = u[0];
    const double* fold = P + kLorenzFold;  // (0.5h)s, h s, (h/6)s, (0.5h)b, h b
    for (int s = 0; s < sub; ++s) {
      const double rx = P[1] - x[2], mbx = -(P[2] * x[2]);
      // the control enters every stage's second component as + u: it is
      // folded into the stage bases x1 + c u (c = h/2, h) instead, and the
      // stages carry k1 - u (two FMAs per substep instead of four DADDs)
      const double x1h = fma(half, uu, x[1]), x1f = fma(h, uu, x[1]);
      // stage 1 at x
      double a0 = x[1] - x[0];
      double k1 = fma(x[0], rx, -x[1]);
      double k2 = fma(x[0], x[1], mbx);
      double acc0 = a0, acc1 = k1, acc2 = k2;
      // stages 2..4 at x + c k (c = h/2, h/2, h): t0, t1 formed, t2 not
#pragma unroll
      for (int stg = 0; stg < 3; ++stg) {
        const double cs = stg < 2 ? fold[0] : fold[1];  // c sigma
        const double c = stg < 2 ? half : h;
        const double cb = stg < 2 ? fold[3] : fold[4];  // c beta
        const double t0 = fma(cs, a0, x[0]);
        const double t1 = fma(c, k1, stg < 2 ? x1h : x1f);
        const double b = fma(-c, k2, rx);                // rho - t2
        const double nk2 = fma(t0, t1, fma(-cb, k2, mbx));  // t0 t1 - beta t2
        a0 = t1 - t0;
        k1 = fma(t0, b, -t1);
        k2 = nk2;
        if (stg < 2) {
          acc0 = fma(2.0, a0, acc0);
          acc1 = fma(2.0, k1, acc1);
          acc2 = fma(2.0, k2, acc2);
        }
      }
      x[0] = fma(fold[2], acc0 + a0, x[0]);
      x[1] = fma(h6, acc1 + k1, x1f);
      x[2] = fma(h6, acc2 + k2, x[2]);
    }
  }
};

#ifndef __CUDACC_RTC__
// Parameter vector a kernel sees: the model's own parameters, then the
// host-folded products of the specialised integrators.
inline void model_params(const gis_model& m, double* out) {
  for (int i = 0; i < GIS_MAX_PARAMS; ++i) out[i] = m.params[i];
  if (m.kind == GIS_LORENZ && m.integrator == GIS_RK4) {
    const StepSizes st = StepSizes::of(m.h);
    out[kLorenzFold + 0] = st.half * m.params[0];
    out[kLorenzFold + 1] = st.h * m.params[0];
    out[kLorenzFold + 2] = st.h6 * m.params[0];
    out[kLorenzFold + 3] = st.half * m.params[2];
    out[kLorenzFold + 4] = st.h * m.params[2];
  }
}

#endif  // !__CUDACC_RTC__

#ifndef __CUDACC_RTC__
// Compile-time dispatch over (kind, n, integrator).  F is a functor template
// `template <int KIND, int N, int INTEG> static void go(Args...)`.
template <template <int, int, int> class F, class... Args>
void dispatch_model(const gis_model& m, Args&&... args) {
  const int k = m.kind, n = m.n, it = m.integrator;
  auto bad = [&]() {
    throw Error{GIS_E_INVALID, "unsupported model (kind " + std::to_string(k) + ", n " +
                                   std::to_string(n) + ", integrator " +
                                   std::to_string(it) + ")"};
  };
  auto ode = [&](auto kind_c, auto n_c) {
    constexpr int K = decltype(kind_c)::value, NN = decltype(n_c)::value;
    if (n != NN) bad();
    if (it == GIS_EULER) F<K, NN, GIS_EULER>::go(args...);
    else if (it == GIS_RK4) F<K, NN, GIS_RK4>::go(args...);
    else if (it == GIS_RHS) F<K, NN, GIS_RHS>::go(args...);
    else bad();
  };
  auto direct = [&](auto kind_c) {
    constexpr int K = decltype(kind_c)::value;
    if (it != GIS_MAP) bad();
    switch (n) {
      case 1: F<K, 1, GIS_MAP>::go(args...); break;
      case 2: F<K, 2, GIS_MAP>::go(args...); break;
      case 3: F<K, 3, GIS_MAP>::go(args...); break;
      case 4: F<K, 4, GIS_MAP>::go(args...); break;
      default: bad();
    }
  };
  using std::integral_constant;
  switch (k) {
    case GIS_IDENTITY: direct(integral_constant<int, GIS_IDENTITY>{}); break;
    case GIS_SHIFT: direct(integral_constant<int, GIS_SHIFT>{}); break;
    case GIS_LINEAR: direct(integral_constant<int, GIS_LINEAR>{}); break;
    case GIS_AFFINE: direct(integral_constant<int, GIS_AFFINE>{}); break;
    case GIS_CSTR: ode(integral_constant<int, GIS_CSTR>{}, integral_constant<int, 2>{}); break;
    case GIS_PENDULUM:
      ode(integral_constant<int, GIS_PENDULUM>{}, integral_constant<int, 2>{}); break;
    case GIS_CSTR_DIMLESS:
      ode(integral_constant<int, GIS_CSTR_DIMLESS>{}, integral_constant<int, 2>{}); break;
    case GIS_LORENZ: ode(integral_constant<int, GIS_LORENZ>{}, integral_constant<int, 3>{}); break;
    case GIS_CARTPOLE:
      ode(integral_constant<int, GIS_CARTPOLE>{}, integral_constant<int, 4>{}); break;
    default: bad();
  }
}

#endif  // !__CUDACC_RTC__

}  // namespace gis
