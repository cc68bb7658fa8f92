// User-defined models: the reference's SystemModel plugin API
// (cg/system.py:52-75, `SystemModel(step=callable)`) reopened without a CPU
// fallback.  A model is given as CUDA C++ source for its vector field (or
// direct map); NVRTC compiles the SAME K1 kernel templates the built-in
// models use (gis_k1.cuh) with that field for sm_100a, once per model, and
// libgis launches the resulting enclose / map kernels exactly where it
// launches the built-in instantiations.  The field is evaluated in the
// reference's operation order (no fused updates, -fmad=false), with CUDA's
// libm for transcendentals.
//
//   form 0 (ODE): body computes f[0..n-1] from x[0..n-1], u[0..m-1], p[...]
//                 and is discretised by Euler or RK4 with the model's substeps
//   form 1 (map): body computes y[0..n-1] (the next state) from x, u, p
//
// NVRTC is loaded with dlopen on first use (libnvrtc.so.12 of the CUDA
// toolkit); the headers it compiles are embedded into libgis at build time
// (build.py -> build_obj/gis_jit_headers.cu), so the library stays
// self-contained.
#include <dlfcn.h>
#include <nvrtc.h>

#include <memory>
#include <type_traits>
#include <mutex>

#include "gis_k1.cuh"

extern const int kGisJitHeaderCount;
extern const char* const kGisJitHeaderNames[];
extern const char* const kGisJitHeaderSources[];

namespace gis {

struct Nvrtc {
  void* h = nullptr;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*add_name)(nvrtcProgram, const char*) = nullptr;
  nvrtcResult (*lowered)(nvrtcProgram, const char*, const char**) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*errstr)(nvrtcResult) = nullptr;
};

static Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so",
                           "/usr/local/cuda/lib64/libnvrtc.so.12"};
    for (const char* nm : names)
      if ((n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!n.h) return;
    auto sym = [&](auto& fn, const char* s) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(n.h, s));
    };
    sym(n.create, "nvrtcCreateProgram");
    sym(n.compile, "nvrtcCompileProgram");
    sym(n.log_size, "nvrtcGetProgramLogSize");
    sym(n.log, "nvrtcGetProgramLog");
    sym(n.cubin_size, "nvrtcGetCUBINSize");
    sym(n.cubin, "nvrtcGetCUBIN");
    sym(n.add_name, "nvrtcAddNameExpression");
    sym(n.lowered, "nvrtcGetLoweredName");
    sym(n.destroy, "nvrtcDestroyProgram");
    sym(n.errstr, "nvrtcGetErrorString");
  });
  GIS_REQUIRE(n.h && n.create && n.compile && n.cubin && n.lowered, GIS_E_CUDA,
              "NVRTC (libnvrtc.so.12) is not available: user-defined models need it");
  return n;
}

struct JitModel {
  std::string body;
  int form = 0, n = 0, m = 0, integ = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t enclose = nullptr, map = nullptr, rhs = nullptr;
};

static std::mutex g_jit_mu;
static std::vector<std::unique_ptr<JitModel>> g_jit;  // id = index + 1

static std::string jit_source(const JitModel& j) {
  const std::string N = std::to_string(j.n);
  std::string s = "#include \"gis_k1.cuh\"\nnamespace gis {\n";
  if (j.form == 0) {
    s += "template <> struct Field<GIS_JIT, " + N + "> {\n"
         "  template <class Tr, bool FUSED = true>\n"
         "  static __device__ __forceinline__ void eval(const double (&x)[" + N + "],\n"
         "      const double* u, const double* p, double (&f)[" + N + "], Tr&) {\n"
         "#line 1 \"user_field\"\n" + j.body + "\n  }\n};\n";
  } else {
    s += "template <> struct Map<GIS_JIT, " + N + "> {\n"
         "  static __device__ __forceinline__ void eval(double (&xs)[" + N + "],\n"
         "      const double* u, const double* p, int) {\n"
         "    double xc[" + N + "], y[" + N + "];\n"
         "    for (int d = 0; d < " + N + "; ++d) { xc[d] = xs[d]; y[d] = xs[d]; }\n"
         "    const double (&x)[" + N + "] = xc;\n"
         "#line 1 \"user_map\"\n" + j.body + "\n"
         "    for (int d = 0; d < " + N + "; ++d) xs[d] = y[d];\n  }\n};\n";
  }
  s += "}  // namespace gis\n";
  return s;
}

struct Compiled {
  std::vector<char> cubin;
  std::string enclose, map, rhs;  // lowered kernel names
};

static Compiled jit_compile_cubin(const JitModel& j) {
  Nvrtc& nv = nvrtc();
  const std::string src = jit_source(j);
  nvrtcProgram prog;
  nvrtcResult r = nv.create(&prog, src.c_str(), "gis_user_model.cu", kGisJitHeaderCount,
                            kGisJitHeaderSources, kGisJitHeaderNames);
  GIS_REQUIRE(r == NVRTC_SUCCESS, GIS_E_CUDA, "nvrtcCreateProgram failed");
  const std::string N = std::to_string(j.n), K = std::to_string(GIS_JIT);
  const std::string e_name =
      "&gis::enclose_kernel<" + K + ", " + N + ", " + std::to_string(j.integ) + ">";
  const std::string m_name = "&gis::map_kernel<" + K + ", " + N + ", " +
                             std::to_string(j.integ) + ">";
  const std::string r_name =
      "&gis::map_kernel<" + K + ", " + N + ", " + std::to_string(GIS_RHS) + ">";
  nv.add_name(prog, e_name.c_str());
  nv.add_name(prog, m_name.c_str());
  if (j.form == 0) nv.add_name(prog, r_name.c_str());
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                        "-default-device"};
  r = nv.compile(prog, 5, opts);
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    nv.destroy(&prog);
    throw Error{GIS_E_INVALID, "user model does not compile (NVRTC):\n" + log};
  }
  size_t cs = 0;
  nv.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  nv.cubin(prog, cubin.data());
  const char *le = nullptr, *lm = nullptr, *lr = nullptr;
  nv.lowered(prog, e_name.c_str(), &le);
  nv.lowered(prog, m_name.c_str(), &lm);
  if (j.form == 0) nv.lowered(prog, r_name.c_str(), &lr);
  Compiled c;
  c.enclose = le ? le : "";
  c.map = lm ? lm : "";
  c.rhs = lr ? lr : "";
  nv.destroy(&prog);
  GIS_REQUIRE(!c.enclose.empty() && !c.map.empty(), GIS_E_CUDA, "NVRTC lost a kernel name");
  c.cubin = std::move(cubin);
  return c;
}

static void jit_compile(JitModel& j) {
  const Compiled c = jit_compile_cubin(j);
  GIS_CUDA(cudaLibraryLoadData(&j.lib, c.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr,
                               0));
  GIS_CUDA(cudaLibraryGetKernel(&j.enclose, j.lib, c.enclose.c_str()));
  GIS_CUDA(cudaLibraryGetKernel(&j.map, j.lib, c.map.c_str()));
  if (j.form == 0) GIS_CUDA(cudaLibraryGetKernel(&j.rhs, j.lib, c.rhs.c_str()));
}

static void check_jit_args(const char* body, int32_t form, int32_t n, int32_t m,
                           int32_t integrator) {
  GIS_REQUIRE(body != nullptr, GIS_E_INVALID, "null argument");
  GIS_REQUIRE(form == 0 || form == 1, GIS_E_INVALID, "form must be 0 (ODE) or 1 (map)");
  GIS_REQUIRE(n >= 1 && n <= GIS_MAX_DIM && m >= 1 && m <= GIS_MAX_DIM, GIS_E_INVALID,
              "n and m must be in [1, 4]");
  GIS_REQUIRE(form == 1 ? integrator == GIS_MAP
                        : (integrator == GIS_EULER || integrator == GIS_RK4),
              GIS_E_INVALID, "ODE models integrate by Euler or RK4; maps use GIS_MAP");
}

static JitModel& jit_model(const gis_model& m) {
  std::lock_guard<std::mutex> lk(g_jit_mu);
  GIS_REQUIRE(m.jit >= 1 && m.jit <= (int)g_jit.size(), GIS_E_INVALID,
              "unknown user model id (gis_jit_register)");
  JitModel& j = *g_jit[m.jit - 1];
  GIS_REQUIRE(j.n == m.n && j.m == m.m, GIS_E_INVALID,
              "user model id does not match the model's dimensions");
  return j;
}

static void launch(cudaKernel_t k, dim3 grid, dim3 block, void** args, size_t smem,
                   gis_ctx* ctx) {
  if (smem > 48 * 1024)
    GIS_CUDA(cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem, ctx->device));
  GIS_CUDA(cudaLaunchKernel((const void*)k, grid, block, args, smem, ctx->stream));
  count_launch(ctx);
}

void jit_enclose(gis_ctx* ctx, const gis_model& m, EncArgs& a) {
  JitModel& j = jit_model(m);
  GIS_REQUIRE(m.integrator == j.integ, GIS_E_INVALID,
              "user model compiled for another integrator");
  const int64_t threads = a.ncells * a.U * a.L;
  if (threads == 0) return;
  const size_t smem = (size_t)(a.U * a.m + 2 * a.S * m.n) * sizeof(double);
  void* args[] = {(void*)&a};
  launch(j.enclose, dim3((unsigned)ceil_div(threads, 256)), dim3(256), args, smem, ctx);
}

void jit_map(gis_ctx* ctx, const gis_model& m, MapArgs& a) {
  JitModel& j = jit_model(m);
  cudaKernel_t k = m.integrator == GIS_RHS ? j.rhs : j.map;
  GIS_REQUIRE(k && (m.integrator == j.integ || m.integrator == GIS_RHS), GIS_E_INVALID,
              "user model compiled for another integrator");
  if (a.N == 0) return;
  void* args[] = {(void*)&a};
  launch(k, dim3((unsigned)ceil_div(a.N, 128)), dim3(128), args, 0, ctx);
}

}  // namespace gis

using namespace gis;

GIS_API int gis_jit_register(gis_ctx* ctx, const char* body, int32_t form, int32_t n, int32_t m,
                             int32_t integrator, int32_t* id) {
  return guarded([&] {
    GIS_REQUIRE(ctx, GIS_E_INVALID, "null context");
    GIS_REQUIRE(id, GIS_E_INVALID, "null argument");
    check_jit_args(body, form, n, m, integrator);
    {
      std::lock_guard<std::mutex> lk(g_jit_mu);
      for (size_t i = 0; i < g_jit.size(); ++i) {
        const JitModel& j = *g_jit[i];
        if (j.body == body && j.form == form && j.n == n && j.m == m && j.integ == integrator) {
          *id = (int32_t)i + 1;
          return;
        }
      }
    }
    auto j = std::make_unique<JitModel>();
    j->body = body;
    j->form = form;
    j->n = n;
    j->m = m;
    j->integ = integrator;
    jit_compile(*j);
    std::lock_guard<std::mutex> lk(g_jit_mu);
    g_jit.push_back(std::move(j));
    *id = (int32_t)g_jit.size();
  });
}

GIS_API int gis_jit_compile_check(const char* body, int32_t form, int32_t n, int32_t m,
                                  int32_t integrator, int64_t* cubin_bytes) {
  return guarded([&] {
    check_jit_args(body, form, n, m, integrator);
    JitModel j;
    j.body = body;
    j.form = form;
    j.n = n;
    j.m = m;
    j.integ = integrator;
    const Compiled c = jit_compile_cubin(j);
    if (cubin_bytes) *cubin_bytes = (int64_t)c.cubin.size();
  });
}
