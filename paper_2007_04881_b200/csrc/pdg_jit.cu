// Runtime specialisation of the element kernel (NVRTC -> sm_100a cubin).
//
// The coefficient fields of one problem are known only at run time (they
// are Python expressions).  The ahead-of-time kernels interpret them from
// bytecode, which costs a dispatch loop + a local-memory stack per field per
// quadrature point and keeps every "has advection / full tensor ..." test a
// runtime branch.  Here the generated policy class (model.py
// ``policy_source``) is compiled together with assemble_body.cuh, so fields
// are inlined expressions and the kind flags are compile-time constants: the
// compiler drops the unused paths, registers and instruction-cache pressure
// fall, and sin(pi*x) etc. are scheduled with the tabulation.
//
// libnvrtc and libcuda are opened with dlopen on first use, so the library
// itself links only against cudart (it must load on GPU-less build hosts).
// Compiled cubins are cached in memory and on disk ($PDG_JIT_CACHE, default
// <libdir>/jit_cache) keyed by the full source + options + a content hash of
// the included headers (PDG_SRC_HASH, set by the Makefile).
#include <dlfcn.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>

#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "assemble_kernel.cuh"
#include "slab_body.cuh"
#include "approach1_body.cuh"

#ifndef PDG_SRC_HASH
#error "PDG_SRC_HASH must be defined by the build (content hash of the kernel headers)"
#endif

namespace pdg {

// ---- minimal driver / NVRTC API surface (resolved with dlsym) ---------------
typedef int CUres;
typedef struct CUmod_st* CUmod;
typedef struct CUfunc_st* CUfunc;
typedef int nvrtcRes;
typedef struct _nvrtcProgram* nvrtcProg;

struct Api {
  bool ok = false;
  std::string why;
  CUres (*cuModuleLoadData)(CUmod*, const void*);
  CUres (*cuModuleGetFunction)(CUfunc*, CUmod, const char*);
  CUres (*cuFuncSetAttribute)(CUfunc, int, int);
  CUres (*cuLaunchKernel)(CUfunc, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                          cudaStream_t, void**, void**);
  CUres (*cuOccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunc, int, size_t);
  nvrtcRes (*nvrtcCreateProgram)(nvrtcProg*, const char*, const char*, int, const char* const*,
                                 const char* const*);
  nvrtcRes (*nvrtcCompileProgram)(nvrtcProg, int, const char* const*);
  nvrtcRes (*nvrtcGetProgramLogSize)(nvrtcProg, size_t*);
  nvrtcRes (*nvrtcGetProgramLog)(nvrtcProg, char*);
  nvrtcRes (*nvrtcGetCUBINSize)(nvrtcProg, size_t*);
  nvrtcRes (*nvrtcGetCUBIN)(nvrtcProg, char*);
  nvrtcRes (*nvrtcDestroyProgram)(nvrtcProg*);
};

constexpr int CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES_ = 8;

static Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* cu = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    void* rtc = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!rtc) rtc = dlopen("libnvrtc.so", RTLD_NOW | RTLD_GLOBAL);
    if (!cu || !rtc) {
      a.why = std::string("cannot dlopen ") + (!cu ? "libcuda.so.1 " : "") + (!rtc ? "libnvrtc.so.12" : "");
      return;
    }
#define PDG_SYM(lib, name)                                               \
  a.name = reinterpret_cast<decltype(a.name)>(dlsym(lib, #name));        \
  if (!a.name) {                                                         \
    a.why = "missing symbol " #name;                                     \
    return;                                                              \
  }
    PDG_SYM(cu, cuModuleLoadData)
    PDG_SYM(cu, cuModuleGetFunction)
    PDG_SYM(cu, cuFuncSetAttribute)
    PDG_SYM(cu, cuLaunchKernel)
    PDG_SYM(cu, cuOccupancyMaxActiveBlocksPerMultiprocessor)
    PDG_SYM(rtc, nvrtcCreateProgram)
    PDG_SYM(rtc, nvrtcCompileProgram)
    PDG_SYM(rtc, nvrtcGetProgramLogSize)
    PDG_SYM(rtc, nvrtcGetProgramLog)
    PDG_SYM(rtc, nvrtcGetCUBINSize)
    PDG_SYM(rtc, nvrtcGetCUBIN)
    PDG_SYM(rtc, nvrtcDestroyProgram)
#undef PDG_SYM
    a.ok = true;
  });
  return a;
}

static std::string lib_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&pdg_abi_version), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    const size_t k = p.rfind('/');
    return k == std::string::npos ? std::string(".") : p.substr(0, k);
  }
  return ".";
}

static uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

struct JitKernel {
  CUmod mod = nullptr;
  CUfunc fn = nullptr;
};

static std::mutex g_mu;
static std::unordered_map<std::string, JitKernel> g_cache;

// PDG_RHS_REGS_MAX for runtime compiles (env override for experiments)
static int jit_rhs_regs_max() {
  const char* v = getenv("PDG_RHS_REGS_MAX");
  return v ? atoi(v) : PDG_RHS_REGS_MAX;
}

// PDG_JIT_WARPS: warps per CTA of the single-warp body (default 4).  Small CTAs
// let the register budget, not the CTA granularity, set the resident warp count.
// Default by dimension (measured r01, same box, cfg4 3D p=2: 4 warps x 3 CTAs
// 10.25 ms, 2 x 6 9.89 ms, 1 x 12 10.38 ms; 2D keeps 4 x 3).
// Large bases (p >= 5 in 2D with advection rows) need so much shared memory per
// warp that 4-warp CTAs leave the SM with a single CTA: the CTA size is then
// chosen for the most resident warps (<= 12, the 168-register budget), ties
// going to the measured default (r02, 250k cfg3 p=6 ADR: 4 warps x 1 CTA
// 48.05 ms, 2 warps x 3 CTAs 44.55 ms; p = 5 and below keep 4-warp CTAs).
// CTAs of w warps that fit one SM's shared memory
static int smem_ctas(int w, int warp_doubles) {
  const double budget = 227.0 * 1024 - 4096;  // per SM, minus a rule-table allowance
  return (int)(budget / ((double)w * warp_doubles * 8.0));
}

static int jit_warps(int dim, int warp_doubles) {
  const char* v = getenv("PDG_JIT_WARPS");
  // 3D kernels that shared memory holds below 12 warps compile with up to 255
  // registers (full_source): 1-warp CTAs then measured best (r02, cfg4 8.66 vs
  // 8.79 ms at 2 warps, 9.03 at 4)
  const int def = dim == 3 ? (smem_ctas(2, warp_doubles) * 2 < 12 ? 1 : 2) : 4;
  if (v) {
    const int w = atoi(v);
    return w >= 1 && w <= 8 ? w : def;
  }
  auto resident = [&](int w) { return std::min(smem_ctas(w, warp_doubles) * w, 12); };
  // switch only for a clear gain (>= 25% more warps): 3D p=2 at 1-warp CTAs
  // would get 9 instead of 8 warps but measured slower (r01: 10.38 vs 9.89 ms)
  int best = def, best_r = resident(def);
  for (int w : {4, 2, 1})
    if (4 * resident(w) >= 5 * resident(def) && resident(w) > best_r) best = w, best_r = resident(w);
  return best;
}

static std::string full_source(const std::string& policy, int dim, int P, bool sym, int kv, int warps,
                               int warp_doubles) {
  // PDG_JIT_MINBLOCKS: minimum resident CTAs per SM the compiler must allow.
  // Default: 12 warps per SM (168 registers; 4-warp CTAs x 3) when shared
  // memory fits them (v2 measured 2/3/4 CTAs -> 11.0/9.2/8.95 ms, v3 3/4 ->
  // 7.47/7.75 ms, 400k cfg5 cells).  When shared memory already holds the SM
  // below 12 warps, no bound: ptxas may use up to 255 registers (r02 same box:
  // cfg3 p=4 / 5 / 6 ADR 6.71 -> 6.01, 17.06 -> 15.41, 45.0 -> 34.5 ms; cfg4 3D
  // 9.53 -> 9.11 ms at 8 instead of 10 warps; register-limited kernels lose:
  // cfg5 6.26 -> 7.30, cfg2 1.25 -> 1.47 ms).
  const char* mb = getenv("PDG_JIT_MINBLOCKS");
  const bool smem_bound = smem_ctas(warps, warp_doubles) * warps < 12;
  const int minblocks = (mb && *mb) ? std::max(1, atoi(mb)) : (smem_bound ? 1 : 12 / warps);
  std::ostringstream os;
  os << "#ifndef PDG_REG_CAPPED\n#define PDG_REG_CAPPED " << (minblocks * warps >= 12 ? 1 : 0) << "\n#endif\n"
     << "#include \"assemble_body.cuh\"\n"
     << "#include \"prepass_body.cuh\"\n"
     << "namespace pdg_jit {\nusing namespace pdg;\n"
     << policy << "\n}\n"
     << "extern \"C\" __global__ void ";
  // PDG_JIT_MAXNREG: a register cap (__maxnreg__) instead of the minimum-CTAs bound
  if (const char* mr = getenv("PDG_JIT_MAXNREG"))
    os << "__maxnreg__(" << atoi(mr) << ")";
  else
    os << "__launch_bounds__(" << 32 * warps << ", " << minblocks << ")";
  os << " pdg_jit_kernel(const __grid_constant__ pdg::KArgs a) {\n"
     << "  pdg::assemble_body<" << dim << ", " << P << ", " << (sym ? "true" : "false")
     << ", pdg_jit::JitCoef, " << kv << ">(a, pdg_jit::JitCoef());\n}\n";
  // the face pre-pass with the same inlined fields (pdg_face_prepass_jit)
  os << "extern \"C\" __global__ void __launch_bounds__(256) pdg_jit_abar(const pdg_mesh m, const pdg_basis B, "
        "const pdg_rules R, const pdg_params prm, double* abar, uint32_t* flags) {\n"
     << "  pdg::elem_abar_body<" << dim << ">(m, B, pdg_jit::JitCoef(), R, prm, abar, flags);\n}\n"
     << "extern \"C\" __global__ void __launch_bounds__(128) pdg_jit_face_prepass(const pdg_mesh m, "
        "const pdg_basis B, const pdg_rules R, const pdg_params prm, const double* abar, double* sigma, "
        "int8_t* flow, uint32_t* flags) {\n"
     << "  pdg::face_prepass_body<" << dim << ">(m, B, pdg_jit::JitCoef(), R, prm, abar, sigma, flow, flags);\n}\n";
  return os.str();
}

static bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return true;
}

// compile (NVRTC, sm_100a) or fetch a module; returns empty string on success, else the error
static std::string get_module(const std::string& src, CUmod& out) {
  Api& A = api();
  if (!A.ok) return "JIT unavailable: " + A.why;
  const std::string dir = lib_dir();
  std::vector<std::string> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                                   "-DPDG_RHS_REGS_MAX=" + std::to_string(jit_rhs_regs_max()),
                                   "-I" + dir + "/csrc",
                                   "-I" + dir + "/../include"};
  // PDG_JIT_DEFINES: extra space-separated -D options (tuning experiments)
  if (const char* defs = getenv("PDG_JIT_DEFINES")) {
    std::istringstream is(defs);
    std::string tok;
    while (is >> tok) opts.push_back(tok);
  }
  // the generated source only #includes the kernel headers, so their content
  // hash (computed by the Makefile) and the ABI version are part of the key:
  // a rebuilt library never loads a cubin compiled from older headers
  std::string key = src + "\n// headers " PDG_SRC_HASH " abi " + std::to_string(PDG_ABI_VERSION);
  for (auto& o : opts) key += "\n" + o;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      out = it->second.mod;
      return "";
    }
  }
  // disk cache: file = 16 hex digits of the key hash; content = key size, key, cubin
  const char* env = getenv("PDG_JIT_CACHE");
  const std::string cdir = env ? std::string(env) : dir + "/jit_cache";
  char hex[32];
  snprintf(hex, sizeof(hex), "%016llx", (unsigned long long)fnv1a(key));
  const std::string cpath = cdir + "/" + hex + ".cubin";
  std::string cubin, blob;
  if (read_file(cpath, blob) && blob.size() > 8) {
    uint64_t klen = 0;
    std::memcpy(&klen, blob.data(), 8);
    if (klen + 8 <= blob.size() && blob.compare(8, klen, key) == 0) cubin = blob.substr(8 + klen);
  }
  if (cubin.empty()) {
    nvrtcProg prog;
    if (A.nvrtcCreateProgram(&prog, src.c_str(), "pdg_jit.cu", 0, nullptr, nullptr) != 0)
      return "nvrtcCreateProgram failed";
    std::vector<const char*> co;
    for (auto& o : opts) co.push_back(o.c_str());
    const nvrtcRes rc = A.nvrtcCompileProgram(prog, (int)co.size(), co.data());
    size_t lsz = 0;
    A.nvrtcGetProgramLogSize(prog, &lsz);
    std::string log(lsz, '\0');
    if (lsz) A.nvrtcGetProgramLog(prog, &log[0]);
    if (rc != 0) {
      A.nvrtcDestroyProgram(&prog);
      return "NVRTC compile failed:\n" + log;
    }
    size_t csz = 0;
    A.nvrtcGetCUBINSize(prog, &csz);
    cubin.resize(csz);
    A.nvrtcGetCUBIN(prog, &cubin[0]);
    A.nvrtcDestroyProgram(&prog);
    // best-effort disk cache (atomic rename)
    std::string cmd = "mkdir -p '" + cdir + "' 2>/dev/null";
    if (system(cmd.c_str()) == 0) {
      const std::string tmp = cpath + ".tmp" + std::to_string((long long)getpid());
      std::ofstream f(tmp, std::ios::binary);
      if (f) {
        const uint64_t klen = key.size();
        f.write(reinterpret_cast<const char*>(&klen), 8);
        f.write(key.data(), (std::streamsize)key.size());
        f.write(cubin.data(), (std::streamsize)cubin.size());
        f.close();
        rename(tmp.c_str(), cpath.c_str());
      }
    }
  }
  cudaFree(nullptr);  // make sure the runtime's primary context is current
  JitKernel k;
  if (A.cuModuleLoadData(&k.mod, cubin.data()) != 0) return "cuModuleLoadData failed";
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_cache[key] = k;
  }
  out = k.mod;
  return "";
}

static std::string get_function(CUmod mod, const char* name, CUfunc& fn) {
  if (api().cuModuleGetFunction(&fn, mod, name) != 0) return std::string("cuModuleGetFunction failed: ") + name;
  return "";
}

static std::string get_kernel(const std::string& policy, int dim, int P, bool sym, const AsmLayout& lay,
                              JitKernel& out) {
  CUmod mod = nullptr;
  std::string err = get_module(full_source(policy, dim, P, sym, lay.kv, jit_warps(dim, lay.warp_doubles), lay.warp_doubles), mod);
  if (!err.empty()) return err;
  out.mod = mod;
  return get_function(mod, "pdg_jit_kernel", out.fn);
}

KArgs make_kargs(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_rules* rules, const pdg_params* params,
                 const pdg_pattern& pat, const pdg_frames* frames, const double* sigma, const int8_t* flow,
                 double* values, int write_cols, double* rhs, uint32_t* flags, int mode);

}  // namespace pdg

using namespace pdg;

extern "C" int pdg_jit_prepare(const pdg_coeffs* coeffs, const char* policy_source, int32_t dim,
                               int32_t max_degree) {
  PDG_TRY {
    if (!coeffs || !policy_source) return fail(PDG_ERR_INVALID, "null argument");
    JitKernel k;
    const AsmLayout lay = make_layout(dim, max_degree, coeffs->diffusion_kind,
                                      coeffs->has_advection || coeffs->has_reaction, jit_rhs_regs_max());
    const std::string err = get_kernel(policy_source, dim, max_degree, symmetric_accumulation(*coeffs), lay, k);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_assemble_jit(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                                const char* policy_source, const pdg_rules* rules, const pdg_params* params,
                                const pdg_pattern* pattern, const pdg_frames* frames, const double* sigma,
                                const int8_t* face_flow, double* values, int32_t write_col_idx, double* rhs,
                                uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    int rc = check_common(mesh, basis, coeffs);
    if (rc) return rc;
    if (!policy_source || !rules || !rules->sqrt_weights || !params || !pattern || !frames || !sigma || !face_flow || !values || !rhs)
      return fail(PDG_ERR_INVALID, "null argument");
    if (write_col_idx && !pattern->col_idx) return fail(PDG_ERR_INVALID, "col_idx not allocated");
    if (!pattern->nbr_rec) return fail(PDG_ERR_INVALID, "interface records missing (pdg_iface_records)");
    JitKernel k;
    const bool sym = symmetric_accumulation(*coeffs);
    const bool has_vr = coeffs->has_advection || coeffs->has_reaction;
    KArgs a = make_kargs(mesh, basis, rules, params, *pattern, frames, sigma, face_flow, values, write_col_idx,
                         rhs, err_flags, 0);
    a.lay = make_layout(mesh->dim, basis->max_degree, coeffs->diffusion_kind, has_vr, jit_rhs_regs_max());
    const std::string err = get_kernel(policy_source, mesh->dim, basis->max_degree, sym, a.lay, k);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    int threads = 32 * jit_warps(mesh->dim, a.lay.warp_doubles);
    // the CTA's rule copy (always reserved: the JIT build may toggle PDG_RULES_SMEM)
    size_t smem = ((size_t)rule_smem_doubles(rules->n_points) + (size_t)a.lay.warp_doubles * (threads / 32)) * 8;
    Api& A = api();
    if (A.cuFuncSetAttribute(k.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES_, (int)smem) != 0)
      return fail(PDG_ERR_CUDA, "cuFuncSetAttribute(max dynamic smem) failed");
    int per_sm = 0;
    if (A.cuOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, threads, smem) != 0 || per_sm < 1) per_sm = 1;
    const int64_t need = (pattern->n_row_elements + threads / 32 - 1) / (threads / 32);
    const int64_t grid = std::min<int64_t>(need, (int64_t)num_sms() * per_sm * 8);
    if (grid <= 0) return PDG_OK;
    void* args[] = {&a};
    if (A.cuLaunchKernel(k.fn, (unsigned)grid, 1, 1, threads, 1, 1, (unsigned)smem, (cudaStream_t)stream, args,
                         nullptr) != 0)
      return fail(PDG_ERR_CUDA, "cuLaunchKernel failed");
    note_launch();
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_face_prepass_jit(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                                    const char* policy_source, const pdg_rules* rules, const pdg_params* params,
                                    double* sigma, int8_t* face_flow, double* elem_abar, uint32_t* err_flags,
                                    pdg_stream stream) {
  PDG_TRY {
    int rc = check_common(mesh, basis, coeffs);
    if (rc) return rc;
    if (!policy_source || !rules || !params || !sigma || !face_flow) return fail(PDG_ERR_INVALID, "null argument");
    const bool iso_var = coeffs->diffusion_kind == PDG_DIFF_ISO && !coeffs->diffusion[0].is_const;
    if (iso_var && !elem_abar) return fail(PDG_ERR_INVALID, "elem_abar scratch required");
    // the module of the element kernel (same policy, dim, degree) carries the pre-pass kernels
    const AsmLayout lay = make_layout(mesh->dim, basis->max_degree, coeffs->diffusion_kind,
                                      coeffs->has_advection || coeffs->has_reaction, jit_rhs_regs_max());
    JitKernel k;
    std::string err = get_kernel(policy_source, mesh->dim, basis->max_degree, symmetric_accumulation(*coeffs), lay, k);
    CUfunc fa = nullptr, ff = nullptr;
    if (err.empty()) err = get_function(k.mod, "pdg_jit_abar", fa);
    if (err.empty()) err = get_function(k.mod, "pdg_jit_face_prepass", ff);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    pdg_mesh m = *mesh;
    pdg_basis B = *basis;
    pdg_rules R = *rules;
    pdg_params prm = *params;
    Api& A = api();
    if (iso_var && mesh->n_elements > 0) {
      void* args[] = {&m, &B, &R, &prm, &elem_abar, &err_flags};
      if (A.cuLaunchKernel(fa, (unsigned)grid_for_warps(mesh->n_elements, 256), 1, 1, 256, 1, 1, 0,
                           (cudaStream_t)stream, args, nullptr) != 0)
        return fail(PDG_ERR_CUDA, "cuLaunchKernel(pdg_jit_abar) failed");
      note_launch();
    }
    if (mesh->n_faces > 0) {
      const double* ab = elem_abar;
      void* args[] = {&m, &B, &R, &prm, &ab, &sigma, &face_flow, &err_flags};
      if (A.cuLaunchKernel(ff, (unsigned)grid_for(mesh->n_faces, 128), 1, 1, 128, 1, 1, 0, (cudaStream_t)stream,
                           args, nullptr) != 0)
        return fail(PDG_ERR_CUDA, "cuLaunchKernel(pdg_jit_face_prepass) failed");
      note_launch();
    }
    return PDG_OK;
  }
  PDG_CATCH
}

// ---------------------------------------------------------------------------
// space-time slabs (slab_body.cuh): one module per (coefficient set, degree,
// family) holding the slab element kernel and the lateral face pre-pass
// ---------------------------------------------------------------------------
namespace pdg {

static int slab_nb(int S, int P, int fam) { return fam ? (P + 1) * binom(P + S, S) : binom(P + S + 1, S + 1); }

// PDG_SLAB_WARPS: warps per CTA of the slab kernel (1, 2 or 4); default by the
// row block's tile count (measured, 200k-prism slabs, family P, r01:
// p=1 1/2/4 warps 4.47/5.74/10.5 ms, p=2 11.3/15.7/25.5, p=3 36.7/39.9/55.2,
// p=4 -/148.7/170.7): one warp up to 3x3 tiles, two up to 6x6, else four
static int slab_warps(int S, int P, int fam) {
  if (const char* v = getenv("PDG_SLAB_WARPS")) {
    const int w = atoi(v);
    if (w == 1 || w == 2 || w == 4) return w;
  }
  const int nt = (slab_nb(S, P, fam) + 7) / 8;
  return nt <= 3 ? 1 : (nt <= 6 ? 2 : 4);
}

static std::string slab_source(const std::string& policy, int S, int P, int fam, int nw) {
  std::ostringstream os;
  os << "#include \"slab_body.cuh\"\n"
     << "namespace pdg_jit {\nusing namespace pdg;\n" << policy << "\n}\n"
     << "extern \"C\" __global__ void __launch_bounds__(" << 32 * nw << ", 1) "
     << "pdg_slab_kernel(const __grid_constant__ pdg::SlabArgs a) {\n"
     << "  pdg::slab_body<" << S << ", " << P << ", " << (fam ? "true" : "false") << ", " << nw
     << ", pdg_jit::JitCoef>(a, pdg_jit::JitCoef());\n}\n"
     << "extern \"C\" __global__ void __launch_bounds__(128) "
     << "pdg_slab_prepass(const __grid_constant__ pdg::SlabArgs a, double* sigma, int8_t* flow) {\n"
     << "  pdg::slab_prepass_body<" << S << ">(a, pdg_jit::JitCoef(), sigma, flow);\n}\n";
  return os.str();
}

static std::string slab_module(const char* policy, int S, int P, int fam, CUmod& mod) {
  const int pmax = fam ? PDG_SLAB_MAX_DEGREE_PQ : PDG_SLAB_MAX_DEGREE;
  if (P < 0 || P > pmax)
    return "slab degree " + std::to_string(P) + " outside the supported range 0.." + std::to_string(pmax) +
           (fam ? " (family PQ)" : " (family P)");
  if (S != 2 && S != 3) return "slab spatial dimension must be 2 or 3";
  return get_module(slab_source(policy, S, P, fam, slab_warps(S, P, fam)), mod);
}

static int slab_check(const pdg_mesh* mesh, const pdg_basis* basis, const char* policy, const pdg_rules* rules,
                      const pdg_params* params, const pdg_slab* slab) {
  if (!mesh || !basis || !policy || !rules || !params || !slab) return fail(PDG_ERR_INVALID, "null argument");
  if (mesh->dim != 2 && mesh->dim != 3) return fail(PDG_ERR_UNSUPPORTED, "slabs need a 2D or 3D spatial mesh");
  if (!slab->time_rules.points || !slab->time_rules.face_offset) return fail(PDG_ERR_INVALID, "time rules missing");
  if (!slab->lateral_tag) return fail(PDG_ERR_INVALID, "lateral tags missing");
  if (slab->table_rows < 4 || slab->table_rows > 10) return fail(PDG_ERR_INVALID, "table_rows must be 4..10");
  if (!(slab->t1 > slab->t0)) return fail(PDG_ERR_INVALID, "slab interval must have positive length");
  if (slab->prev_values && (!slab->prev_dof_offset || !slab->prev_box))
    return fail(PDG_ERR_INVALID, "previous slab data incomplete");
  return PDG_OK;
}

static SlabArgs slab_args(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_rules* rules,
                          const pdg_params* params, const pdg_slab* slab, const pdg_frames* frames,
                          const double* sigma, const int8_t* flow, uint32_t* flags) {
  SlabArgs a;
  std::memset(&a, 0, sizeof(a));
  a.m = *mesh;
  a.B = *basis;
  a.R = *rules;
  a.prm = *params;
  a.sl = *slab;
  a.T = slab->time_rules;
  a.sframe = frames->simplex;
  a.fframe = frames->facet;
  a.erec = frames->element;
  a.sigma = sigma;
  a.flow = flow;
  a.flags = flags;
  return a;
}

}  // namespace pdg

extern "C" int pdg_slab_prepare(const char* policy_source, int32_t spatial_dim, int32_t max_degree,
                                int32_t family) {
  PDG_TRY {
    if (!policy_source) return fail(PDG_ERR_INVALID, "null argument");
    CUmod mod = nullptr;
    const std::string err = slab_module(policy_source, spatial_dim, max_degree, family, mod);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_slab_prepass(const pdg_mesh* mesh, const pdg_basis* basis, const char* policy_source,
                                const pdg_rules* rules, const pdg_params* params, const pdg_slab* slab,
                                const pdg_frames* frames, double* sigma, int8_t* face_flow, uint32_t* err_flags,
                                pdg_stream stream) {
  PDG_TRY {
    int rc = slab_check(mesh, basis, policy_source, rules, params, slab);
    if (rc) return rc;
    if (!frames || !frames->simplex || !frames->facet || !sigma || !face_flow)
      return fail(PDG_ERR_INVALID, "null argument");
    if (mesh->n_faces == 0) return PDG_OK;
    CUmod mod = nullptr;
    std::string err = slab_module(policy_source, mesh->dim, basis->max_degree, slab->family, mod);
    CUfunc fn = nullptr;
    if (err.empty()) err = get_function(mod, "pdg_slab_prepass", fn);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    SlabArgs a = slab_args(mesh, basis, rules, params, slab, frames, sigma, face_flow, err_flags);
    void* args[] = {&a, &sigma, &face_flow};
    if (api().cuLaunchKernel(fn, (unsigned)grid_for(mesh->n_faces, 128), 1, 1, 128, 1, 1, 0, (cudaStream_t)stream,
                             args, nullptr) != 0)
      return fail(PDG_ERR_CUDA, "cuLaunchKernel(pdg_slab_prepass) failed");
    note_launch();
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_slab_assemble(const pdg_mesh* mesh, const pdg_basis* basis, const char* policy_source,
                                 const pdg_rules* rules, const pdg_params* params, const pdg_slab* slab,
                                 const pdg_pattern* pattern, const pdg_frames* frames, const double* sigma,
                                 const int8_t* face_flow, double* values, double* rhs, uint32_t* err_flags,
                                 pdg_stream stream) {
  PDG_TRY {
    int rc = slab_check(mesh, basis, policy_source, rules, params, slab);
    if (rc) return rc;
    if (!pattern || !frames || !frames->simplex || !frames->facet || !frames->element || !sigma || !face_flow ||
        !values || !rhs)
      return fail(PDG_ERR_INVALID, "null argument");
    if (!pattern->nbr_ptr || !pattern->nbr_elem || !pattern->nbr_iface || !pattern->row_len ||
        !pattern->elem_val_offset)
      return fail(PDG_ERR_INVALID, "pattern not built (pdg_adjacency / pdg_pattern_offsets)");
    if (!pattern->nbr_rec) return fail(PDG_ERR_INVALID, "interface records missing (pdg_iface_records)");
    if (pattern->col_dof) return fail(PDG_ERR_UNSUPPORTED, "slab assembly of a sub-mesh (col_dof) is not supported");
    if (pattern->n_row_elements <= 0) return PDG_OK;
    const int S = mesh->dim, P = basis->max_degree, fam = slab->family, nw = slab_warps(S, P, fam);
    CUmod mod = nullptr;
    std::string err = slab_module(policy_source, S, P, fam, mod);
    CUfunc fn = nullptr;
    if (err.empty()) err = get_function(mod, "pdg_slab_kernel", fn);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    SlabArgs a = slab_args(mesh, basis, rules, params, slab, frames, sigma, face_flow, err_flags);
    a.pat = *pattern;
    a.values = values;
    a.rhs = rhs;
    const int nb = slab_nb(S, P, fam), nt = (nb + 7) / 8;
    const size_t smem = slab_smem_bytes(slab->table_rows, nt * 8, nt, nw);
    Api& A = api();
    if (A.cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES_, (int)smem) != 0)
      return fail(PDG_ERR_CUDA, "cuFuncSetAttribute(max dynamic smem) failed");
    int per_sm = 0;
    if (A.cuOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * nw, smem) != 0 || per_sm < 1) per_sm = 1;
    const int64_t grid = std::min<int64_t>(pattern->n_row_elements, (int64_t)num_sms() * per_sm);
    void* args[] = {&a};
    if (A.cuLaunchKernel(fn, (unsigned)grid, 1, 1, 32 * nw, 1, 1, (unsigned)smem, (cudaStream_t)stream, args,
                         nullptr) != 0)
      return fail(PDG_ERR_CUDA, "cuLaunchKernel(pdg_slab_kernel) failed");
    note_launch();
    return PDG_OK;
  }
  PDG_CATCH
}

// ---------------------------------------------------------------------------
// Approach 1 (approach1_body.cuh): item emission, one warp per work item
// ---------------------------------------------------------------------------
namespace pdg {

static std::string a1_source(const std::string& policy, int dim, int P, int nw) {
  std::ostringstream os;
  os << "#include \"approach1_body.cuh\"\n"
     << "namespace pdg_jit {\nusing namespace pdg;\n" << policy << "\n}\n"
     << "extern \"C\" __global__ void __launch_bounds__(" << 32 * nw << ") "
     << "pdg_a1_kernel(const __grid_constant__ pdg::A1Args a) {\n"
     << "  pdg::approach1_body<" << dim << ", " << P << ", pdg_jit::JitCoef>(a, pdg_jit::JitCoef());\n}\n";
  return os.str();
}

static int a1_warps(int dim, int P) {
  const int nb = binom(P + dim, dim), nbp = ((nb + 7) / 8) * 8;
  const size_t per = (size_t)a1_warp_doubles(dim, nbp) * 8;
  int w = (int)std::min<size_t>(4, (200 * 1024) / per);
  return w < 1 ? 1 : w;
}

}  // namespace pdg

extern "C" int pdg_a1_emit(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                           const char* policy_source, const pdg_rules* rules, const pdg_params* params,
                           const pdg_frames* frames, const double* sigma, const int8_t* face_flow,
                           const pdg_a1_items* items, uint64_t* keys, double* vals, uint64_t* load_keys,
                           double* load_vals, uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    int rc = check_common(mesh, basis, coeffs);
    if (rc) return rc;
    if (!policy_source || !rules || !params || !frames || !frames->simplex || !frames->facet || !frames->element ||
        !sigma || !face_flow || !items || !keys || !vals || !load_keys || !load_vals)
      return fail(PDG_ERR_INVALID, "null argument");
    const int64_t n_items = items->n_volume + items->n_interior + items->n_boundary;
    if (n_items <= 0) return PDG_OK;
    if (!items->stripe_offset || !items->load_offset || (items->n_volume && !items->volume_element) ||
        (items->n_interior + items->n_boundary > 0 && (!items->face || !items->facet_row)))
      return fail(PDG_ERR_INVALID, "work item arrays missing");
    const int dim = mesh->dim, P = basis->max_degree, nw = a1_warps(dim, P);
    CUmod mod = nullptr;
    std::string err = get_module(a1_source(policy_source, dim, P, nw), mod);
    CUfunc fn = nullptr;
    if (err.empty()) err = get_function(mod, "pdg_a1_kernel", fn);
    if (!err.empty()) return fail(PDG_ERR_UNSUPPORTED, err);
    A1Args a;
    std::memset(&a, 0, sizeof(a));
    a.m = *mesh;
    a.B = *basis;
    a.R = *rules;
    a.prm = *params;
    a.it = *items;
    a.sframe = frames->simplex;
    a.fframe = frames->facet;
    a.erec = frames->element;
    a.sigma = sigma;
    a.flow = face_flow;
    a.keys = keys;
    a.vals = vals;
    a.load_keys = load_keys;
    a.load_vals = load_vals;
    a.n_cols = items->n_cols;
    a.flags = err_flags;
    if (items->n_cols <= 0) return fail(PDG_ERR_INVALID, "n_cols must be positive");
    const int nb = binom(P + dim, dim), nbp = ((nb + 7) / 8) * 8;
    const size_t smem = (size_t)a1_warp_doubles(dim, nbp) * 8 * nw;
    Api& A = api();
    if (A.cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES_, (int)smem) != 0)
      return fail(PDG_ERR_CUDA, "cuFuncSetAttribute(max dynamic smem) failed");
    int per_sm = 0;
    if (A.cuOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * nw, smem) != 0 || per_sm < 1) per_sm = 1;
    const int64_t need = (n_items + nw - 1) / nw;
    const int64_t grid = std::min<int64_t>(need, (int64_t)num_sms() * per_sm * 8);
    void* args[] = {&a};
    if (A.cuLaunchKernel(fn, (unsigned)grid, 1, 1, 32 * nw, 1, 1, (unsigned)smem, (cudaStream_t)stream, args,
                         nullptr) != 0)
      return fail(PDG_ERR_CUDA, "cuLaunchKernel(pdg_a1_kernel) failed");
    note_launch();
    return PDG_OK;
  }
  PDG_CATCH
}
