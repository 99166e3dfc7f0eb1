// Runtime compilation of template-specialised kernels (NVRTC -> sm_100a CUBIN -> driver module).
// NVRTC is dlopen'ed and the driver API is reached through cudaGetDriverEntryPoint, so the
// library loads (and its host-only entry points work) on machines without a GPU or NVRTC.
#include "jit.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace fastilu {

namespace {

struct Api {
  bool ok = false;
  std::string why;
  // NVRTC
  nvrtcResult (*CreateProgram)(nvrtcProgram *, const char *, const char *, int,
                               const char *const *, const char *const *) = nullptr;
  nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char *const *) = nullptr;
  nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t *) = nullptr;
  nvrtcResult (*GetCUBIN)(nvrtcProgram, char *) = nullptr;
  nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t *) = nullptr;
  nvrtcResult (*GetProgramLog)(nvrtcProgram, char *) = nullptr;
  nvrtcResult (*DestroyProgram)(nvrtcProgram *) = nullptr;
  // driver
  CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, unsigned, CUstream, void **, void **) = nullptr;
  CUresult (*FuncGetAttribute)(int *, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int *, CUfunction, int,
                                                        size_t) = nullptr;
};

Api &api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *cands[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                           "libnvrtc.so"};
    void *h = nullptr;
    for (const char *c : cands)
      if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
      a.why = "libnvrtc not found";
      return;
    }
#define NV(f) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nvrtc" #f))
    NV(CreateProgram);
    NV(CompileProgram);
    NV(GetCUBINSize);
    NV(GetCUBIN);
    NV(GetProgramLogSize);
    NV(GetProgramLog);
    NV(DestroyProgram);
#undef NV
#define DR(f)                                                                             \
  {                                                                                        \
    void *p = nullptr;                                                                     \
    cudaDriverEntryPointQueryResult q;                                                     \
    if (cudaGetDriverEntryPoint("cu" #f, &p, cudaEnableDefault, &q) == cudaSuccess &&      \
        q == cudaDriverEntryPointSuccess)                                                  \
      a.f = reinterpret_cast<decltype(a.f)>(p);                                            \
  }
    DR(ModuleLoadData);
    DR(ModuleGetFunction);
    DR(LaunchKernel);
    DR(FuncGetAttribute);
    DR(OccupancyMaxActiveBlocksPerMultiprocessor);
#undef DR
    a.ok = a.CreateProgram && a.CompileProgram && a.GetCUBINSize && a.GetCUBIN &&
           a.DestroyProgram && a.ModuleLoadData && a.ModuleGetFunction && a.LaunchKernel &&
           a.FuncGetAttribute && a.OccupancyMaxActiveBlocksPerMultiprocessor;
    if (!a.ok) a.why = "NVRTC or driver entry points missing";
  });
  return a;
}

std::mutex g_mu;
std::map<std::pair<int, std::string>, CUfunction> g_cache;

}  // namespace

bool jit_available(std::string *why) {
  Api &a = api();
  if (!a.ok && why) *why = a.why;
  return a.ok;
}

int jit_get(const std::string &src, const char *name, int device, void **fn, std::string *log) {
  Api &a = api();
  if (!a.ok) {
    if (log) *log = a.why;
    return 1;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(device, src);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *fn = (void *)it->second;
    return 0;
  }
  nvrtcProgram prog;
  if (a.CreateProgram(&prog, src.c_str(), "fastilu_tsell.cu", 0, nullptr, nullptr) !=
      NVRTC_SUCCESS)
    return 2;
  const char *opts[] = {"--gpu-architecture=sm_100a", "-default-device", "-lineinfo",
                        "--std=c++17"};
  nvrtcResult cr = a.CompileProgram(prog, 4, opts);
  if (cr != NVRTC_SUCCESS) {
    if (log && a.GetProgramLogSize && a.GetProgramLog) {
      size_t n = 0;
      a.GetProgramLogSize(prog, &n);
      std::string l(n, '\0');
      a.GetProgramLog(prog, &l[0]);
      *log = l;
    }
    a.DestroyProgram(&prog);
    return 3;
  }
  size_t n = 0;
  a.GetCUBINSize(prog, &n);
  std::vector<char> cubin(n);
  a.GetCUBIN(prog, cubin.data());
  a.DestroyProgram(&prog);
  cudaSetDevice(device);
  cudaFree(nullptr);  // make sure the primary context is current
  CUmodule mod;
  if (a.ModuleLoadData(&mod, cubin.data()) != CUDA_SUCCESS) return 4;
  CUfunction f;
  if (a.ModuleGetFunction(&f, mod, name) != CUDA_SUCCESS) return 5;
  g_cache[key] = f;
  *fn = (void *)f;
  return 0;
}

int jit_launch(void *fn, int grid, int block, void *stream, void **args) {
  Api &a = api();
  return a.LaunchKernel((CUfunction)fn, grid, 1, 1, block, 1, 1, 0, (CUstream)stream, args,
                        nullptr) == CUDA_SUCCESS
             ? 0
             : 1;
}

int jit_func_info(void *fn, int *regs, int *local_bytes, int block, int *blocks_per_sm) {
  Api &a = api();
  CUfunction f = (CUfunction)fn;
  if (regs) a.FuncGetAttribute(regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
  if (local_bytes) a.FuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
  if (blocks_per_sm) a.OccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, block, 0);
  return 0;
}

}  // namespace fastilu
