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

DeviceGuard::DeviceGuard(int device) {
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (device >= 0 && device != prev) cudaSetDevice(device);
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
}

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
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*TensorMapEncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill) = nullptr;
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
    DR(FuncSetAttribute);
    DR(TensorMapEncodeTiled);
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
  auto key = std::make_pair(device, std::string(name) + '\n' + src);  // a source may hold
                                                                         // several kernels
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
  DeviceGuard dg_(device);
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

int jit_set_smem(void *fn, int bytes) {
  Api &a = api();
  if (!a.FuncSetAttribute) return 1;
  // a request above the opt-in limit is a configuration that does not fit: report it without
  // issuing the failing driver call
  int dev = 0, mx = 0;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess &&
      bytes > mx)
    return 3;
  return a.FuncSetAttribute((CUfunction)fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                            bytes) == CUDA_SUCCESS
             ? 0
             : 2;
}

int jit_launch_smem(void *fn, int grid, int block, int smem, void *stream, void **args) {
  Api &a = api();
  return a.LaunchKernel((CUfunction)fn, grid, 1, 1, block, 1, 1, (unsigned)smem,
                        (CUstream)stream, args, nullptr) == CUDA_SUCCESS
             ? 0
             : 1;
}

int jit_occupancy(void *fn, int block, int smem, int *blocks_per_sm) {
  Api &a = api();
  *blocks_per_sm = 0;
  return a.OccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, (CUfunction)fn, block,
                                                     (size_t)smem) == CUDA_SUCCESS
             ? 0
             : 1;
}

int jit_tmap_sell(void *out, const double *base, int W, long long nsl, int box_cols,
                  int box_slices) {
  Api &a = api();
  if (!a.TensorMapEncodeTiled) return 1;
  if ((reinterpret_cast<uintptr_t>(out) & 63) || (reinterpret_cast<uintptr_t>(base) & 15))
    return 2;
  const cuuint64_t dims[3] = {32, (cuuint64_t)W, (cuuint64_t)nsl};
  const cuuint64_t strides[2] = {256, (cuuint64_t)W * 256};
  const cuuint32_t box[3] = {32, (cuuint32_t)box_cols, (cuuint32_t)box_slices};
  const cuuint32_t estr[3] = {1, 1, 1};
  return a.TensorMapEncodeTiled(reinterpret_cast<CUtensorMap *>(out),
                                CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides,
                                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 3;
}

int jit_tmap_sell_cm(void *out, const double *base, int W, long long nsl, int box_cols,
                     int box_slices) {
  Api &a = api();
  if (!a.TensorMapEncodeTiled) return 1;
  if ((reinterpret_cast<uintptr_t>(out) & 63) || (reinterpret_cast<uintptr_t>(base) & 15))
    return 2;
  const cuuint64_t dims[3] = {32, (cuuint64_t)nsl, (cuuint64_t)W};
  const cuuint64_t strides[2] = {(cuuint64_t)W * 256, 256};
  const cuuint32_t box[3] = {32, (cuuint32_t)box_slices, (cuuint32_t)box_cols};
  const cuuint32_t estr[3] = {1, 1, 1};
  return a.TensorMapEncodeTiled(reinterpret_cast<CUtensorMap *>(out),
                                CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides,
                                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 3;
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
