// Runtime compilation of generated kernels (jit.cpp).
#pragma once
#include <string>

namespace fastilu {

// RAII guard for the calling thread's current CUDA device: switches to `device` (if >= 0 and
// different) and restores the caller's device on scope exit, so no ABI entry point leaves the
// caller on another GPU.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device);
  ~DeviceGuard();
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;
};

bool jit_available(std::string *why);
// Compiles (cached per device and source) and returns the CUfunction `name`; 0 on success,
// otherwise an error code with the NVRTC log in *log.
int jit_get(const std::string &src, const char *name, int device, void **fn, std::string *log);
int jit_launch(void *fn, int grid, int block, void *stream, void **args);
int jit_func_info(void *fn, int *regs, int *local_bytes, int block, int *blocks_per_sm);
// Dynamic shared memory: raise the function's limit to `bytes`, launch with `smem` bytes and
// query the resident blocks per SM at that size.
int jit_set_smem(void *fn, int bytes);
int jit_launch_smem(void *fn, int grid, int block, int smem, void *stream, void **args);
int jit_occupancy(void *fn, int block, int smem, int *blocks_per_sm);
// 3D TMA tensor map (128 bytes, 64-byte aligned `out`) over a template-SELL array of fp64:
// dims {32 rows of a slice, W columns, nsl slices}, strides {256 B, W * 256 B}, box
// {32, box_cols, box_slices}; out-of-range boxes are zero-filled.  0 on success.
int jit_tmap_sell(void *out, const double *base, int W, long long nsl, int box_cols,
                  int box_slices);
// The same tensor over the SELL layout with the slice and column dimensions swapped (dims {32
// rows, nsl slices, W columns}, box {32, box_slices, box_cols}): a box lands column-major in
// shared memory, [column][slice][32 rows] (kStagedColMajor).  Swapped argument order of the box
// coordinates in the kernel: {0, slice, column}.
int jit_tmap_sell_cm(void *out, const double *base, int W, long long nsl, int box_cols,
                     int box_slices);

}  // namespace fastilu
