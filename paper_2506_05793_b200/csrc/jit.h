// Runtime compilation of generated kernels (jit.cpp).
#pragma once
#include <string>

namespace fastilu {

bool jit_available(std::string *why);
// Compiles (cached per device and source) and returns the CUfunction `name`; 0 on success,
// otherwise an error code with the NVRTC log in *log.
int jit_get(const std::string &src, const char *name, int device, void **fn, std::string *log);
int jit_launch(void *fn, int grid, int block, void *stream, void **args);
int jit_func_info(void *fn, int *regs, int *local_bytes, int block, int *blocks_per_sm);

}  // namespace fastilu
