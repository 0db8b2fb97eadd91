// Host-side utilities: error state, CUDA driver entry points (resolved at run time through
// cudaGetDriverEntryPoint so the library loads on a machine without a GPU driver).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

namespace tgp {

void set_error(const char* fmt, ...);
const char* get_error();

struct Driver {
  bool ok = false;
  decltype(&cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
  decltype(&cuStreamWaitValue32) streamWaitValue32 = nullptr;
  decltype(&cuStreamWriteValue32) streamWriteValue32 = nullptr;
};
// Resolves the driver entry points once; returns nullptr (with tgp_last_error set) on failure.
const Driver* driver();

}  // namespace tgp

#define TGP_CUDA_TRY(expr)                                                                          \
  do {                                                                                              \
    cudaError_t _e = (expr);                                                                        \
    if (_e != cudaSuccess) {                                                                        \
      ::tgp::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e));         \
      return TGP_E_CUDA;                                                                            \
    }                                                                                               \
  } while (0)

#define TGP_CU_TRY(expr)                                                                            \
  do {                                                                                              \
    CUresult _r = (expr);                                                                           \
    if (_r != CUDA_SUCCESS) {                                                                       \
      ::tgp::set_error("%s:%d: %s: CUresult %d", __FILE__, __LINE__, #expr, (int)_r);               \
      return TGP_E_CUDA;                                                                            \
    }                                                                                               \
  } while (0)

#define TGP_TRY(expr)                  \
  do {                                 \
    int _s = (expr);                   \
    if (_s != 0) return (tgp_status)_s; \
  } while (0)
