// wt_host.h -- host-side helpers shared by the C-ABI translation units
// (wt_capi.cu, wt_ops.cu): the thread's last error, status macros, device setup.
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "../../include/wt_b200.h"

extern thread_local std::string g_err;
extern thread_local int64_t g_err_index;
int fail(int code, const std::string& msg);
int setup_device(int device);   // cudaSetDevice + a warm stream-ordered pool
int sm_count(int device);

#define CU(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      return fail(e_ == cudaErrorMemoryAllocation ? WT_ERR_OOM : WT_ERR_CUDA,           \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    }                                                                                   \
  } while (0)
#define TRY(call)               \
  do {                          \
    int s_ = (call);            \
    if (s_ != WT_OK) return s_; \
  } while (0)
