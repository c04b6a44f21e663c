// Thread-local error state behind tp_last_error() and the status-code helpers.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "trainplan/capi.h"

namespace gptb200 {

inline std::string& last_error() {
  thread_local std::string msg;
  return msg;
}

inline int set_error(int code, const std::string& msg) {
  last_error() = msg;
  return code;
}

inline int clear_error() {
  last_error().clear();
  return TP_OK;
}

inline int set_cuda_error(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaErrorMemoryAllocation)
    return set_error(TP_ERR_OOM, std::string(where) + ": " + cudaGetErrorString(e));
  return set_error(TP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace gptb200
