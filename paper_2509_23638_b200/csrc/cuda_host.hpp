// Host-side CUDA runtime helpers (usable from g++ translation units).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "common.hpp"

namespace ps {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(PS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define PS_CUDA(call) ::ps::cuda_check((call), #call)
// Launch check: catches configuration errors immediately (no device sync).
#define PS_LAUNCH_CHECK(name) ::ps::cuda_check(cudaGetLastError(), name)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

}  // namespace ps
