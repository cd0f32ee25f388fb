// zeus_internal.h -- host-side error plumbing shared by the C-ABI entry points.
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>

#include "../../include/zeus_b200.h"

namespace zeus {

// Records a message for zeus_last_error() (thread-local) and returns `code`.
int set_error(int code, const char* fmt, ...);
inline int clear_error() { return set_error(ZEUS_OK, ""); }

// Checks the most recent launch / API call.
inline int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return set_error(ZEUS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return ZEUS_OK;
}
inline int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int current_sm_count();
// byte offset of the PsoXchg descriptor inside a rank's exchange block (pso.cu)
size_t xchg_desc_offset(int d, int world);

}  // namespace zeus
