// hod_ce.cu — copy-engine data movement over NVLink (peer-mapped addresses).
//
// A device-to-device cudaMemcpyAsync between a local and a peer-mapped
// (symmetric-memory) address is executed by the GPU's copy engines, not by
// SMs: the bytes cross NVLink while every SM stays free for the reduction /
// AdamW kernels (or the backward GEMMs).  Used by the "ce" RS/AG path.
#include "hod_common.cuh"

extern "C" {

int hod_ce_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return HOD_OK;
  if (!dst || !src) { hod::set_error("hod_ce_copy: null pointer"); return HOD_EINVAL; }
  return hod::cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice,
                                          static_cast<cudaStream_t>(stream)),
                          "hod_ce_copy");
}

}  // extern "C"
