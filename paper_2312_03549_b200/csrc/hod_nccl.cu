// hod_nccl.cu — C1/C2/C3 collectives over NCCL (NVLink 5 / NVSwitch).
//
// Thin wrappers: one communicator per GroupPlan DP row (groups.py:137-148)
// plus an optional world communicator for the clip norm.  Built against the
// NCCL headers of the pip wheel torch loads (2.28.x) and linked to the same
// libnccl.so.2 soname, so the process holds exactly one NCCL.
#include <nccl.h>
#include <string.h>

#include "hod_common.cuh"

namespace {

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return HOD_OK;
  hod::set_error("%s: %s (ncclResult %d)", what, ncclGetErrorString(r), static_cast<int>(r));
  return HOD_ENCCL;
}

}  // namespace

extern "C" {

int hod_nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  if (!out) { hod::set_error("hod_nccl_unique_id: null"); return HOD_EINVAL; }
  ncclUniqueId id;
  const int rc = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(out, id.internal, 128);
  return HOD_OK;
}

int hod_nccl_comm_init(const uint8_t id[128], int nranks, int rank, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
    hod::set_error("hod_nccl_comm_init: bad arguments (nranks=%d rank=%d)", nranks, rank);
    return HOD_EINVAL;
  }
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ncclComm_t c = nullptr;
  const int rc = nccl_status(ncclCommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm = c;
  return HOD_OK;
}

int hod_comm_destroy(void* comm) {
  if (!comm) return HOD_OK;
  return nccl_status(ncclCommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

int hod_comm_async_error(void* comm) {
  if (!comm) { hod::set_error("hod_comm_async_error: null"); return HOD_EINVAL; }
  ncclResult_t async = ncclSuccess;
  const int rc = nccl_status(ncclCommGetAsyncError(static_cast<ncclComm_t>(comm), &async),
                             "ncclCommGetAsyncError");
  if (rc) return rc;
  return nccl_status(async, "NCCL communicator (asynchronous error)");
}

int hod_reduce_scatter_bf16(const void* send, void* recv, size_t recvcount, void* comm, void* stream) {
  if (!send || !recv || !comm) { hod::set_error("hod_reduce_scatter_bf16: null"); return HOD_EINVAL; }
  return nccl_status(ncclReduceScatter(send, recv, recvcount, ncclBfloat16, ncclSum,
                                       static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)),
                     "ncclReduceScatter");
}

int hod_all_gather_bf16(const void* send, void* recv, size_t sendcount, void* comm, void* stream) {
  if (!send || !recv || !comm) { hod::set_error("hod_all_gather_bf16: null"); return HOD_EINVAL; }
  return nccl_status(ncclAllGather(send, recv, sendcount, ncclBfloat16, static_cast<ncclComm_t>(comm),
                                   static_cast<cudaStream_t>(stream)),
                     "ncclAllGather");
}

int hod_all_reduce_f32(float* buf, size_t n, void* comm, void* stream) {
  if (!buf || !comm) { hod::set_error("hod_all_reduce_f32: null"); return HOD_EINVAL; }
  return nccl_status(ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm),
                                   static_cast<cudaStream_t>(stream)),
                     "ncclAllReduce");
}

}  // extern "C"
