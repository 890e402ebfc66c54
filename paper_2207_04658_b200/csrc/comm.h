// comm.h -- point-to-point exchanges of the slab decomposition over NCCL (loaded at
// run time with dlopen, so libqmpm has no link-time NCCL dependency).  Internal.
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace qmpm {

struct NcclComm;  // opaque (ncclComm_t + rank layout)

// 128-byte NCCL unique id
bool nccl_unique_id(unsigned char id[128], std::string& err);
NcclComm* nccl_connect(const unsigned char id[128], int nranks, int rank, std::string& err);
void nccl_destroy(NcclComm* c);

// One grouped exchange with the two z-neighbours (rank - 1 = down, rank + 1 = up).
// Each direction: send `send_bytes` from `send`, receive `recv_bytes` into `recv`
// (pointers may be null / sizes zero when the neighbour does not exist).
struct P2P {
  const void* send_dn;
  size_t send_dn_bytes;
  const void* send_up;
  size_t send_up_bytes;
  void* recv_dn;  // from rank - 1
  size_t recv_dn_bytes;
  void* recv_up;  // from rank + 1
  size_t recv_up_bytes;
};
bool nccl_exchange(NcclComm* c, const P2P& x, cudaStream_t st, std::string& err);
// in-place all-reduce (max) of one device uint32 over every rank (the sticky status)
bool nccl_allreduce_max_u32(NcclComm* c, unsigned int* v, cudaStream_t st, std::string& err);

}  // namespace qmpm
