// NCCL inside libsdrt: the halo exchange of face traces between the
// ranks of an element-partitioned run.  NCCL is loaded at run time (dlopen of
// libnccl.so.2, reusing the copy the process already has, e.g. torch's), so the library
// itself has no link-time NCCL dependency and loads on hosts without it; the comm
// entry points return SDRT_E_NCCL there.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace sdrt {

struct NcclComm;  // opaque: communicator + the library's comm stream and events

// 128-byte unique id (rank 0); throws std::runtime_error("nccl: ...") on failure
void nccl_unique_id(uint8_t id[128]);
// communicator over nranks ranks for this process's current CUDA device
NcclComm* nccl_comm_create(const uint8_t id[128], int rank, int nranks);
void nccl_comm_destroy(NcclComm* c);
cudaStream_t nccl_comm_stream(NcclComm* c);
cudaEvent_t nccl_comm_event(NcclComm* c, int k);  // k = 0: "packed", 1: "exchanged"
// grouped point-to-point on the comm stream: for each i, send n_send[i] doubles from
// sbuf[i] to peer_send[i] and receive n_recv[i] doubles into rbuf[i] from peer_recv[i];
// calls are posted in index order on every rank (NCCL matches per peer pair in order)
void nccl_exchange(NcclComm* c, int n, const double* const* sbuf, const int64_t* n_send, const int* peer_send,
                   double* const* rbuf, const int64_t* n_recv, const int* peer_recv);
// in-place min-reduction of one uint64 device value over all ranks, on stream st
void nccl_allreduce_min_u64(NcclComm* c, unsigned long long* d_val, cudaStream_t st);

}  // namespace sdrt
