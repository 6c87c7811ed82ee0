// Native NCCL transport of the subdomain-partitioned DDM (hs_nccl.cpp).
#pragma once

#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>
#include <nccl.h>

#include "hs_common.hpp"

namespace hsb {

int nccl_version();                                          // throws Error(kCuda) without libnccl
void nccl_unique_id(unsigned char out[NCCL_UNIQUE_ID_BYTES]);  // ncclGetUniqueId

// One communicator over the ranks of a partitioned solver (one GPU each).
struct NcclComm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  NcclComm(const unsigned char id[NCCL_UNIQUE_ID_BYTES], int rank, int world);
  ~NcclComm();
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  // one message to / from each listed peer (offsets and counts in doubles), one NCCL group on s
  void exchange(int npeers, const int* peers, const std::int64_t* soff, const std::int64_t* scnt,
                const std::int64_t* roff, const std::int64_t* rcnt, const double* send, double* recv, cudaStream_t s);
  void allreduce(double* buf, std::int64_t count, cudaStream_t s);  // in place, sum
  void allgather(const double* send, double* recv, std::int64_t count, cudaStream_t s);
};

}  // namespace hsb
