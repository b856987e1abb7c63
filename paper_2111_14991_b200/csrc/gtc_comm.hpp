// Exchange layer of candidate-axis sharding (gtc_comm_*, include/gridtune_cuda.h).
//
// One operation: an all-gather of a small device buffer, enqueued on the
// caller's stream without a host synchronisation, so a sharded gtc_run_steps
// chunk runs its per-iteration exchanges (the variance-total
// accumulators and the selection records) in stream order with its kernels.
// Two transports:
//  - NCCL (ncclAllGather over NVLink/NVSwitch), one rank per process/GPU;
//    libnccl is opened at run time (dlopen), so the library loads without it;
//  - an in-process group of shards driven by one host thread each (peer
//    copies + CUDA events), for one process driving several devices -- and
//    several shards on one device (the single-GPU parity tests).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

struct gtc_comm {
  int rank = 0;
  int nranks = 1;
  virtual ~gtc_comm() = default;
  // recv[i * bytes, (i + 1) * bytes) = rank i's send buffer, for every rank,
  // in stream order on `stream` (device buffers).  Returns a GTC_* status.
  virtual int allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) = 0;
  virtual const char* kind() const = 0;
};
