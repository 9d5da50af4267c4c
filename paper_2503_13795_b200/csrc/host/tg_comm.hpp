// tg_comm.hpp — internal interface of the NCCL exchange (tg_comm.cpp).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#include "tg_abi.h"

namespace tgcomm {

/// Sets the thread-local tg_last_error message (defined in tg_abi.cpp).
tg_status fail_status(tg_status s, const std::string& msg);

/// NCCL could be bound (dlopen); err says why not.
bool available(std::string& err);
/// In-place ncclAllReduce(sum) of `count` scalars on `st`.
bool allreduce_sum(void* buf, std::size_t count, tg_dtype dtype, void* comm, cudaStream_t st, std::string& err);
/// ncclCommCount, -1 on failure.
int comm_size(void* comm);
/// dlsym of the bound NCCL library (nullptr when absent or not exported).
void* nccl_symbol(const char* name);

}  // namespace tgcomm
