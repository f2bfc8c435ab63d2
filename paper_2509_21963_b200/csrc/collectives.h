// collectives.h — NCCL for the column-sharded engine, loaded at run time (dlopen): the library
// has no link-time NCCL dependency, and in a process that already uses NCCL (torch.distributed)
// it shares that process's libnccl.so.2.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

namespace itercur_b200 {

struct NcclApi {
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int*);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
  const char* (*GetErrorString)(ncclResult_t);
};

// nullptr when no libnccl.so.2 can be loaded (nccl_load_error() says why)
const NcclApi* nccl_api();
const char* nccl_load_error();

}  // namespace itercur_b200
