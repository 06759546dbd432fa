#pragma once
#include <cstddef>
#include <cuda_runtime.h>

// Minimal NCCL declarations (ABI-compatible with nccl.h 2.x) so no NCCL header or
// library is needed at build time.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { dgNcclFloat64 = 8 };

namespace dg {

struct NcclApi {
    ncclResult_t (*ncclGetUniqueId)(ncclUniqueId*);
    ncclResult_t (*ncclCommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*ncclCommDestroy)(ncclComm_t);
    ncclResult_t (*ncclCommGetAsyncError)(ncclComm_t, ncclResult_t*);
    const char* (*ncclGetErrorString)(ncclResult_t);
    ncclResult_t (*ncclSend)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*ncclRecv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*ncclGroupStart)();
    ncclResult_t (*ncclGroupEnd)();
    ncclResult_t (*ncclCommCount)(const ncclComm_t, int*);   // optional
};

const NcclApi* nccl_api();   // nullptr if NCCL cannot be loaded

}  // namespace dg
