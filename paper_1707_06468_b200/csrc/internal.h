// Library-internal helpers (error state, common launch constants).
#pragma once
#include <cuda_runtime.h>

#include "../../include/proxsaga.h"

int ps_fail(int code, const char *msg);
int ps_cuda_fail(cudaError_t e, const char *where);

// return the library status of a failed CUDA call
#define CK(call, where)                                                    \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) return ps_cuda_fail(_e, where);             \
    } while (0)
