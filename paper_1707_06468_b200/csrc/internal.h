// Library-internal helpers (error state, common launch constants).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/proxsaga.h"

int ps_fail(int code, const char *msg);
int ps_cuda_fail(cudaError_t e, const char *where);

// return the library status of a failed CUDA call
#define CK(call, where)                                                    \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) return ps_cuda_fail(_e, where);             \
    } while (0)

// NVTX range over a library entry point (visible in nsys / ncu --nvtx timelines):
// K1/K2 = ps_run (deterministic replay / asynchronous solve), K3 = objective,
// K4 = gradient / fixed-point residual / resync, K5 = prepare, K8 = dual.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
