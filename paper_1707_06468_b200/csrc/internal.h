// Library-internal helpers (error state, common launch constants).
#pragma once
#include <cuda_runtime.h>

#include "../../include/proxsaga.h"

int ps_fail(int code, const char *msg);
int ps_cuda_fail(cudaError_t e, const char *where);
