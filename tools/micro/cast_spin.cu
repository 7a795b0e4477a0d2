// Micro test: fp64 shared-memory atomicAdd (ATOMS.CAST.SPIN loop) mixed with
// ATOMS.EXCH takes by other warps, as in the staged-column pending
// accumulators.  Integer-valued doubles keep every sum exact, so
// added == taken + left over must hold bit for bit.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double take(unsigned a) {
  double v; asm volatile("atom.shared.exch.b64 %0, [%1], 0;" : "=d"(v) : "r"(a) : "memory"); return v; }
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(double *out, int iters, int nslot) {
  extern __shared__ double s[];
  const unsigned base = (unsigned)__cvta_generic_to_shared(s);
  for (int i = threadIdx.x; i < 2 * nslot; i += blockDim.x) s[i] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double added = 0.0, taken = 0.0;
  unsigned st = 1234567u * (threadIdx.x + 1) + blockIdx.x;
  for (int it = 0; it < iters; it++) {
    st = st * 1664525u + 1013904223u;
    // lanes pick distinct slots: rotate a warp-uniform offset
    const int slot = (int)(((st >> 8) & 0x7fu) * 0) + ((it * 7 + w * 3 + lane) % nslot);
    const double v = (double)((st >> 20) & 15u) + 1.0;
    if (MODE == 0) atomicAdd(s + slot, v);
    if (MODE == 1) { atomicAdd(s + slot, v); atomicAdd(s + nslot + slot, v); }
    added += v * (MODE == 1 ? 2.0 : 1.0);
    if ((it % 24) == w % 24) {  // this warp flushes: lane l takes slots l, l+32, ...
      __syncwarp();
      for (int q = lane; q < nslot; q += 32) { taken += take(base + 8u * q); if (MODE == 1) taken += take(base + 8u * (nslot + q)); }
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) { double rem = 0; for (int i = 0; i < 2 * nslot; i++) rem += s[i]; atomicAdd(out + 2, rem); }
  atomicAdd(out + 0, added); atomicAdd(out + 1, taken);
}
int main() {
  double *d; cudaMalloc(&d, 3 * sizeof(double));
  for (int mode = 0; mode < 2; mode++) for (int nslot : {64, 512}) {
    cudaMemset(d, 0, 3 * sizeof(double));
    if (mode == 0) k<0><<<148, 1024, 2 * nslot * 8>>>(d, 20000, nslot); else k<1><<<148, 1024, 2 * nslot * 8>>>(d, 20000, nslot);
    double h[3]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d nslot %d: added %.0f taken+left %.0f diff %.0f (%s)\n", mode, nslot, h[0], h[1] + h[2], h[0] - h[1] - h[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
