// Shared-memory atomic throughput on sm_100a: fp64 CAS-loop add, u32 native add,
// u32 add x2 (split fixed point), plain LDS/STS, for 32 warps x 1 CTA/SM,
// each lane hitting a random slot among H (Zipf-ish: slot = (r*r) % H biased to head).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash(uint32_t x){ x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int MODE>
__global__ void __launch_bounds__(1024,1) k(int iters, int H, int active, double *out) {
  extern __shared__ double sm[];
  for (int s = threadIdx.x; s < 4*H; s += blockDim.x) sm[s] = 0;
  __syncthreads();
  uint32_t st = hash(threadIdx.x + 7919u * blockIdx.x);
  const int lane = threadIdx.x & 31;
  double acc = 0;
  for (int it = 0; it < iters; it++) {
    st = hash(st + it);
    // skewed slot: head-heavy
    uint32_t r = st % 1024u; uint32_t slot = (r * r) >> 11;  // in [0,512)
    slot = (slot * 7u + lane * 13u) % (uint32_t)H;        // lanes of a warp distinct-ish
    if (lane < active) {
      if (MODE == 0) atomicAdd(&sm[slot], 1.0);
      else if (MODE == 1) atomicAdd(reinterpret_cast<unsigned*>(sm) + slot, 1u);
      else if (MODE == 2) { atomicAdd(reinterpret_cast<unsigned*>(sm) + 2*slot, 1u); atomicAdd(reinterpret_cast<unsigned*>(sm) + 2*slot + 1, 3u); }
      else if (MODE == 3) { acc += sm[slot]; }
      else if (MODE == 4) { double2 v = reinterpret_cast<double2*>(sm)[slot]; acc += v.x + v.y; }
      else if (MODE == 5) { volatile double *p = &sm[slot]; *p = *p + 1.0; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0] + acc;
}
int main() {
  double *out; cudaMalloc(&out, 1024 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char *names[] = {"f64 CAS add", "u32 add", "2x u32 add", "LDS.64", "LDS.128", "LDS+STS f64"};
  for (int H : {512, 1024}) for (int active : {15, 32}) for (int m = 0; m < 6; m++) {
    int iters = 20000; size_t smem = 4 * H * 8;
    void (*f)(int,int,int,double*) = m==0?k<0>:m==1?k<1>:m==2?k<2>:m==3?k<3>:m==4?k<4>:k<5>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    f<<<sms, 1024, smem>>>(10, H, active, out);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); f<<<sms, 1024, smem>>>(iters, H, active, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double cyc = ms * 1e-3 * 1.965e9;
    double per_warp_instr = cyc / (iters * 32.0);  // SM cycles per warp-instruction (32 warps/SM)
    printf("H=%4d active=%2d %-12s  %.3f ms  %.2f SM-cycles per warp-op  %.3f per lane-op  %s\n", H, active, names[m], ms,
           per_warp_instr, per_warp_instr / active, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
