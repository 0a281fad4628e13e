// Microbenchmark: cost of a warp softmax + top-2 (the decode kernel's phase-0
// decision) in isolation, with/without a large dynamic smem footprint and with
// the other warps parked at a CTA barrier.  Development aid, not product code.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float wsum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void k(float* out, unsigned long long* t, int E, int kk, int mode) {
  extern __shared__ float sm[];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 64) sm[threadIdx.x] = 0.1f * threadIdx.x;
  __syncthreads();
  unsigned long long t0 = clock64(), t1 = 0, t2 = 0;
  if (warp == 0) {
    float z = lane < E ? sm[lane] : 0.f;
    float m = lane < E ? z : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float e = lane < E ? expf(z - m) : 0.f;
    float p = lane < E ? e / wsum(e) : 0.f;
    t1 = clock64();
    bool taken = lane >= E;
    int sel = -1;
    for (int j = 0; j < kk; ++j) {
      float bv = taken ? -INFINITY : p;
      int bi = taken ? 0x7fffffff : lane;
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == j) sel = bi;
      if (lane == bi) taken = true;
    }
    t2 = clock64();
    if (lane < kk) out[blockIdx.x * 8 + lane] = sel + p;
  }
  if (mode == 1) __syncthreads();
  if (threadIdx.x == 0) { t[blockIdx.x * 2] = t1 - t0; t[blockIdx.x * 2 + 1] = t2 - t1; }
}
int main() {
  float* out; unsigned long long* t; cudaMalloc(&out, 148 * 8 * 4); cudaMalloc(&t, 148 * 16);
  unsigned long long h[296];
  for (int smem : {4096, 220 * 1024}) for (int mode : {0, 1}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int it = 0; it < 3; ++it) k<<<148, 256, smem>>>(out, t, 8, 2, mode);
    cudaDeviceSynchronize();
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long a = 0, b = 0;
    for (int i = 0; i < 148; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
    printf("smem=%6d barrier=%d  softmax %llu cycles, top2 %llu cycles (mean over 148 CTAs) err=%s\n",
           smem, mode, a / 148, b / 148, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
