// Microbenchmark: cost of release fences at gpu vs sys scope after a burst
// of 16-byte stores (local HBM).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fence_cost.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int MODE>
__global__ void k(int4* buf, int nst, unsigned long long* out) {
  const int tid = threadIdx.x;
  int4 v = make_int4(tid, 1, 2, 3);
  __syncthreads();
  uint64_t t0 = gt();
  for (int i = 0; i < nst; ++i) buf[(size_t)blockIdx.x * nst * blockDim.x + i * blockDim.x + tid] = v;
  __syncthreads();
  uint64_t t1 = gt();
  if (tid == 0) {
    if (MODE == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (MODE == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (MODE == 2) asm volatile("fence.sc.sys;" ::: "memory");
    if (MODE == 3) asm volatile("fence.sc.gpu;" ::: "memory");
  }
  __syncthreads();
  uint64_t t2 = gt();
  if (tid == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t1; }
}
int main() {
  int4* buf; unsigned long long* out;
  cudaMalloc(&buf, 512ull << 20); cudaMalloc(&out, 4096 * 16);
  unsigned long long h[2 * 148];
  const char* names[] = {"acq_rel.gpu", "acq_rel.sys", "sc.sys", "sc.gpu"};
  for (int nst : {0, 1, 4, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      for (int rep = 0; rep < 3; ++rep) {
        if (mode == 0) k<0><<<128, 512>>>(buf, nst, out);
        if (mode == 1) k<1><<<128, 512>>>(buf, nst, out);
        if (mode == 2) k<2><<<128, 512>>>(buf, nst, out);
        if (mode == 3) k<3><<<128, 512>>>(buf, nst, out);
      }
      cudaMemcpy(h, out, sizeof(unsigned long long) * 2 * 128, cudaMemcpyDeviceToHost);
      double st = 0, fe = 0;
      for (int b = 0; b < 128; ++b) { st += h[2 * b]; fe += h[2 * b + 1]; }
      printf("stores/thread=%2d %-12s store-phase %7.0f ns  fence %7.0f ns (avg over CTAs)\n", nst, names[mode], st / 128, fe / 128);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
