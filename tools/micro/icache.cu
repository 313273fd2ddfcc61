// Instruction-fetch cost of straight-line code run once per SM: a kernel
// with ~N KB of unrolled independent FADDs, timed with %globaltimer per CTA.
// Launch 1 after an L2 flush (cold), launch 2 right after (warm).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int N>
__global__ void k(float* out, unsigned long long* ts) {
  float a = threadIdx.x, b = 1.0f, c = 2.0f, d = 3.0f;
  uint64_t t0 = gt();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    asm volatile("add.f32 %0, %0, %1;" : "+f"(a) : "f"(b));
    asm volatile("add.f32 %0, %0, %1;" : "+f"(c) : "f"(d));
  }
  uint64_t t1 = gt();
  if (threadIdx.x == 0) ts[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + c;
}
int main() {
  float* out; unsigned long long* ts; char* flush;
  cudaMalloc(&out, 1 << 22); cudaMalloc(&ts, 4096 * 8); cudaMalloc(&flush, 512 << 20);
  unsigned long long h[148];
  auto run = [&](auto kern, const char* name, int ninstr) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      kern<<<148, 512>>>(out, ts);          // cold (after L2 flush)
      cudaMemcpy(h, ts, 148 * 8, cudaMemcpyDeviceToHost);
      double cold = 0; for (int i = 0; i < 148; ++i) cold += h[i]; cold /= 148;
      kern<<<148, 512>>>(out, ts);          // warm
      cudaMemcpy(h, ts, 148 * 8, cudaMemcpyDeviceToHost);
      double warm = 0; for (int i = 0; i < 148; ++i) warm += h[i]; warm /= 148;
      printf("%-10s ~%6d instr (%4d KB): cold %8.0f ns  warm %8.0f ns\n", name, ninstr, ninstr * 16 / 1024, cold, warm);
    }
  };
  run(k<512>, "1K", 1024);
  run(k<2048>, "4K", 4096);
  run(k<4096>, "8K", 8192);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
