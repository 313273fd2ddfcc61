// NVLink peer-write micro for the dispatch's store pattern: 128 CTAs, one
// token row each held in registers (one 16-byte piece per thread), stored
// to `rpc` randomly placed rows of a peer buffer.  Question: does a row
// stride that is not a multiple of 128 B (the fp8 DSv3 row is 7168 + 224 =
// 7392 B) cost link throughput against a 128-B aligned stride (7424 B)?
// Kernel time with CUDA events (host ahead of the GPU behind a spin
// kernel), median of 20; with `fence`, each CTA ends with a system fence
// and a remote counter add, as the dispatch's signal does.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/peer_rows tools/micro/peer_rows.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void spin(long long ns) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0; while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}

__global__ void __launch_bounds__(512, 1) rows(const uint8_t* __restrict__ src, uint8_t* dst, const int* perm,
                                               int rpc, int row_bytes, int stride, int fence,
                                               unsigned long long* ctr, unsigned long long* span) {
  const int n16 = row_bytes / 16, t = threadIdx.x;
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  uint4 v = make_uint4(0, 0, 0, 0);
  if (t < n16) v = reinterpret_cast<const uint4*>(src + (size_t)blockIdx.x * row_bytes)[t];
  for (int k = 0; k < rpc; ++k) {
    const int r = perm[blockIdx.x * rpc + k];
    if (t < n16) *reinterpret_cast<uint4*>(dst + (size_t)r * stride + 16 * t) = v;
  }
  if (fence) {
    __syncthreads();
    if (t == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" :: "l"(ctr) : "memory");
    }
  }
  if (t == 0 && span) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    span[2 * blockIdx.x] = g0;
    span[2 * blockIdx.x + 1] = g1;
  }
}

// spin, optionally keeping the link busy: one thread stores 16 B into the
// peer buffer every ~`gap` ns while it spins
__global__ void spin_peer(long long ns, uint4* peer, long long gap) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0, last = t0; unsigned i = 0;
  while (t - t0 < ns) {
    if (peer && t - last >= gap) { peer[(i++) & 1023] = make_uint4(i, i, i, i); last = t; }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
}

static uint4* g_keep = nullptr;
static long long g_gap = 0;

// the dispatch token role's shape: 256 threads hold the row as two 16-byte
// chunks each; the CTA stores `rpc` remote and `lpc` local rows (local HBM)
__global__ void __launch_bounds__(512, 1) rows2(const uint8_t* __restrict__ src, uint8_t* dst, uint8_t* ldst,
                                                const int* perm, int rpc, int lpc, int row_bytes,
                                                unsigned long long* ctr, unsigned long long* span, int mode = 2,
                                                unsigned long long* lctr = nullptr) {
  const int n16 = row_bytes / 16, t = threadIdx.x - 256;
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (t >= 0) {
    uint4 v[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    for (int u = 0; u < 2; ++u)
      if (t + 256 * u < n16) v[u] = reinterpret_cast<const uint4*>(src + (size_t)blockIdx.x * row_bytes)[t + 256 * u];
    for (int u = 0; u < 2; ++u)
      if (t + 256 * u < n16)
        for (int k = 0; k < rpc + lpc; ++k) {
          const int r = perm[blockIdx.x * 8 + k];
          uint8_t* base = k < rpc ? dst : ldst;
          *reinterpret_cast<uint4*>(base + (size_t)r * row_bytes + 16 * (t + 256 * u)) = v[u];
        }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode >= 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (mode >= 2) asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" :: "l"(ctr) : "memory");
    if (mode >= 3) {
      asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" :: "l"(ctr + 1) : "memory");
      asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" :: "l"(lctr) : "memory");
      asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" :: "l"(lctr + 1) : "memory");
    }
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    span[2 * blockIdx.x] = g0;
    span[2 * blockIdx.x + 1] = g1;
  }
}

template <typename F>
static float timed(F launch, cudaStream_t st) {
  std::vector<float> ts;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 23; ++k) {
    spin_peer<<<1, 1, 0, st>>>(50000, g_keep, g_gap);
    cudaEventRecord(e0, st); launch(); cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (k >= 3) ts.push_back(ms * 1e3f);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main() {
  int n = 0; cudaGetDeviceCount(&n);
  const int peer = n > 1 ? 1 : 0;
  cudaSetDevice(0);
  if (peer) cudaDeviceEnablePeerAccess(1, 0);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int T = 128;
  uint8_t* src; cudaMalloc(&src, (size_t)T * 8192); cudaMemset(src, 5, (size_t)T * 8192);
  unsigned long long* ctr;
  cudaSetDevice(peer);
  uint8_t* dst; cudaMalloc(&dst, (size_t)T * 8 * 8192 + 4096);
  cudaMalloc(&ctr, 64); cudaMemset(ctr, 0, 64);
  cudaSetDevice(0);
  int* perm; cudaMalloc(&perm, T * 8 * sizeof(int));
  unsigned long long* span; cudaMalloc(&span, 2 * T * 8);
  uint4* keep; cudaSetDevice(peer); cudaMalloc(&keep, 1024 * 16); cudaSetDevice(0);
  for (long long gap : {0LL}) {
  g_keep = gap ? keep : nullptr; g_gap = gap;
  printf("## link keep-alive during the idle spin: %s (gap %lld ns)\n", gap ? "on" : "off", gap);
  printf("# 128 CTAs x 512 threads, one row per CTA in registers -> rpc rows of a cuda:%d buffer (random slots); us, median of 20\n", peer);
  printf("%4s %6s %7s %6s %9s %9s %8s %9s %8s\n", "rpc", "row", "stride", "fence", "MB", "us", "GB/s", "span_us", "GB/s");
  std::mt19937 rng(1);
  for (int rpc : {4, 6, 8}) {
    std::vector<int> h(T * rpc);
    for (int i = 0; i < T * rpc; ++i) h[i] = i;
    std::shuffle(h.begin(), h.end(), rng);
    cudaMemcpy(perm, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice);
    for (int row : {7392}) {
      for (int stride : {row}) {
        for (int fence : {0, 1}) {
          const float us = timed([&] { rows<<<T, 512, 0, st>>>(src, dst, perm, rpc, row, stride, fence, ctr, nullptr); }, st);
          // device-clock span: first CTA start -> last CTA end (after its fence)
          std::vector<double> sp;
          for (int k = 0; k < 20; ++k) {
            spin_peer<<<1, 1, 0, st>>>(50000, g_keep, g_gap);
            rows<<<T, 512, 0, st>>>(src, dst, perm, rpc, row, stride, fence, ctr, span);
            cudaStreamSynchronize(st);
            std::vector<unsigned long long> h(2 * T);
            cudaMemcpy(h.data(), span, 2 * T * 8, cudaMemcpyDeviceToHost);
            unsigned long long a = ~0ull, b = 0;
            for (int c = 0; c < T; ++c) { a = std::min(a, h[2 * c]); b = std::max(b, h[2 * c + 1]); }
            sp.push_back((b - a) / 1e3);
          }
          std::sort(sp.begin(), sp.end());
          const double mb = (double)T * rpc * row / 1e6;
          printf("%4d %6d %7d %6d %9.2f %9.2f %8.0f %9.2f %8.0f\n", rpc, row, stride, fence, mb, us, mb * 1e3 / us,
                 sp[10], mb * 1e3 / sp[10]);
        }
      }
    }
  }
  }
  if (peer) {
    // both directions at once: GPU 1 runs the same kernel into a buffer on
    // GPU 0 while GPU 0 writes into GPU 1 (an EP=2 dispatch does this)
    cudaSetDevice(1);
    cudaDeviceEnablePeerAccess(0, 0);
    cudaStream_t st1; cudaStreamCreateWithFlags(&st1, cudaStreamNonBlocking);
    uint8_t* src1; cudaMalloc(&src1, (size_t)T * 8192); cudaMemset(src1, 6, (size_t)T * 8192);
    int* perm1; cudaMalloc(&perm1, T * 8 * sizeof(int));
    unsigned long long* span1; cudaMalloc(&span1, 2 * T * 8);
    cudaSetDevice(0);
    uint8_t* dst0; cudaMalloc(&dst0, (size_t)T * 8 * 8192 + 4096);
    unsigned long long* ctr0; cudaMalloc(&ctr0, 64);
    // a shared start flag on GPU 0: both spin kernels release together
    std::mt19937 rng2(2);
    printf("## bidirectional (GPU0 -> GPU1 and GPU1 -> GPU0 at once), fenced, device-clock span per direction\n");
    printf("%4s %9s %9s %9s\n", "rpc", "MB/dir", "span0_us", "span1_us");
    for (int rpc : {4, 6, 8}) {
      std::vector<int> h(T * rpc);
      for (int i = 0; i < T * rpc; ++i) h[i] = i;
      std::shuffle(h.begin(), h.end(), rng2);
      cudaMemcpy(perm, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice);
      cudaSetDevice(1); cudaMemcpy(perm1, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice); cudaSetDevice(0);
      std::vector<double> s0, s1;
      for (int k = 0; k < 20; ++k) {
        cudaSetDevice(0); spin_peer<<<1, 1, 0, st>>>(200000, nullptr, 0);
        cudaSetDevice(1); spin_peer<<<1, 1, 0, st1>>>(200000, nullptr, 0);
        cudaSetDevice(0); rows<<<T, 512, 0, st>>>(src, dst, perm, rpc, 7392, 7392, 1, ctr, span);
        cudaSetDevice(1); rows<<<T, 512, 0, st1>>>(src1, dst0, perm1, rpc, 7392, 7392, 1, ctr0, span1);
        cudaStreamSynchronize(st1); cudaSetDevice(0); cudaStreamSynchronize(st);
        for (int g = 0; g < 2; ++g) {
          std::vector<unsigned long long> hh(2 * T);
          if (g) cudaSetDevice(1);
          cudaMemcpy(hh.data(), g ? span1 : span, 2 * T * 8, cudaMemcpyDeviceToHost);
          cudaSetDevice(0);
          unsigned long long a = ~0ull, b = 0;
          for (int c = 0; c < T; ++c) { a = std::min(a, hh[2 * c]); b = std::max(b, hh[2 * c + 1]); }
          (g ? s1 : s0).push_back((b - a) / 1e3);
        }
      }
      std::sort(s0.begin(), s0.end()); std::sort(s1.begin(), s1.end());
      printf("%4d %9.2f %9.2f %9.2f\n", rpc, (double)T * rpc * 7392 / 1e6, s0[10], s1[10]);
    }
    // the dispatch's mix: 256 threads x 2 chunks, 4 remote + 4 local rows per CTA, both directions
    uint8_t* loc0; cudaMalloc(&loc0, (size_t)T * 8 * 8192);
    cudaSetDevice(1); uint8_t* loc1; cudaMalloc(&loc1, (size_t)T * 8 * 8192); cudaSetDevice(0);
    printf("## dispatch mix (256 thr x 2 chunks, rpc remote + lpc local rows per CTA, both directions); mode 0 no fence, 1 fence.sys, 2 + 1 remote red, 3 + 2 remote + 2 local reds\n");
    printf("%4s %4s %4s %9s %9s\n", "mode", "rpc", "lpc", "span0_us", "span1_us");
    unsigned long long* lc0; cudaMalloc(&lc0, 64);
    cudaSetDevice(1); unsigned long long* lc1; cudaMalloc(&lc1, 64); cudaSetDevice(0);
    for (int mode : {0, 1, 2, 3})
    for (int rl : {44, 80}) {
      const int rpc = rl / 10, lpc = rl % 10;
      std::vector<int> h(T * 8);
      for (int c = 0; c < T; ++c) for (int k = 0; k < 8; ++k) h[c * 8 + k] = k < rpc ? c * rpc + k : c * 8 + k;
      // remote slots shuffled
      cudaMemcpy(perm, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice);
      cudaSetDevice(1); cudaMemcpy(perm1, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice); cudaSetDevice(0);
      std::vector<double> s0, s1;
      for (int k = 0; k < 20; ++k) {
        cudaSetDevice(0); spin_peer<<<1, 1, 0, st>>>(200000, nullptr, 0);
        cudaSetDevice(1); spin_peer<<<1, 1, 0, st1>>>(200000, nullptr, 0);
        cudaSetDevice(0); rows2<<<T, 512, 0, st>>>(src, dst, loc0, perm, rpc, lpc, 7392, ctr, span, mode, lc0);
        cudaSetDevice(1); rows2<<<T, 512, 0, st1>>>(src1, dst0, loc1, perm1, rpc, lpc, 7392, ctr0, span1, mode, lc1);
        cudaStreamSynchronize(st1); cudaSetDevice(0); cudaStreamSynchronize(st);
        for (int g = 0; g < 2; ++g) {
          std::vector<unsigned long long> hh(2 * T);
          if (g) cudaSetDevice(1);
          cudaMemcpy(hh.data(), g ? span1 : span, 2 * T * 8, cudaMemcpyDeviceToHost);
          cudaSetDevice(0);
          unsigned long long a = ~0ull, b = 0;
          for (int c = 0; c < T; ++c) { a = std::min(a, hh[2 * c]); b = std::max(b, hh[2 * c + 1]); }
          (g ? s1 : s0).push_back((b - a) / 1e3);
        }
      }
      std::sort(s0.begin(), s0.end()); std::sort(s1.begin(), s1.end());
      printf("%4d %4d %4d %9.2f %9.2f   (max CTA end, us; p90 %.2f)\n", mode, rpc, lpc, s0[10], s1[10], s0[18]);
    }
  }
  return 0;
}
