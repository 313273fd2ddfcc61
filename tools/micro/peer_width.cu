// NVLink peer-write micro: does the store width (16 B vs 32 B per thread)
// or the number of bytes in flight per warp change the time to move a
// decode-sized buffer from cuda:0 HBM into cuda:1 HBM?  Kernel time with
// CUDA events (host ahead of the GPU behind a spin kernel), median of 20.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/peer_width tools/micro/peer_width.cu
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

// W = bytes per store (16 or 32); U = stores in flight per thread per pass
template <int W, int U>
__global__ void __launch_bounds__(512, 1) copy(const uint8_t* __restrict__ s, uint8_t* d, size_t n) {
  const size_t nv = n / W;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  for (size_t b = tid; b < nv; b += nt * U) {
    if constexpr (W == 16) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) if (b + u * nt < nv) v[u] = reinterpret_cast<const uint4*>(s)[b + u * nt];
#pragma unroll
      for (int u = 0; u < U; ++u) if (b + u * nt < nv) reinterpret_cast<uint4*>(d)[b + u * nt] = v[u];
    } else {
      uint32_t r[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (b + u * nt < nv) {
          const uint8_t* p = s + (b + u * nt) * 32;
          asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                         "=r"(r[u][6]), "=r"(r[u][7]) : "l"(p));
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (b + u * nt < nv) {
          uint8_t* q = d + (b + u * nt) * 32;
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(q), "r"(r[u][0]), "r"(r[u][1]),
                       "r"(r[u][2]), "r"(r[u][3]), "r"(r[u][4]), "r"(r[u][5]), "r"(r[u][6]), "r"(r[u][7]) : "memory");
        }
    }
  }
}

// one warp per 8-KiB page: page p of the source to slot perm[p] of the peer
// buffer (the KV stream's access pattern without its step loop)
__global__ void __launch_bounds__(256, 1) pages(const uint8_t* __restrict__ s, uint8_t* d, const int* perm, int np) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < np; p += nw) {
    const uint4* sp = reinterpret_cast<const uint4*>(s + (size_t)p * 8192);
    uint4* dp = reinterpret_cast<uint4*>(d + (size_t)perm[p] * 8192);
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = sp[lane + 32 * u];
#pragma unroll
    for (int u = 0; u < 16; ++u) dp[lane + 32 * u] = v[u];
  }
}

__global__ void __launch_bounds__(256, 1) pages2(const uint8_t* __restrict__ s, uint8_t* d, const int* sperm,
                                                 const int* perm, int np) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < np; p += nw) {
    const uint4* sp = reinterpret_cast<const uint4*>(s + (size_t)sperm[p] * 8192);
    uint4* dp = reinterpret_cast<uint4*>(d + (size_t)perm[p] * 8192);
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = sp[lane + 32 * u];
#pragma unroll
    for (int u = 0; u < 16; ++u) dp[lane + 32 * u] = v[u];
  }
}

template <typename F>
static float timed(F launch, cudaStream_t st) {
  std::vector<float> ts;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 23; ++k) {
    spin<<<1, 1, 0, st>>>(50000);
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
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  size_t sizes[] = {3784704, 7340032, 16777216, 67108864};
  printf("# peer write cuda:0 -> cuda:%d, grid %d x 512, us (median of 20)\n", peer, sms);
  printf("%12s %10s %10s %10s %10s %10s\n", "bytes", "16Bx4", "16Bx8", "32Bx2", "32Bx4", "CE");
  for (size_t nb : sizes) {
    uint8_t *s, *d;
    cudaSetDevice(0); cudaMalloc(&s, nb); cudaMemset(s, 3, nb);
    cudaSetDevice(peer); cudaMalloc(&d, nb);
    cudaSetDevice(0);
    float a = timed([&] { copy<16, 4><<<sms, 512, 0, st>>>(s, d, nb); }, st);
    float b = timed([&] { copy<16, 8><<<sms, 512, 0, st>>>(s, d, nb); }, st);
    float c = timed([&] { copy<32, 2><<<sms, 512, 0, st>>>(s, d, nb); }, st);
    float e = timed([&] { copy<32, 4><<<sms, 512, 0, st>>>(s, d, nb); }, st);
    float ce = timed([&] { cudaMemcpyPeerAsync(d, peer, s, 0, nb, st); }, st);
    printf("%12zu %10.2f %10.2f %10.2f %10.2f %10.2f   (GB/s at best %.0f)\n", nb, a, b, c, e, ce,
           nb / (std::min(std::min(a, b), std::min(c, e)) * 1e-6) / 1e9);
    cudaFree(s); cudaSetDevice(peer); cudaFree(d); cudaSetDevice(0);
  }
  // grid-size sweep: is the peer-write rate set per SM (store injection)?
  printf("# grid sweep, 16Bx4, 512 threads per CTA, us (median of 20)\n%12s", "bytes");
  const int grids[] = {32, 64, 96, 128, 148, 296};
  for (int g : grids) printf(" %9d", g);
  printf("\n");
  for (size_t nb : {(size_t)3784704, (size_t)67108864}) {
    uint8_t *s, *d;
    cudaSetDevice(0); cudaMalloc(&s, nb); cudaMemset(s, 3, nb);
    cudaSetDevice(peer); cudaMalloc(&d, nb);
    cudaSetDevice(0);
    printf("%12zu", nb);
    for (int g : grids) printf(" %9.2f", timed([&] { copy<16, 4><<<g, 512, 0, st>>>(s, d, nb); }, st));
    printf("\n");
    cudaFree(s); cudaSetDevice(peer); cudaFree(d); cudaSetDevice(0);
  }
  // SM copy and copy engine at once, each on half of 256 MB (two streams):
  // is 655 GB/s a per-engine limit or the link's?
  {
    const size_t nb = 256ull << 20, half = nb / 2;
    uint8_t *s, *d;
    cudaSetDevice(0); cudaMalloc(&s, nb); cudaMemset(s, 3, nb);
    cudaSetDevice(peer); cudaMalloc(&d, nb);
    cudaSetDevice(0);
    cudaStream_t st2; cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, j; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&j);
    std::vector<float> tb, ts, tc;
    for (int k = 0; k < 13; ++k) {
      spin<<<1, 1, 0, st>>>(50000);
      cudaEventRecord(e0, st);
      cudaStreamWaitEvent(st2, e0, 0);
      copy<16, 4><<<sms, 512, 0, st>>>(s, d, half);
      cudaMemcpyPeerAsync(d + half, peer, s + half, 0, half, st2);
      cudaEventRecord(j, st2);
      cudaStreamWaitEvent(st, j, 0);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (k >= 3) tb.push_back(ms * 1e3f);
    }
    float t_sm = timed([&] { copy<16, 4><<<sms, 512, 0, st>>>(s, d, nb); }, st);
    float t_ce = timed([&] { cudaMemcpyPeerAsync(d, peer, s, 0, nb, st); }, st);
    std::sort(tb.begin(), tb.end());
    printf("# 256 MB to the peer: SM copy %.1f us (%.0f GB/s), copy engine %.1f us (%.0f GB/s), "
           "half each at once %.1f us (%.0f GB/s)\n", t_sm, nb / (t_sm * 1e-6) / 1e9, t_ce,
           nb / (t_ce * 1e-6) / 1e9, tb[tb.size() / 2], nb / (tb[tb.size() / 2] * 1e-6) / 1e9);
  }
  // scattered 8-KiB pages: 256 MB as 32768 pages into a 1 GiB peer pool
  {
    const int np = 32768;
    uint8_t *s, *d;
    cudaSetDevice(0); cudaMalloc(&s, (size_t)np * 8192); cudaMemset(s, 3, (size_t)np * 8192);
    cudaSetDevice(peer); cudaMalloc(&d, 4ull * np * 8192);
    cudaSetDevice(0);
    std::vector<int> h(4 * np);
    for (int i = 0; i < 4 * np; ++i) h[i] = i;
    std::mt19937 rng(3); std::shuffle(h.begin(), h.end(), rng);
    int* perm; cudaMalloc(&perm, np * sizeof(int));
    cudaMemcpy(perm, h.data(), np * sizeof(int), cudaMemcpyHostToDevice);
    std::vector<int> seq(np); for (int i = 0; i < np; ++i) seq[i] = i;
    int* ident; cudaMalloc(&ident, np * sizeof(int));
    cudaMemcpy(ident, seq.data(), np * sizeof(int), cudaMemcpyHostToDevice);
    const double nb = (double)np * 8192;
    // and over a 10 GiB pool (the KV request's size): 256 MB into slots
    // spread over 10 GiB of the peer, sources spread over 10 GiB locally
    {
      const size_t big = 10ull << 30;
      uint8_t *sb, *db;
      cudaSetDevice(0); cudaMalloc(&sb, big);
      cudaSetDevice(peer); cudaMalloc(&db, big);
      cudaSetDevice(0);
      const int nslots = (int)(big / 8192);
      std::vector<int> hs(nslots);
      for (int i = 0; i < nslots; ++i) hs[i] = i;
      std::shuffle(hs.begin(), hs.end(), rng);
      int* pb; cudaMalloc(&pb, np * sizeof(int));
      cudaMemcpy(pb, hs.data(), np * sizeof(int), cudaMemcpyHostToDevice);
      float tb = timed([&] { pages<<<sms, 256, 0, st>>>(s, db, pb, np); }, st);
      printf("# 256 MB as 8-KiB pages into random slots of a 10 GiB peer pool: %.1f us (%.0f GB/s)\n", tb,
             nb / (tb * 1e-6) / 1e9);
      std::shuffle(hs.begin(), hs.end(), rng);
      int* sp2; cudaMalloc(&sp2, np * sizeof(int));
      cudaMemcpy(sp2, hs.data(), np * sizeof(int), cudaMemcpyHostToDevice);
      float tb2 = timed([&] { pages2<<<sms, 256, 0, st>>>(sb, db, sp2, pb, np); }, st);
      printf("# ... and from random pages of a 10 GiB local pool: %.1f us (%.0f GB/s)\n", tb2,
             nb / (tb2 * 1e-6) / 1e9);
      // the whole 10 GiB (the KV request's duration), contiguous pages in order
      {
        const int nall = (int)(big / 8192);
        std::vector<int> id(nall); for (int i = 0; i < nall; ++i) id[i] = i;
        int* pid; cudaMalloc(&pid, (size_t)nall * sizeof(int));
        cudaMemcpy(pid, id.data(), (size_t)nall * sizeof(int), cudaMemcpyHostToDevice);
        std::vector<float> tt;
        for (int k = 0; k < 4; ++k) {
          cudaEvent_t a0, a1; cudaEventCreate(&a0); cudaEventCreate(&a1);
          cudaEventRecord(a0, st);
          pages2<<<sms, 256, 0, st>>>(sb, db, pid, pid, nall);
          cudaEventRecord(a1, st);
          cudaStreamSynchronize(st);
          float ms; cudaEventElapsedTime(&ms, a0, a1); tt.push_back(ms);
        }
        std::sort(tt.begin(), tt.end());
        printf("# the whole 10 GiB as 8-KiB pages in one pass: %.2f ms (%.0f GB/s)\n", tt[1],
               (double)big / (tt[1] * 1e-3) / 1e9);
      }
      cudaFree(sb); cudaSetDevice(peer); cudaFree(db); cudaSetDevice(0);
    }
    for (int g : {sms, 2 * sms}) {
      float tr = timed([&] { pages<<<g, 256, 0, st>>>(s, d, perm, np); }, st);
      float ti = timed([&] { pages<<<g, 256, 0, st>>>(s, d, ident, np); }, st);
      printf("# 256 MB as 8-KiB pages, one warp each, grid %d x 256: random slots %.1f us (%.0f GB/s), "
             "in order %.1f us (%.0f GB/s)\n", g, tr, nb / (tr * 1e-6) / 1e9, ti, nb / (ti * 1e-6) / 1e9);
    }
  }
  return 0;
}
