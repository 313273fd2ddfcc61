// Generic WriteImm + ImmCounter primitives over NVLink peer memory: the
// B200 form of TransferEngine.submit_single_write / submit_paged_writes /
// submit_scatter / submit_barrier / expect_imm_count (engine.py:397-619,
// 138-205) and the data path of the paged KV-cache transfer (kvcache.py:
// 477-507) and the RL weight publication (weights.py:370-387, 570-590).
//
// A write is a list of pages (page i: src_base + src_offset + src_idx[i] *
// src_stride -> dst_base + dst_offset + dst_idx[i] * dst_stride, page_len
// bytes).  Pages are cut into pieces of at most kPiece bytes; CTAs take
// pieces round-robin and move them with TMA bulk copies (cp.async.bulk
// global -> shared -> global, mbarrier-tracked, double buffered) when the
// addresses are 16-byte aligned, 16-byte vector copies otherwise.  When the
// last CTA has finished (ticket), it releases one increment on the
// destination's ImmCounter slot -- exactly once per operation and only
// after the whole payload is visible, as engine.py:9-17 requires.
#include "txb_common.cuh"
#include "txb_tma.cuh"

namespace txb {

constexpr int kCopyThreads = 256;
constexpr int kPiece = 16 * 1024;  // bytes per TMA piece (one smem stage)
constexpr int kStages = 8;

struct PieceRef {
  const uint8_t* src;
  uint8_t* dst;
  uint32_t bytes;
};

__device__ __forceinline__ PieceRef piece_of(const txb_pages& j, int64_t k, int64_t per_page) {
  const int64_t page = k / per_page, piece = k - page * per_page;
  const int64_t si = j.src_idx ? j.src_idx[page] : page;
  const int64_t di = j.dst_idx ? j.dst_idx[page] : page;
  const int64_t off = piece * kPiece;
  const int64_t rem = j.page_len - off;
  PieceRef p;
  p.src = reinterpret_cast<const uint8_t*>(j.src_base) + j.src_offset + si * j.src_stride + off;
  p.dst = reinterpret_cast<uint8_t*>(j.dst_base) + j.dst_offset + di * j.dst_stride + off;
  p.bytes = (uint32_t)(rem < kPiece ? rem : kPiece);
  return p;
}

__global__ void __launch_bounds__(kCopyThreads, 1) k_copy_pages(txb_pages j) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t last;
  const int64_t per_page = (j.page_len + kPiece - 1) / kPiece;
  const int64_t total = j.npages * per_page;
  const bool tma = j.use_tma != 0;
  if (tma) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // thread 0 drives a kStages-deep TMA pipeline over this CTA's pieces
    if (threadIdx.x == 0) {
      uint32_t phase[kStages] = {};
      const int64_t k0 = blockIdx.x;
      // prologue: fill the stages
      for (int s = 0; s < kStages && k0 + (int64_t)s * gridDim.x < total; ++s) {
        const PieceRef p = piece_of(j, k0 + (int64_t)s * gridDim.x, per_page);
        mbar_expect_tx(&bars[s], p.bytes);
        tma_load(stage + s * kPiece, p.src, p.bytes, &bars[s]);
      }
      for (int64_t it = 0, k = k0; k < total; ++it, k += gridDim.x) {
        const int s = (int)(it % kStages);
        const PieceRef p = piece_of(j, k, per_page);
        mbar_wait(&bars[s], phase[s]);
        phase[s] ^= 1u;
        tma_store(p.dst, stage + s * kPiece, p.bytes);
        const int64_t kn = k + (int64_t)kStages * gridDim.x;
        if (kn < total) {
          tma_store_wait_read<kStages>();  // the stage stored kStages-1 pieces ago is free
          const PieceRef q = piece_of(j, kn, per_page);
          mbar_expect_tx(&bars[s], q.bytes);
          tma_load(stage + s * kPiece, q.src, q.bytes, &bars[s]);
        }
      }
      tma_store_wait_all();
      // order the async-proxy global writes before the generic release below
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  } else {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t k = (int64_t)blockIdx.x * nw + warp; k < total; k += (int64_t)gridDim.x * nw) {
      const PieceRef p = piece_of(j, k, per_page);
      const int w = vec_width(p.src, p.dst, p.bytes);
      if (w == 16) {
        // a whole 16-KiB piece is 32 int4 per lane: all loads in flight
        // before the first store
        const int4* s = reinterpret_cast<const int4*>(p.src);
        int4* d = reinterpret_cast<int4*>(p.dst);
        const int nv = (int)(p.bytes >> 4);
        constexpr int U = kPiece / 512;
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (lane + 32 * u < nv) v[u] = s[lane + 32 * u];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (lane + 32 * u < nv) d[lane + 32 * u] = v[u];
      } else {
        copy_row(p.dst, p.src, p.bytes, lane, 32);
      }
    }
  }
  // completion: the last CTA releases one increment on the ImmCounter slot
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_release(j.single_device != 0);
    last = (atomicAdd(j.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *j.ticket = 0;
    if (j.imm_ctr) {
      fence_release(j.single_device != 0);
      red_relaxed_sys_add(j.imm_ctr, 1);
    }
  }
}

// Zero-length write carrying an immediate (barrier leg, engine.py:599-619).
__global__ void k_imm_add(uint64_t* const* ctrs, int n, uint64_t v, int single_device) {
  if (threadIdx.x == 0) fence_release(single_device != 0);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) red_relaxed_sys_add(ctrs[i], v);
}

// Device-side expectation: block the stream until *ctr >= threshold (the
// consumer-side ImmFlag for GPU work queued behind it).
__global__ void k_imm_wait(const uint64_t* ctr, uint64_t threshold, uint64_t timeout_ns, uint32_t* err) {
  if (threadIdx.x == 0) {
    const uint64_t dl = globaltimer() + timeout_ns;
    if (!spin_ge(ctr, threshold, dl) && err) atomicOr(err, TXB_EV_WAIT_IMM);
  }
}

// Device clock sample (%globaltimer, ns) into *out: brackets a stream's
// work in the same clock domain as the kernels' phase stamps.
__global__ void k_globaltimer(uint64_t* out) {
  if (threadIdx.x == 0) *out = globaltimer();
}

// Per-tensor fp8 quantisation of bf16 words (weights.prepare narrowing,
// weights.py:383-387 -> kernels.fp8_quantize over the whole tensor):
// pass 1 reduces amax over finite values into *amax_bits (non-negative
// floats order like their bit patterns), pass 2 encodes with
// scale = amax/448 (1.0 when 0) and writes the f32 scale footer.
__global__ void k_amax_bf16(const uint16_t* __restrict__ x, int64_t n, uint32_t* amax_bits) {
  float m = 0.f;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t n8 = vec ? n / 8 : 0;
  // 16-byte loads, two in flight per thread per pass
  for (int64_t c = tid; c < n8; c += 2 * nthr) {
    uint4 v[2];
    v[0] = reinterpret_cast<const uint4*>(x)[c];
    if (c + nthr < n8) v[1] = reinterpret_cast<const uint4*>(x)[c + nthr];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && c + nthr >= n8) break;
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[u]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = __uint_as_float(w[k] << 16), b = __uint_as_float(w[k] & 0xFFFF0000u);
        if (isfinite(a)) m = fmaxf(m, fabsf(a));
        if (isfinite(b)) m = fmaxf(m, fabsf(b));
      }
    }
  }
  for (int64_t i = 8 * n8 + tid; i < n; i += nthr) {
    const float v = bf16_to_f(x[i]);
    if (isfinite(v)) m = fmaxf(m, fabsf(v));
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, __float_as_uint(m));
}

// x / scale correctly rounded (div_rn_by: reciprocal multiply + two FMA
// corrections, bit-identical to the IEEE division), e4m3 RNE satfinite;
// 16-byte loads of 8 bf16, 8-byte stores of 8 fp8.
__global__ void k_quant_bf16_fp8(const uint16_t* __restrict__ x, int64_t n, const uint32_t* amax_bits,
                                 uint8_t* __restrict__ out) {
  const float amax = __uint_as_float(*amax_bits);
  const float scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  const float rs = __frcp_rn(scale);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && ((reinterpret_cast<uintptr_t>(out) & 7) == 0);
  const int64_t n8 = vec ? n / 8 : 0;
  for (int64_t c = tid; c < n8; c += nthr) {
    const uint4 v = reinterpret_cast<const uint4*>(x)[c];
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
    uint32_t o[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float f0 = __uint_as_float(w[2 * q] << 16), f1 = __uint_as_float(w[2 * q] & 0xFFFF0000u);
      const float f2 = __uint_as_float(w[2 * q + 1] << 16), f3 = __uint_as_float(w[2 * q + 1] & 0xFFFF0000u);
      o[q] = fp8x2(div_rn_by(f0, scale, rs), div_rn_by(f1, scale, rs)) |
             (fp8x2(div_rn_by(f2, scale, rs), div_rn_by(f3, scale, rs)) << 16);
    }
    reinterpret_cast<uint2*>(out)[c] = make_uint2(o[0], o[1]);
  }
  for (int64_t i = 8 * n8 + tid; i < n; i += nthr)
    out[i] = (uint8_t)(fp8x2(div_rn_by(bf16_to_f(x[i]), scale, rs), 0.f) & 0xFF);
  if (blockIdx.x == 0 && threadIdx.x < 4) out[n + threadIdx.x] = (uint8_t)(__float_as_uint(scale) >> (8 * threadIdx.x));
}

static int sms(int) {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

}  // namespace txb

using namespace txb;

extern "C" {

int txb_imm_table_slots(void) { return TXB_IMM_SLOTS; }

int txb_copy_pages(const txb_pages* j, int grid, void* stream) {
  if (!j || !j->ticket) {
    set_error("txb_copy_pages: null job or ticket");
    return TXB_ERR_TRANSFER;
  }
  if (j->npages < 0 || j->page_len < 0) {
    set_error("negative page count or length");
    return TXB_ERR_TRANSFER;
  }
  DeviceFor on_dev(stream, j->src_base);
  txb_pages job = *j;
  const int64_t per_page = job.page_len > 0 ? (job.page_len + kPiece - 1) / kPiece : 0;
  const int64_t total = job.npages * per_page;
  if (grid <= 0) {
    const int64_t want = job.use_tma ? total : (total + 7) / 8;
    const int cap = sms(0);
    grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  }
  if (total == 0) job.npages = 0;
  const size_t smem = job.use_tma ? (size_t)kStages * kPiece : 0;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && (dev < 0 || dev >= 64 || !attr_set[dev])) {
    TXB_CUDA(cudaFuncSetAttribute(k_copy_pages, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kStages * kPiece)));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  k_copy_pages<<<grid, kCopyThreads, smem, (cudaStream_t)stream>>>(job);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_imm_add(uint64_t* const* ctrs, int n, uint64_t value, int single_device, void* stream) {
  DeviceFor on_dev(stream, ctrs);
  if (n <= 0) return TXB_OK;
  k_imm_add<<<1, 128, 0, (cudaStream_t)stream>>>(ctrs, n, value, single_device);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_imm_wait(const uint64_t* ctr, uint64_t threshold, uint64_t timeout_ns, uint32_t* err, void* stream) {
  DeviceFor on_dev(stream, ctr);
  k_imm_wait<<<1, 32, 0, (cudaStream_t)stream>>>(ctr, threshold, timeout_ns, err);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_globaltimer(uint64_t* out, void* stream) {
  DeviceFor on_dev(stream, out);
  k_globaltimer<<<1, 32, 0, (cudaStream_t)stream>>>(out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_fp8_quantize_tensor(const uint16_t* x, int64_t n, uint32_t* amax_scratch, uint8_t* out, void* stream) {
  DeviceFor on_dev(stream, x);
  cudaStream_t st = (cudaStream_t)stream;
  TXB_CUDA(cudaMemsetAsync(amax_scratch, 0, sizeof(uint32_t), st));
  int64_t g = (n + 255) / 256;
  const int grid = (int)(g < 1 ? 1 : (g > 4 * sms(0) ? 4 * sms(0) : g));
  k_amax_bf16<<<grid, 256, 0, st>>>(x, n, amax_scratch);
  k_quant_bf16_fp8<<<grid, 256, 0, st>>>(x, n, amax_scratch, out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

}  // extern "C"
