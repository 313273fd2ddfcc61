// Standalone codec kernels: the "cuda" entry of the reference kernel
// registry (kernels.implementations(), kernels.py:245-264) and the device
// versions of moe.encode_tokens / decode_tokens (moe.py:231-262).
#include "txb_rows.cuh"

namespace txb {

template <int SRC, int ELEM>
__global__ void __launch_bounds__(256, 1)
k_encode_rows(const void* __restrict__ x, int64_t n, int H, int scales, int64_t P, uint8_t* __restrict__ out) {
  __shared__ float red[33];
  __shared__ uint8_t* dst[1];
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (threadIdx.x == 0) dst[0] = out + t * P;
    __syncthreads();
    encode_store_row<SRC, ELEM>(x, t, H, scales, P, dst, 1, red);
    __syncthreads();
  }
}

template <int ELEM>
__global__ void __launch_bounds__(256, 1)
k_decode_rows(const uint8_t* __restrict__ rows, int64_t n, int H, int64_t P, float* __restrict__ out) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const uint8_t* r = rows + t * P;
    float scale = 1.f;
    if (ELEM == 1) {
      const uint8_t* sp = r + H;
      scale = __uint_as_float((uint32_t)sp[0] | ((uint32_t)sp[1] << 8) | ((uint32_t)sp[2] << 16) |
                              ((uint32_t)sp[3] << 24));
    }
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      float v;
      if (ELEM == 1) {
        v = __fmul_rn(fp8x2_to_f2((uint16_t)r[h]).x, scale);  // kernels.py:139-141
      } else if (ELEM == 2) {
        v = bf16_to_f((uint16_t)(r[2 * h] | (r[2 * h + 1] << 8)));
      } else {
        uint32_t u = 0;
        for (int q = 0; q < 4; ++q) u |= (uint32_t)r[4 * h + q] << (8 * q);
        v = __uint_as_float(u);
      }
      out[t * H + h] = v;
    }
  }
}

__global__ void __launch_bounds__(256, 1)
k_pack_rows(const uint8_t* __restrict__ src, int64_t width, const int64_t* __restrict__ rows, int64_t k,
            uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < k; i += nw)
    copy_row(out + i * width, src + rows[i] * width, width, lane, 32);
}

__global__ void __launch_bounds__(256, 1)
k_weighted_combine(const float* __restrict__ y, int64_t hidden, const int64_t* __restrict__ pos,
                   const float* __restrict__ w, int64_t n, int topk, float* __restrict__ out) {
  combine_rows<4>(reinterpret_cast<const uint8_t*>(y), hidden * 4, nullptr, 0, (int)hidden, pos, nullptr, w, n,
                  topk, out, 0, blockIdx.x, gridDim.x);
}

__global__ void k_fp8_encode(const float* __restrict__ x, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(fp8x2(x[i], 0.f) & 0xFF);
}

__global__ void k_fp8_decode(const uint8_t* __restrict__ b, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fp8x2_to_f2((uint16_t)b[i]).x;
}

__global__ void k_bf16_encode(const float* __restrict__ x, int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = bf16_rne(x[i]);
}

static int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 4096) g = 4096;
  return (int)g;
}

unsigned int check_failures_codec() {
#ifdef TXB_CHECKED
  return read_check_fail();
#else
  return 0;
#endif
}

cudaError_t preload_codec() {
  cudaError_t e = cudaSuccess;
  for (cudaError_t r : {touch(k_encode_rows<TXB_SRC_F32, 1>), touch(k_encode_rows<TXB_SRC_F32, 2>),
                        touch(k_encode_rows<TXB_SRC_F32, 4>), touch(k_encode_rows<TXB_SRC_BF16, 1>),
                        touch(k_encode_rows<TXB_SRC_BF16, 2>), touch(k_encode_rows<TXB_SRC_BF16, 4>),
                        touch(k_decode_rows<1>), touch(k_decode_rows<2>), touch(k_decode_rows<4>),
                        touch(k_pack_rows), touch(k_weighted_combine), touch(k_fp8_encode), touch(k_fp8_decode),
                        touch(k_bf16_encode)})
    if (r != cudaSuccess) e = r;
  return e;
}

}  // namespace txb

using namespace txb;

extern "C" {

int txb_encode_rows(const void* values, int src_kind, int64_t n, int32_t hidden, int32_t elem_size,
                    int32_t scales, void* out, void* stream) {
  DeviceFor on_dev(stream, out);
  if (n <= 0) return TXB_OK;
  if (elem_size == 1 && scales < 1) {
    set_error("quantized payloads need at least one scale slot");
    return TXB_ERR_PROTOCOL;
  }
  const int64_t P = (int64_t)hidden * elem_size + 4LL * scales;
  const int grid = grid_for(n, 1);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* o = (uint8_t*)out;
#define TXB_ENC(SRC, ELEM) k_encode_rows<SRC, ELEM><<<grid, 256, 0, st>>>(values, n, hidden, scales, P, o)
  const bool f32 = src_kind == TXB_SRC_F32;
  if (src_kind != TXB_SRC_F32 && src_kind != TXB_SRC_BF16) {
    set_error("encode source must be f32 or bf16 values");
    return TXB_ERR_PROTOCOL;
  }
  switch (elem_size) {
    case 1: if (f32) TXB_ENC(TXB_SRC_F32, 1); else TXB_ENC(TXB_SRC_BF16, 1); break;
    case 2: if (f32) TXB_ENC(TXB_SRC_F32, 2); else TXB_ENC(TXB_SRC_BF16, 2); break;
    case 4: if (f32) TXB_ENC(TXB_SRC_F32, 4); else TXB_ENC(TXB_SRC_BF16, 4); break;
    default: set_error("element size %d not in (1, 2, 4)", elem_size); return TXB_ERR_PROTOCOL;
  }
#undef TXB_ENC
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_decode_rows(const void* rows, int64_t n, int32_t hidden, int32_t elem_size, int32_t scales, float* out,
                    void* stream) {
  DeviceFor on_dev(stream, out);
  if (n <= 0) return TXB_OK;
  const int64_t P = (int64_t)hidden * elem_size + 4LL * scales;
  const int grid = grid_for(n, 1);
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* r = (const uint8_t*)rows;
  switch (elem_size) {
    case 1: k_decode_rows<1><<<grid, 256, 0, st>>>(r, n, hidden, P, out); break;
    case 2: k_decode_rows<2><<<grid, 256, 0, st>>>(r, n, hidden, P, out); break;
    case 4: k_decode_rows<4><<<grid, 256, 0, st>>>(r, n, hidden, P, out); break;
    default: set_error("element size %d not in (1, 2, 4)", elem_size); return TXB_ERR_PROTOCOL;
  }
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_pack_rows(const void* src, int64_t width, const int64_t* rows, int64_t k, void* out, void* stream) {
  DeviceFor on_dev(stream, out);
  if (k <= 0) return TXB_OK;
  k_pack_rows<<<grid_for(k, 8), 256, 0, (cudaStream_t)stream>>>((const uint8_t*)src, width, rows, k, (uint8_t*)out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_weighted_combine(const float* y, int64_t hidden, const int64_t* pos, const float* w, int64_t n, int32_t topk,
                         float* out, void* stream) {
  DeviceFor on_dev(stream, out);
  if (n <= 0) return TXB_OK;
  if (topk > kMaxTopk) {
    set_error("topk %d above the supported %d", topk, kMaxTopk);
    return TXB_ERR_PROTOCOL;
  }
  k_weighted_combine<<<grid_for(n, 1), 256, 0, (cudaStream_t)stream>>>(y, hidden, pos, w, n, topk, out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_fp8_encode(const float* x, int64_t n, uint8_t* out, void* stream) {
  DeviceFor on_dev(stream, out);
  if (n <= 0) return TXB_OK;
  k_fp8_encode<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, n, out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_fp8_decode(const uint8_t* b, int64_t n, float* out, void* stream) {
  DeviceFor on_dev(stream, out);
  if (n <= 0) return TXB_OK;
  k_fp8_decode<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(b, n, out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_bf16_encode(const float* x, int64_t n, uint16_t* out, void* stream) {
  DeviceFor on_dev(stream, out);
  if (n <= 0) return TXB_OK;
  k_bf16_encode<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, n, out);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

}  // extern "C"
