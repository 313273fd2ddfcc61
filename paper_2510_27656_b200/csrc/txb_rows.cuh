// Row codecs shared by the MoE kernels and the standalone codec kernels:
// wire-row encode (encode_tokens, moe.py:231-246 / kernels.fp8_quantize,
// kernels.py:129-136) and the weighted combine (kernels.py:206-242).
#pragma once

#include "txb_common.cuh"

namespace txb {

constexpr int kMaxTopk = 64;

template <int SRC>
__device__ __forceinline__ void load_vals(const void* x, int64_t off, float* v, int cnt) {
  if constexpr (SRC == TXB_SRC_F32) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + off);
#pragma unroll
    for (int k = 0; k < cnt / 4; ++k) {
      const float4 a = p[k];
      v[4 * k] = a.x; v[4 * k + 1] = a.y; v[4 * k + 2] = a.z; v[4 * k + 3] = a.w;
    }
  } else {
    // bf16 -> f32 is exact (kernels.bf16_decode, kernels.py:153-154)
    const uint2* p = reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(x) + off);
#pragma unroll
    for (int k = 0; k < cnt / 4; ++k) {
      const uint2 a = p[k];
      v[4 * k] = __uint_as_float(a.x << 16);
      v[4 * k + 1] = __uint_as_float(a.x & 0xFFFF0000u);
      v[4 * k + 2] = __uint_as_float(a.y << 16);
      v[4 * k + 3] = __uint_as_float(a.y & 0xFFFF0000u);
    }
  }
}

__device__ __forceinline__ float load_val(const void* x, int src, int64_t off) {
  return src == TXB_SRC_F32 ? reinterpret_cast<const float*>(x)[off]
                            : bf16_to_f(reinterpret_cast<const uint16_t*>(x)[off]);
}

// Encode one token row (values -> wire row) and store it to `nd` destination
// rows.  ELEM: 1 fp8 (per-row scale), 2 bf16, 4 f32.  The data part is
// produced in 16-byte chunks when hidden*ELEM is a multiple of 16 and the
// source is 16-byte aligned; otherwise element by element.
template <int SRC, int ELEM>
__device__ void encode_store_row(const void* x, int64_t t, int H, int scales, int64_t P,
                                 uint8_t* const* dst, int nd, float* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t rowoff = t * (int64_t)H;
  float scale = 1.0f;
  if (ELEM == 1) {
    float amax = 0.f;
    for (int h = tid; h < H; h += nt) {
      const float v = load_val(x, SRC, rowoff + h);
      if (isfinite(v)) amax = fmaxf(amax, fabsf(v));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((tid & 31) == 0) red[tid >> 5] = amax;
    __syncthreads();
    if (tid < 32) {
      float a = tid < (nt >> 5) ? red[tid] : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
      if (tid == 0) red[32] = a;
    }
    __syncthreads();
    amax = red[32];
    scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;  // kernels.py:133-134
  }
  constexpr int EPC = 16 / ELEM;  // elements per 16-byte output chunk
  const int64_t srcbytes = (SRC == TXB_SRC_F32 ? 4 : 2);
  // 16-byte output chunks need 16-byte aligned destination rows (P % 16) and
  // an aligned source chunk (4 or more source elements per load)
  const int64_t salign = (EPC * srcbytes) >= 16 ? 16 : EPC * srcbytes;
  const bool vec = ((H * ELEM) % 16 == 0) && (P % 16 == 0) &&
                   (((reinterpret_cast<uintptr_t>(x) + rowoff * srcbytes) % salign) == 0);
  if (vec) {
    const int nchunk = H / EPC;
    for (int c = tid; c < nchunk; c += nt) {
      float v[EPC];
      load_vals<SRC>(x, rowoff + (int64_t)c * EPC, v, EPC);
      uint4 o;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
      if (ELEM == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t lo = fp8x2(__fdiv_rn(v[4 * q], scale), __fdiv_rn(v[4 * q + 1], scale));
          const uint32_t hi = fp8x2(__fdiv_rn(v[4 * q + 2], scale), __fdiv_rn(v[4 * q + 3], scale));
          ow[q] = lo | (hi << 16);
        }
      } else if (ELEM == 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) ow[q] = (uint32_t)bf16_rne(v[2 * q]) | ((uint32_t)bf16_rne(v[2 * q + 1]) << 16);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) ow[q] = __float_as_uint(v[q]);
      }
      for (int j = 0; j < nd; ++j) reinterpret_cast<uint4*>(dst[j])[c] = o;
    }
  } else {
    for (int h = tid; h < H; h += nt) {
      const float v = load_val(x, SRC, rowoff + h);
      for (int j = 0; j < nd; ++j) {
        if (ELEM == 1) {
          dst[j][h] = (uint8_t)(fp8x2(__fdiv_rn(v, scale), 0.f) & 0xFF);
        } else if (ELEM == 2) {
          const uint16_t b = bf16_rne(v);
          dst[j][2 * h] = (uint8_t)(b & 0xFF);
          dst[j][2 * h + 1] = (uint8_t)(b >> 8);
        } else {
          const uint32_t b = __float_as_uint(v);
          for (int q = 0; q < 4; ++q) dst[j][4 * h + q] = (uint8_t)(b >> (8 * q));
        }
      }
    }
  }
  // scale slots: f32 scale in slot 0 for fp8, all other bytes zero (moe.py:241-245)
  const int tailb = 4 * scales;
  if (tailb) {
    const int64_t d0 = (int64_t)H * ELEM;
    const uint32_t sbits = ELEM == 1 ? __float_as_uint(scale) : 0u;
    for (int b = tid; b < tailb; b += nt) {
      const uint8_t val = b < 4 ? (uint8_t)(sbits >> (8 * b)) : (uint8_t)0;
      for (int j = 0; j < nd; ++j) dst[j][d0 + b] = val;
    }
  }
}

template <int ELEM>
__device__ __forceinline__ void load8(const uint8_t* row, int64_t h0, float* v) {
  if (ELEM == 1) {
    const uint2 b = *reinterpret_cast<const uint2*>(row + h0);
    const uint32_t w[2] = {b.x, b.y};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float2 lo = fp8x2_to_f2((uint16_t)(w[q] & 0xFFFF));
      const float2 hi = fp8x2_to_f2((uint16_t)(w[q] >> 16));
      v[4 * q] = lo.x; v[4 * q + 1] = lo.y; v[4 * q + 2] = hi.x; v[4 * q + 3] = hi.y;
    }
  } else if (ELEM == 2) {
    const uint4 b = *reinterpret_cast<const uint4*>(row + 2 * h0);
    const uint32_t w[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[2 * q] = __uint_as_float(w[q] << 16);
      v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
    }
  } else {
    const float4 a = *reinterpret_cast<const float4*>(row + 4 * h0);
    const float4 b = *reinterpret_cast<const float4*>(row + 4 * h0 + 16);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <int ELEM>
__device__ __forceinline__ float load1(const uint8_t* row, int64_t h) {
  if (ELEM == 1) {
    const uint8_t b = row[h];
    return fp8x2_to_f2((uint16_t)b).x;
  } else if (ELEM == 2) {
    return bf16_to_f((uint16_t)(row[2 * h] | (row[2 * h + 1] << 8)));
  } else {
    uint32_t u = 0;
    for (int q = 0; q < 4; ++q) u |= (uint32_t)row[4 * h + q] << (8 * q);
    return __uint_as_float(u);
  }
}

// out[t] = sum_j w[t,j] * y[pos[t,j]], j ascending from 0.0, separately rounded
// multiply and add (kernels.py:214-226); fp8 rows are dequantised first as
// e4m3 * f32 scale (kernels.py:139-141).
template <int ELEM>
__device__ void combine_rows(const uint8_t* base, int64_t Pc, int H, const int64_t* pos, const float* w,
                             int64_t n, int R, void* out, int out_bf16) {
  __shared__ const uint8_t* rowp[kMaxTopk];
  __shared__ float ws[kMaxTopk];
  __shared__ float sc[kMaxTopk];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (tid < R) {
      const int64_t p = pos[t * R + tid];
      rowp[tid] = base + p * Pc;
      ws[tid] = w[t * R + tid];
      float scale = 1.f;
      if (ELEM == 1) {
        const uint8_t* sp = base + p * Pc + H;
        uint32_t u = (uint32_t)sp[0] | ((uint32_t)sp[1] << 8) | ((uint32_t)sp[2] << 16) | ((uint32_t)sp[3] << 24);
        scale = __uint_as_float(u);
      }
      sc[tid] = scale;
    }
    __syncthreads();
    const bool vec = (H % 8 == 0) && ((Pc & 15) == 0) && ((reinterpret_cast<uintptr_t>(base) & 15) == 0);
    if (vec) {
      for (int c = tid; c < H / 8; c += nt) {
        float acc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = 0.f;
        for (int j = 0; j < R; ++j) {
          float v[8];
          load8<ELEM>(rowp[j], (int64_t)c * 8, v);
          const float wj = ws[j], sj = sc[j];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float y = ELEM == 1 ? __fmul_rn(v[k], sj) : v[k];
            acc[k] = __fadd_rn(acc[k], __fmul_rn(wj, y));
          }
        }
        if (out_bf16) {
          uint4 o;
          uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
          for (int q = 0; q < 4; ++q) ow[q] = (uint32_t)bf16_rne(acc[2 * q]) | ((uint32_t)bf16_rne(acc[2 * q + 1]) << 16);
          reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(out) + t * H)[c] = o;
        } else {
          float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + t * H) + 2 * c;
          o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
      }
    } else {
      for (int h = tid; h < H; h += nt) {
        float acc = 0.f;
        for (int j = 0; j < R; ++j) {
          const float v = load1<ELEM>(rowp[j], h);
          const float y = ELEM == 1 ? __fmul_rn(v, sc[j]) : v;
          acc = __fadd_rn(acc, __fmul_rn(ws[j], y));
        }
        if (out_bf16) reinterpret_cast<uint16_t*>(out)[t * H + h] = bf16_rne(acc);
        else reinterpret_cast<float*>(out)[t * H + h] = acc;
      }
    }
    __syncthreads();
  }
}

}  // namespace txb
