// Row codecs shared by the MoE kernels and the standalone codec kernels:
// wire-row encode (encode_tokens, moe.py:231-246 / kernels.fp8_quantize,
// kernels.py:129-136) and the weighted combine (kernels.py:206-242).
#pragma once

#include "txb_common.cuh"

namespace txb {

constexpr int kMaxTopk = 64;

// Load `cnt` (multiple of 4) consecutive source values as f32.
template <int SRC>
__device__ __forceinline__ void load_vals(const void* x, int64_t off, float* v, int cnt) {
  if constexpr (SRC == TXB_SRC_F32) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + off);
#pragma unroll
    for (int k = 0; k < cnt / 4; ++k) {
      const float4 a = p[k];
      v[4 * k] = a.x; v[4 * k + 1] = a.y; v[4 * k + 2] = a.z; v[4 * k + 3] = a.w;
    }
  } else if (cnt % 8 == 0) {
    // bf16 -> f32 is exact (kernels.bf16_decode, kernels.py:153-154)
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(x) + off);
#pragma unroll
    for (int k = 0; k < cnt / 8; ++k) {
      const uint4 a = p[k];
      const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[8 * k + 2 * q] = __uint_as_float(w[q] << 16);
        v[8 * k + 2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
      }
    }
  } else {
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

// Block-wide max of non-negative floats; every thread gets the result.
__device__ __forceinline__ float block_max(float v, float* red, const Grp& g = Grp::cta()) {
  const int tid = g.tid, nt = g.nt;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((tid & 31) == 0) red[tid >> 5] = v;
  g.sync();
  if (tid < 32) {
    float a = tid < ((nt + 31) >> 5) ? red[tid] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (tid == 0) red[32] = a;
  }
  g.sync();
  const float r = red[32];
  g.sync();
  return r;
}

// One 16-byte output chunk from EPC = 16/ELEM values.
template <int ELEM>
__device__ __forceinline__ uint4 encode_chunk(const float* v, float scale) {
  uint4 o;
  uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
  if constexpr (ELEM == 1) {
    // x / f32(scale) correctly rounded, then e4m3 RNE satfinite
    const float rs = __frcp_rn(scale);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = fp8x2(div_rn_by(v[4 * q], scale, rs), div_rn_by(v[4 * q + 1], scale, rs));
      const uint32_t hi = fp8x2(div_rn_by(v[4 * q + 2], scale, rs), div_rn_by(v[4 * q + 3], scale, rs));
      ow[q] = lo | (hi << 16);
    }
  } else if constexpr (ELEM == 2) {
#pragma unroll
    for (int q = 0; q < 4; ++q) ow[q] = (uint32_t)bf16_rne(v[2 * q]) | ((uint32_t)bf16_rne(v[2 * q + 1]) << 16);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) ow[q] = __float_as_uint(v[q]);
  }
  return o;
}

// Encode one token row (values -> wire row) and store it to `nd` destination
// rows.  ELEM: 1 fp8 (per-row scale), 2 bf16, 4 f32.
//   fast path (hidden*ELEM % 16 == 0, 16-byte aligned rows, <= 2 chunks per
//   thread): the row is read from HBM once into registers, the per-row amax
//   is reduced across the block, and each 16-byte chunk is stored to all
//   destinations;
//   general path: element by element (arbitrary hidden / payload sizes).
template <int SRC, int ELEM>
__device__ __noinline__ void encode_store_row(const void* x, int64_t t, int H, int scales, int64_t P,
                                 uint8_t* const* dst, int nd, float* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t rowoff = t * (int64_t)H;
  constexpr int EPC = 16 / ELEM;  // elements per 16-byte output chunk
  const int64_t srcbytes = (SRC == TXB_SRC_F32 ? 4 : 2);
  const int64_t salign = (EPC * srcbytes) >= 16 ? 16 : EPC * srcbytes;
  const int nchunk = H / EPC;
  const bool vec = ((H * ELEM) % 16 == 0) && (P % 16 == 0) && nchunk <= 2 * nt &&
                   (((reinterpret_cast<uintptr_t>(x) + rowoff * srcbytes) % salign) == 0);
  float scale = 1.0f;
  if (vec) {
    float v[2][EPC];
    float amax = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = tid + u * nt;
      if (c < nchunk) {
        load_vals<SRC>(x, rowoff + (int64_t)c * EPC, v[u], EPC);
        if constexpr (ELEM == 1) {
#pragma unroll
          for (int k = 0; k < EPC; ++k)
            if (isfinite(v[u][k])) amax = fmaxf(amax, fabsf(v[u][k]));
        }
      }
    }
    if constexpr (ELEM == 1) {
      amax = block_max(amax, red);
      scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;  // kernels.py:133-134
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = tid + u * nt;
      if (c < nchunk) {
        const uint4 o = encode_chunk<ELEM>(v[u], scale);
        for (int j = 0; j < nd; ++j) reinterpret_cast<uint4*>(dst[j])[c] = o;
      }
    }
  } else {
    if constexpr (ELEM == 1) {
      float amax = 0.f;
      for (int h = tid; h < H; h += nt) {
        const float v = load_val(x, SRC, rowoff + h);
        if (isfinite(v)) amax = fmaxf(amax, fabsf(v));
      }
      amax = block_max(amax, red);
      scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;
    }
    for (int h = tid; h < H; h += nt) {
      const float v = load_val(x, SRC, rowoff + h);
      for (int j = 0; j < nd; ++j) {
        if constexpr (ELEM == 1) {
          dst[j][h] = (uint8_t)(fp8x2(__fdiv_rn(v, scale), 0.f) & 0xFF);
        } else if constexpr (ELEM == 2) {
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
    if ((d0 & 3) == 0) {
      for (int b = tid; b < scales; b += nt) {
        const uint32_t val = b == 0 ? sbits : 0u;
        for (int j = 0; j < nd; ++j) reinterpret_cast<uint32_t*>(dst[j] + d0)[b] = val;
      }
    } else {
      for (int b = tid; b < tailb; b += nt) {
        const uint8_t val = b < 4 ? (uint8_t)(sbits >> (8 * b)) : (uint8_t)0;
        for (int j = 0; j < nd; ++j) dst[j][d0 + b] = val;
      }
    }
  }
}

// Pre-encoded row held in registers: thread `tid` owns 16-byte chunks
// c = tid and c = tid + blockDim.x of the wire row.  Lets a kernel read and
// encode its token before the layout is known and store it afterwards.
struct RowRegs {
  uint4 c[2];
  float scale;
  int nchunk;  // chunks of the data part (values) or of the whole row (raw)
  bool ok;     // false: shape not eligible, use encode_store_row later
};

// A 16-byte global load the compiler keeps where it is written (asm
// volatile): the row loads are issued first so their HBM latency overlaps the
// work that follows, instead of being sunk next to their first use.
__device__ __forceinline__ uint4 ldg_pinned(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Raw source bytes of a thread's (up to) two chunks, loaded before they are
// needed so the HBM latency overlaps other work (route counting).
struct RowRaw {
  uint4 r[2][4];
  int nchunk;
  bool ok;
};

template <int SRC, int ELEM>
__device__ __forceinline__ void load_row_raw(const void* x, int64_t t, int H, int64_t P, RowRaw& rr,
                                             const Grp& g = Grp::cta()) {
  const int tid = g.tid, nt = g.nt;
  rr.ok = false;
  if constexpr (SRC == TXB_SRC_ROWS) {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(x) + t * P;
    rr.nchunk = (int)(P >> 4);
    if ((P & 15) || (reinterpret_cast<uintptr_t>(src) & 15) || rr.nchunk > 2 * nt) return;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = tid + u * nt;
      if (c < rr.nchunk) rr.r[u][0] = ldg_pinned(reinterpret_cast<const uint4*>(src) + c);
    }
  } else {
    constexpr int EPC = 16 / ELEM;
    constexpr int SB = SRC == TXB_SRC_F32 ? 4 : 2;  // source bytes per element
    constexpr int CB = EPC * SB;                     // source bytes per chunk (8..64)
    const int64_t rowoff = t * (int64_t)H;
    const int64_t salign = CB >= 16 ? 16 : CB;
    rr.nchunk = H / EPC;
    if (((H * ELEM) % 16) || (P % 16) || rr.nchunk > 2 * nt ||
        ((reinterpret_cast<uintptr_t>(x) + rowoff * SB) % salign))
      return;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(x) + rowoff * SB;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = tid + u * nt;
      if (c < rr.nchunk) {
        if constexpr (CB >= 16) {
#pragma unroll
          for (int k = 0; k < CB / 16; ++k) rr.r[u][k] = ldg_pinned(reinterpret_cast<const uint4*>(src + (int64_t)c * CB) + k);
        } else {
          const uint2 v = *reinterpret_cast<const uint2*>(src + (int64_t)c * CB);
          rr.r[u][0] = make_uint4(v.x, v.y, 0, 0);
        }
      }
    }
  }
  rr.ok = true;
}

// Finish a raw row into encoded chunks (per-row amax reduce for fp8).
template <int SRC, int ELEM>
__device__ void finish_row_regs(const RowRaw& rr, RowRegs& r, float* red, const Grp& g = Grp::cta()) {
  const int tid = g.tid, nt = g.nt;
  r.ok = rr.ok;
  r.nchunk = rr.nchunk;
  r.scale = 1.0f;
  if (!rr.ok) return;
  if constexpr (SRC == TXB_SRC_ROWS) {
    r.c[0] = rr.r[0][0];
    r.c[1] = rr.r[1][0];
  } else {
    constexpr int EPC = 16 / ELEM;
    float v[2][EPC];
    float amax = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&rr.r[u][0]);
#pragma unroll
      for (int k = 0; k < EPC; ++k) {
        if constexpr (SRC == TXB_SRC_F32) v[u][k] = __uint_as_float(w[k]);
        else v[u][k] = __uint_as_float((k & 1) ? (w[k >> 1] & 0xFFFF0000u) : (w[k >> 1] << 16));
      }
      if constexpr (ELEM == 1) {
        if (tid + u * nt < rr.nchunk) {
#pragma unroll
          for (int k = 0; k < EPC; ++k)
            if (isfinite(v[u][k])) amax = fmaxf(amax, fabsf(v[u][k]));
        }
      }
    }
    if constexpr (ELEM == 1) {
      amax = block_max(amax, red, g);
      r.scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;  // kernels.py:133-134
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (tid + u * nt < rr.nchunk) r.c[u] = encode_chunk<ELEM>(v[u], r.scale);
  }
}

// Store a RowRegs row to nd destination rows (plus the scale slots); null
// destinations are skipped (copies stored in another pass).
template <int SRC, int ELEM>
__device__ void store_row_regs(const RowRegs& r, int H, int scales, uint8_t* const* dst, int nd,
                               const Grp& g = Grp::cta()) {
  const int tid = g.tid, nt = g.nt;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = tid + u * nt;
    if (c < r.nchunk)
      for (int j = 0; j < nd; ++j)
        if (dst[j]) reinterpret_cast<uint4*>(dst[j])[c] = r.c[u];
  }
  if constexpr (SRC != TXB_SRC_ROWS) {
    const int64_t d0 = (int64_t)H * ELEM;  // 16-byte aligned on this path
    const uint32_t sbits = ELEM == 1 ? __float_as_uint(r.scale) : 0u;
    for (int b = tid; b < scales; b += nt)
      for (int j = 0; j < nd; ++j)
        if (dst[j]) reinterpret_cast<uint32_t*>(dst[j] + d0)[b] = b == 0 ? sbits : 0u;
  }
}

// ----------------------------------------------------------------- combine

// Raw 8-element chunk of one wire row, loaded before any arithmetic so the
// R loads of a chunk are in flight together.
template <int ELEM>
struct Chunk8 {
  uint4 a, b;  // ELEM 1: a.x,a.y; ELEM 2: a; ELEM 4: a,b
};

template <int ELEM>
__device__ __forceinline__ Chunk8<ELEM> load_chunk8(const uint8_t* row, int64_t h0) {
  Chunk8<ELEM> c;
  if constexpr (ELEM == 1) {
    const uint2 v = *reinterpret_cast<const uint2*>(row + h0);
    c.a = make_uint4(v.x, v.y, 0, 0);
  } else if constexpr (ELEM == 2) {
    c.a = *reinterpret_cast<const uint4*>(row + 2 * h0);
  } else {
    c.a = *reinterpret_cast<const uint4*>(row + 4 * h0);
    c.b = *reinterpret_cast<const uint4*>(row + 4 * h0 + 16);
  }
  return c;
}

template <int ELEM>
__device__ __forceinline__ void unpack_chunk8(const Chunk8<ELEM>& c, float* v) {
  if constexpr (ELEM == 1) {
    const uint32_t w[2] = {c.a.x, c.a.y};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float2 lo = fp8x2_to_f2((uint16_t)(w[q] & 0xFFFF));
      const float2 hi = fp8x2_to_f2((uint16_t)(w[q] >> 16));
      v[4 * q] = lo.x; v[4 * q + 1] = lo.y; v[4 * q + 2] = hi.x; v[4 * q + 3] = hi.y;
    }
  } else if constexpr (ELEM == 2) {
    const uint32_t w[4] = {c.a.x, c.a.y, c.a.z, c.a.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[2 * q] = __uint_as_float(w[q] << 16);
      v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
    }
  } else {
    v[0] = __uint_as_float(c.a.x); v[1] = __uint_as_float(c.a.y);
    v[2] = __uint_as_float(c.a.z); v[3] = __uint_as_float(c.a.w);
    v[4] = __uint_as_float(c.b.x); v[5] = __uint_as_float(c.b.y);
    v[6] = __uint_as_float(c.b.z); v[7] = __uint_as_float(c.b.w);
  }
}

template <int ELEM>
__device__ __forceinline__ float load1(const uint8_t* row, int64_t h) {
  if constexpr (ELEM == 1) {
    return fp8x2_to_f2((uint16_t)row[h]).x;
  } else if constexpr (ELEM == 2) {
    return bf16_to_f((uint16_t)(row[2 * h] | (row[2 * h + 1] << 8)));
  } else {
    uint32_t u = 0;
    for (int q = 0; q < 4; ++q) u |= (uint32_t)row[4 * h + q] << (8 * q);
    return __uint_as_float(u);
  }
}

constexpr int kCombBatch = 8;  // rows of one chunk loaded together

// out[t] = sum_j w[t,j] * y[t,j], j ascending from 0.0, separately rounded
// multiply and add (kernels.py:214-226); fp8 rows are dequantised first as
// e4m3 * f32 scale (kernels.py:139-141).  Row y[t,j] is out_rows +
// gidx[t,j]*ld when gidx[t,j] >= 0 (a copy this rank served itself, read in
// place from the expert outputs) and comb + pos[t,j]*Pc otherwise.  Each
// thread owns 8-element chunks; the rows of a chunk are fetched in batches
// of kCombBatch before the accumulation so their memory latencies overlap.
// Per-token row pointers, weights and (fp8) scales, staged in shared memory.
struct CombTok {
  const uint8_t* rowp[kMaxTopk];
  float ws[kMaxTopk];
  float sc[kMaxTopk];
  bool local[kMaxTopk];  // row served by this rank (readable before the wait)
};

// Row of copy j of token t: out_rows + gidx*ld when this rank served it
// (read in place), else comb + pos*Pc.  Needs only metadata, so it can run
// before the rows have arrived.
__device__ __forceinline__ void combine_prep(CombTok& ct, const uint8_t* comb, int64_t Pc, const uint8_t* out_rows,
                                             int64_t ld, const int64_t* pos, const int32_t* gidx, const float* w,
                                             int64_t t, int R) {
  const int tid = threadIdx.x;
  if (tid < R) {
    const int32_t gi = gidx ? gidx[t * R + tid] : -1;
    ct.rowp[tid] = gi >= 0 ? out_rows + (int64_t)gi * ld : comb + pos[t * R + tid] * Pc;
    if (w) ct.ws[tid] = w[t * R + tid];
    ct.local[tid] = gi >= 0;
  }
}

// out[t] = sum_j w[t,j] * y[t,j], j ascending from 0.0, separately rounded
// multiply and add (kernels.py:214-226); fp8 rows are dequantised first as
// e4m3 * f32 scale (kernels.py:139-141).  Each thread owns 8-element chunks;
// the rows of a chunk are fetched in batches of kCombBatch before the
// accumulation so their memory latencies overlap.  Expects combine_prep(t)
// and a barrier before the call.
template <int ELEM>
__device__ void combine_token(CombTok& ct, int64_t Pc, const uint8_t* comb, int H, int R, int64_t t, void* dst,
                              int out_bf16, bool vec) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (ELEM == 1) {
    if (tid < R) {
      const uint8_t* sp = ct.rowp[tid] + H;
      const uint32_t u = (uint32_t)sp[0] | ((uint32_t)sp[1] << 8) | ((uint32_t)sp[2] << 16) | ((uint32_t)sp[3] << 24);
      ct.sc[tid] = __uint_as_float(u);
    }
    __syncthreads();
  }
  const uint8_t* const* rowp = ct.rowp;
  const float* ws = ct.ws;
  const float* sc = ct.sc;
  if (vec) {
    // two 8-element chunks per thread per pass (c, c + nt) for 1- and
    // 2-byte rows: 2*kCombBatch independent loads in flight per thread
    constexpr int CPT = ELEM == 4 ? 1 : 2;
    for (int c0 = tid; c0 < H / 8; c0 += CPT * nt) {
      float acc[CPT][8];
#pragma unroll
      for (int p = 0; p < CPT; ++p)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[p][k] = 0.f;
      for (int j0 = 0; j0 < R; j0 += kCombBatch) {
        Chunk8<ELEM> raw[CPT][kCombBatch];
#pragma unroll
        for (int p = 0; p < CPT; ++p)
#pragma unroll
          for (int u = 0; u < kCombBatch; ++u)
            if (j0 + u < R && c0 + p * nt < H / 8)
              raw[p][u] = load_chunk8<ELEM>(rowp[j0 + u], (int64_t)(c0 + p * nt) * 8);
#pragma unroll
        for (int p = 0; p < CPT; ++p)
#pragma unroll
          for (int u = 0; u < kCombBatch; ++u) {
            if (j0 + u < R) {
              float v[8];
              unpack_chunk8<ELEM>(raw[p][u], v);
              const float wj = ws[j0 + u], sj = sc[j0 + u];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float y = ELEM == 1 ? __fmul_rn(v[k], sj) : v[k];
                acc[p][k] = __fadd_rn(acc[p][k], __fmul_rn(wj, y));
              }
            }
          }
      }
#pragma unroll
      for (int p = 0; p < CPT; ++p) {
        const int c = c0 + p * nt;
        if (c >= H / 8) continue;
        if (out_bf16) {
          uint4 o;
          uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            ow[q] = (uint32_t)bf16_rne(acc[p][2 * q]) | ((uint32_t)bf16_rne(acc[p][2 * q + 1]) << 16);
          reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + t * H)[c] = o;
        } else {
          float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + t * H) + 2 * c;
          o[0] = make_float4(acc[p][0], acc[p][1], acc[p][2], acc[p][3]);
          o[1] = make_float4(acc[p][4], acc[p][5], acc[p][6], acc[p][7]);
        }
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
      if (out_bf16) reinterpret_cast<uint16_t*>(dst)[t * H + h] = bf16_rne(acc);
      else reinterpret_cast<float*>(dst)[t * H + h] = acc;
    }
  }
}

// Decode fast path (R <= kCombBatch, 8-element chunks vectorisable): the
// rows this rank served itself are loaded BEFORE the completion wait, the
// returned rows after it; the sum then runs in the reference order.  The
// wait itself is done by `wait_fn` (thread 0 spins, then a barrier).
// The weights (an input, usually cold) are fetched after the row loads are
// in flight; the wait's barrier publishes them.
template <int ELEM, typename Wait>
__device__ bool combine_token_split(CombTok& ct, int H, int R, int64_t t, const float* w, void* dst, int out_bf16,
                                    Wait wait_fn) {
  const int tid = threadIdx.x, nt = blockDim.x;
  constexpr int CPT = ELEM == 4 ? 1 : 2;
  const int c0 = tid;
  Chunk8<ELEM> raw[CPT][kCombBatch];
#pragma unroll
  for (int p = 0; p < CPT; ++p)
#pragma unroll
    for (int u = 0; u < kCombBatch; ++u)
      if (u < R && ct.local[u] && c0 + p * nt < H / 8)
        raw[p][u] = load_chunk8<ELEM>(ct.rowp[u], (int64_t)(c0 + p * nt) * 8);
  if (w && tid >= nt - 32 && tid - (nt - 32) < R) ct.ws[tid - (nt - 32)] = w[t * R + tid - (nt - 32)];
  if (!wait_fn()) return false;
#pragma unroll
  for (int p = 0; p < CPT; ++p)
#pragma unroll
    for (int u = 0; u < kCombBatch; ++u)
      if (u < R && !ct.local[u] && c0 + p * nt < H / 8)
        raw[p][u] = load_chunk8<ELEM>(ct.rowp[u], (int64_t)(c0 + p * nt) * 8);
  if (ELEM == 1) {
    if (tid < R) {
      const uint8_t* sp = ct.rowp[tid] + H;
      const uint32_t v = (uint32_t)sp[0] | ((uint32_t)sp[1] << 8) | ((uint32_t)sp[2] << 16) | ((uint32_t)sp[3] << 24);
      ct.sc[tid] = __uint_as_float(v);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < CPT; ++p) {
    const int c = c0 + p * nt;
    if (c >= H / 8) continue;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
    for (int u = 0; u < kCombBatch; ++u) {
      if (u < R) {
        float v[8];
        unpack_chunk8<ELEM>(raw[p][u], v);
        const float wj = ct.ws[u], sj = ct.sc[u];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float y = ELEM == 1 ? __fmul_rn(v[k], sj) : v[k];
          acc[k] = __fadd_rn(acc[k], __fmul_rn(wj, y));
        }
      }
    }
    if (out_bf16) {
      uint4 o;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) ow[q] = (uint32_t)bf16_rne(acc[2 * q]) | ((uint32_t)bf16_rne(acc[2 * q + 1]) << 16);
      reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + t * H)[c] = o;
    } else {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + t * H) + 2 * c;
      o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
  return true;
}

template <int ELEM>
__device__ bool combine_vec(int64_t Pc, const uint8_t* comb, const uint8_t* out_rows, int64_t ld, int H,
                            const int32_t* gidx) {
  return (H % 8 == 0) && ((Pc & 15) == 0) && ((reinterpret_cast<uintptr_t>(comb) & 15) == 0) &&
         (!gidx || (((ld & 15) == 0) && ((reinterpret_cast<uintptr_t>(out_rows) & 15) == 0)));
}

template <int ELEM>
__device__ void combine_rows(const uint8_t* comb, int64_t Pc, const uint8_t* out_rows, int64_t ld, int H,
                             const int64_t* pos, const int32_t* gidx, const float* w, int64_t n, int R,
                             void* dst, int out_bf16, int cta, int ncta) {
  __shared__ CombTok ct;
  const bool vec = combine_vec<ELEM>(Pc, comb, out_rows, ld, H, gidx);
  for (int64_t t = cta; t < n; t += ncta) {
    combine_prep(ct, comb, Pc, out_rows, ld, pos, gidx, w, t, R);
    __syncthreads();
    combine_token<ELEM>(ct, Pc, comb, H, R, t, dst, out_bf16, vec);
    __syncthreads();
  }
}

}  // namespace txb
