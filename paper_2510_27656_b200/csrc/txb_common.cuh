// Shared device helpers for libtxb200 (sm_100a).
//
// Memory-model primitives used for the order-free completion protocol:
//   - payload: plain (weak) 16-byte st.global to peer addresses over NVLink;
//   - completion: __syncthreads() then one thread issues fence.sc.sys and a
//     red.release.sys add (counters) or st.release.sys (tags) on the peer;
//   - waiter: ld.acquire.sys spin with a %globaltimer deadline.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/txb200.h"

namespace txb {

// ------------------------------------------------------------ error string

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define TXB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::txb::cuda_fail(_e, #call); \
  } while (0)

// Entry points that take a caller's stream launch on the device that stream
// belongs to; for the legacy default stream (handle 0, shared by every
// device) on the device that owns `p`.  Without this a call made while
// another device is current would run on that device and reach the
// buffers over NVLink.  The caller's current device is restored on return.
struct DeviceFor {
  int prev = -1;
  DeviceFor(void* stream, const void* p) {
    cudaGetDevice(&prev);
    int dev = -1;
    // inside a stream capture only capture-safe calls are allowed: the
    // capturing stream fixes the device, so leave it alone
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (stream && cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone) {
      prev = -1;
      return;
    }
    cudaGetLastError();
    if (stream && cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &dev) == cudaSuccess) {
      if (dev != prev) cudaSetDevice(dev);
      return;
    }
    cudaGetLastError();
    cudaPointerAttributes at;
    if (p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice &&
        at.device != prev)
      cudaSetDevice(at.device);
    cudaGetLastError();
  }
  ~DeviceFor() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Entry points that name their device explicitly (a rank's shape, a region)
// make it current for the call and restore the caller's device on return,
// so a call never leaves torch's current device pointing at another rank.
struct OnDevice {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit OnDevice(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev != prev) err = cudaSetDevice(dev);
  }
  ~OnDevice() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define TXB_ON_DEVICE(dev)                                      \
  ::txb::OnDevice _on_dev(dev);                                 \
  if (_on_dev.err != cudaSuccess) return ::txb::cuda_fail(_on_dev.err, "cudaSetDevice")

// Loading every kernel up front (txb_preload).  Under CUDA's lazy module
// loading (the default since 12.2) the first launch of a kernel loads it,
// and that load did not complete while a persistent kernel of this library
// was polling a word on the device (tools/debug/clock_probe.py): the first
// clock write of a KV stream never landed.  cudaFuncGetAttributes loads the
// function without launching it.
template <typename K>
inline cudaError_t touch(K kernel) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(kernel));
}
cudaError_t preload_engine();
cudaError_t preload_moe();
cudaError_t preload_codec();
unsigned int check_failures_engine();
unsigned int check_failures_moe();
unsigned int check_failures_codec();

// ------------------------------------------------------------ checked build
//
// `make checked` builds libtxb200_checked.so with -DTXB_CHECKED: every index
// a kernel computes before a store or load through it (grouped row, combine
// slot, private-slab slot, shared-memory table extent) is bounds-checked on
// the device.  A failed check prints the site, latches bit 0 of
// g_txb_check_fail (read with txb_check_failures) and skips the access --
// the pool's compute-sanitizer substitute (profiles/r02/README.md).  The
// release build compiles the checks out.
#ifdef TXB_CHECKED
// one flag per translation unit (no relocatable device code needed); each
// unit reports its own through check_failures_<unit>() (txb_check_failures)
static __device__ unsigned int g_txb_check_fail = 0;
static inline unsigned int read_check_fail() {
  unsigned int v = 0;
  cudaMemcpyFromSymbol(&v, g_txb_check_fail, sizeof(v));
  return v;
}
#define TXB_ASSERT(cond)                                                                      \
  (__builtin_expect(!(cond), 0)                                                               \
       ? (atomicOr(&::txb::g_txb_check_fail, 1u),                                             \
          printf("txb check failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,       \
                 (int)blockIdx.x, (int)threadIdx.x, #cond),                                   \
          false)                                                                              \
       : true)
// TXB_ASSERT_V: the same, printing up to four integer values of the site
#define TXB_ASSERT_V(cond, a, b, c, d)                                                        \
  (__builtin_expect(!(cond), 0)                                                               \
       ? (atomicOr(&::txb::g_txb_check_fail, 1u),                                             \
          printf("txb check failed %s:%d block %d thread %d: %s [%lld %lld %lld %lld]\n",     \
                 __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x, #cond, (long long)(a), \
                 (long long)(b), (long long)(c), (long long)(d)),                             \
          false)                                                                              \
       : true)
#else
#define TXB_ASSERT(cond) true
#define TXB_ASSERT_V(cond, a, b, c, d) true
#endif

// ------------------------------------------------------------ PTX wrappers

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_release_sys_add(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_relaxed_sys_add(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One release fence for a batch of relaxed signals: fence.acq_rel.sys
// followed by relaxed stores/reds forms the release pattern of the PTX
// memory model, so N destination counters cost one system-scope MEMBAR
// instead of one per red.release.
__device__ __forceinline__ void fence_acqrel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ void fence_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }

// Release fence at the narrowest scope that covers every rank: .gpu when the
// whole mesh lives on this device (~0.2-0.9 us), .sys across GPUs (~2 us).
__device__ __forceinline__ void fence_release(bool gpu_only) {
  if (gpu_only) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else asm volatile("fence.acq_rel.sys;" ::: "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Spin until *p >= target (acquire, system scope) or the deadline passes.
__device__ __forceinline__ bool spin_ge(const uint64_t* p, uint64_t target, uint64_t deadline) {
  uint32_t it = 0;
  while (ld_acquire_sys(p) < target) {
    if (((++it) & 255u) == 0 && globaltimer() > deadline) return ld_acquire_sys(p) >= target;
  }
  return true;
}

// ------------------------------------------------------------ region layout

// Per-rank flag block at region offset off_flags (4 KiB aligned).
// route_tag/done are written by peers (single writer per slot, monotone);
// tok_ctr/comb_ctr receive release-adds from every peer; the rest is local.
struct Flags {
  uint64_t route_tag[2][TXB_MAX_RANKS];  // [step parity][source] = step
  uint64_t done[TXB_MAX_RANKS];          // [peer] = last step whose reads of this region finished (published by the peer's next route phase)
  uint64_t tok_ctr;                      // rows received (dispatch)
  uint64_t comb_ctr;                     // rows received (combine)
  uint64_t priv_ctr[2];                  // [step parity] speculative private rows received
  uint64_t pad0[4];
  // local-only state (written by this rank's kernels, in stream order)
  uint64_t step;         // last completed step (every kernel of step k reads k-1)
  uint64_t tok_target;   // cumulative expected tok_ctr
  uint64_t comb_target;  // cumulative expected comb_ctr
  uint32_t err;          // TXB_EV_* latch
  uint32_t ticket;       // last-CTA detection at the end of a step
  uint64_t bar_epoch;    // local epoch of txb_moe_barrier
  uint32_t gbar_count;   // grid barrier of the cooperative kernels (local)
  uint32_t gbar_gen;
  uint32_t send_cnt;     // grouped rows to return to other ranks (this step)
  uint32_t pad2;
  uint64_t gbar_arrive;  // monotone grid-barrier counter (+TXB_MAX_CTAS per barrier)
  uint64_t bar[TXB_MAX_RANKS];  // [peer] = last barrier epoch peer reached
  uint32_t phase_cnt[16];       // send-list fill per phase (large batches, this step)
  // speculative private rows (moe.py:556-582): cumulative expected
  // priv_ctr per step parity (advanced at the end of each step by that
  // step's count, priv_step, which the dispatch books once the route
  // matrix is known)
  uint64_t priv_target[2];
  uint64_t priv_step;
  uint64_t pad3;
  // Per-source lanes, for the timeout diagnostics only (moe.py:874-899):
  // every signal also adds its count to the slot of its source rank, and
  // the receiver books the cumulative count it expects from each source,
  // so a timeout names the ranks that have not delivered.  The waits use
  // the aggregate counters above.
  uint64_t tok_src[TXB_MAX_RANKS];     // [source] token rows received (peer-written)
  uint64_t comb_src[TXB_MAX_RANKS];    // [source] combine rows received (peer-written)
  uint64_t priv_src[TXB_MAX_RANKS];    // [source] private rows received (peer-written)
  uint64_t tok_src_t[TXB_MAX_RANKS];   // [source] cumulative expected (local)
  uint64_t comb_src_t[TXB_MAX_RANKS];
  uint64_t priv_src_t[TXB_MAX_RANKS];
};

__host__ __device__ inline Flags* flags_of(void* region, const txb_moe_shape& s) {
  return reinterpret_cast<Flags*>(reinterpret_cast<char*>(region) + s.off_flags);
}
// Route matrix words: (step tag << 32) | count.  A word is one 8-byte
// single-copy-atomic store, so a reader that sees the tag of this step also
// sees its count -- the route exchange needs no fence on either side.
__host__ __device__ inline uint64_t* route_of(void* region, const txb_moe_shape& s, int slot) {
  return reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(region) + s.off_route) +
         (size_t)slot * s.ranks * s.experts;
}
__host__ __device__ inline uint8_t* grouped_of(void* region, const txb_moe_shape& s) {
  return reinterpret_cast<uint8_t*>(region) + s.off_grouped;
}
__host__ __device__ inline uint8_t* comb_of(void* region, const txb_moe_shape& s) {
  return reinterpret_cast<uint8_t*>(region) + s.off_comb;
}

// Per-token completion (large batches, see txb_moe.cu: kTokWaitMin), placed
// after the combine rows: tokc[T] u64 -- rows of token t returned to this
// rank (release-adds from the expert ranks), tokt[T] u64 -- cumulative
// expected tokc (local), srctok[G] i32 -- origin token index of each grouped
// row (written by the origin with the row during the dispatch).
__host__ __device__ inline uint64_t tok_offset(const txb_moe_shape& s) {
  return (s.off_comb + (uint64_t)s.comb_rows * (uint64_t)s.comb_bytes + 255) / 256 * 256;
}
__host__ __device__ inline uint64_t* tokc_of(void* region, const txb_moe_shape& s) {
  return reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(region) + tok_offset(s));
}
__host__ __device__ inline uint64_t* tokt_of(void* region, const txb_moe_shape& s) {
  return tokc_of(region, s) + s.max_tokens;
}
__host__ __device__ inline int32_t* srctok_of(void* region, const txb_moe_shape& s) {
  return reinterpret_cast<int32_t*>(tokc_of(region, s) + 2 * (uint64_t)s.max_tokens);
}

// Speculative private slabs (PrivateBufferConfig, moe.py:92-102, 556-582):
// rows [2 parity][N source][priv_tokens][P] at off_priv, then the origin
// token index of each row, i32 [2][N][priv_tokens] (for per-token combine
// completion).  A source stores the first priv_tokens rows of its slab for
// this rank here before the route exchange has finished; the receiver moves
// them to their grouped rows once the layout is known.  Step parity double
// buffering makes the early stores safe without a wait: a source writes
// parity p at step k only after it saw this rank's end-of-step k-2 barrier.
__host__ __device__ inline uint8_t* priv_rows_of(void* region, const txb_moe_shape& s, int parity, int src) {
  return reinterpret_cast<uint8_t*>(region) + s.off_priv +
         ((uint64_t)(parity * s.ranks + src) * (uint64_t)s.priv_tokens) * (uint64_t)s.payload_bytes;
}
__host__ __device__ inline int32_t* privsrc_of(void* region, const txb_moe_shape& s, int parity, int src) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(region) + s.off_priv +
                                    2ull * s.ranks * s.priv_tokens * (uint64_t)s.payload_bytes) +
         (uint64_t)(parity * s.ranks + src) * s.priv_tokens;
}

// ------------------------------------------------------------- block scan

// Exclusive prefix sum of a[0..len) (int32, shared memory) in place; every
// thread of the block must call it.  Returns the total.  `tmp` needs 33
// ints.  Out of line: one copy of the code serves every call site (the
// fused kernels are instruction-fetch bound when the code balloons).
// A thread group that synchronises on its own hardware barrier: the whole
// CTA (barrier 0, what __syncthreads uses) or a warp-aligned role of it on a
// named barrier, so two roles of one CTA can run different phases at once.
struct Grp {
  int tid, nt, bar;
  __device__ static Grp cta() { return Grp{(int)threadIdx.x, (int)blockDim.x, 0}; }
  __device__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nt) : "memory"); }
};

static __device__ __forceinline__ int block_scan_i32_body(int* a, int len, int* tmp, const Grp& g) {
  const int nt = g.nt, tid = g.tid;
  const int per = (len + nt - 1) / nt;
  const int lo = min(len, tid * per), hi = min(len, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += a[i];
  const int lane = tid & 31, warp = tid >> 5;
  int x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  g.sync();
  if (warp == 0) {
    const int nw = (nt + 31) >> 5;
    int w = lane < nw ? tmp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) tmp[lane] = w;  // inclusive warp totals
    if (lane == nw - 1) tmp[32] = w;
  }
  g.sync();
  int run = (x - sum) + (warp ? tmp[warp - 1] : 0);
  for (int i = lo; i < hi; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  const int total = tmp[32];
  g.sync();
  return total;
}

static __device__ __noinline__ int block_scan_i32(int* a, int len, int* tmp) {
  return block_scan_i32_body(a, len, tmp, Grp::cta());
}

// Call-site choice: INL = inline copy (a straight-line decode path, where a
// call into cold out-of-line code costs an instruction-fetch miss per
// call), else the shared out-of-line copy.
template <bool INL>
__device__ __forceinline__ int block_scan(int* a, int len, int* tmp, const Grp& g) {
  if constexpr (INL) return block_scan_i32_body(a, len, tmp, g);
  else return block_scan_i32(a, len, tmp);  // whole CTA only
}

// ------------------------------------------------------------- row copy

__device__ __forceinline__ int vec_width(const void* a, const void* b, int64_t bytes) {
  uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | (uintptr_t)bytes;
  if ((m & 15) == 0) return 16;
  if ((m & 7) == 0) return 8;
  if ((m & 3) == 0) return 4;
  return 1;
}

// Copy `bytes` from src to dst with the widest vector the alignment allows;
// the calling group is `nthr` threads with index `t`.
static __device__ __noinline__ void copy_row(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t bytes,
                                      int t, int nthr) {
  const int w = vec_width(dst, src, bytes);
  if (w == 16) {
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    const int64_t nv = bytes >> 4;
    int64_t i = t;
    for (; i + 3 * nthr < nv; i += 4 * nthr) {
      const int4 a = s[i], b = s[i + nthr], c = s[i + 2 * nthr], e = s[i + 3 * nthr];
      d[i] = a; d[i + nthr] = b; d[i + 2 * nthr] = c; d[i + 3 * nthr] = e;
    }
    for (; i < nv; i += nthr) d[i] = s[i];
  } else if (w >= 4) {
    const int* s = reinterpret_cast<const int*>(src);
    int* d = reinterpret_cast<int*>(dst);
    for (int64_t i = t; i < (bytes >> 2); i += nthr) d[i] = s[i];
  } else {
    for (int64_t i = t; i < bytes; i += nthr) dst[i] = src[i];
  }
}

static __device__ __noinline__ void zero_row(uint8_t* dst, int64_t bytes, int t, int nthr) {
  const int w = vec_width(dst, dst, bytes);
  if (w == 16) {
    const int4 z = make_int4(0, 0, 0, 0);
    for (int64_t i = t; i < (bytes >> 4); i += nthr) reinterpret_cast<int4*>(dst)[i] = z;
  } else if (w >= 4) {
    for (int64_t i = t; i < (bytes >> 2); i += nthr) reinterpret_cast<int*>(dst)[i] = 0;
  } else {
    for (int64_t i = t; i < bytes; i += nthr) dst[i] = 0;
  }
}

// -------------------------------------------------------------- codecs

// e4m3 RNE satfinite; NaN -> 0x7F regardless of sign (kernels.py:65-76).
__device__ __forceinline__ uint32_t fp8x2(float a, float b) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(b), "f"(a));
  uint32_t v = r;
  if (isnan(a)) v = (v & 0xFF00u) | 0x7Fu;
  if (isnan(b)) v = (v & 0x00FFu) | 0x7F00u;
  return v;
}

// Exact e4m3 -> f32 (every e4m3 value is an f16 value).
__device__ __forceinline__ float2 fp8x2_to_f2(uint16_t v) {
  uint32_t h2;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(v));
  __half2_raw raw;
  raw.x = (unsigned short)(h2 & 0xFFFF);
  raw.y = (unsigned short)(h2 >> 16);
  return __half22float2(*reinterpret_cast<__half2*>(&raw));
}

// x / s rounded to nearest even, given r = RN(1/s): a multiply and two
// Markstein corrections (the residual x - q*s is exact in an FMA; once q is
// within an ulp of x/s, RN(q + residual * r) is the correctly rounded
// quotient when nothing over- or underflows).  One correction is not
// enough: RN(x * r) can be two ulps off.  Quotients outside the safe
// normal range, zeros, infinities and NaNs take the IEEE division.
// Bit-identical to __fdiv_rn; checked exhaustively on the GPU through the
// fp8 encode (tests/test_moe_gpu.py).
static __device__ __noinline__ float div_rn_slow(float x, float s) { return __fdiv_rn(x, s); }

__device__ __forceinline__ float div_rn_by(float x, float s, float r) {
  const float q0 = __fmul_rn(x, r);
  const float q1 = __fmaf_rn(__fmaf_rn(-q0, s, x), r, q0);
  const float q = __fmaf_rn(__fmaf_rn(-q1, s, x), r, q1);
  const float a = fabsf(q);
  return (a >= 0x1p-120f && a <= 0x1p120f) ? q : div_rn_slow(x, s);
}

// bf16 RNE with the reference NaN rule 0x7FC0|hi (kernels.py:144-150).
__device__ __forceinline__ uint16_t bf16_rne(float x) {
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x007FFFFFu)) return (uint16_t)(0x7FC0u | (b >> 16));
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

__device__ __forceinline__ float bf16_to_f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

}  // namespace txb
