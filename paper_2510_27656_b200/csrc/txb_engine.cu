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
constexpr int kPiece = 8 * 1024;   // bytes per piece (a KV page; one TMA stage)
constexpr int kWarpStages = 2;     // TMA stages per issuing warp
constexpr int kCopyWarps = kCopyThreads / 32;
constexpr int kMaxJobs = TXB_MAX_JOBS;

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

// One piece by one warp with 16-byte vectors: all loads in flight before
// the first store.
__device__ __forceinline__ void warp_copy_piece(const PieceRef& p, int lane) {
  if (vec_width(p.src, p.dst, p.bytes) == 16) {
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

// The pieces k = first, first + stride, ... < total of one warp.  TMA: lane
// 0 of every warp drives its own kWarpStages-deep bulk-copy pipeline
// (global -> shared -> global, mbarrier-tracked loads, bulk-group stores),
// so eight issuers per CTA keep pieces in flight; vector: the warp copies
// each piece with 16-byte loads and stores.
template <typename PieceFn>
__device__ __forceinline__ void warp_copy_range(int64_t first, int64_t stride, int64_t total, bool tma,
                                                uint8_t* stage, uint64_t* bars, uint32_t* phase, PieceFn piece) {
  const int lane = threadIdx.x & 31;
  if (!tma) {
    #pragma unroll 1
    for (int64_t k = first; k < total; k += stride) warp_copy_piece(piece(k), lane);
    return;
  }
  if (lane != 0) return;
  #pragma unroll 1
  for (int s = 0; s < kWarpStages && first + (int64_t)s * stride < total; ++s) {
    const PieceRef p = piece(first + (int64_t)s * stride);
    mbar_expect_tx(&bars[s], p.bytes);
    tma_load(stage + s * kPiece, p.src, p.bytes, &bars[s]);
  }
  int64_t it = 0;
  #pragma unroll 1
  for (int64_t k = first; k < total; k += stride, ++it) {
    const int s = (int)(it % kWarpStages);
    const PieceRef p = piece(k);
    mbar_wait(&bars[s], phase[s]);
    phase[s] ^= 1u;
    tma_store(p.dst, stage + s * kPiece, p.bytes);
    const int64_t kn = k + (int64_t)kWarpStages * stride;
    if (kn < total) {
      tma_store_wait_read<kWarpStages>();  // the stage stored kWarpStages-1 pieces ago is free
      const PieceRef q = piece(kn);
      mbar_expect_tx(&bars[s], q.bytes);
      tma_load(stage + s * kPiece, q.src, q.bytes, &bars[s]);
    }
  }
  tma_store_wait_all();
  // order the async-proxy global writes before the generic release that follows
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void init_warp_bars(uint64_t* bars, bool tma) {
  if (tma && (threadIdx.x & 31) == 0) {
    for (int s = 0; s < kWarpStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

// Every submitted write of one launch (a single write, a paged write, or
// all the per-peer slices of a scatter): pieces of all jobs are numbered
// through the prefix `start`, CTAs take them round-robin, and each job
// completes on its own -- a CTA adds the pieces it moved of job i to job
// i's ticket after a release fence; the CTA that brings the ticket to the
// job's piece count resets it and releases one increment on that job's
// ImmCounter slot, exactly once per write and only after its whole payload
// is visible (engine.py:9-17).
struct JobSet {
  txb_pages job[kMaxJobs];
  int64_t start[kMaxJobs + 1];
  int32_t njobs;
  int32_t use_tma;
};

__device__ __forceinline__ int job_of(const JobSet& js, int64_t k) {
  int lo = 0, hi = js.njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (js.start[mid] <= k) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kCopyThreads, 2) k_copy_jobs(const __grid_constant__ JobSet js) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[kCopyWarps * kWarpStages];
  __shared__ uint32_t done[kMaxJobs];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tma = js.use_tma != 0;
  for (int i = threadIdx.x; i < js.njobs; i += blockDim.x) done[i] = 0;
  init_warp_bars(bars + warp * kWarpStages, tma);
  __syncthreads();
  const int64_t total = js.start[js.njobs];
  uint32_t phase[kWarpStages] = {};
  auto piece = [&](int64_t k) {
    const int i = job_of(js, k);
    const txb_pages& j = js.job[i];
    return piece_of(j, k - js.start[i], (j.page_len + kPiece - 1) / kPiece);
  };
  const int64_t first = (int64_t)blockIdx.x * kCopyWarps + warp, stride = (int64_t)gridDim.x * kCopyWarps;
  warp_copy_range(first, stride, total, tma, stage + (size_t)warp * kWarpStages * kPiece,
                  bars + warp * kWarpStages, phase, piece);
  if (lane == 0)
    for (int64_t k = first; k < total; k += stride) atomicAdd(&done[job_of(js, k)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    bool any = false;
    for (int i = 0; i < js.njobs; ++i) any |= done[i] != 0;
    bool gpu_only = true;
    for (int i = 0; i < js.njobs; ++i) gpu_only &= js.job[i].single_device != 0;
    if (any) fence_release(gpu_only);
    for (int i = 0; i < js.njobs; ++i) {
      const txb_pages& j = js.job[i];
      const uint32_t need = (uint32_t)(js.start[i + 1] - js.start[i]);
      // zero-piece jobs (a zero-length write carrying an immediate) are
      // completed by CTA 0
      const uint32_t mine = need == 0 ? (blockIdx.x == 0 ? 1u : 0u) : done[i];
      if (!mine) continue;
      const uint32_t old = need == 0 ? 0u : atomicAdd(j.ticket, mine);
      if (old + mine == (need == 0 ? 1u : need)) {
        if (need) *j.ticket = 0;
        if (j.imm_ctr) {
          fence_release(j.single_device != 0);
          red_relaxed_sys_add(j.imm_ctr, 1);
        }
      }
    }
  }
}

// Fallback clock write (GPU-scope release; the readers are kernels of the
// same GPU and acquire).
__global__ void k_write_value(uint64_t* p, uint64_t v) {
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ bool spin_ge_gpu(const uint64_t* p, uint64_t target, uint64_t deadline) {
  uint32_t it = 0;
  while (ld_acquire_gpu(p) < target) {
    if (((++it) & 255u) == 0 && globaltimer() > deadline) return ld_acquire_gpu(p) >= target;
  }
  return true;
}

// Persistent paged stream (the KV-cache layer-by-layer transfer,
// kvcache.py:477-507, with the LayerClock of kvcache.py:317-334 on the
// device): step k (0-based) of the request moves pages_per_step pages
// (indices [k*pages_per_step, (k+1)*pages_per_step) of the index arrays)
// as soon as *clock >= clock_base + k + 1 -- the compute stream advances the
// clock after each layer, no host in the loop -- and the warp that finishes
// a step last releases one increment on the request's ImmCounter slot.
//
// Every warp runs on its own (no CTA barrier): the request's pieces are
// dealt round-robin across steps, and completion is booked per warp in
// batches of kStreamBatch pieces -- one release fence (which waits for the
// warp's stores to land) covers the batch, then one ticket increment per
// piece on its step; the increment that brings a step's ticket to its piece
// count releases the receipt.  A warp that reaches a step the clock has not
// released yet books what it has first, so receipts never wait on a future
// layer.  The fence is the only drain, and no other warp waits for it.
constexpr int kStreamBatch = 32;

__global__ void __launch_bounds__(kCopyThreads, 1) k_kv_stream(const __grid_constant__ txb_stream_job ks) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bars[kCopyWarps * kWarpStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tma = ks.use_tma != 0;
  init_warp_bars(bars + warp * kWarpStages, tma);
  uint32_t phase[kWarpStages] = {};
  const int64_t per_page = (ks.page_len + kPiece - 1) / kPiece;
  const int64_t total = ks.pages_per_step * per_page;
  const uint32_t nwarps = gridDim.x * kCopyWarps;
  const int64_t gw = (int64_t)blockIdx.x * kCopyWarps + warp;
  const uint64_t dl = globaltimer() + ks.timeout_ns;
  // The request's pieces are numbered across steps (step k holds pieces
  // [k*total, (k+1)*total)) and dealt round-robin to the warps, so every
  // warp stays busy across step boundaries (per step, 1024 pages on 1184
  // warps left 160 warps idle and every warp re-entered the step loop per
  // page: 583 GB/s, against 697 for the same scattered pages copied in one
  // pass -- tools/micro/peer_width.cu).  A step's ticket counts its pieces.
  const int64_t all = (int64_t)ks.nsteps * total;
  if (total == 0) {  // steps without pages still release their receipts, in clock order
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int k = 0; k < ks.nsteps; ++k) {
        if (!spin_ge_gpu(ks.clock, ks.clock_base + (uint64_t)k + 1, dl)) {
          if (ks.err) atomicOr(ks.err, TXB_EV_WAIT_IMM);
          return;
        }
        if (ks.imm_ctr) red_relaxed_sys_add(ks.imm_ctr, 1);
      }
    return;
  }
  int64_t pend_q0 = 0;
  int npend = 0;      // pieces pend_q0, pend_q0 + nwarps, ... copied, not yet booked
  uint64_t seen = 0;  // clock value this warp has already acquired
  auto book = [&]() {
    if (npend == 0) return;
    __syncwarp();
    // one fence (a warp instruction) makes the batch's stores visible, then
    // the lanes book its pieces in parallel: a serial loop of returning
    // atomics on one lane cost a round trip per piece
    fence_release(ks.single_device != 0);
    const int kb0 = (int)(pend_q0 / total);
    const int64_t qb0 = pend_q0 - (int64_t)kb0 * total;
    for (int i = lane; i < npend; i += 32) {
      const int kb = kb0 + (int)((qb0 + (int64_t)i * nwarps) / total);
      if (atomicAdd(&ks.tickets[kb], 1u) == (uint32_t)total - 1) {
        ks.tickets[kb] = 0;
        if (ks.imm_ctr) {
          fence_release(ks.single_device != 0);
          red_relaxed_sys_add(ks.imm_ctr, 1);
        }
      }
    }
    __syncwarp();
    npend = 0;
  };
  // the page indices of a warp's next piece are loaded one piece ahead (a
  // dependent round trip per 8-KiB piece otherwise); (step, piece in step)
  // advance incrementally -- 64-bit divisions per piece made this kernel
  // execute 6x the instructions of a plain page copy (ncu, round 2)
  const int32_t tot32 = (int32_t)total, pp32 = (int32_t)per_page, nw32 = (int32_t)nwarps;
  auto advance = [&](int& k, int32_t& qs) {
    qs += nw32;
    while (qs >= tot32) {
      qs -= tot32;
      ++k;
    }
  };
  auto idx_of = [&](int k, int32_t qs, int64_t& sidx, int64_t& didx) {
    if (k >= ks.nsteps) return;
    const int64_t row = (int64_t)k * ks.pages_per_step + (pp32 == 1 ? qs : qs / pp32);
    sidx = ks.src_idx[row];
    didx = ks.dst_idx[row];
  };
  int k = (int)(gw / total);
  int32_t qs = (int32_t)(gw - (int64_t)k * total);
  int64_t s_cur = 0, d_cur = 0;
  idx_of(k, qs, s_cur, d_cur);
  #pragma unroll 1
  for (int64_t q = gw; q < all; q += nwarps) {
    int kn = k;
    int32_t qsn = qs;
    advance(kn, qsn);
    int64_t s_nxt = 0, d_nxt = 0;
    idx_of(kn, qsn, s_nxt, d_nxt);
    const uint64_t want = ks.clock_base + (uint64_t)k + 1;
    if (seen < want) {  // the clock is read only when the cached value runs out
      uint32_t ok = 1;
      if (lane == 0) {
        seen = ld_acquire_gpu(ks.clock);
        if (seen < want) ok = 2;  // not released yet: book the finished pieces before waiting
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok == 2) {
        book();
        if (lane == 0) {
          ok = spin_ge_gpu(ks.clock, want, dl) ? 1u : 0u;
          if (!ok && ks.err) atomicOr(ks.err, TXB_EV_WAIT_IMM);
          seen = ld_acquire_gpu(ks.clock);
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) return;
      }
      seen = __shfl_sync(0xffffffffu, seen, 0);
    }
    const int32_t pc = pp32 == 1 ? 0 : qs % pp32;
    const int64_t off = (int64_t)pc * kPiece, rem = ks.page_len - off;
    PieceRef p;
    p.src = reinterpret_cast<const uint8_t*>(ks.src) + s_cur * ks.page_len + off;
    p.dst = reinterpret_cast<uint8_t*>(ks.dst) + d_cur * ks.page_len + off;
    p.bytes = (uint32_t)(rem < kPiece ? rem : kPiece);
    s_cur = s_nxt;
    d_cur = d_nxt;
    k = kn;
    qs = qsn;
    if (!tma) {
      warp_copy_piece(p, lane);
    } else {
      warp_copy_range(0, 1, 1, true, stage + (size_t)warp * kWarpStages * kPiece, bars + warp * kWarpStages, phase,
                      [&](int64_t) { return p; });
    }
    __syncwarp();
    if (npend == 0) pend_q0 = q;
    if (++npend == kStreamBatch) book();
  }
  book();
}

// Full-u32 ImmCounter table (ImmCounterTable, engine.py:138-205): keys
// u64[TXB_IMM_SLOTS] (0 = empty, else imm + 1) then counts u64[SLOTS].
// Open addressing with linear probing; a slot is claimed with a system-scope
// CAS, so the owner and every sender (over NVLink) converge on the same slot
// for an imm whoever arrives first.  Keys are never removed.
__device__ __forceinline__ uint32_t imm_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void k_imm_probe(uint64_t* keys, uint32_t imm, int insert, int64_t* out) {
  if (threadIdx.x != 0) return;
  const uint64_t key = (uint64_t)imm + 1;
  uint32_t h = imm_hash(imm) & (TXB_IMM_SLOTS - 1);
  for (int i = 0; i < TXB_IMM_SLOTS; ++i, h = (h + 1) & (TXB_IMM_SLOTS - 1)) {
    unsigned long long cur;
    if (insert) {
      asm volatile("atom.cas.sys.global.b64 %0, [%1], %2, %3;"
                   : "=l"(cur) : "l"(keys + h), "l"(0ull), "l"(key) : "memory");
    } else {
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(cur) : "l"(keys + h) : "memory");
    }
    if (cur == key || (insert && cur == 0)) {
      *out = h;
      return;
    }
    if (cur == 0) break;  // lookup: an empty slot ends the probe sequence
  }
  *out = -1;
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
// Pass 1: four 16-byte loads in flight per thread per pass (the HBM needs
// ~6.5 MB in flight at full rate), one block reduction, one atomic per CTA
// (a per-warp atomic put ~4700 same-address atomics on one L2 slice).
constexpr int kQU = 4;
__global__ void __launch_bounds__(256) k_amax_bf16(const uint16_t* __restrict__ x, int64_t n, uint32_t* amax_bits) {
  __shared__ float red[8];
  float m = 0.f;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t n8 = vec ? n / 8 : 0;
  for (int64_t c = tid; c < n8; c += kQU * nthr) {
    uint4 v[kQU];
#pragma unroll
    for (int u = 0; u < kQU; ++u)
      if (c + u * nthr < n8) v[u] = reinterpret_cast<const uint4*>(x)[c + u * nthr];
#pragma unroll
    for (int u = 0; u < kQU; ++u) {
      if (c + u * nthr >= n8) break;
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
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (threadIdx.x == 0) atomicMax(amax_bits, __float_as_uint(a));
  }
}

// x / scale correctly rounded (div_rn_by: reciprocal multiply + two FMA
// corrections, bit-identical to the IEEE division), e4m3 RNE satfinite;
// 16-byte loads of 8 bf16 (four in flight per thread), 8-byte stores of 8 fp8.
__global__ void __launch_bounds__(256) k_quant_bf16_fp8(const uint16_t* __restrict__ x, int64_t n,
                                                        const uint32_t* amax_bits, uint8_t* __restrict__ out) {
  const float amax = __uint_as_float(*amax_bits);
  const float scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  const float rs = __frcp_rn(scale);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && ((reinterpret_cast<uintptr_t>(out) & 7) == 0);
  const int64_t n8 = vec ? n / 8 : 0;
  for (int64_t c0 = tid; c0 < n8; c0 += kQU * nthr) {
    uint4 v[kQU];
#pragma unroll
    for (int u = 0; u < kQU; ++u)
      if (c0 + u * nthr < n8) v[u] = reinterpret_cast<const uint4*>(x)[c0 + u * nthr];
#pragma unroll
    for (int u = 0; u < kQU; ++u) {
      const int64_t c = c0 + u * nthr;
      if (c >= n8) break;
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[u]);
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

unsigned int check_failures_engine() {
#ifdef TXB_CHECKED
  return read_check_fail();
#else
  return 0;
#endif
}

cudaError_t preload_engine() {
  cudaError_t e = cudaSuccess;
  for (cudaError_t r : {touch(k_copy_jobs), touch(k_write_value), touch(k_kv_stream), touch(k_imm_probe),
                        touch(k_imm_add), touch(k_imm_wait), touch(k_globaltimer), touch(k_amax_bf16),
                        touch(k_quant_bf16_fp8)})
    if (r != cudaSuccess) e = r;
  return e;
}

}  // namespace txb

using namespace txb;

extern "C" {

int txb_imm_table_slots(void) { return TXB_IMM_SLOTS; }

static int launch_jobs(JobSet& js, int grid, void* stream) {
  int64_t total = 0;
  js.start[0] = 0;
  bool sd = true;
  for (int i = 0; i < js.njobs; ++i) {
    const txb_pages& j = js.job[i];
    if (!j.ticket) {
      set_error("copy job %d: null ticket", i);
      return TXB_ERR_TRANSFER;
    }
    if (j.npages < 0 || j.page_len < 0) {
      set_error("copy job %d: negative page count or length", i);
      return TXB_ERR_TRANSFER;
    }
    const int64_t per_page = j.page_len > 0 ? (j.page_len + kPiece - 1) / kPiece : 0;
    total += j.npages * per_page;
    js.start[i + 1] = total;
    sd &= j.single_device != 0;
  }
  js.use_tma = 1;
  for (int i = 0; i < js.njobs; ++i) js.use_tma &= js.job[i].use_tma != 0;
  if (grid <= 0) {
    const int64_t want = (total + kCopyWarps - 1) / kCopyWarps;
    const int cap = (js.use_tma ? 1 : 2) * sms(0);  // two CTAs per SM unless TMA stages fill the smem
    grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  }
  const size_t smem = js.use_tma ? (size_t)kCopyWarps * kWarpStages * kPiece : 0;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && (dev < 0 || dev >= 64 || !attr_set[dev])) {
    TXB_CUDA(cudaFuncSetAttribute(k_copy_jobs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kCopyWarps * kWarpStages * kPiece)));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  (void)sd;
  k_copy_jobs<<<grid, kCopyThreads, smem, (cudaStream_t)stream>>>(js);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_copy_pages(const txb_pages* j, int grid, void* stream) {
  if (!j) {
    set_error("txb_copy_pages: null job");
    return TXB_ERR_TRANSFER;
  }
  DeviceFor on_dev(stream, j->src_base);
  static thread_local JobSet js;
  js.njobs = 1;
  js.job[0] = *j;
  return launch_jobs(js, grid, stream);
}

int txb_copy_jobs(const txb_pages* jobs, int njobs, int grid, void* stream) {
  if (!jobs || njobs < 1 || njobs > kMaxJobs) {
    set_error("txb_copy_jobs: %d jobs outside 1..%d", njobs, kMaxJobs);
    return TXB_ERR_TRANSFER;
  }
  DeviceFor on_dev(stream, jobs[0].src_base);
  static thread_local JobSet js;
  js.njobs = njobs;
  for (int i = 0; i < njobs; ++i) js.job[i] = jobs[i];
  return launch_jobs(js, grid, stream);
}

int txb_kv_stream(const txb_stream_job* ks, int grid, void* stream) {
  if (!ks || !ks->tickets || !ks->clock || !ks->src_idx || !ks->dst_idx) {
    set_error("txb_kv_stream: null job, tickets, clock or page indices");
    return TXB_ERR_TRANSFER;
  }
  if (ks->nsteps < 0 || ks->pages_per_step < 0 || ks->page_len <= 0) {
    set_error("txb_kv_stream: bad step / page counts");
    return TXB_ERR_TRANSFER;
  }
  DeviceFor on_dev(stream, ks->src);
  if (grid <= 0) grid = sms(0);  // one CTA per SM (two measured 2% slower, profiles/r02/README.md)
  const size_t smem = ks->use_tma ? (size_t)kCopyWarps * kWarpStages * kPiece : 0;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && (dev < 0 || dev >= 64 || !attr_set[dev])) {
    TXB_CUDA(cudaFuncSetAttribute(k_kv_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kCopyWarps * kWarpStages * kPiece)));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  k_kv_stream<<<grid, kCopyThreads, smem, (cudaStream_t)stream>>>(*ks);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_read_u64(const uint64_t* const* ptrs, int n, uint64_t* out) {
  if (n <= 0) return TXB_OK;
  if (!ptrs || !out || n > 64) {
    set_error("txb_read_u64: null arguments or more than 64 words");
    return TXB_ERR_TRANSFER;
  }
  DeviceFor on_dev(nullptr, ptrs[0]);
  static thread_local cudaStream_t side[64] = {nullptr};
  static thread_local uint64_t* host[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  const int d = dev >= 0 && dev < 64 ? dev : 0;
  if (!side[d]) TXB_CUDA(cudaStreamCreateWithFlags(&side[d], cudaStreamNonBlocking));
  if (!host[d]) TXB_CUDA(cudaHostAlloc(&host[d], 64 * sizeof(uint64_t), cudaHostAllocPortable));
  for (int i = 0; i < n; ++i)
    TXB_CUDA(cudaMemcpyAsync(host[d] + i, ptrs[i], sizeof(uint64_t), cudaMemcpyDeviceToHost, side[d]));
  TXB_CUDA(cudaStreamSynchronize(side[d]));
  for (int i = 0; i < n; ++i) out[i] = host[d][i];
  return TXB_OK;
}

int txb_imm_slot(uint64_t* table, uint32_t imm, int insert, int64_t* out_slot) {
  if (!table || !out_slot) {
    set_error("txb_imm_slot: null table or output");
    return TXB_ERR_TRANSFER;
  }
  DeviceFor on_dev(nullptr, table);
  static thread_local cudaStream_t side[64] = {nullptr};
  static thread_local int64_t* host_out[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  const int d = dev >= 0 && dev < 64 ? dev : 0;
  if (!side[d]) TXB_CUDA(cudaStreamCreateWithFlags(&side[d], cudaStreamNonBlocking));
  if (!host_out[d]) TXB_CUDA(cudaHostAlloc(&host_out[d], sizeof(int64_t), cudaHostAllocMapped | cudaHostAllocPortable));
  int64_t* dptr = nullptr;
  TXB_CUDA(cudaHostGetDevicePointer(&dptr, host_out[d], 0));
  *host_out[d] = -2;
  k_imm_probe<<<1, 32, 0, side[d]>>>(table, imm, insert, dptr);
  TXB_CUDA(cudaGetLastError());
  TXB_CUDA(cudaStreamSynchronize(side[d]));
  *out_slot = *host_out[d];
  if (*out_slot < 0 && insert) {
    set_error("ImmCounter table full (%d slots)", TXB_IMM_SLOTS);
    return TXB_ERR_TRANSFER;
  }
  return TXB_OK;
}

// Stream memory operations (the device layer clock): the copy stream waits
// in the GPU front end until a u64 word reaches a value, the compute stream
// writes the word -- no SM and no host thread involved.  Through the driver
// entry points (cuStreamWaitValue64 / cuStreamWriteValue64); a one-thread
// kernel stands in where the driver lacks 64-bit stream memory operations.
typedef int (*PFN_wait64)(void*, uint64_t, uint64_t, unsigned int);
typedef int (*PFN_write64)(void*, uint64_t, uint64_t, unsigned int);

static bool stream_memops(PFN_wait64* w, PFN_write64* wr) {
  static int state = -1;
  static PFN_wait64 fw = nullptr;
  static PFN_write64 fwr = nullptr;
  if (state < 0) {
    cudaDriverEntryPointQueryResult q1, q2;
    void* a = nullptr;
    void* b = nullptr;
    const bool ok = cudaGetDriverEntryPoint("cuStreamWaitValue64", &a, cudaEnableDefault, &q1) == cudaSuccess &&
                    cudaGetDriverEntryPoint("cuStreamWriteValue64", &b, cudaEnableDefault, &q2) == cudaSuccess &&
                    q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && a && b;
    cudaGetLastError();
    int dev = 0, attr = 0;
    cudaGetDevice(&dev);
    // CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS = 118 (cudaDevAttr has no alias)
    cudaDeviceGetAttribute(&attr, (cudaDeviceAttr)118, dev);
    cudaGetLastError();
    state = ok && attr ? 1 : 0;
    if (state) {
      fw = reinterpret_cast<PFN_wait64>(a);
      fwr = reinterpret_cast<PFN_write64>(b);
    }
    if (getenv("TXB_NO_STREAM_MEMOPS")) state = 0;
  }
  *w = fw;
  *wr = fwr;
  return state == 1;
}

int txb_stream_write_value64(uint64_t* addr, uint64_t value, void* stream) {
  DeviceFor on_dev(stream, addr);
  PFN_wait64 w;
  PFN_write64 wr;
  if (stream_memops(&w, &wr)) {
    const int rc = wr(stream, (uint64_t)(uintptr_t)addr, value, 0 /* CU_STREAM_WRITE_VALUE_DEFAULT: fenced */);
    if (rc == 0) return TXB_OK;
  }
  k_write_value<<<1, 32, 0, (cudaStream_t)stream>>>(addr, value);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_stream_wait_value64(const uint64_t* addr, uint64_t value, uint64_t timeout_ns, uint32_t* err, void* stream) {
  DeviceFor on_dev(stream, addr);
  PFN_wait64 w;
  PFN_write64 wr;
  if (stream_memops(&w, &wr)) {
    const int rc = w(stream, (uint64_t)(uintptr_t)addr, value, 0x1 /* CU_STREAM_WAIT_VALUE_GEQ */);
    if (rc == 0) return TXB_OK;
  }
  k_imm_wait<<<1, 32, 0, (cudaStream_t)stream>>>(addr, value, timeout_ns, err);
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
