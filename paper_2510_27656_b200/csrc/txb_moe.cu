// MoE expert-parallel dispatch/combine over one-sided peer stores and an
// order-free completion counter (the WriteImm + ImmCounter design of
// arXiv 2510.27656 section 6, reference: railtx/moe.py).
//
// One step on rank `me` is five stream-ordered kernels:
//   k_route      count row + stable per-expert ranks + pos; the own count
//                row is stored into every peer's route matrix and a step tag
//                is release-published (reference: route scatter, imm_route).
//   k_dispatch   acquire-waits for all route rows and for every peer's
//                previous-step barrier, derives the layout and stores each
//                token copy (optionally encoded: fp8 per-token scale / bf16)
//                directly at its final grouped row on the owning rank, then
//                release-adds the row count to that rank's token counter.
//   k_recv       builds rows/sources/return-slot metadata and zero padding,
//                then acquire-waits for the expected number of rows.
//   k_comb_send  stores every valid grouped output row back into its
//                source's combine buffer at the originating send slot,
//                release-adds counts, and (last CTA) publishes the step
//                barrier tag to every peer (buffer-reuse barrier, moe.dbar).
//   k_comb_recv  acquire-waits for n*R rows, fp32 weighted sum per token.
//
// Completion is counted, never ordered: a waiter only compares a monotone
// counter with a cumulative threshold, so delivery order across NVLink is
// irrelevant (engine.py:9-17 / ImmCounterTable engine.py:138-205).
#include <cstdio>

#include "txb_rows.cuh"

namespace txb {

constexpr int kGroupPad = 8;     // moe.py:27
constexpr int kRouteThreads = 1024;
constexpr int kMaxExperts = 1536;  // route-kernel shared-memory bound (33*E*4 B)

__device__ __forceinline__ int64_t load_route(const void* r, int i32, int64_t i) {
  return i32 ? (int64_t) reinterpret_cast<const int32_t*>(r)[i] : reinterpret_cast<const int64_t*>(r)[i];
}

__device__ __forceinline__ int64_t pad_up(int64_t x) { return (x + kGroupPad - 1) / kGroupPad * kGroupPad; }

// ---------------------------------------------------------------- k_route

__global__ void __launch_bounds__(kRouteThreads)
k_route(txb_moe_shape s, const void* __restrict__ routes, int i32, int64_t n,
        void* const* __restrict__ peers, void* region, int32_t* __restrict__ rank_out,
        int64_t* __restrict__ pos) {
  extern __shared__ uint32_t sm[];
  const int E = s.experts, R = s.topk, N = s.ranks;
  uint32_t* hist = sm;       // [E]   running per-expert counts
  uint32_t* wc = sm + E;     // [32][E] per-warp counts, then exclusive bases
  __shared__ uint32_t bad;
  __shared__ uint32_t tmp[33];
  __shared__ uint64_t step_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  Flags* f = flags_of(region, s);
  if (tid == 0) {
    bad = 0;
    step_sh = f->step + 1;
  }
  for (int e = tid; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int64_t M = n * R;
  for (int64_t base = 0; base < M; base += blockDim.x) {
    for (int i = tid; i < nwarps * E; i += blockDim.x) wc[i] = 0;
    __syncthreads();
    const int64_t i = base + tid;
    int e = -1;
    if (i < M) {
      const int64_t v = load_route(routes, i32, i);
      if (v < 0 || v >= E) {
        atomicOr(&bad, TXB_EV_ROUTE_RANGE);
      } else {
        e = (int)v;
        const int64_t t = i / R;
        const int j = (int)(i - t * R);
        for (int jj = 0; jj < j; ++jj)
          if (load_route(routes, i32, t * R + jj) == v) atomicOr(&bad, TXB_EV_ROUTE_DUP);
      }
    }
    // stable rank among equal experts inside the warp, then across warps
    const uint32_t peers_mask = __match_any_sync(0xffffffffu, e);
    const int lr = __popc(peers_mask & lanemask_lt());
    if (e >= 0 && lr == 0) wc[warp * E + e] = __popc(peers_mask);
    __syncthreads();
    for (int x = tid; x < E; x += blockDim.x) {
      uint32_t run = hist[x];
      for (int w = 0; w < nwarps; ++w) {
        const uint32_t c = wc[w * E + x];
        wc[w * E + x] = run;
        run += c;
      }
      hist[x] = run;
    }
    __syncthreads();
    if (e >= 0) rank_out[i] = (int32_t)(wc[warp * E + e] + lr);
    __syncthreads();
  }
  const uint32_t b = bad;
  if (b) {
    for (int e = tid; e < E; e += blockDim.x) hist[e] = 0;  // publish an empty row
  }
  for (int e = tid; e < E; e += blockDim.x) wc[e] = hist[e];
  __syncthreads();
  block_excl_scan<uint32_t>(wc, E, tmp);
  // pos[t,j] = first send slot of expert e + stable rank (moe.py:514-521)
  for (int64_t i = tid; i < M; i += blockDim.x) {
    const int64_t v = load_route(routes, i32, i);
    pos[i] = b ? -1 : (int64_t)wc[(int)v] + rank_out[i];
  }
  // route-row scatter: own counts into every rank's matrix row `me`
  const uint64_t step = step_sh;
  const int slot = (int)(step & 1);
  for (int idx = tid; idx < N * E; idx += blockDim.x) {
    const int d = idx / E, e = idx - d * E;
    route_of(peers[d], s, slot)[(size_t)s.me * E + e] = hist[e];
  }
  __syncthreads();
  if (tid == 0) {
    fence_sys();
    for (int d = 0; d < N; ++d) st_release_sys(&flags_of(peers[d], s)->route_tag[slot][s.me], step);
    f->step = step;
    f->comb_target += b ? 0 : (uint64_t)M;
    if (b) atomicOr(&f->err, b);
  }
}

// ------------------------------------------------------------- k_dispatch

constexpr int kDispThreads = 512;

template <int SRC, int ELEM>
__global__ void __launch_bounds__(kDispThreads)
k_dispatch(txb_moe_shape s, const void* __restrict__ x, int64_t n, const void* __restrict__ routes,
           int i32, const int32_t* __restrict__ rank_in, void* const* __restrict__ peers, void* region,
           uint64_t timeout_ns) {
  extern __shared__ int64_t dsm[];
  const int N = s.ranks, E = s.experts, L = s.local_experts, R = s.topk;
  int64_t* baseg = dsm;      // [E] grouped base row on the owner for (me, expert)
  int64_t* padded = dsm + E; // [E+1] scan scratch
  __shared__ int64_t tmp[33];
  __shared__ uint32_t cnt[TXB_MAX_RANKS];
  __shared__ uint8_t* dstp[kMaxTopk];
  __shared__ uint32_t fail;
  __shared__ float red[33];
  __shared__ uint64_t recv_me;
  const int tid = threadIdx.x;
  Flags* f = flags_of(region, s);
  const uint64_t step = *reinterpret_cast<volatile uint64_t*>(&f->step);
  const int slot = (int)(step & 1);
  if (tid == 0) {
    fail = 0;
    recv_me = 0;
  }
  for (int q = tid; q < N; q += blockDim.x) cnt[q] = 0;
  __syncthreads();
  // wait: every route row of this step, every peer past the previous step
  if (tid < 32) {
    const uint64_t dl = globaltimer() + timeout_ns;
    for (int q = tid; q < N; q += 32) {
      if (!spin_ge(&f->route_tag[slot][q], step, dl)) atomicOr(&fail, TXB_EV_WAIT_ROUTE);
      if (!spin_ge(&f->done[q], step - 1, dl)) atomicOr(&fail, TXB_EV_WAIT_BARRIER);
    }
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) atomicOr(&f->err, fail);
    return;
  }
  // layout (compute_layout + grouped order, moe.py:200-225, 699-716)
  const uint32_t* C = route_of(region, s, slot);
  for (int e = tid; e < E; e += blockDim.x) {
    int64_t col = 0, pre = 0;
    for (int q = 0; q < N; ++q) {
      const uint32_t c = C[(size_t)q * E + e];
      col += c;
      if (q < s.me) pre += c;
    }
    padded[e] = pad_up(col);
    baseg[e] = pre;
    if (blockIdx.x == 0 && e / L == s.me) atomicAdd((unsigned long long*)&recv_me, (unsigned long long)col);
  }
  __syncthreads();
  const int64_t tot = block_excl_scan<int64_t>(padded, E, tmp);
  if (tid == 0) padded[E] = tot;
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) baseg[e] += padded[e] - padded[(e / L) * L];
  for (int d = tid; d < N; d += blockDim.x) {
    const int64_t need = padded[(d + 1) * L] - padded[d * L];
    if (need > s.grouped_rows) atomicOr(&fail, TXB_EV_CAPACITY);
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) atomicOr(&f->err, fail);
    return;
  }
  if (blockIdx.x == 0 && tid == 0) f->tok_target += recv_me;
  const int64_t P = s.payload_bytes;
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (tid < R) {
      const int e = (int)load_route(routes, i32, t * R + tid);
      const int d = e / L;
      const int64_t g = baseg[e] + rank_in[t * R + tid];
      dstp[tid] = grouped_of(peers[d], s) + g * P;
      atomicAdd(&cnt[d], 1u);
    }
    __syncthreads();
    if constexpr (SRC == TXB_SRC_ROWS) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(x) + t * P;
      const int w = vec_width(src, dstp[0], P);
      if (w == 16) {
        const int64_t nv = P >> 4;
        for (int64_t v = tid; v < nv; v += blockDim.x) {
          const int4 val = reinterpret_cast<const int4*>(src)[v];
          for (int j = 0; j < R; ++j) reinterpret_cast<int4*>(dstp[j])[v] = val;
        }
      } else {
        for (int j = 0; j < R; ++j) copy_row(dstp[j], src, P, tid, blockDim.x);
      }
    } else {
      encode_store_row<SRC, ELEM>(x, t, s.hidden, s.scales, P, dstp, R, red);
    }
    __syncthreads();
  }
  // completion: per-destination release-add of the rows this CTA stored
  if (tid == 0) {
    fence_sys();
    for (int d = 0; d < N; ++d)
      if (cnt[d]) red_release_sys_add(&flags_of(peers[d], s)->tok_ctr, cnt[d]);
  }
}

// ----------------------------------------------------------------- k_recv

constexpr int kRecvThreads = 256;

// Receive side: every CTA derives the (small) per-(source, local expert)
// tables from the route matrix, then the grid walks the grouped rows with
// one warp per row: metadata by lane 0, zero fill of padding rows by the
// whole warp.  CTA 0 finally acquire-waits for the token receipts.
__global__ void __launch_bounds__(kRecvThreads)
k_recv(txb_moe_shape s, void* region, int64_t* __restrict__ rows, int64_t* __restrict__ sources,
       int32_t* __restrict__ ret, int64_t* __restrict__ info, uint64_t timeout_ns) {
  extern __shared__ int64_t rsm[];
  const int N = s.ranks, E = s.experts, L = s.local_experts, me = s.me;
  int64_t* a = rsm;                    // [N][L] counts into my experts
  int64_t* rowbase = a + N * L;        // [N*L+1] flattened exclusive prefix = recv slot base
  int64_t* retbase = rowbase + N * L + 1;  // [N][L] send slot base on the source
  int64_t* gstart = retbase + N * L;   // [L+1] group starts (padded)
  int64_t* gsize = gstart + L + 1;     // [L]
  int64_t* srcpre = gsize + L;         // [L][N+1] prefix over sources within a group
  int64_t* pre_all = srcpre + L * (N + 1);  // [N] sum_{e' < me*L} C[q][e']
  __shared__ int64_t tmp[33];
  const int tid = threadIdx.x, nt = blockDim.x;
  Flags* f = flags_of(region, s);
  const uint64_t step = *reinterpret_cast<volatile uint64_t*>(&f->step);
  const int slot = (int)(step & 1);
  const uint32_t* C = route_of(region, s, slot);
  for (int i = tid; i < N * L; i += nt) {
    const int q = i / L, le = i - q * L;
    a[i] = C[(size_t)q * E + me * L + le];
    rowbase[i] = a[i];
  }
  for (int q = tid; q < N; q += nt) pre_all[q] = 0;
  __syncthreads();
  if (me > 0) {
    for (int i = tid; i < N * me * L; i += nt) {
      const int q = i / (me * L), e = i - q * (me * L);
      atomicAdd((unsigned long long*)&pre_all[q], (unsigned long long)C[(size_t)q * E + e]);
    }
  }
  for (int le = tid; le < L; le += nt) {
    int64_t run = 0;
    for (int q = 0; q < N; ++q) {
      srcpre[le * (N + 1) + q] = run;
      run += a[q * L + le];
    }
    srcpre[le * (N + 1) + N] = run;
    gsize[le] = run;
    gstart[le] = pad_up(run);
  }
  __syncthreads();
  const int64_t padded_total = block_excl_scan<int64_t>(gstart, L, tmp);
  // recv slot base: recv_start[me][q] + sum_{le'<le} a[q][le'] is exactly the
  // exclusive prefix of a[] flattened source-major (moe.py:178-184, 204-213)
  const int64_t recv_total = block_excl_scan<int64_t>(rowbase, N * L, tmp);
  if (tid == 0) {
    gstart[L] = padded_total;
    rowbase[N * L] = recv_total;
  }
  __syncthreads();
  for (int i = tid; i < N * L; i += nt) {
    const int q = i / L;
    retbase[i] = pre_all[q] + (rowbase[i] - rowbase[q * L]);
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int le = tid; le < L; le += nt) {
      info[le] = gsize[le];
      info[L + le] = gstart[le];
    }
    if (tid == 0) {
      info[2 * L] = padded_total;
      info[2 * L + 1] = recv_total;
    }
  }
  const int64_t P = s.payload_bytes;
  uint8_t* G = grouped_of(region, s);
  const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
  for (int64_t g = (int64_t)blockIdx.x * nwarp + warp; g < padded_total; g += (int64_t)gridDim.x * nwarp) {
    int lo = 0, hi = L - 1;  // last le with gstart[le] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (gstart[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const int le = lo;
    const int64_t k = g - gstart[le];
    if (k >= gsize[le]) {
      if (lane == 0) {
        rows[g] = -1;
        sources[g] = -1;
        ret[g] = -1;
      }
      zero_row(G + g * P, P, lane, 32);  // padding rows are zero (moe.py:719)
    } else if (lane == 0) {
      const int64_t* sp = srcpre + le * (N + 1);
      int q = 0;
      while (sp[q + 1] <= k) ++q;
      const int64_t kk = k - sp[q];
      rows[g] = rowbase[q * L + le] + kk;
      sources[g] = q;
      ret[g] = (int32_t)(retbase[q * L + le] + kk);
    }
  }
  // acquire-wait for every expected row (token immediate count)
  if (blockIdx.x == 0 && tid == 0) {
    const uint64_t dl = globaltimer() + timeout_ns;
    if (!spin_ge(&f->tok_ctr, f->tok_target, dl)) atomicOr(&f->err, TXB_EV_WAIT_TOKEN);
    info[2 * L + 2] = (int64_t)*reinterpret_cast<volatile uint32_t*>(&f->err);
  }
}

// ------------------------------------------------------------ k_comb_send

constexpr int kCombThreads = 512;

__global__ void __launch_bounds__(kCombThreads)
k_comb_send(txb_moe_shape s, const uint8_t* __restrict__ out, int64_t ld, void* const* __restrict__ peers,
            void* region, const int64_t* __restrict__ sources, const int32_t* __restrict__ ret,
            const int64_t* __restrict__ info) {
  __shared__ uint32_t cnt[TXB_MAX_RANKS];
  const int N = s.ranks, L = s.local_experts, tid = threadIdx.x;
  Flags* f = flags_of(region, s);
  for (int q = tid; q < N; q += blockDim.x) cnt[q] = 0;
  __syncthreads();
  const int64_t total = info[2 * L];
  const int64_t Pc = s.comb_bytes;
  const int lane = tid & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (tid >> 5); g < total; g += nw) {
    const int64_t q = sources[g];
    if (q < 0) continue;
    copy_row(comb_of(peers[q], s) + (int64_t)ret[g] * Pc, out + g * ld, Pc, lane, 32);
    if (lane == 0) atomicAdd(&cnt[q], 1u);
  }
  __syncthreads();
  if (tid == 0) {
    fence_sys();
    for (int q = 0; q < N; ++q)
      if (cnt[q]) red_release_sys_add(&flags_of(peers[q], s)->comb_ctr, cnt[q]);
    const uint32_t t = atomicAdd(&f->ticket, 1u);
    if (t == gridDim.x - 1) {
      f->ticket = 0;
      fence_sys();
      const uint64_t step = *reinterpret_cast<volatile uint64_t*>(&f->step);
      for (int q = 0; q < N; ++q) st_release_sys(&flags_of(peers[q], s)->done[s.me], step);
    }
  }
}

// ------------------------------------------------------------ k_comb_recv

constexpr int kCombRecvThreads = 512;

template <int ELEM>
__global__ void __launch_bounds__(kCombRecvThreads)
k_comb_recv(txb_moe_shape s, void* region, const int64_t* __restrict__ pos, const float* __restrict__ w,
            int64_t n, void* out, int out_bf16, uint64_t timeout_ns) {
  __shared__ uint32_t ok;
  Flags* f = flags_of(region, s);
  if (threadIdx.x == 0) {
    const uint64_t dl = globaltimer() + timeout_ns;
    ok = spin_ge(&f->comb_ctr, f->comb_target, dl) ? 1u : 0u;
    if (!ok) atomicOr(&f->err, TXB_EV_WAIT_COMBINE);
  }
  __syncthreads();
  if (!ok) return;
  combine_rows<ELEM>(comb_of(region, s), s.comb_bytes, s.hidden, pos, w, n, s.topk, out, out_bf16);
}

// -------------------------------------------------------------- k_barrier

// All-rank device barrier (the reference's submit_barrier with one imm per
// peer, engine.py:599-619): publish my epoch into every peer's slot, then
// acquire-wait until every peer's epoch has reached mine.
__global__ void k_barrier(txb_moe_shape s, void* const* __restrict__ peers, void* region, uint64_t timeout_ns) {
  Flags* f = flags_of(region, s);
  __shared__ uint64_t ep;
  __shared__ uint32_t fail;
  if (threadIdx.x == 0) {
    ep = f->bar_epoch + 1;
    f->bar_epoch = ep;
    fail = 0;
  }
  __syncthreads();
  const int N = s.ranks;
  for (int q = threadIdx.x; q < N; q += blockDim.x) st_release_sys(&flags_of(peers[q], s)->bar[s.me], ep);
  const uint64_t dl = globaltimer() + timeout_ns;
  for (int q = threadIdx.x; q < N; q += blockDim.x)
    if (!spin_ge(&f->bar[q], ep, dl)) atomicOr(&fail, TXB_EV_WAIT_BARRIER);
  __syncthreads();
  if (threadIdx.x == 0 && fail) atomicOr(&f->err, fail);
}

// ------------------------------------------------------------------ host

static int sm_count(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

static uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

static int check_shape(const txb_moe_shape* s) {
  if (!s) {
    set_error("null shape");
    return TXB_ERR_PROTOCOL;
  }
  if (s->payload_bytes <= 0 || s->region_bytes == 0) {
    set_error("shape not planned (call txb_moe_plan)");
    return TXB_ERR_PROTOCOL;
  }
  return TXB_OK;
}

}  // namespace txb

using namespace txb;

extern "C" {

int txb_moe_plan(txb_moe_shape* s) {
  if (!s) {
    set_error("null shape");
    return TXB_ERR_PROTOCOL;
  }
  // RoutingSpec.__post_init__ (moe.py:52-70)
  if (s->ranks < 1) { set_error("rank count must be positive"); return TXB_ERR_PROTOCOL; }
  if (s->ranks > TXB_MAX_RANKS) { set_error("rank count %d above %d", s->ranks, TXB_MAX_RANKS); return TXB_ERR_PROTOCOL; }
  if (s->experts < 1 || s->experts % s->ranks) {
    set_error("expert count %d is not a positive multiple of %d ranks", s->experts, s->ranks);
    return TXB_ERR_PROTOCOL;
  }
  if (s->topk < 1 || s->topk > s->experts) { set_error("topk %d outside 1..%d", s->topk, s->experts); return TXB_ERR_PROTOCOL; }
  if (s->max_tokens < 1) { set_error("max_tokens must be positive"); return TXB_ERR_PROTOCOL; }
  if (s->hidden < 1) { set_error("hidden size must be positive"); return TXB_ERR_PROTOCOL; }
  if (s->elem_size != 1 && s->elem_size != 2 && s->elem_size != 4) {
    set_error("element size %d not in (1, 2, 4)", s->elem_size);
    return TXB_ERR_PROTOCOL;
  }
  if (s->scales < 0) { set_error("scale count must be non-negative"); return TXB_ERR_PROTOCOL; }
  if (s->elem_size == 1 && s->scales < 1) { set_error("quantized payloads need at least one scale slot"); return TXB_ERR_PROTOCOL; }
  if (s->comb_elem_size == 0) { s->comb_elem_size = s->elem_size; s->comb_scales = s->scales; }
  if (s->comb_elem_size != 1 && s->comb_elem_size != 2 && s->comb_elem_size != 4) {
    set_error("combine element size %d not in (1, 2, 4)", s->comb_elem_size);
    return TXB_ERR_PROTOCOL;
  }
  if (s->comb_scales < 0 || (s->comb_elem_size == 1 && s->comb_scales < 1)) {
    set_error("combine rows need a non-negative scale count (>=1 for fp8)");
    return TXB_ERR_PROTOCOL;
  }
  if (s->topk > kMaxTopk) { set_error("topk %d above the supported %d", s->topk, kMaxTopk); return TXB_ERR_PROTOCOL; }
  if (s->experts > kMaxExperts) { set_error("expert count %d above the supported %d", s->experts, kMaxExperts); return TXB_ERR_PROTOCOL; }
  if (s->me < 0 || s->me >= s->ranks) { set_error("rank %d outside 0..%d", s->me, s->ranks - 1); return TXB_ERR_PROTOCOL; }
  const int64_t N = s->ranks, T = s->max_tokens, R = s->topk;
  s->local_experts = s->experts / s->ranks;
  const int64_t L = s->local_experts;
  s->payload_bytes = (int64_t)s->hidden * s->elem_size + 4LL * s->scales;
  s->comb_bytes = (int64_t)s->hidden * s->comb_elem_size + 4LL * s->comb_scales;
  s->capacity = N * T * (R > L ? R : L);
  // a token sends at most min(R, L) copies to one destination
  s->grouped_rows = N * T * (R < L ? R : L) + L * (kGroupPad - 1);
  s->comb_rows = T * R > 0 ? T * R : 1;
  uint64_t off = 0;
  s->off_flags = off;
  off = align_up(off + sizeof(Flags), 4096);
  s->off_route = off;
  off = align_up(off + 2ull * N * s->experts * 4, 4096);
  s->off_grouped = off;
  off = align_up(off + (uint64_t)s->grouped_rows * s->payload_bytes, 4096);
  s->off_comb = off;
  off = align_up(off + (uint64_t)s->comb_rows * s->comb_bytes, 4096);
  s->region_bytes = off;
  return TXB_OK;
}

int txb_moe_route(const txb_moe_shape* s, const void* routes, int routes_i32, int64_t n, void* const* peers,
                  void* region, int32_t* rank_scratch, int64_t* pos, uint64_t timeout_ns, void* stream) {
  (void)timeout_ns;
  if (int rc = check_shape(s)) return rc;
  if (n < 0 || n > s->max_tokens) {
    set_error("%lld tokens exceed the %d-token limit", (long long)n, s->max_tokens);
    return TXB_ERR_PROTOCOL;
  }
  TXB_CUDA(cudaSetDevice(s->device));
  const size_t smem = (size_t)(1 + kRouteThreads / 32) * s->experts * sizeof(uint32_t);
  if (smem > 48 * 1024) TXB_CUDA(cudaFuncSetAttribute(k_route, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_route<<<1, kRouteThreads, smem, (cudaStream_t)stream>>>(*s, routes, routes_i32, n, peers, region,
                                                             rank_scratch, pos);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_moe_dispatch(const txb_moe_shape* s, const void* x, int src_kind, int64_t n, const void* routes,
                     int routes_i32, const int32_t* rank_scratch, void* const* peers, void* region,
                     uint64_t timeout_ns, int grid, void* stream) {
  if (int rc = check_shape(s)) return rc;
  TXB_CUDA(cudaSetDevice(s->device));
  if (grid <= 0) {
    const int64_t g = n < 1 ? 1 : n;
    grid = (int)(g < 4 * sm_count(s->device) ? g : 4 * sm_count(s->device));
  }
  const size_t smem = (size_t)(2 * s->experts + 1) * sizeof(int64_t);
  cudaStream_t st = (cudaStream_t)stream;
#define TXB_LAUNCH_D(SRC, ELEM)                                                                   \
  do {                                                                                            \
    auto kfn = k_dispatch<SRC, ELEM>;                                                             \
    if (smem > 48 * 1024) TXB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kfn<<<grid, kDispThreads, smem, st>>>(*s, x, n, routes, routes_i32, rank_scratch, peers, region, timeout_ns); \
  } while (0)
  if (src_kind == TXB_SRC_ROWS) {
    TXB_LAUNCH_D(TXB_SRC_ROWS, 1);
  } else if (src_kind == TXB_SRC_F32 || src_kind == TXB_SRC_BF16) {
    const bool f32 = src_kind == TXB_SRC_F32;
    switch (s->elem_size) {
      case 1: if (f32) TXB_LAUNCH_D(TXB_SRC_F32, 1); else TXB_LAUNCH_D(TXB_SRC_BF16, 1); break;
      case 2: if (f32) TXB_LAUNCH_D(TXB_SRC_F32, 2); else TXB_LAUNCH_D(TXB_SRC_BF16, 2); break;
      default: if (f32) TXB_LAUNCH_D(TXB_SRC_F32, 4); else TXB_LAUNCH_D(TXB_SRC_BF16, 4); break;
    }
  } else {
    set_error("unknown source kind %d", src_kind);
    return TXB_ERR_PROTOCOL;
  }
#undef TXB_LAUNCH_D
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_moe_dispatch_recv(const txb_moe_shape* s, void* region, int64_t* rows, int64_t* sources,
                          int32_t* ret_slot, int64_t* info, uint64_t timeout_ns, void* stream) {
  if (int rc = check_shape(s)) return rc;
  TXB_CUDA(cudaSetDevice(s->device));
  const int N = s->ranks, L = s->local_experts;
  const size_t smem = (size_t)(3 * N * L + 1 + 2 * L + 1 + L * (N + 1) + N) * sizeof(int64_t);
  if (smem > 48 * 1024) TXB_CUDA(cudaFuncSetAttribute(k_recv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t maxrows = s->grouped_rows;
  const int64_t wpb = kRecvThreads / 32;
  int grid = (int)((maxrows + wpb - 1) / wpb);
  if (grid > 2 * sm_count(s->device)) grid = 2 * sm_count(s->device);
  if (grid < 1) grid = 1;
  k_recv<<<grid, kRecvThreads, smem, (cudaStream_t)stream>>>(*s, region, rows, sources, ret_slot, info, timeout_ns);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_moe_combine_send(const txb_moe_shape* s, const void* outputs, int64_t ld, void* const* peers, void* region,
                         const int64_t* sources, const int32_t* ret_slot, const int64_t* info, int grid,
                         void* stream) {
  if (int rc = check_shape(s)) return rc;
  TXB_CUDA(cudaSetDevice(s->device));
  if (grid <= 0) {
    const int64_t rows = s->grouped_rows;
    const int64_t want = (rows + (kCombThreads / 32) - 1) / (kCombThreads / 32);
    const int cap = 2 * sm_count(s->device);
    grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  }
  k_comb_send<<<grid, kCombThreads, 0, (cudaStream_t)stream>>>(*s, (const uint8_t*)outputs, ld, peers, region,
                                                                 sources, ret_slot, info);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_moe_combine_recv(const txb_moe_shape* s, void* region, const int64_t* pos, const float* weights, int64_t n,
                         void* out, int out_bf16, uint64_t timeout_ns, void* stream) {
  if (int rc = check_shape(s)) return rc;
  TXB_CUDA(cudaSetDevice(s->device));
  int grid = (int)(n < 1 ? 1 : (n < 4 * sm_count(s->device) ? n : 4 * sm_count(s->device)));
  cudaStream_t st = (cudaStream_t)stream;
  switch (s->comb_elem_size) {
    case 1: k_comb_recv<1><<<grid, kCombRecvThreads, 0, st>>>(*s, region, pos, weights, n, out, out_bf16, timeout_ns); break;
    case 2: k_comb_recv<2><<<grid, kCombRecvThreads, 0, st>>>(*s, region, pos, weights, n, out, out_bf16, timeout_ns); break;
    default: k_comb_recv<4><<<grid, kCombRecvThreads, 0, st>>>(*s, region, pos, weights, n, out, out_bf16, timeout_ns); break;
  }
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_moe_barrier(const txb_moe_shape* s, void* const* peers, void* region, uint64_t timeout_ns, void* stream) {
  if (int rc = check_shape(s)) return rc;
  TXB_CUDA(cudaSetDevice(s->device));
  k_barrier<<<1, 128, 0, (cudaStream_t)stream>>>(*s, peers, region, timeout_ns);
  TXB_CUDA(cudaGetLastError());
  return TXB_OK;
}

int txb_moe_status(const txb_moe_shape* s, void* region, uint32_t* err, uint64_t* counters, int64_t ncounters) {
  if (int rc = check_shape(s)) return rc;
  TXB_CUDA(cudaSetDevice(s->device));
  // read on a private non-blocking stream so the snapshot never waits for
  // (or serialises with) kernels that are spinning on other streams
  static thread_local cudaStream_t side[64] = {nullptr};
  const int dev = s->device >= 0 && s->device < 64 ? s->device : 0;
  if (!side[dev]) TXB_CUDA(cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking));
  Flags h;
  TXB_CUDA(cudaMemcpyAsync(&h, flags_of(region, *s), sizeof(Flags), cudaMemcpyDeviceToHost, side[dev]));
  TXB_CUDA(cudaStreamSynchronize(side[dev]));
  if (err) *err = h.err;
  if (counters) {
    const int N = s->ranks;
    uint64_t buf[5 + 3 * TXB_MAX_RANKS];
    int k = 0;
    buf[k++] = h.step;
    buf[k++] = h.tok_ctr;
    buf[k++] = h.tok_target;
    buf[k++] = h.comb_ctr;
    buf[k++] = h.comb_target;
    for (int p = 0; p < 2; ++p)
      for (int q = 0; q < N; ++q) buf[k++] = h.route_tag[p][q];
    for (int q = 0; q < N; ++q) buf[k++] = h.done[q];
    for (int i = 0; i < k && i < ncounters; ++i) counters[i] = buf[i];
  }
  return TXB_OK;
}

}  // extern "C"
