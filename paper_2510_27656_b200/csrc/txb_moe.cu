// MoE expert-parallel dispatch/combine over one-sided peer stores and an
// order-free completion counter (the WriteImm + ImmCounter design of
// arXiv 2510.27656 section 6; reference: railtx/moe.py).
//
// A step is built from six phases (device functions below):
//   P1 route    per-expert counts + stable per-copy ranks + pos; the own
//               count row is stored into every peer's route matrix as
//               (step tag | count) words (reference: route scatter, imm_route)
//   P2 wait     acquire every route word of this step and every peer's
//               end-of-previous-step barrier (buffer reuse, moe.dbar)
//   P3 layout   compute_layout + grouped order from the route matrix
//   P4 tokens   each token copy is encoded (fp8 per-token scale / bf16 / raw)
//               and stored straight into its final grouped row on the owner;
//               per-destination row counts are added to the owner's token
//               counter after one release fence (the ImmCounter)
//   P5 recv     rows / sources / return-slot metadata, zeroed padding rows,
//               then acquire-wait for the expected number of token rows
//   C1 send     every valid grouped output row returns to its source's
//               combine buffer at the originating send slot (rows whose
//               source is this rank are read in place by C2)
//   C2 combine  acquire-wait for the returned rows, fp32 weighted sum per
//               token, last CTA publishes the end-of-step barrier tag
//
// Kernels:  split path  k_route(P1) k_dispatch(P2-P4) k_recv(P5)
//                       k_comb_send(C1) k_comb_recv(C2)
//           fused path  k_dispatch_fused(P1-P5) k_combine_fused(C1-C2),
//                       cooperative launches (one wave, every CTA resident).
// k_dispatch_fused<..., DECODE=true> is the decode-batch specialisation (one
// token per CTA, read and encoded before the route exchange, direct counts):
// it carries only the code that path executes, because a once-per-SM kernel
// of this kind is bound by instruction fetch when the code balloons.
// The split path is used when several ranks share one GPU (host-gated
// emulation: no kernel may spin on a rank queued behind it).
//
// Completion is counted, never ordered: a waiter compares a monotone
// counter with a cumulative threshold, so delivery order across NVLink is
// irrelevant (engine.py:9-17, ImmCounterTable engine.py:138-205).
#include <cstddef>
#include <cstdlib>
#include <cstdio>

#include "txb_rows.cuh"

namespace txb {

constexpr int kGroupPad = 8;       // moe.py:27
constexpr int kMaxExperts = 1536;  // shared-memory bound of the route phase
constexpr int kThreads = 512;      // block size of the main kernels
constexpr int kRouteThreads = 1024;
constexpr int kMaxOwn = 64;        // copies per CTA of the direct-count path
// Per-token combine completion for large batches (max_tokens above this, on
// every rank alike): each expert rank's warps return whole rows, fence and
// release-add a per-origin-token counter, so the origin reduces a token as
// soon as its rows are in instead of after the last row of the step.  Every
// dispatch kernel books the expected count (tokt) so the counters stay in
// step whichever path a step takes.
constexpr int kTokWaitMin = 256;
__host__ __device__ inline bool tok_mode(const txb_moe_shape& s) {
  return s.max_tokens > kTokWaitMin && s.ranks > 1;
}
// Per-token combine completion (tokc / tokt / srctok) runs with tok_mode.
// Measured at decode size (EP=2, DSv3 shape; profiles/r02/README.md):
// counting 2-KiB chunks per origin token, one fence per warp, made the
// returns take 18 us instead of 6-11 -- the system-scope fences of a CTA's
// warps do not overlap -- and a token's rows come from ~56 CTAs, so it
// completes with the slowest of them anyway.  Decode keeps one fence per
// CTA and the step's global combine counter.
__host__ __device__ inline bool per_token(const txb_moe_shape& s) { return tok_mode(s); }
// Completion unit of a returned row on tokc: its 2-KiB chunks.
constexpr int kChunk = 2048;
__host__ __device__ inline int comb_chunks(const txb_moe_shape& s) { return (int)((s.comb_bytes + kChunk - 1) / kChunk); }

// Bookkeeping adds to this rank's flags (targets, per-source diagnostics):
// a fire-and-forget reduction, not a load-add-store whose load is a round
// trip on the issuing CTA's critical path.
__device__ __forceinline__ void add_flag(uint64_t* p, uint64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

__device__ __forceinline__ int pad_up(int x) { return (x + kGroupPad - 1) / kGroupPad * kGroupPad; }

// Programmatic dependent launch (sm_90+): let the next kernel on the stream
// be scheduled now / wait for the previous one to complete.  Both are no-ops
// when the launch carries no programmatic dependency.
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Optional phase stamps for profiling (txb_moe_bufs.prof, [grid][32]).
__device__ __forceinline__ void stamp(const txb_moe_bufs& b, int k) {
  if (b.prof && threadIdx.x == 0) b.prof[blockIdx.x * 32 + k] = globaltimer();
}

__device__ __forceinline__ uint64_t cur_step(Flags* f) {
  return *reinterpret_cast<volatile uint64_t*>(&f->step) + 1;
}

// Shared-memory footprint of the phases (bytes), carved from one dynamic
// buffer and reused phase to phase; all tables are int32.
__host__ __device__ inline size_t smem_route(int E, int nwarps) { return (size_t)(1 + nwarps) * E * 4 + 16; }
__host__ __device__ inline size_t smem_layout(int E) { return (size_t)(2 * E + 1) * 4; }
__host__ __device__ inline size_t smem_recv(int N, int L) {
  return (size_t)(3 * N * L + 2 + 2 * L + L * (N + 1) + N + N + (N + 1)) * 4;
}
__host__ __device__ inline size_t smem_cmat(int N, int E) { return ((size_t)N * E * 4 + 15) / 16 * 16; }
// layout scratch [0, recv_offset), receive tables [recv_offset, cmat_offset),
// route matrix copy (Cs) after them; the route-count phase overlaps all
__host__ __device__ inline size_t recv_offset(const txb_moe_shape& s) {
  return (smem_layout(s.experts) + 15) / 16 * 16;
}
__host__ __device__ inline size_t cmat_offset(const txb_moe_shape& s) {
  return recv_offset(s) + (smem_recv(s.ranks, s.local_experts) + 15) / 16 * 16;
}

// large batches: the per-copy destination pointers after the route matrix
__host__ __device__ inline size_t flat_offset(const txb_moe_shape& s) {
  return (cmat_offset(s) + smem_cmat(s.ranks, s.experts) + 15) / 16 * 16;
}

// decode, one rank: [histogram E | staged ids n*R] then the receive tables
__host__ __device__ inline size_t solo_recv_offset(const txb_moe_shape& s, int64_t n) {
  return ((size_t)(s.experts + n * s.topk) * 4 + 16 + 15) / 16 * 16;
}

struct Shared {  // static shared state of one CTA
  uint32_t bad, fail, lfail, recv_me, direct;  // lfail: dispatch_layout's own flag (it follows wait_routes
                                               // with no barrier between: a shared flag would be reset
                                               // while slow threads still read wait_routes' result)
  int tmp[33];
  float red[33];
  uint32_t cnt[TXB_MAX_RANKS];   // rows stored per destination (token / combine counter)
  uint32_t pcnt[TXB_MAX_RANKS];  // speculative private rows stored per destination
  int32_t sst[TXB_MAX_RANKS];    // send_start[me][d]: first slab slot of destination d
  uint8_t* dstp[kMaxTopk];       // grouped-row destination of each own copy (null: private)
  uint8_t* pdst[kMaxTopk];       // private-slab destination of each own copy (null: none)
  uint32_t own_rank[kMaxOwn];
  int32_t own_e[kMaxOwn];
  int32_t own_i[kMaxOwn];
};

// ------------------------------------------------------------------- P1

// Direct counts: shared atomics (order-free) for the histogram; the stable
// rank of each of this CTA's copies (token order within an expert, the
// (local_expert, t, j) slab order of moe.py:514-521) is the number of
// earlier copies with its expert, counted afterwards by one warp per copy
// with ballots over the batch's expert ids (staged as int32 in `rv`, m
// entries of shared memory).  Validation (moe.py:142-155): range, and
// duplicates within a token -- R-1 shuffles when R divides 32 (a token's
// copies sit in consecutive lanes), loads otherwise.
// Stable rank of each of this CTA's nw copies: one warp per copy counts the
// earlier entries of the batch with the same expert (ballots over rv).
__device__ __forceinline__ void own_ranks(const int32_t* rv, int32_t* rank_out, int nw, Shared& sh, const Grp& g) {
  const int lane = g.tid & 31, warp = g.tid >> 5, nwarp = g.nt >> 5;
  #pragma unroll 1
  for (int k = warp; k < nw; k += nwarp) {
    const int e = sh.own_e[k], lim = sh.own_i[k];
    int cnt = 0;
#pragma unroll 8
    for (int b0 = 0; b0 < lim; b0 += 32) {
      const int q = b0 + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, q < lim && rv[q] == e));
    }
    if (lane == 0) rank_out[lim] = cnt;
    if (lane == 0) sh.own_rank[k] = (uint32_t)cnt;
  }
}

// with_ranks = false: histogram, staging and validation only (the caller
// runs own_ranks on another warp group).
// Duplicates within a token (moe.py:152-154) over the staged ids: each id
// against the token's earlier ones (out-of-range ids are -1, already
// latched).  Returns TXB_EV_ROUTE_DUP or 0 for the calling thread's share.
__device__ __forceinline__ uint32_t staged_dups(const int32_t* rv, int m, int R, const Grp& g) {
  bool dup = false;
  #pragma unroll 1
  for (int i = g.tid; i < m; i += g.nt) {
    const int j = i % R, v = rv[i];
    #pragma unroll 1
    for (int jj = i - j; jj < i; ++jj) dup |= v >= 0 && rv[jj] == v;
  }
  return dup ? TXB_EV_ROUTE_DUP : 0u;
}

// check_dups = false (the decode kernels, one token per CTA): the pass over
// the whole batch (~1.8 us measured on the routing role's critical path) is
// replaced by own_token_dups in the token role, which checks the CTA's own
// token while its row load is in flight.  A duplicate cannot send a store out
// of bounds -- every CTA counts the same ids -- so the step completes, and
// dispatch_recv reads the rank's error word after the kernel.
__device__ __forceinline__ void own_token_dups(const txb_moe_shape& s, const int64_t* routes, int64_t n,
                                               int cta, uint32_t* err, const Grp& g) {
  const int R = s.topk, E = s.experts;
  if (g.tid >= 32 || cta >= n) return;
  const int lane = g.tid;
  if (R <= 32) {
    int v = -1 - lane;  // lane-unique when unused or out of range (range is checked elsewhere)
    if (lane < R) {
      const int64_t x = routes[(int64_t)cta * R + lane];
      if (x >= 0 && x < E) v = (int)x;
    }
    int same = 0;
    #pragma unroll 1
    for (int j = 0; j < R; ++j) same += __shfl_sync(0xffffffffu, v, j) == v;
    if (__any_sync(0xffffffffu, lane < R && same > 1) && lane == 0) atomicOr(err, TXB_EV_ROUTE_DUP);
  } else if (lane == 0) {
    const int64_t* r = routes + (int64_t)cta * R;
    bool dup = false;
    #pragma unroll 1
    for (int j = 1; j < R; ++j)
      #pragma unroll 1
      for (int jj = 0; jj < j; ++jj) dup |= r[j] == r[jj];
    if (dup) atomicOr(err, TXB_EV_ROUTE_DUP);
  }
}
__device__ uint32_t route_counts_direct(const txb_moe_shape& s, const int64_t* routes, int64_t n, uint32_t* hist,
                                        int32_t* rv, int32_t* rank_out, int cta, int ncta, Shared& sh,
                                        const txb_moe_bufs& bufs, const Grp& g, bool with_ranks = true,
                                        bool check_dups = true) {
  const int E = s.experts, R = s.topk, tid = g.tid;
  const int m = (int)(n * R);
  const int nmine = n > cta ? (int)((n - cta + ncta - 1) / ncta) : 0;
  const int nw = nmine * R;
  // issue every route load this thread needs (its own copies and up to
  // kPre entries of the batch) before the first barrier
  constexpr int kPre = 4;
  const int nt = g.nt;
  const bool pre_ok = m <= kPre * nt;
  int64_t pre[kPre];
#pragma unroll
  for (int u = 0; u < kPre; ++u) pre[u] = (pre_ok && u * nt + tid < m) ? routes[u * nt + tid] : -1;
  #pragma unroll 1
  for (int e = tid; e < E; e += nt) hist[e] = 0;
  #pragma unroll 1
  for (int k = tid; k < nw; k += nt) {
    const int i = (cta + (k / R) * ncta) * R + (k % R);
    const int64_t v = routes[i];
    sh.own_e[k] = (v >= 0 && v < E) ? (int)v : -1;
    sh.own_i[k] = i;
  }
  if (tid == 0) {
    sh.bad = 0;
    sh.direct = 1;
  }
  g.sync();
  stamp(bufs, 19);

  // one entry: stage its id, count it, flag a range error (a short body:
  // this code runs cold once per CTA per step, so its size is its cost)
  auto entry = [&](int i, int64_t v) {
    if (i >= m) return;
    const bool in_range = v >= 0 && v < E;
    rv[i] = in_range ? (int)v : -1;
    if (in_range) atomicAdd(&hist[(int)v], 1u);
    else atomicOr(&sh.bad, TXB_EV_ROUTE_RANGE);
  };
  if (pre_ok) {
#pragma unroll
    for (int u = 0; u < kPre; ++u)
      if (u * nt < m) entry(u * nt + tid, pre[u]);
  } else {
    #pragma unroll 1
    for (int base = 0; base < m; base += nt) {
      const int i = base + tid;
      entry(i, i < m ? routes[i] : -1);
    }
  }
  g.sync();
  stamp(bufs, 22);
  if (check_dups) {
    const uint32_t d = staged_dups(rv, m, R, g);
    if (d) atomicOr(&sh.bad, d);
  }
  stamp(bufs, 27);
  if (with_ranks) own_ranks(rv, rank_out, nw, sh, g);
  g.sync();
  stamp(bufs, 28);
  const uint32_t b = sh.bad;
  if (b)
    #pragma unroll 1
    for (int e = tid; e < E; e += nt) hist[e] = 0;  // publish an empty row
  g.sync();
  return b;
}

// Chunked counts for large batches: per chunk of blockDim copies a warp
// match + per-warp counts + a scan over warps per expert give the stable
// ranks; copies of tokens t with t % ncta == cta get their rank stored.
__device__ __noinline__ uint32_t route_counts_chunked(const txb_moe_shape& s, const int64_t* routes, int64_t n,
                                                     uint32_t* hist, uint32_t* wc, int32_t* rank_out, int cta,
                                                     int ncta, Shared& sh) {
  const int E = s.experts, R = s.topk;
  const int tid = threadIdx.x, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (tid == 0) {
    sh.bad = 0;
    sh.direct = 0;
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
      const int64_t v = routes[i];
      if (v < 0 || v >= E) {
        atomicOr(&sh.bad, TXB_EV_ROUTE_RANGE);
      } else {
        e = (int)v;
        const int64_t t = i / R;
        for (int64_t q = t * R; q < i; ++q)
          if (routes[q] == v) atomicOr(&sh.bad, TXB_EV_ROUTE_DUP);
      }
    }
    const uint32_t same = __match_any_sync(0xffffffffu, e);
    const int lr = __popc(same & lanemask_lt());
    if (e >= 0 && lr == 0) wc[warp * E + e] = __popc(same);
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
    if (e >= 0 && (int)((i / R) % ncta) == cta) rank_out[i] = (int32_t)(wc[warp * E + e] + lr);
    __syncthreads();
  }
  const uint32_t b = sh.bad;
  if (b)
    for (int e = tid; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  return b;
}

// Grid barrier for cooperative launches (every CTA resident): one release
// atomic per CTA on a monotone 64-bit counter and an acquire poll.  CTA 0
// adds K - (ncta - 1) and every other CTA 1, so each barrier raises the
// counter by exactly K = TXB_MAX_CTAS whatever the grid size: every CTA of
// barrier j sees old in [jK, (j+1)K) and waits for (j+1)K.  One atomic hop,
// no reset (the last arriver does not have to bump a generation word).
__device__ void grid_sync(Flags* f, int ncta) {
  __syncthreads();
  if (threadIdx.x == 0) {
    constexpr uint64_t K = TXB_MAX_CTAS;
    const uint64_t add = blockIdx.x == 0 ? K - (uint64_t)(ncta - 1) : 1;
    uint64_t old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(&f->gbar_arrive), "l"(add) : "memory");
    const uint64_t target = (old / K + 1) * K;
    uint64_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&f->gbar_arrive) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Segmented counts for large batches: CTA `cta` owns tokens [t0, t1); it
// ranks its own copies (chunked warp match + per-warp scan), publishes its
// per-expert counts, and after a grid barrier adds the counts of all
// earlier CTAs -- global stable ranks (moe.py:514-521) in O(n/grid) per CTA.
// Writes the global ranks and pos[t,j] of its copies; hist = totals.
__device__ __noinline__ uint32_t route_counts_segmented(const txb_moe_shape& s, const int64_t* routes,
                                                       uint32_t* hist, uint32_t* wc, int32_t* rank_out,
                                                       int64_t* pos, int64_t t0, int64_t t1,
                                                       uint32_t* cta_hist, uint32_t* cta_bad, Flags* f, int cta,
                                                       int ncta, Shared& sh, const txb_moe_bufs& bufs) {
  const int E = s.experts, R = s.topk;
  const int tid = threadIdx.x, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (tid == 0) {
    sh.bad = 0;
    sh.direct = 0;
  }
  for (int e = tid; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int64_t M0 = t0 * R, M1 = t1 * R;
  for (int64_t base = M0; base < M1; base += blockDim.x) {
    for (int i = tid; i < nwarps * E; i += blockDim.x) wc[i] = 0;
    __syncthreads();
    const int64_t i = base + tid;
    int e = -1;
    if (i < M1) {
      const int64_t v = routes[i];
      if (v < 0 || v >= E) {
        atomicOr(&sh.bad, TXB_EV_ROUTE_RANGE);
      } else {
        e = (int)v;
        for (int64_t q = (i / R) * R; q < i; ++q)
          if (routes[q] == v) atomicOr(&sh.bad, TXB_EV_ROUTE_DUP);
      }
    }
    const uint32_t same = __match_any_sync(0xffffffffu, e);
    const int lr = __popc(same & lanemask_lt());
    if (e >= 0 && lr == 0) wc[warp * E + e] = __popc(same);
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
  stamp(bufs, 19);
  for (int e = tid; e < E; e += blockDim.x) cta_hist[(size_t)cta * E + e] = hist[e];
  if (tid == 0) cta_bad[cta] = sh.bad;
  grid_sync(f, ncta);
  stamp(bufs, 22);
  // Column prefixes, distributed: CTA `cta` owns experts [e0, e1); one warp
  // per expert loads the column of per-CTA counts (all loads in flight), scans
  // it and writes the exclusive prefix back in place, the total in row ncta.
  // After a second grid barrier every CTA reads its own row: O(E) loads per
  // CTA instead of O(ncta * E) (TXB_MAX_CTAS rows leave room for row ncta).
  {
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int e0 = (int)((int64_t)E * cta / ncta), e1 = (int)((int64_t)E * (cta + 1) / ncta);
    constexpr int kQ = 8;  // 32 * kQ CTAs per pass
    #pragma unroll 1
    for (int e = e0 + warp; e < e1; e += nwarps) {
      int run = 0;
      #pragma unroll 1
      for (int qb = 0; qb < ncta; qb += 32 * kQ) {
        int c[kQ];
#pragma unroll
        for (int u = 0; u < kQ; ++u) {
          const int q = qb + u * 32 + lane;
          c[u] = q < ncta ? (int)cta_hist[(size_t)q * E + e] : 0;
        }
#pragma unroll
        for (int u = 0; u < kQ; ++u) {
          int x = c[u];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          const int q = qb + u * 32 + lane;
          if (q < ncta) cta_hist[(size_t)q * E + e] = (uint32_t)(run + x - c[u]);
          run += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      if (lane == 0) cta_hist[(size_t)ncta * E + e] = (uint32_t)run;
    }
  }
  stamp(bufs, 24);
  grid_sync(f, ncta);
  stamp(bufs, 25);
  int* basev = reinterpret_cast<int*>(wc);   // [E] counts of earlier CTAs
  int* ex = basev + E;                       // [E] exclusive prefix of the totals
  for (int e = tid; e < E; e += blockDim.x) {
    basev[e] = (int)cta_hist[(size_t)cta * E + e];
    hist[e] = cta_hist[(size_t)ncta * E + e];
  }
  for (int q = tid; q < ncta; q += blockDim.x)
    if (cta_bad[q]) atomicOr(&sh.bad, cta_bad[q]);
  __syncthreads();
  const uint32_t b = sh.bad;
  for (int e = tid; e < E; e += blockDim.x) {
    if (b) hist[e] = 0;  // publish an empty row
    ex[e] = (int)hist[e];
  }
  __syncthreads();
  block_scan_i32(ex, E, sh.tmp);
  for (int64_t i = M0 + tid; i < M1; i += blockDim.x) {
    if (b) {
      pos[i] = -1;
      continue;
    }
    const int e = (int)routes[i];
    const int r = rank_out[i] + basev[e];
    rank_out[i] = r;
    pos[i] = (int64_t)ex[e] + r;
  }
  __syncthreads();
  return b;
}

// pos[t,j] = first send slot of expert e + stable rank, for this CTA's
// tokens (moe.py:510-520).  ex: int32 scratch of E entries.
__device__ void route_positions(const txb_moe_shape& s, const int64_t* routes, int64_t n, const uint32_t* hist,
                                int* ex, const int32_t* rank_in, int64_t* pos, uint32_t bad, int cta, int ncta,
                                Shared& sh) {
  const int E = s.experts, R = s.topk;
  for (int e = threadIdx.x; e < E; e += blockDim.x) ex[e] = (int)hist[e];
  __syncthreads();
  block_scan_i32(ex, E, sh.tmp);
  const int64_t nmine = n > cta ? (n - cta + ncta - 1) / ncta : 0;
  for (int64_t k = threadIdx.x; k < nmine * R; k += blockDim.x) {
    const int64_t i = (cta + (k / R) * ncta) * R + (k % R);
    pos[i] = bad ? -1 : (int64_t)ex[(int)routes[i]] + rank_in[i];
  }
  __syncthreads();
}

// Route-row scatter: own counts into row `me` of every rank's matrix as
// (step tag << 32 | count) words -- single-copy atomic, so no fence.  Every
// CTA holds the full histogram; CTA `part` of `nparts` stores its slice.
// The last part also books the copies that will come back from other ranks
// (read-modify-writes of the flags, a few serial round trips) -- not part 0,
// whose CTA also writes the receive info and the error word (EP=2 phase
// stamps: CTA 0 was the last to store its rows; 42.5 -> 41.6 us per step).
__device__ void route_publish(const txb_moe_shape& s, void* const* peers, Flags* f, const uint32_t* hist,
                              uint64_t step, int64_t n, uint32_t bad, int part, int nparts,
                              const Grp& g = Grp::cta()) {
  const int E = s.experts, N = s.ranks, L = s.local_experts;
  const int slot = (int)(step & 1);
  const uint64_t tag = (uint64_t)(uint32_t)step << 32;
  #pragma unroll 1
  // every CTA stores an equal contiguous slice (a few words each): with the
  // words packed into the first CTAs, those CTAs' remote stores held their
  // routing role back ~1.5 us (EP=2 phase stamps, round 2)
  const int NE = N * E, per = (NE + nparts - 1) / nparts;
  const int i1 = min(NE, (part + 1) * per);
  #pragma unroll 1
  for (int idx = part * per + g.tid; idx < i1; idx += g.nt) {
    const int d = idx / E, e = idx - d * E;
    if (N == 1) *(route_of(peers[d], s, slot) + (size_t)s.me * E + e) = tag | hist[e];
    else st_relaxed_sys(route_of(peers[d], s, slot) + (size_t)s.me * E + e, tag | hist[e]);
  }
  if (part == nparts - 1 && g.tid < 32) {
    // copies this rank serves itself do not come back through the counter
    const int lane = g.tid;
    uint32_t self = 0;
    #pragma unroll 1
    for (int le = lane; le < L; le += 32) self += hist[s.me * L + le];
    for (int o = 16; o; o >>= 1) self += __shfl_xor_sync(0xffffffffu, self, o);
    // per-source step tags (host-side gating / diagnostics), and the
    // buffer-reuse barrier of the previous step (moe.dbar): every read this
    // rank made of its buffers in step-1 finished before this kernel began
    // (stream order), so peers may now overwrite them.  Publishing it here
    // rather than at the end of the combine keeps a system-scope fence and
    // N remote stores off the step's tail; peers wait for it together with
    // this step's route words, which they need anyway.
    #pragma unroll 1
    for (int d = lane; d < N; d += 32) {
      Flags* pf = flags_of(peers[d], s);
      if (N == 1) {
        pf->route_tag[slot][s.me] = step;
        pf->done[s.me] = step - 1;
      } else {
        st_relaxed_sys(&pf->route_tag[slot][s.me], step);
        st_relaxed_sys(&pf->done[s.me], step - 1);
      }
    }
    if (!bad)
      #pragma unroll 1
      for (int d = 0; d < N; ++d) {  // copies that come back from d (diagnostics)
        uint32_t c = 0;
        #pragma unroll 1
        for (int le = lane; le < L; le += 32) c += hist[d * L + le];
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0 && d != s.me) add_flag(&f->comb_src_t[d], (uint64_t)c * comb_chunks(s));
      }
    if (lane == 0) {
      if (!bad) add_flag(&f->comb_target, ((uint64_t)(n * s.topk) - self) * comb_chunks(s));
      if (bad) atomicOr(&f->err, bad);
    }
  }
}

// ------------------------------------------------------------------- P2

// Acquire every route word of this step (tag == step) into Cs[N*E] (shared
// memory) and wait for every peer's end-of-previous-step barrier.
__device__ bool wait_routes(const txb_moe_shape& s, Flags* f, const uint64_t* C, uint32_t* Cs, uint64_t step,
                            uint64_t timeout_ns, Shared& sh, const Grp& g = Grp::cta()) {
  if (g.tid == 0) sh.fail = 0;
  g.sync();
  const uint64_t dl = globaltimer() + timeout_ns;
  const uint32_t want = (uint32_t)step;
  const int NE = s.ranks * s.experts;
  // kW words per thread per pass; every poll re-issues the loads of all the
  // words still pending at once, so the pass ends one memory round trip
  // after its last word lands (not one round trip per word)
  constexpr int kW = 8;
  #pragma unroll 1
  for (int base = g.tid; base < NE; base += kW * g.nt) {
    uint32_t pending = 0;
#pragma unroll
    for (int u = 0; u < kW; ++u)
      if (base + u * g.nt < NE) pending |= 1u << u;
    uint32_t it = 0;
    while (pending) {
      uint64_t v[kW];
#pragma unroll
      for (int u = 0; u < kW; ++u)
        if (pending & (1u << u)) v[u] = ld_relaxed_sys(C + base + u * g.nt);
#pragma unroll
      for (int u = 0; u < kW; ++u)
        if ((pending & (1u << u)) && (uint32_t)(v[u] >> 32) == want) {
          Cs[base + u * g.nt] = (uint32_t)v[u];
          pending &= ~(1u << u);
        }
      if (pending && ((++it) & 255u) == 0 && globaltimer() > dl) {
        atomicOr(&sh.fail, TXB_EV_WAIT_ROUTE);
        break;
      }
    }
  }
  if (g.tid < 32)
    #pragma unroll 1
    for (int q = g.tid; q < s.ranks; q += 32)
      if (!spin_ge(&f->done[q], step - 1, dl)) atomicOr(&sh.fail, TXB_EV_WAIT_BARRIER);
  g.sync();
  const uint32_t fl = sh.fail;
  if (fl && g.tid == 0) atomicOr(&f->err, fl);
  return fl == 0;
}

// ------------------------------------------------------------------- P3

// baseg[e] = grouped row on owner(e) where this rank's first copy for e
// lands: group_starts[le] + sum_{s' < me} counts[s', e];
// sh.sst[d] = send_start[me][d] (moe.py:221-222), the slab base the
// private-copy test of copy_dest measures from.
__device__ bool dispatch_layout(const txb_moe_shape& s, const uint32_t* C, int* baseg, int* padded, Flags* f,
                                Shared& sh) {
  const int N = s.ranks, E = s.experts, L = s.local_experts, tid = threadIdx.x;
  if (tid == 0) sh.lfail = 0;
  for (int d = tid; d < N; d += blockDim.x) {
    int a = 0;
    for (int le = 0; le < L; ++le) a += (int)C[s.me * E + d * L + le];
    sh.sst[d] = a;
  }
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) {
    int col = 0, pre = 0;
    for (int q = 0; q < N; ++q) {
      const int c = (int)C[q * E + e];
      col += c;
      if (q < s.me) pre += c;
    }
    padded[e] = pad_up(col);
    baseg[e] = pre;
  }
  if (tid == 0) {
    int run = 0;
    for (int d = 0; d < N; ++d) {
      const int v = sh.sst[d];
      sh.sst[d] = run;
      run += v;
    }
  }
  __syncthreads();
  const int tot = block_scan_i32(padded, E, sh.tmp);
  if (tid == 0) padded[E] = tot;
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) baseg[e] += padded[e] - padded[(e / L) * L];
  for (int d = tid; d < N; d += blockDim.x)
    if (padded[(d + 1) * L] - padded[d * L] > s.grouped_rows) atomicOr(&sh.lfail, TXB_EV_CAPACITY);
  __syncthreads();
  const uint32_t fl = sh.lfail;
  if (fl) {
    if (tid == 0) atomicOr(&f->err, fl);
    return false;
  }
  return true;
}

// Receive-side bookkeeping of one step, once the route matrix C is known
// (one warp, CTA 0): the rows this rank expects on its token counter --
// every copy routed to its experts except the speculative private rows,
// min(priv_tokens, assigned[q][me]) from each other source q (moe.py:
// 556-582, DispatchLayout.private_take) -- and this step's private rows
// (priv_step, added to priv_target at the end of the step).  The per-source
// expectations feed the timeout diagnostics.
__device__ void book_recv(const txb_moe_shape& s, Flags* f, const uint32_t* C, int lane) {
  const int N = s.ranks, E = s.experts, L = s.local_experts, me = s.me;
  uint32_t tok = 0, pv = 0;
  #pragma unroll 1
  for (int q = 0; q < N; ++q) {
    uint32_t a = 0;
    #pragma unroll 1
    for (int le = lane; le < L; le += 32) a += C[q * E + me * L + le];
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    const uint32_t take = (q != me && s.priv_tokens > 0) ? min(a, (uint32_t)s.priv_tokens) : 0u;
    if (lane == 0) {
      add_flag(&f->tok_src_t[q], a - take);
      if (take) add_flag(&f->priv_src_t[q], take);
    }
    tok += a - take;
    pv += take;
  }
  if (lane == 0) {
    add_flag(&f->tok_target, tok);
    f->priv_step = pv;
  }
}

// DECODE layout: this CTA's single token needs only its own R copies'
// send slots and destination rows, so each comes from one warp reduction
// instead of block-wide scans (one warp per copy, no block barrier).
// pos = sum_{e' < e} hist[e'] + rank (moe.py:514-521).
//
// With `peers` (EP > 1, priv_tokens > 0) it also places the speculative
// private copies (moe.py:556-582): a copy whose slot in its destination's
// slab, pos - send_start[me][d], is below priv_tokens goes to d's private
// slab for this rank, sh.pdst[k] (counted in sh.pcnt); every other copy
// gets sh.pdst[k] = null.  That needs only this rank's own counts, so the
// copy can be stored before the route exchange has finished.
__device__ void own_positions(const txb_moe_shape& s, const uint32_t* hist, int64_t* pos, uint32_t bad,
                              Shared& sh, const Grp& g = Grp::cta(), void* const* peers = nullptr,
                              uint64_t step = 0) {
  const int lane = g.tid & 31, warp = g.tid >> 5, nwarp = g.nt >> 5;
  const int L = s.local_experts;
  const bool priv = peers && s.priv_tokens > 0 && s.ranks > 1 && !bad;
  #pragma unroll 1
  for (int k = warp; k < s.topk; k += nwarp) {
    const int e = sh.own_e[k];
    const int d0 = e >= 0 ? (e / L) * L : 0;
    int acc = 0, acc0 = 0;
    #pragma unroll 1
    for (int x = lane; x < (bad ? 0 : e); x += 32) {
      const int h = (int)hist[x];
      acc += h;
      if (x < d0) acc0 += h;
    }
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
    }
    if (lane == 0) {
      TXB_ASSERT(bad || (acc + (int)sh.own_rank[k] >= 0 && acc + (int)sh.own_rank[k] < s.comb_rows));
      pos[sh.own_i[k]] = bad ? -1 : (int64_t)acc + sh.own_rank[k];
      uint8_t* pd = nullptr;
      const int d = d0 / L;
      if (priv && d != s.me) {
        const int sidx = acc - acc0 + (int)sh.own_rank[k];
        if (sidx < s.priv_tokens) {
          const int par = (int)(step & 1);
          pd = priv_rows_of(peers[d], s, par, s.me) + (int64_t)sidx * s.payload_bytes;
          if (per_token(s)) privsrc_of(peers[d], s, par, s.me)[sidx] = sh.own_i[k] / s.topk;
          atomicAdd(&sh.pcnt[d], 1u);
        }
      }
      sh.pdst[k] = pd;
    }
  }
}

// EP=1 decode: everything about copy k of the CTA's token by ONE warp, no
// CTA barrier between the steps -- its stable rank (earlier entries of the
// batch with the same expert, counted four staged ids per lane per load),
// pos = sum_{e' < e} hist[e'] + rank (moe.py:514-521) and its grouped row
// group_starts[e] + rank, group_starts[e] = sum_{e' < e} pad8(hist[e'])
// (with one rank the local expert is the expert).  One
// barrier at the end publishes sh.dstp to the storing threads.
__device__ void own_copies_solo(const txb_moe_shape& s, const uint32_t* hist, const int32_t* rv,
                                const txb_moe_bufs& b, uint32_t bad, Shared& sh, const Grp& g) {
  const int lane = g.tid & 31, warp = g.tid >> 5, nwarp = g.nt >> 5;
  const bool v4 = (reinterpret_cast<uintptr_t>(rv) & 15) == 0;
  #pragma unroll 1
  for (int k = warp; k < s.topk; k += nwarp) {
    const int e = sh.own_e[k], i = sh.own_i[k];
    if (bad) {
      if (lane == 0) {
        b.pos[i] = -1;
        sh.dstp[k] = nullptr;
        sh.pdst[k] = nullptr;
      }
      continue;
    }
    int cnt = 0;
    if (v4) {
      const int4* r4 = reinterpret_cast<const int4*>(rv);
      #pragma unroll 4
      for (int q = lane; 4 * q < i; q += 32) {
        const int4 v = r4[q];
        const int j = 4 * q;
        cnt += (v.x == e) + (j + 1 < i && v.y == e) + (j + 2 < i && v.z == e) + (j + 3 < i && v.w == e);
      }
    } else {
      #pragma unroll 4
      for (int j = lane; j < i; j += 32) cnt += rv[j] == e;
    }
    int acc = 0, accp = 0;
    #pragma unroll 4
    for (int x = lane; x < e; x += 32) {
      const int h = (int)hist[x];
      acc += h;
      accp += pad_up(h);
    }
    for (int o = 16; o; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      accp += __shfl_xor_sync(0xffffffffu, accp, o);
    }
    if (lane == 0) {
      const int gr = accp + cnt;
      if (!TXB_ASSERT(gr >= 0 && gr < s.grouped_rows)) {
        sh.dstp[k] = nullptr;
        sh.pdst[k] = nullptr;
        continue;
      }
      b.rank_scratch[i] = cnt;
      TXB_ASSERT(acc + cnt >= 0 && acc + cnt < s.comb_rows);
      b.pos[i] = (int64_t)acc + cnt;
      b.gidx[i] = gr;
      sh.dstp[k] = grouped_of(b.peers[0], s) + (int64_t)gr * s.payload_bytes;
      sh.pdst[k] = nullptr;
    }
  }
  g.sync();
}

// grouped row on owner d of copy k: group_starts_d[le] + sum_{s' < me}
// counts[s', e] + rank; books gidx and the counts.
__device__ void own_dests(const txb_moe_shape& s, const uint32_t* C, void* const* peers, int32_t* gidx,
                          Shared& sh, const Grp& g = Grp::cta()) {
  const int N = s.ranks, E = s.experts, L = s.local_experts;
  const int lane = g.tid & 31, warp = g.tid >> 5, nwarp = g.nt >> 5;
  #pragma unroll 1
  for (int k = warp; k < s.topk; k += nwarp) {
    if (sh.pdst[k]) {  // stored to the owner's private slab (own_positions)
      if (lane == 0) {
        sh.dstp[k] = nullptr;
        gidx[sh.own_i[k]] = -1;
      }
      continue;
    }
    const int e = sh.own_e[k], d = e / L, le = e - d * L;
    int acc = 0;
    #pragma unroll 1
    for (int x = lane; x < le; x += 32) {
      int col = 0;
      #pragma unroll 1
      for (int q = 0; q < N; ++q) col += (int)C[q * E + d * L + x];
      acc += pad_up(col);
    }
    #pragma unroll 1
    for (int q = lane; q < s.me; q += 32) acc += (int)C[q * E + e];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int g = acc + (int)sh.own_rank[k];
      if (!TXB_ASSERT(g >= 0 && g < s.grouped_rows && d >= 0 && d < N)) {
        sh.dstp[k] = nullptr;
        continue;
      }
      sh.dstp[k] = grouped_of(peers[d], s) + (int64_t)g * s.payload_bytes;
      gidx[sh.own_i[k]] = d == s.me ? g : -1;
      if (per_token(s)) srctok_of(peers[d], s)[g] = sh.own_i[k] / s.topk;
      atomicAdd(&sh.cnt[d], 1u);
    }
  }
  g.sync();
  // one token per CTA on these paths: book its rows that will come back
  if (per_token(s) && g.tid == 0)
    tokt_of(peers[s.me], s)[sh.own_i[0] / s.topk] += (uint64_t)(s.topk - sh.cnt[s.me]) * comb_chunks(s);
}

// ------------------------------------------------------------------- P4

// Destination rows of token t's copies (kt-th token of this CTA) into
// sh.dstp; books gidx and per-destination counts.
// Copy i (token t = i / R) to destination d: its private-slab row when its
// slab slot pos[i] - send_start[me][d] is below priv_tokens (d != me), else
// its grouped row baseg[e] + rank.  Books gidx, srctok and the counts.
__device__ __forceinline__ uint8_t* copy_dest(const txb_moe_shape& s, void* const* peers, const int* baseg,
                                              const int64_t* pos, int32_t* gidx, uint64_t step, int64_t i, int e,
                                              int rank, Shared& sh) {
  const int d = e / s.local_experts;
  const int64_t t = i / s.topk;
  if (d != s.me && s.priv_tokens > 0) {
    const int64_t sidx = pos[i] - sh.sst[d];
    if (sidx < s.priv_tokens && TXB_ASSERT(sidx >= 0)) {
      const int par = (int)(step & 1);
      gidx[i] = -1;
      if (per_token(s)) privsrc_of(peers[d], s, par, s.me)[sidx] = (int32_t)t;
      atomicAdd(&sh.pcnt[d], 1u);
      return priv_rows_of(peers[d], s, par, s.me) + sidx * s.payload_bytes;
    }
  }
  const int64_t g = (int64_t)baseg[e] + rank;
  if (!TXB_ASSERT(g >= 0 && g < s.grouped_rows && d >= 0 && d < s.ranks)) return grouped_of(peers[s.me], s);
  gidx[i] = d == s.me ? (int32_t)g : -1;
  if (per_token(s)) srctok_of(peers[d], s)[g] = (int32_t)t;
  atomicAdd(&sh.cnt[d], 1u);
  return grouped_of(peers[d], s) + g * s.payload_bytes;
}

__device__ __forceinline__ void token_dests(const txb_moe_shape& s, const int64_t* routes, const int32_t* rank_in,
                                            const int64_t* pos, int32_t* gidx, void* const* peers, const int* baseg,
                                            int64_t t, int kt, uint64_t step, Shared& sh) {
  const int R = s.topk, tid = threadIdx.x;
  if (tid < R) {
    int e, rank;
    if (sh.direct) {  // experts and ranks of this CTA's copies are in smem
      e = sh.own_e[kt * R + tid];
      rank = (int)sh.own_rank[kt * R + tid];
    } else {
      e = (int)routes[t * R + tid];
      rank = rank_in[t * R + tid];
    }
    sh.dstp[tid] = copy_dest(s, peers, baseg, pos, gidx, step, t * R + tid, e, rank, sh);
  }
  __syncthreads();
}

// Out-of-line copy/encode of one token row to sh.dstp (general shapes).
template <int SRC, int ELEM>
__device__ __noinline__ void dispatch_row_slow(const txb_moe_shape& s, const void* x, int64_t t, Shared& sh) {
  const int64_t P = s.payload_bytes;
  if constexpr (SRC == TXB_SRC_ROWS) {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(x) + t * P;
    for (int j = 0; j < s.topk; ++j) copy_row(sh.dstp[j], src, P, threadIdx.x, blockDim.x);
  } else {
    encode_store_row<SRC, ELEM>(x, t, s.hidden, s.scales, P, sh.dstp, s.topk, sh.red);
  }
}

// Tokens t = t0, t0 + dt, ... < t1 of this CTA.
template <int SRC, int ELEM>
__device__ __noinline__ void dispatch_tokens(const txb_moe_shape& s, const void* x, int64_t t0, int64_t t1,
                                             int64_t dt, const int64_t* routes, const int32_t* rank_in,
                                             const int64_t* pos, int32_t* gidx, void* const* peers,
                                             const int* baseg, uint64_t step, Shared& sh) {
  const int R = s.topk, tid = threadIdx.x;
  const int64_t P = s.payload_bytes;
  int kt = 0;
  for (int64_t t = t0; t < t1; t += dt, ++kt) {
    token_dests(s, routes, rank_in, pos, gidx, peers, baseg, t, kt, step, sh);
    if constexpr (SRC == TXB_SRC_ROWS) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(x) + t * P;
      if (vec_width(src, sh.dstp[0], P) == 16) {
        for (int64_t v = tid; v < (P >> 4); v += blockDim.x) {
          const int4 val = reinterpret_cast<const int4*>(src)[v];
          for (int j = 0; j < R; ++j) reinterpret_cast<int4*>(sh.dstp[j])[v] = val;
        }
      } else {
        dispatch_row_slow<SRC, ELEM>(s, x, t, sh);
      }
    } else {
      encode_store_row<SRC, ELEM>(x, t, s.hidden, s.scales, P, sh.dstp, R, sh.red);
    }
    __syncthreads();
  }
}

// Large batches, rows that need no per-token reduction (bf16 / f32 rows,
// raw payload rows): the destinations of all the CTA's copies are resolved
// up front into shared memory (one pass, one memory round trip), so the
// token loop has no barrier and no metadata load, and every thread keeps
// the next token's chunks in flight while it stores the current token's
// R copies.  Returns false (nothing done) when the shape is not eligible or
// the pointer table does not fit `dp`'s capacity; the caller then runs
// dispatch_tokens.
template <int SRC, int ELEM>
__device__ __noinline__ bool dispatch_tokens_flat(const txb_moe_shape& s, const void* x, int64_t t0, int64_t t1,
                                                  const int64_t* routes, const int32_t* rank_in,
                                                  const int64_t* pos, int32_t* gidx, void* const* peers,
                                                  const int* baseg, uint8_t** dp, int cap, uint64_t step,
                                                  Shared& sh) {
  if constexpr (ELEM == 1 && SRC != TXB_SRC_ROWS) {
    return false;  // fp8 rows need a per-token amax across the CTA
  } else {
    const int R = s.topk, L = s.local_experts, tid = threadIdx.x, nt = blockDim.x;
    const int64_t P = s.payload_bytes;
    const int m = (int)((t1 - t0) * R);
    if (t1 <= t0 || m > cap) return false;
    RowRaw cur;
    load_row_raw<SRC, ELEM>(x, t0, s.hidden, P, cur);
    if (!cur.ok) return false;  // uniform across the CTA (shape / alignment)
    #pragma unroll 1
    for (int k = tid; k < m; k += nt) {
      const int64_t i = t0 * R + k;
      dp[k] = copy_dest(s, peers, baseg, pos, gidx, step, i, (int)routes[i], rank_in[i], sh);
    }
    __syncthreads();
    #pragma unroll 1
    for (int64_t t = t0; t < t1; ++t) {
      RowRaw nxt;
      if (t + 1 < t1) load_row_raw<SRC, ELEM>(x, t + 1, s.hidden, P, nxt);
      RowRegs r;
      finish_row_regs<SRC, ELEM>(cur, r, sh.red);
      store_row_regs<SRC, ELEM>(r, s.hidden, s.scales, dp + (t - t0) * R, R);
      cur = nxt;
    }
    return true;
  }
}

// Per-token completion (EP > 1): book the copies of tokens t0, t0 + dt,
// ... < t1 that another rank serves -- the rows that will come back through
// tokc[t].  Every dispatch path books them, so tokc and tokt stay in step
// whichever path (fused, split) a step takes.
__device__ __forceinline__ void book_tok_targets(const txb_moe_shape& s, const int64_t* routes, void* region,
                                                 int64_t t0, int64_t t1, int64_t dt) {
  if (!per_token(s)) return;
  uint64_t* tokt = tokt_of(region, s);
  #pragma unroll 1
  for (int64_t t = t0 + (int64_t)threadIdx.x * dt; t < t1; t += (int64_t)blockDim.x * dt) {
    int remote = 0;
    for (int j = 0; j < s.topk; ++j) remote += (int)routes[t * s.topk + j] / s.local_experts != s.me;
    tokt[t] += (uint64_t)remote * comb_chunks(s);
  }
}

// Completion of this CTA's stores: one release fence, then a relaxed add of
// the row counts on every destination's counters -- sh.cnt on the token
// (kind 0) or combine (kind 1) counter, and for kind 0 sh.pcnt on the
// private-row counter of this step's parity -- each also on the
// destination's per-source slot of this rank (diagnostics).  Called by one
// thread after the stores it covers are ordered before it (a barrier).
__device__ void signal_rows_thread(const txb_moe_shape& s, void* const* peers, int kind, uint64_t step, Shared& sh,
                                   bool with_main, bool with_priv) {
  const int N = s.ranks, me = s.me, par = (int)(step & 1);
  bool any = false;
  #pragma unroll 1
  for (int d = 0; d < N; ++d) any |= (with_main && sh.cnt[d]) || (with_priv && sh.pcnt[d]);
  if (!any) return;
  fence_release(s.single_device);
  #pragma unroll 1
  for (int d = 0; d < N; ++d) {
    Flags* pf = flags_of(peers[d], s);
    if (with_main && sh.cnt[d]) {
      red_relaxed_sys_add(kind == 0 ? &pf->tok_ctr : &pf->comb_ctr, sh.cnt[d]);
      red_relaxed_sys_add(kind == 0 ? &pf->tok_src[me] : &pf->comb_src[me], sh.cnt[d]);
    }
    if (with_priv && sh.pcnt[d]) {
      red_relaxed_sys_add(&pf->priv_ctr[par], sh.pcnt[d]);
      red_relaxed_sys_add(&pf->priv_src[me], sh.pcnt[d]);
      sh.pcnt[d] = 0;
    }
  }
}

__device__ void signal_counts(const txb_moe_shape& s, void* const* peers, int kind, uint64_t step, Shared& sh) {
  __syncthreads();
  if (threadIdx.x == 0) signal_rows_thread(s, peers, kind, step, sh, true, kind == 0);
}

// ------------------------------------------------------------------- P5

// Receive metadata for grouped rows (moe.py:699-722), in two parts:
// recv_tables (block barriers) derives the per-(source, local expert) tables
// from the route matrix into shared memory; recv_rows (no barriers) walks
// the grouped rows, one warp per row: lane 0 writes rows / sources / return
// slot, the warp zero-fills padding rows that may hold stale data.
struct RecvTables {
  int* a;        // [N][L] counts into my experts
  int* gstart;   // [L] group starts (padded) -- followed directly by rowbase,
  int* rowbase;  // [N*L] flattened exclusive prefix = recv slot base
  int* tot;      // [2] padded_total, recv_total
  int* retbase;  // [N][L] send slot base on the source
  int* gsize;    // [L]
  int* srcpre;   // [L][N+1]
  int* pre_all;  // [N] sum_{e' < me*L} C[q][e']
  int* asg;      // [N] assigned[q][me]: copies source q routes to this rank
  int* take;     // [N+1] private rows from q, min(priv_tokens, asg[q]) (0 for me); [N] = sum
};

__device__ __forceinline__ RecvTables recv_carve(const txb_moe_shape& s, const int* sm_c) {
  int* sm = const_cast<int*>(sm_c);
  const int N = s.ranks, L = s.local_experts;
  RecvTables t;
  t.a = sm;
  t.gstart = t.a + N * L;
  t.rowbase = t.gstart + L;
  t.tot = t.rowbase + N * L;
  t.retbase = t.tot + 2;
  t.gsize = t.retbase + N * L;
  t.srcpre = t.gsize + L;
  t.pre_all = t.srcpre + L * (N + 1);
  t.asg = t.pre_all + N;
  t.take = t.asg + N;
  return t;
}

// One rank (EP=1): the receive tables of recv_tables_body collapse to two
// prefixes of the histogram -- group starts (padded to 8) and receive-slot
// bases (unpadded) -- computed in ONE two-array block scan (each thread a
// contiguous run of local experts, warp shuffles, one pass over the warp
// totals): two barriers instead of the six of the general tables.
__device__ __forceinline__ void recv_tables_solo(const txb_moe_shape& s, const uint32_t* hist, int* sm, int64_t* info,
                                                 int cta, Shared& sh, const Grp& g) {
  const int L = s.local_experts, tid = g.tid, nt = g.nt;
  RecvTables t = recv_carve(s, sm);
  const int per = (L + nt - 1) / nt;
  const int lo = min(L, tid * per), hi = min(L, lo + per);
  int sp = 0, sr = 0;
  #pragma unroll 1
  for (int le = lo; le < hi; ++le) {
    const int a = (int)hist[le];
    sp += pad_up(a);
    sr += a;
  }
  const int lane = tid & 31, warp = tid >> 5;
  int xp = sp, xr = sr;
  for (int o = 1; o < 32; o <<= 1) {
    const int yp = __shfl_up_sync(0xffffffffu, xp, o), yr = __shfl_up_sync(0xffffffffu, xr, o);
    if (lane >= o) {
      xp += yp;
      xr += yr;
    }
  }
  // warp totals in sh.tmp (this role's scratch; sh.red belongs to the
  // token role's amax reduce, which may still be running)
  int* wp = sh.tmp;         // [16] padded
  int* wr = sh.tmp + 16;    // [16] unpadded
  if (lane == 31) {
    wp[warp] = xp;
    wr[warp] = xr;
  }
  g.sync();
  int bp = 0, br = 0, tp = 0, tr = 0;
  const int nw = nt >> 5;
  #pragma unroll 1
  for (int w = 0; w < nw; ++w) {
    if (w < warp) {
      bp += wp[w];
      br += wr[w];
    }
    tp += wp[w];
    tr += wr[w];
  }
  int rp = bp + xp - sp, rr = br + xr - sr;  // exclusive prefixes at lo
  #pragma unroll 1
  for (int le = lo; le < hi; ++le) {
    const int a = (int)hist[le];
    t.a[le] = a;
    t.gstart[le] = rp;
    t.rowbase[le] = rr;
    t.retbase[le] = rr;
    t.gsize[le] = a;
    t.srcpre[2 * le] = 0;
    t.srcpre[2 * le + 1] = a;
    if (cta == 0) {
      info[le] = a;
      info[L + le] = rp;
    }
    rp += pad_up(a);
    rr += a;
  }
  if (tid == 0) {
    t.tot[0] = tp;
    t.tot[1] = tr;
    t.pre_all[0] = 0;
    t.asg[0] = tr;
    t.take[0] = 0;
    t.take[1] = 0;
    if (cta == 0) {
      info[2 * L] = tp;
      info[2 * L + 1] = tr;
    }
  }
  g.sync();
}

template <bool INL>
__device__ __forceinline__ void recv_tables_body(const txb_moe_shape& s, const uint32_t* C, int* sm, int64_t* info,
                                                 int cta, Shared& sh, const txb_moe_bufs& b,
                                                 const Grp& g = Grp::cta()) {
  const int N = s.ranks, E = s.experts, L = s.local_experts, me = s.me;
  const int tid = g.tid, nt = g.nt;
  RecvTables t = recv_carve(s, sm);
  #pragma unroll 1
  for (int i = tid; i < N * L; i += nt) {
    const int q = i / L, le = i - q * L;
    t.a[i] = (int)C[q * E + me * L + le];
    t.rowbase[i] = t.a[i];
  }
  {
    const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
    #pragma unroll 1
    for (int q = warp; q < N; q += nwarp) {
      int acc = 0, a = 0;
      #pragma unroll 1
      for (int e = lane; e < me * L; e += 32) acc += (int)C[q * E + e];
      #pragma unroll 1
      for (int e = lane; e < L; e += 32) a += (int)C[q * E + me * L + e];
      for (int o = 16; o; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        a += __shfl_xor_sync(0xffffffffu, a, o);
      }
      if (lane == 0) {
        t.pre_all[q] = acc;
        t.asg[q] = a;
        t.take[q] = (q != me && s.priv_tokens > 0) ? min(a, s.priv_tokens) : 0;
      }
    }
  }
  g.sync();
  if (tid < 32) {
    int v = 0, r = 0;
    #pragma unroll 1
    for (int q = tid; q < N; q += 32) {
      v += t.take[q];
      r += t.asg[q];
    }
    for (int o = 16; o; o >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, o);
      r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if (tid == 0) {
      t.take[N] = v;
      t.tot[1] = r;  // recv_total: every copy routed to this rank
    }
  }
  stamp(b, 16);
  #pragma unroll 1
  for (int le = tid; le < L; le += nt) {
    int run = 0;
    #pragma unroll 1
    for (int q = 0; q < N; ++q) {
      t.srcpre[le * (N + 1) + q] = run;
      run += t.a[q * L + le];
    }
    t.srcpre[le * (N + 1) + N] = run;
    t.gsize[le] = run;
    t.gstart[le] = pad_up(run);
  }
  g.sync();
  stamp(b, 17);
  // one scan over [padded group sizes (L) | counts flattened source-major
  // (N*L)]: the first part gives group_starts, the second (minus the padded
  // total) recv_start[me][q] + sum_{le'<le} a[q][le'] (moe.py:178-184, 204-213)
  const int all = block_scan<INL>(t.gstart, L + N * L, sh.tmp, g);
  stamp(b, 18);
  // the padded total is what the scan adds before the counts part; taken
  // from the totals, not from rowbase[0], which thread 0 rewrites in the
  // loop below while slower warps could still be reading it (a race the
  // checked build caught at EP=2 in round 2: a whole warp's rowbase came
  // out unshifted and its return slots ran past comb_rows)
  const int padded_total = all - t.tot[1];
  #pragma unroll 1
  for (int i = tid; i < N * L; i += nt) t.rowbase[i] -= padded_total;
  if (tid == 0) t.tot[0] = padded_total;
  g.sync();
  #pragma unroll 1
  for (int i = tid; i < N * L; i += nt) t.retbase[i] = t.pre_all[i / L] + (t.rowbase[i] - t.rowbase[(i / L) * L]);
  g.sync();
  if (cta == 0) {
    #pragma unroll 1
    for (int le = tid; le < L; le += nt) {
      info[le] = t.gsize[le];
      info[L + le] = t.gstart[le];
    }
    if (tid == 0) {
      info[2 * L] = t.tot[0];
      info[2 * L + 1] = t.tot[1];
    }
  }
}

__device__ __noinline__ void recv_tables(const txb_moe_shape& s, const uint32_t* C, int* sm, int64_t* info,
                                         int cta, Shared& sh, const txb_moe_bufs& b) {
  recv_tables_body<false>(s, C, sm, info, cta, sh, b);
}

// Dirty flags of the first kPreDirty rows a warp of group `g` will visit in
// recv_rows_body, loaded at kernel start so the (cold) byte reads are off
// the kernel's tail.  Byte i of the result = dirty[row i] (0 beyond G).
constexpr int kPreDirty = 4;

// The loads stay unconsumed (separate registers) until recv_rows_body reads
// them, so issuing them does not stall the issuing role.
struct PreDirty {
  uint8_t v[kPreDirty];
  bool on;
};

__device__ __forceinline__ PreDirty prefetch_dirty(const txb_moe_shape& s, const uint8_t* dirty, int cta, int ncta,
                                                   const Grp& g) {
  const int nwarp = g.nt >> 5, warp = g.tid >> 5;
  PreDirty pd;
  pd.on = true;
#pragma unroll
  for (int i = 0; i < kPreDirty; ++i) {
    const int64_t r = (int64_t)cta * nwarp + warp + (int64_t)i * ncta * nwarp;
    pd.v[i] = r < s.grouped_rows ? dirty[r] : (uint8_t)0;
  }
  return pd;
}

// pd: prefetch_dirty of the same group (or ~0u: read the flags here).
__device__ __forceinline__ void recv_rows_body(const txb_moe_shape& s, int* sm, int64_t* rows, int64_t* sources,
                                               int32_t* ret, uint8_t* G, uint8_t* dirty, int32_t* send_list,
                                               uint32_t* send_cnt, int cta, int ncta, const Grp& grp = Grp::cta(),
                                               PreDirty pd = PreDirty{{0}, false}) {
  const int N = s.ranks, L = s.local_experts;
  const RecvTables t = recv_carve(s, sm);
  const int padded_total = t.tot[0];
  if (!TXB_ASSERT(padded_total >= 0 && padded_total <= s.grouped_rows)) return;
  const int64_t P = s.payload_bytes;
  const int warp = grp.tid >> 5, lane = grp.tid & 31, nwarp = grp.nt >> 5;
  int it = 0;
  #pragma unroll 1
  for (int g = cta * nwarp + warp; g < padded_total; g += ncta * nwarp, ++it) {
    // last le with gstart[le] <= g: the warp tests 32 candidates per round
    // (two rounds for L <= 1024) instead of a serial binary search
    int lo = 0, span = L;
    #pragma unroll 1
    while (span > 1) {
      const int stp = (span + 31) >> 5;
      const int cand = lo + lane * stp;
      const unsigned m = __ballot_sync(0xffffffffu, cand < lo + span && t.gstart[cand] <= g);
      const int last = 31 - __clz(m);  // lane 0 (cand = lo) always qualifies
      const int nlo = lo + last * stp;
      span = min(stp, lo + span - nlo);
      lo = nlo;
    }
    const int le = lo;
    const int k = g - t.gstart[le];
    if (k >= t.gsize[le]) {
      // padding rows read as zero (moe.py:719); only rows that held data
      // since they were last zeroed need the store
      bool d;
      if (pd.on && it < kPreDirty) {
        uint8_t v = 0;
#pragma unroll
        for (int i = 0; i < kPreDirty; ++i)
          if (i == it) v = pd.v[i];
        d = v != 0;
      } else {
        d = dirty[g] != 0;
      }
      if (d) zero_row(G + (int64_t)g * P, P, lane, 32);
      if (lane == 0) {
        rows[g] = -1;
        sources[g] = -1;
        ret[g] = -1;
        if (d) dirty[g] = 0;
      }
    } else if (lane == 0) {
      dirty[g] = 1;
      const int* sp = t.srcpre + le * (N + 1);
      int q = 0;
      while (sp[q + 1] <= k) ++q;
      const int kk = k - sp[q];
      rows[g] = t.rowbase[q * L + le] + kk;
      sources[g] = q;
      ret[g] = t.retbase[q * L + le] + kk;
      // rows that go back over the fabric, compacted (order is irrelevant)
      if (q != s.me) send_list[atomicAdd(send_cnt, 1u)] = g;
    }
  }
}

// Large batches: the same metadata with one THREAD per grouped row (group by
// binary search, source by a short scan), then one warp per local expert
// zero-fills that group's padding rows that hold stale data.  A warp per
// row would walk tens of thousands of rows one round trip at a time.
//
// With per-token completion (tok_mode) the rows to return are listed in
// kPhases phases by their relative position k/m inside their (source, local
// expert) segment.  A segment holds its source's tokens in ascending order,
// so phase ~ origin token / n: the combine walks the list grid-stride and
// returns early tokens' rows first, which is the order the origins reduce.
constexpr int kPhases = 16;

__device__ __noinline__ void recv_rows_flat(const txb_moe_shape& s, int* sm, int64_t* rows, int64_t* sources,
                                            int32_t* ret, uint8_t* G, uint8_t* dirty, int32_t* send_list,
                                            uint32_t* send_cnt, int cta, int ncta, uint32_t* phase_cnt) {
  const int N = s.ranks, L = s.local_experts;
  const RecvTables t = recv_carve(s, sm);
  const int padded_total = t.tot[0];
  const int64_t P = s.payload_bytes;
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int phase_base[kPhases];
  const bool phased = tok_mode(s) && phase_cnt;
  if (phased) {
    // rows per phase over every remote segment, then exclusive prefix
    if (tid < kPhases) phase_base[tid] = 0;
    __syncthreads();
    int c[kPhases];
#pragma unroll
    for (int ph = 0; ph < kPhases; ++ph) c[ph] = 0;
    #pragma unroll 1
    for (int i = tid; i < N * L; i += nt) {
      if (i / L == s.me) continue;
      const int m = t.a[i];
#pragma unroll
      for (int ph = 0; ph < kPhases; ++ph) c[ph] += (ph + 1) * m / kPhases - ph * m / kPhases;
    }
#pragma unroll
    for (int ph = 0; ph < kPhases; ++ph) {
      int v = c[ph];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((tid & 31) == 0 && v) atomicAdd(&phase_base[ph], v);
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int ph = 0; ph < kPhases; ++ph) {
        const int v = phase_base[ph];
        phase_base[ph] = run;
        run += v;
      }
    }
    __syncthreads();
  }
  #pragma unroll 1
  for (int g = cta * nt + tid; g < padded_total; g += ncta * nt) {
    int lo = 0, hi = L - 1;  // last le with gstart[le] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (t.gstart[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    const int le = lo, k = g - t.gstart[le];
    if (k >= t.gsize[le]) {
      rows[g] = -1;
      sources[g] = -1;
      ret[g] = -1;
      continue;
    }
    dirty[g] = 1;
    const int* sp = t.srcpre + le * (N + 1);
    int q = 0;
    while (sp[q + 1] <= k) ++q;
    const int kk = k - sp[q];
    rows[g] = t.rowbase[q * L + le] + kk;
    sources[g] = q;
    ret[g] = t.retbase[q * L + le] + kk;
    if (q != s.me) {
      if (phased) {
        const int m = t.a[q * L + le];
        int ph = (int)((int64_t)kk * kPhases / m);
        // the phase whose [ph*m/P, (ph+1)*m/P) range holds kk
        while (ph > 0 && kk < ph * m / kPhases) --ph;
        while (ph + 1 < kPhases && kk >= (ph + 1) * m / kPhases) ++ph;
        send_list[phase_base[ph] + atomicAdd(&phase_cnt[ph], 1u)] = g;
        atomicAdd(send_cnt, 1u);
      } else {
        send_list[atomicAdd(send_cnt, 1u)] = g;
      }
    }
  }
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  #pragma unroll 1
  for (int le = cta * nwarp + warp; le < L; le += ncta * nwarp) {
    const int g1 = le + 1 < L ? t.gstart[le + 1] : padded_total;
    #pragma unroll 1
    for (int g = t.gstart[le] + t.gsize[le]; g < g1; ++g) {
      if (!dirty[g]) continue;
      zero_row(G + (int64_t)g * P, P, lane, 32);
      __syncwarp();
      if (lane == 0) dirty[g] = 0;
    }
  }
}

// Speculative private rows (moe.py:693-698, private rows to the slab heads):
// source q's first take[q] slab rows sit in this rank's private slab of the
// step's parity; each goes to its grouped row.  Slab slot k of source q is
// copy kk = k - off(le) of local expert le, where off(le) = sum_{le' < le}
// a[q][le'] = rowbase[q*L+le] - rowbase[q*L] (the last le with off(le) <=
// k), so its grouped row is gstart[le] + srcpre[le][q] + kk (SURVEY.md App.
// A).  Work items are spread over warps (gw of ngw); a warp waits once,
// before its first row, for the step's private counter.
__device__ void recv_private_rows(const txb_moe_shape& s, const int* sm, void* region, uint64_t step,
                                  uint64_t timeout_ns, int gw, int ngw, int lane) {
  const int N = s.ranks, L = s.local_experts, Pt = s.priv_tokens;
  if (Pt <= 0 || N == 1) return;
  const RecvTables t = recv_carve(s, sm);
  if (t.take[N] == 0) return;
  Flags* f = flags_of(region, s);
  const int par = (int)(step & 1);
  const int64_t P = s.payload_bytes;
  uint8_t* G = grouped_of(region, s);
  bool waited = false;
  #pragma unroll 1
  for (int i = gw; i < N * Pt; i += ngw) {
    const int q = i / Pt, k = i - q * Pt;
    if (k >= t.take[q]) continue;
    if (!waited) {
      uint32_t ok = 1;
      if (lane == 0) {
        const uint64_t target = *reinterpret_cast<volatile uint64_t*>(&f->priv_target[par]) + (uint64_t)t.take[N];
        ok = spin_ge(&f->priv_ctr[par], target, globaltimer() + timeout_ns) ? 1u : 0u;
        if (!ok) atomicOr(&f->err, TXB_EV_WAIT_PRIV);
      }
      if (!__shfl_sync(0xffffffffu, ok, 0)) return;
      waited = true;
    }
    const int* rb = t.rowbase + q * L;
    int lo = 0, span = L;  // last le with off(le) <= k, 32 candidates per round
    #pragma unroll 1
    while (span > 1) {
      const int stp = (span + 31) >> 5;
      const int cand = lo + lane * stp;
      const unsigned m = __ballot_sync(0xffffffffu, cand < lo + span && rb[cand] - rb[0] <= k);
      const int last = 31 - __clz(m);
      const int nlo = lo + last * stp;
      span = min(stp, lo + span - nlo);
      lo = nlo;
    }
    const int le = lo, kk = k - (rb[le] - rb[0]);
    const int g = t.gstart[le] + t.srcpre[le * (N + 1) + q] + kk;
    if (!TXB_ASSERT(g >= 0 && g < s.grouped_rows && kk >= 0)) continue;
    const uint8_t* src = priv_rows_of(region, s, par, q) + (int64_t)k * P;
    uint8_t* dst = G + (int64_t)g * P;
    if ((P & 15) == 0) {
      const int4* sv = reinterpret_cast<const int4*>(src);
      int4* dv = reinterpret_cast<int4*>(dst);
      const int n16 = (int)(P >> 4);
      #pragma unroll 1
      for (int c0 = 0; c0 < n16; c0 += 128) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + lane + 32 * u < n16) v[u] = sv[c0 + lane + 32 * u];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + lane + 32 * u < n16) dv[c0 + lane + 32 * u] = v[u];
      }
    } else {
      copy_row(dst, src, P, lane, 32);
    }
    if (lane == 0 && per_token(s)) srctok_of(region, s)[g] = privsrc_of(region, s, par, q)[k];
  }
}

// The step's error word into info (what dispatch_recv reads); also on the
// early-return paths, where CTA 0 has latched its own failure.
__device__ void publish_err(Flags* f, int64_t* info, int L) {
  if (threadIdx.x == 0) info[2 * L + 2] = (int64_t)*reinterpret_cast<volatile uint32_t*>(&f->err);
}

__device__ void wait_tokens(Flags* f, int64_t* info, int L, uint64_t timeout_ns) {
  if (threadIdx.x == 0) {
    const uint64_t dl = globaltimer() + timeout_ns;
    // the target was raised by an atomic add (add_flag) at L2: read it there
    const uint64_t target = *reinterpret_cast<volatile uint64_t*>(&f->tok_target);
    if (!spin_ge(&f->tok_ctr, target, dl)) atomicOr(&f->err, TXB_EV_WAIT_TOKEN);
    info[2 * L + 2] = (int64_t)*reinterpret_cast<volatile uint32_t*>(&f->err);
  }
}

// ------------------------------------------------------------------- C1

// Rows are moved in 2 KiB chunks (kChunk; one warp, four 16-byte loads per
// lane in flight before the four peer stores) so a step's return traffic
// spreads over every warp of the grid instead of one warp per 14 KiB row.
// The combine counter counts CHUNKS (comb_chunks(s) per row): a row's
// chunks may be stored by two CTAs (each CTA takes a contiguous run of
// chunks), and each CTA can only vouch for the chunks it stored itself --
// counting the row once, at its first chunk, let an origin read a row whose
// tail another CTA had not yet delivered (an intermittent combine mismatch
// at EP=2, found in round 2).

__device__ void combine_send_rows(const txb_moe_shape& s, Flags* f, const uint8_t* out, int64_t ld,
                                  void* const* peers, const int64_t* sources, const int32_t* ret,
                                  const int32_t* send_list, int cta, int ncta, Shared& sh) {
  const int N = s.ranks, tid = threadIdx.x;
  #pragma unroll 1
  for (int q = tid; q < N; q += blockDim.x) sh.cnt[q] = 0;
  __syncthreads();
  if (N == 1) return;  // every row is this rank's own: read in place by C2
  // rows that return over the fabric (compacted by the receive phase)
  const int total = (int)*reinterpret_cast<volatile uint32_t*>(&f->send_cnt);
  const int64_t Pc = s.comb_bytes;
  const int lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const bool vec = (Pc % 16 == 0) && (ld % 16 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (per_token(s)) {
    // per-token completion (large batches): each warp returns whole rows in
    // list (phase) order, fences once per kBatch rows, then release-adds
    // each row's count (comb_chunks(s), the unit of tokc) on its origin
    // token's counter.  Every row shape takes this branch (rows that are not
    // 16-byte vectorisable are copied with copy_row), because the origin's
    // reduce waits on tokc whenever per_token holds.
    constexpr int kBatch = 4;
    const int32_t* srct = srctok_of(peers[s.me], s);
    const int cpr = comb_chunks(s);
    // warp-major numbering: consecutive rows go to different CTAs (SMs)
    const int gw = warp * ncta + cta, ngw = ncta * nwarp;
    int pend_q = 0, pend_t = 0, pend_n = 0, npend = 0;
    auto flush = [&]() {
      __syncwarp();
      if (lane == 0 && npend) fence_acqrel_sys();
      #pragma unroll 1
      for (int k = 0; k < npend; ++k) {
        const int qk = __shfl_sync(0xffffffffu, pend_q, k), tk = __shfl_sync(0xffffffffu, pend_t, k);
        const int nk = __shfl_sync(0xffffffffu, pend_n, k);
        if (lane == 0) red_relaxed_sys_add(tokc_of(peers[qk], s) + tk, (uint64_t)nk);
      }
      npend = 0;
    };
    #pragma unroll 1
    for (int r = gw; r < total; r += ngw) {
      const int g = send_list[r];
      const int q = (int)sources[g];
      const int64_t nb = Pc;
      const uint8_t* src = out + (int64_t)g * ld;
      if (!TXB_ASSERT_V(q >= 0 && q < N && ret[g] >= 0 && ret[g] < s.comb_rows, r, total, g, ((int64_t)q << 32) | (uint32_t)ret[g])) continue;
      uint8_t* dst = comb_of(peers[q], s) + (int64_t)ret[g] * Pc;
      if (vec) {
        const int4* sv = reinterpret_cast<const int4*>(src);
        int4* dv = reinterpret_cast<int4*>(dst);
        const int n16 = (int)(nb >> 4);
        #pragma unroll 1
        for (int c0 = 0; c0 < n16; c0 += 256) {
          int4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c0 + lane + 32 * u < n16) v[u] = sv[c0 + lane + 32 * u];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c0 + lane + 32 * u < n16) dv[c0 + lane + 32 * u] = v[u];
        }
      } else {
        copy_row(dst, src, nb, lane, 32);
      }
      if (lane == npend) {
        pend_q = q;
        pend_t = srct[g];
        pend_n = cpr;
      }
      if (lane == 0) atomicAdd(&sh.cnt[q], (uint32_t)cpr);
      if (++npend == kBatch) flush();
    }
    flush();
    return;
  }
  if (vec) {
    // each CTA takes one contiguous run of chunks (whole rows, in order), its
    // warps interleaved over it: per-CTA shares equal to within one chunk,
    // and each CTA's peer writes stay sequential
    const int cpr = (int)((Pc + kChunk - 1) / kChunk);
    const int items = total * cpr;
    const int it1 = (int)((int64_t)items * (cta + 1) / ncta);
    #pragma unroll 1
    for (int it = (int)((int64_t)items * cta / ncta) + warp; it < it1; it += nwarp) {
      const int r = it / cpr, c = it - r * cpr;
      const int g = send_list[r];
      const int q = (int)sources[g];
      const int4* src = reinterpret_cast<const int4*>(out + (int64_t)g * ld + (int64_t)c * kChunk);
      if (!TXB_ASSERT_V(q >= 0 && q < N && ret[g] >= 0 && ret[g] < s.comb_rows, r, total, g, ((int64_t)q << 32) | (uint32_t)ret[g])) continue;
      int4* dst = reinterpret_cast<int4*>(comb_of(peers[q], s) + (int64_t)ret[g] * Pc + (int64_t)c * kChunk);
      const int n16 = (int)(min((int64_t)kChunk, Pc - (int64_t)c * kChunk) >> 4);
      int4 v[kChunk / 512];
#pragma unroll
      for (int u = 0; u < kChunk / 512; ++u)
        if (lane + 32 * u < n16) v[u] = src[lane + 32 * u];
#pragma unroll
      for (int u = 0; u < kChunk / 512; ++u)
        if (lane + 32 * u < n16) dst[lane + 32 * u] = v[u];
      if (lane == 0) atomicAdd(&sh.cnt[q], 1u);  // every chunk: the counter counts chunks
    }
    return;
  }
  #pragma unroll 1
  for (int r = cta * nwarp + warp; r < total; r += ncta * nwarp) {
    const int g = send_list[r];
    const int q = (int)sources[g];
    if (!TXB_ASSERT_V(q >= 0 && q < N && ret[g] >= 0 && ret[g] < s.comb_rows, r, total, g, ((int64_t)q << 32) | (uint32_t)ret[g])) continue;
    copy_row(comb_of(peers[q], s) + (int64_t)ret[g] * Pc, out + (int64_t)g * ld, Pc, lane, 32);
    if (lane == 0) atomicAdd(&sh.cnt[q], (uint32_t)comb_chunks(s));
  }
}

// ------------------------------------------------------------------- C2

// Wait for the returned rows, then reduce this CTA's tokens.  The first
// token's row pointers and weights are staged before the wait.
// Wait for the returned rows, then reduce this CTA's tokens.  The first
// token's row pointers and weights are staged before the wait; on the
// decode path (one token per CTA, R <= 8, H % 8 == 0 rows) the rows this
// rank served itself are already loaded into registers when the wait ends.
// The combine's per-token staging (row pointers, weights, scales); one per CTA.
static __shared__ CombTok s_comb_ct;

template <int ELEM>
__device__ bool combine_reduce(const txb_moe_shape& s, Flags* f, const uint8_t* comb, const uint8_t* out,
                               int64_t ld, const int64_t* pos, const int32_t* gidx, const float* w, int64_t n,
                               void* dst, int out_bf16, uint64_t timeout_ns, int cta, int ncta, Shared& sh,
                               uint64_t* prof = nullptr, void* region = nullptr, bool ws_ready = false) {
  CombTok& ct = s_comb_ct;
  const int64_t Pc = s.comb_bytes;
  const int H = s.hidden, R = s.topk;
  const bool vec = combine_vec<ELEM>(Pc, comb, out, ld, H, gidx);
  const bool split = vec && R <= kCombBatch && cta < n && H / 8 <= 2 * (int)blockDim.x && n <= ncta;
  if (cta < n) combine_prep(ct, comb, Pc, out, ld, pos, gidx, split ? nullptr : w, cta, R);
  // EP=1: every row is this rank's own and already written (stream order)
  const bool solo = s.ranks == 1;
  // fused path at EP > 1 (`region`): each token waits for its own rows only
  // (tokc[t] >= tokt[t]), so reducing overlaps the other tokens' returns
  const bool per_tok = region && per_token(s);
  auto wait = [&]() -> bool {
    if (threadIdx.x == 0) {
      if (solo) {
        sh.fail = 0;
      } else {
        const uint64_t dl = globaltimer() + timeout_ns;
        const bool ok = per_tok ? spin_ge(tokc_of(region, s) + cta, tokt_of(region, s)[cta], dl)
                                : spin_ge(&f->comb_ctr, *reinterpret_cast<volatile uint64_t*>(&f->comb_target), dl);
        sh.fail = ok ? 0u : TXB_EV_WAIT_COMBINE;
        if (sh.fail) atomicOr(&f->err, sh.fail);
      }
      if (prof) prof[blockIdx.x * 32 + 23] = globaltimer();
    }
    __syncthreads();
    return sh.fail == 0;
  };
  if (split) {
    __syncthreads();  // ct staged
    if (!combine_token_split<ELEM>(ct, H, R, cta, ws_ready ? nullptr : w, dst, out_bf16, wait)) return false;
    __syncthreads();
    return true;
  }
  if (!per_tok && !wait()) return false;
  const uint64_t* tokc = per_tok ? tokc_of(region, s) : nullptr;
  const uint64_t* tokt = per_tok ? tokt_of(region, s) : nullptr;
  const uint64_t dl = globaltimer() + timeout_ns;
  #pragma unroll 1
  for (int64_t t = cta; t < n; t += ncta) {
    if (t != cta) combine_prep(ct, comb, Pc, out, ld, pos, gidx, w, t, R);
    if (per_tok && threadIdx.x == 0) {
      sh.fail = spin_ge(tokc + t, tokt[t], dl) ? 0u : TXB_EV_WAIT_COMBINE;
      if (sh.fail) atomicOr(&f->err, sh.fail);
    }
    __syncthreads();
    if (per_tok && sh.fail) return false;
    combine_token<ELEM>(ct, Pc, comb, H, R, t, dst, out_bf16, vec);
    __syncthreads();
  }
  return true;
}

// End of step: the last CTA (ticket) resets the step's scratch counters and
// advances the local step counter.  The buffer-reuse barrier tag (done) is
// published by the next step's route phase (route_publish), so the tail of
// the combine carries no fence and no remote store.
__device__ void end_of_step(Flags* f, int ncta) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // the fields the last CTA updates are loaded before the ticket: nothing
    // changes them during the combine, and the kernel's tail (the next
    // step's dispatch waits on it) then carries one round trip, the ticket
    const uint64_t step = cur_step(f);
    const uint64_t pstep = *reinterpret_cast<volatile uint64_t*>(&f->priv_step);
    const uint64_t ptgt = *reinterpret_cast<volatile uint64_t*>(&f->priv_target[step & 1]);
    const uint32_t t = atomicAdd(&f->ticket, 1u);
    if (t == (uint32_t)ncta - 1) {
      f->ticket = 0;
      f->send_cnt = 0;
      if (pstep) {
        f->priv_target[step & 1] = ptgt + pstep;
        f->priv_step = 0;
      }
      for (int ph = 0; ph < kPhases; ++ph) f->phase_cnt[ph] = 0;
      *reinterpret_cast<volatile uint64_t*>(&f->step) = step;
    }
  }
}

// ------------------------------------------------------------ split kernels

__global__ void __launch_bounds__(kRouteThreads)
k_route(txb_moe_shape s, txb_moe_bufs b, const int64_t* __restrict__ routes, int64_t n) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  uint32_t* hist = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* wc = hist + ((s.experts + 3) & ~3);
  Flags* f = flags_of(b.region, s);
  const uint64_t step = cur_step(f);
  const uint32_t bad = route_counts_chunked(s, routes, n, hist, wc, b.rank_scratch, 0, 1, sh);
  route_positions(s, routes, n, hist, reinterpret_cast<int*>(wc), b.rank_scratch, b.pos, bad, 0, 1, sh);
  route_publish(s, b.peers, f, hist, step, n, bad, 0, 1);
}

template <int SRC, int ELEM>
__global__ void __launch_bounds__(kThreads, 1)
k_dispatch(txb_moe_shape s, txb_moe_bufs b, const void* __restrict__ x, int64_t n,
           const int64_t* __restrict__ routes, uint64_t timeout_ns) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  Flags* f = flags_of(b.region, s);
  const uint64_t step = cur_step(f);
  uint32_t* C = reinterpret_cast<uint32_t*>(dsm + cmat_offset(s));
  if (!wait_routes(s, f, route_of(b.region, s, (int)(step & 1)), C, step, timeout_ns, sh)) return;
  int* baseg = reinterpret_cast<int*>(dsm);
  if (!dispatch_layout(s, C, baseg, baseg + s.experts, f, sh)) return;
  if (blockIdx.x == 0 && threadIdx.x < 32) book_recv(s, f, C, threadIdx.x);
  if (*reinterpret_cast<volatile uint32_t*>(&f->err) & (TXB_EV_ROUTE_RANGE | TXB_EV_ROUTE_DUP)) return;
  for (int q = threadIdx.x; q < s.ranks; q += blockDim.x) sh.cnt[q] = sh.pcnt[q] = 0;
  if (threadIdx.x == 0) sh.direct = 0;
  __syncthreads();
  dispatch_tokens<SRC, ELEM>(s, x, blockIdx.x, n, gridDim.x, routes, b.rank_scratch, b.pos, b.gidx, b.peers, baseg,
                             step, sh);
  book_tok_targets(s, routes, b.region, blockIdx.x, n, gridDim.x);
  signal_counts(s, b.peers, 0, step, sh);
}

__global__ void __launch_bounds__(kThreads, 1)
k_recv(txb_moe_shape s, txb_moe_bufs b, uint64_t timeout_ns) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  Flags* f = flags_of(b.region, s);
  const uint64_t step = cur_step(f);
  uint32_t* C = reinterpret_cast<uint32_t*>(dsm + cmat_offset(s));
  if (!wait_routes(s, f, route_of(b.region, s, (int)(step & 1)), C, step, timeout_ns, sh)) return;
  int* rt = reinterpret_cast<int*>(dsm + recv_offset(s));
  recv_tables(s, C, rt, b.info, blockIdx.x, sh, b);
  recv_rows_flat(s, rt, b.rows, b.sources, b.ret_slot, grouped_of(b.region, s), b.dirty, b.send_list,
                 &f->send_cnt, blockIdx.x, gridDim.x, nullptr);
  {
    const int nw = blockDim.x >> 5;
    recv_private_rows(s, rt, b.region, step, timeout_ns, blockIdx.x * nw + (threadIdx.x >> 5), gridDim.x * nw,
                      threadIdx.x & 31);
  }
  __syncthreads();
  if (blockIdx.x == 0) wait_tokens(f, b.info, s.local_experts, timeout_ns);
}

__global__ void __launch_bounds__(kThreads, 1)
k_comb_send(txb_moe_shape s, txb_moe_bufs b, const uint8_t* __restrict__ out, int64_t ld) {
  __shared__ Shared sh;
  Flags* f = flags_of(b.region, s);
  combine_send_rows(s, f, out, ld, b.peers, b.sources, b.ret_slot, b.send_list, blockIdx.x, gridDim.x, sh);
  signal_counts(s, b.peers, 1, cur_step(f), sh);
}

template <int ELEM>
__global__ void __launch_bounds__(kThreads, 1)
k_comb_recv(txb_moe_shape s, txb_moe_bufs b, const uint8_t* __restrict__ out, int64_t ld,
            const float* __restrict__ w, int64_t n, void* dst, int out_bf16, uint64_t timeout_ns) {
  __shared__ Shared sh;
  Flags* f = flags_of(b.region, s);
  combine_reduce<ELEM>(s, f, comb_of(b.region, s), out, ld, b.pos, b.gidx, w, n, dst, out_bf16, timeout_ns,
                       blockIdx.x, gridDim.x, sh);
  end_of_step(f, gridDim.x);
}

// ------------------------------------------------------------ fused kernels

// Route + dispatch + receive in one cooperative launch.  Every CTA counts
// all n*R copies redundantly (no grid barrier), the CTAs publish slices of
// the count row, every CTA acquires the route matrix, derives the layout,
// stores its tokens and signals; then the grid fills the receive metadata
// and CTA 0 waits for the incoming rows.
// DECODE (n == grid, vectorisable rows, R | 32, <= kMaxOwn copies per CTA):
// the CTA's single token is read and encoded into registers before the
// route exchange and stored once the layout is known.
template <int SRC, int ELEM, bool DECODE>
__global__ void __launch_bounds__(kThreads, 1)
k_dispatch_fused(txb_moe_shape s, txb_moe_bufs b, const void* __restrict__ x, int64_t n,
                 const int64_t* __restrict__ routes, uint64_t timeout_ns) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  Flags* f = flags_of(b.region, s);
  const uint64_t step = cur_step(f);
  const int cta = blockIdx.x, ncta = gridDim.x;
  uint32_t* hist = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* wc = hist + ((s.experts + 3) & ~3);
  uint32_t* C = reinterpret_cast<uint32_t*>(dsm + cmat_offset(s));
  int* rt = reinterpret_cast<int*>(dsm + recv_offset(s));
  const bool solo = s.ranks == 1;
  stamp(b, 0);
  grid_dep_launch();
  if constexpr (DECODE) {
    RowRegs pre;
    RowRaw raw;
    // issue the token's loads first; route counting runs while they land
    load_row_raw<SRC, ELEM>(x, cta, s.hidden, s.payload_bytes, raw);
    const uint32_t bad = route_counts_direct(s, routes, n, hist, reinterpret_cast<int32_t*>(hist + s.experts),
                                             b.rank_scratch, cta, ncta, sh, b, Grp::cta());
    stamp(b, 14);
    finish_row_regs<SRC, ELEM>(raw, pre, sh.red);
    stamp(b, 1);
    for (int q = threadIdx.x; q < s.ranks; q += blockDim.x) sh.cnt[q] = sh.pcnt[q] = 0;
    __syncthreads();
    route_publish(s, b.peers, f, hist, step, n, bad, cta, ncta);
    own_positions(s, hist, b.pos, bad, sh, Grp::cta(), b.peers, step);
    stamp(b, 2);
    // EP=1: the route matrix is this CTA's own histogram and the kernel
    // boundary orders the stores before any reader -- no exchange, fence,
    // counter or wait (the published row still feeds last_layout)
    const uint32_t* Cm = hist;
    if (!solo) {
      if (!wait_routes(s, f, route_of(b.region, s, (int)(step & 1)), C, step, timeout_ns, sh)) {
        if (cta == 0) publish_err(f, b.info, s.local_experts);
        return;
      }
      Cm = C;
    }
    stamp(b, 3);
    if (!bad) {
      own_dests(s, Cm, b.peers, b.gidx, sh);
      // private copies (late on this path) and grouped rows in one pass
      if (threadIdx.x < s.topk && sh.pdst[threadIdx.x]) sh.dstp[threadIdx.x] = sh.pdst[threadIdx.x];
      __syncthreads();
      stamp(b, 15);
      if (pre.ok) store_row_regs<SRC, ELEM>(pre, s.hidden, s.scales, sh.dstp, s.topk);
      else dispatch_row_slow<SRC, ELEM>(s, x, cta, sh);
    }
    stamp(b, 5);
    // the receive tables overlap the stores in flight; the fence follows
    recv_tables_body<true>(s, Cm, rt, b.info, cta, sh, b);
    stamp(b, 4);
    if (!solo) {
      if (cta == 0 && threadIdx.x < 32) book_recv(s, f, Cm, threadIdx.x);
      signal_counts(s, b.peers, 0, step, sh);
    }
  } else {
    // contiguous token range per CTA, segmented counting with a grid barrier
    const int64_t chunk = (n + ncta - 1) / ncta;
    const int64_t t0 = n < cta * chunk ? n : cta * chunk, t1 = n < t0 + chunk ? n : t0 + chunk;
    const uint32_t bad = route_counts_segmented(s, routes, hist, wc, b.rank_scratch, b.pos, t0, t1, b.cta_hist,
                                                b.cta_bad, f, cta, ncta, sh, b);
    stamp(b, 1);
    route_publish(s, b.peers, f, hist, step, n, bad, cta, ncta);
    stamp(b, 2);
    // EP=1: the totals are the route matrix (copied out of `hist`, which
    // the layout below overwrites)
    const uint32_t* Cm = C;
    if (solo) {
      for (int e = threadIdx.x; e < s.experts; e += blockDim.x) C[e] = hist[e];
      __syncthreads();
    } else {
      if (!wait_routes(s, f, route_of(b.region, s, (int)(step & 1)), C, step, timeout_ns, sh)) {
        if (cta == 0) publish_err(f, b.info, s.local_experts);
        return;
      }
      Cm = C;
    }
    stamp(b, 3);
    int* baseg = reinterpret_cast<int*>(dsm);
    if (!dispatch_layout(s, Cm, baseg, baseg + s.experts, f, sh)) {
      if (cta == 0) publish_err(f, b.info, s.local_experts);
      return;
    }
    if (!solo && cta == 0 && threadIdx.x < 32) book_recv(s, f, Cm, threadIdx.x);
    recv_tables(s, Cm, rt, b.info, cta, sh, b);
    for (int q = threadIdx.x; q < s.ranks; q += blockDim.x) sh.cnt[q] = sh.pcnt[q] = 0;
    __syncthreads();
    stamp(b, 4);
    if (!bad) {
      // destination pointer table after the route matrix copy, sized by the
      // host through the dynamic shared-memory size
      uint32_t dyn;
      asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
      const size_t fo = flat_offset(s);
      const int cap = dyn > fo ? (int)((dyn - fo) / sizeof(uint8_t*)) : 0;
      if (!dispatch_tokens_flat<SRC, ELEM>(s, x, t0, t1, routes, b.rank_scratch, b.pos, b.gidx, b.peers, baseg,
                                           reinterpret_cast<uint8_t**>(dsm + fo), cap, step, sh))
        dispatch_tokens<SRC, ELEM>(s, x, t0, t1, 1, routes, b.rank_scratch, b.pos, b.gidx, b.peers, baseg, step,
                                   sh);
      book_tok_targets(s, routes, b.region, t0, t1, 1);
    }
    stamp(b, 5);
    if (!solo) signal_counts(s, b.peers, 0, step, sh);
  }
  // thread 0 fences and signals while the other warps fill the metadata
  stamp(b, 6);
  if constexpr (DECODE)
    recv_rows_body(s, rt, b.rows, b.sources, b.ret_slot, grouped_of(b.region, s), b.dirty, b.send_list,
                   &f->send_cnt, cta, ncta);
  else
    recv_rows_flat(s, rt, b.rows, b.sources, b.ret_slot, grouped_of(b.region, s), b.dirty, b.send_list,
                   &f->send_cnt, cta, ncta, f->phase_cnt);
  {
    const int nw = blockDim.x >> 5;
    recv_private_rows(s, rt, b.region, step, timeout_ns, cta * nw + (threadIdx.x >> 5), ncta * nw, threadIdx.x & 31);
  }
  stamp(b, 7);
  __syncthreads();
  if (cta == 0) {
    // EP=1: every CTA counted every route, so CTA 0 has latched any route
    // error itself; the grid's end publishes the rows
    if (!solo) wait_tokens(f, b.info, s.local_experts, timeout_ns);
    else publish_err(f, b.info, s.local_experts);
  }
  stamp(b, 8);
}

// Decode dispatch with two warp roles on named barriers, so phases that do
// not depend on each other run at once instead of one after another:
//   routing (warps 0-7, barrier 1): count, publish, positions, route
//     acquire, destinations; hand-off (barrier 3); receive tables;
//   token (warps 8-15, barrier 2): load + amax + encode the CTA's token
//     while the routing role counts; hand-off; store the copies while the
//     routing role builds the receive tables.
// Then the whole CTA signals, fills the receive metadata and waits.
// Eligible when the row fits the token role's registers (<= 2 chunks per
// thread) and every route id fits the staging area (host checks).
constexpr int kRouteRole = kThreads / 2;

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Producer side of a hand-off: the routing role marks its arrival and runs
// on; the token role's bar.sync on the same barrier completes once both
// roles are in, and sees the routing role's shared-memory writes (arrive
// synchronizes with the completing sync in the PTX memory model).
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

//
// SOLO (one rank): the route matrix is this CTA's histogram, so the roles
// split differently right after it: the token role ranks its copies and
// derives positions and destinations, then stores; the routing role
// publishes the row and builds the receive tables and rows meanwhile.  Both
// halves start from the histogram instead of the receive metadata waiting
// for the destinations.
template <int SRC, int ELEM>
__device__ __forceinline__ void dispatch_roles_solo(const txb_moe_shape& s, const txb_moe_bufs& b, const void* x,
                                                    int64_t n, const int64_t* routes, Flags* f, uint64_t step,
                                                    uint8_t* dsm, Shared& sh) {
  __shared__ uint32_t bad_s;
  const int cta = blockIdx.x, ncta = gridDim.x;
  uint32_t* hist = reinterpret_cast<uint32_t*>(dsm);
  int32_t* rv = reinterpret_cast<int32_t*>(hist + s.experts);
  // the receive tables are built while the token role still reads the
  // staged ids: they live after them (solo_recv_offset), not over them
  int* rt = reinterpret_cast<int*>(dsm + solo_recv_offset(s, n));
  if (threadIdx.x >= kRouteRole) {
    const Grp tg{(int)threadIdx.x - kRouteRole, kThreads - kRouteRole, 2};
    RowRaw raw;
    RowRegs pre;
    load_row_raw<SRC, ELEM>(x, cta, s.hidden, s.payload_bytes, raw, tg);
    own_token_dups(s, routes, n, cta, &f->err, tg);  // while the row load is in flight
    finish_row_regs<SRC, ELEM>(raw, pre, sh.red, tg);
    if (b.prof && tg.tid == 0) b.prof[blockIdx.x * 32 + 1] = globaltimer();
    for (int q = tg.tid; q < s.ranks; q += tg.nt) sh.cnt[q] = 0;
    named_sync(3, kThreads);  // histogram, staged ids and own copies ready
    const uint32_t bad = bad_s;
    own_copies_solo(s, hist, rv, b, bad, sh, tg);
    if (!bad) {
      if (b.prof && tg.tid == 0) b.prof[blockIdx.x * 32 + 15] = globaltimer();
      store_row_regs<SRC, ELEM>(pre, s.hidden, s.scales, sh.dstp, s.topk, tg);
    }
    if (b.prof && tg.tid == 0) b.prof[blockIdx.x * 32 + 20] = globaltimer();

  } else {
    const Grp rg{(int)threadIdx.x, kRouteRole, 1};
    const uint32_t bad = route_counts_direct(s, routes, n, hist, rv, b.rank_scratch, cta, ncta, sh, b, rg, false,
                                             /*check_dups=*/false);
    const PreDirty pd = prefetch_dirty(s, b.dirty, cta, ncta, rg);  // after the route loads
    if (rg.tid == 0) bad_s = bad;
    named_arrive(3, kThreads);
    stamp(b, 14);
    route_publish(s, b.peers, f, hist, step, n, bad, cta, ncta, rg);
    recv_tables_solo(s, hist, rt, b.info, cta, sh, rg);
    stamp(b, 4);
    recv_rows_body(s, rt, b.rows, b.sources, b.ret_slot, grouped_of(b.region, s), b.dirty, b.send_list,
                   &f->send_cnt, cta, ncta, rg, pd);
    stamp(b, 7);
  }
  __syncthreads();
  stamp(b, 5);
  if (cta == 0) publish_err(f, b.info, s.local_experts);
  stamp(b, 8);
}

template <int SRC, int ELEM, bool SOLO>
__global__ void __launch_bounds__(kThreads, 1)
k_dispatch_roles(txb_moe_shape s, txb_moe_bufs b, const void* __restrict__ x, int64_t n,
                 const int64_t* __restrict__ routes, uint64_t timeout_ns) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  __shared__ uint32_t skip, fail;  // routing -> token: no stores / route acquire failed
  Flags* f = flags_of(b.region, s);
  const uint64_t step = cur_step(f);
  const int cta = blockIdx.x, ncta = gridDim.x;
  // the CTA that books the step's counter targets and waits for the tokens:
  // the last one, so CTA 0 (receive info, error word) carries no more
  const int bk = ncta - 1;
  uint32_t* hist = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* C = reinterpret_cast<uint32_t*>(dsm + cmat_offset(s));
  int* rt = reinterpret_cast<int*>(dsm + recv_offset(s));
  const bool solo = s.ranks == 1;
#ifdef TXB_CHECKED
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const size_t need = SOLO ? solo_recv_offset(s, n) + smem_recv(s.ranks, s.local_experts)
                             : cmat_offset(s) + smem_cmat(s.ranks, s.experts);
    // the staged ids must end before the receive tables in the EP=1 kernel,
    // where the two are live at once
    if (!TXB_ASSERT(need <= dyn && (!SOLO || (size_t)(s.experts + n * s.topk) * 4 + 16 <= solo_recv_offset(s, n))))
      return;
  }
#endif
  stamp(b, 0);
  grid_dep_launch();
  if constexpr (SOLO) {
    dispatch_roles_solo<SRC, ELEM>(s, b, x, n, routes, f, step, dsm, sh);
    return;
  }
  if (threadIdx.x >= kRouteRole) {
    const Grp tg{(int)threadIdx.x - kRouteRole, kThreads - kRouteRole, 2};
    RowRaw raw;
    RowRegs pre;
    load_row_raw<SRC, ELEM>(x, cta, s.hidden, s.payload_bytes, raw, tg);
    own_token_dups(s, routes, n, cta, &f->err, tg);  // while the row load is in flight
    finish_row_regs<SRC, ELEM>(raw, pre, sh.red, tg);
    if (b.prof && tg.tid == 0) b.prof[blockIdx.x * 32 + 1] = globaltimer();
    // speculative private copies (moe.py:556-582): their destinations need
    // only this rank's own counts, so they are stored while the route
    // exchange is still in flight; they are counted with the main rows by
    // the CTA's one release fence at the end (a second fence here would
    // hold the whole CTA at the hand-off barrier for its drain)
    named_sync(4, kThreads);  // private destinations are in sh.pdst
    if (s.priv_tokens > 0) {
      store_row_regs<SRC, ELEM>(pre, s.hidden, s.scales, sh.pdst, s.topk, tg);
      if (b.prof && tg.tid == 0) b.prof[blockIdx.x * 32 + 26] = globaltimer();
    }
    named_sync(3, kThreads);  // destinations are in sh.dstp
    if (!skip) store_row_regs<SRC, ELEM>(pre, s.hidden, s.scales, sh.dstp, s.topk, tg);
    if (b.prof && tg.tid == 0) b.prof[blockIdx.x * 32 + 20] = globaltimer();
  } else {
    const Grp rg{(int)threadIdx.x, kRouteRole, 1};
    for (int q = rg.tid; q < s.ranks; q += rg.nt) sh.cnt[q] = sh.pcnt[q] = 0;
    // the count row is published as soon as the histogram is complete; the
    // stable ranks of the CTA's copies are counted while it travels.  The
    // staged ids `rv` overlap the receive tables `rt` (written after
    // hand-off 3), so only this role reads them, and only before then.
    int32_t* rv = reinterpret_cast<int32_t*>(hist + s.experts);
    const uint32_t bad = route_counts_direct(s, routes, n, hist, rv, b.rank_scratch, cta, ncta, sh, b, rg, false,
                                             /*check_dups=*/false);
    const PreDirty pd = prefetch_dirty(s, b.dirty, cta, ncta, rg);  // after the route loads
    route_publish(s, b.peers, f, hist, step, n, bad, cta, ncta, rg);
    stamp(b, 14);
    if (!bad) {
      const int nw = (n > cta ? (int)((n - cta + ncta - 1) / ncta) : 0) * s.topk;
      own_ranks(rv, b.rank_scratch, nw, sh, rg);
      rg.sync();
    }
    own_positions(s, hist, b.pos, bad, sh, rg, b.peers, step);
    rg.sync();
    named_arrive(4, kThreads);
    stamp(b, 2);
    const uint32_t* Cm = hist;
    bool ok = true;
    if (!solo) {
      ok = wait_routes(s, f, route_of(b.region, s, (int)(step & 1)), C, step, timeout_ns, sh, rg);
      Cm = C;
    } else {
      rg.sync();  // counters zeroed before own_dests adds to them
    }
    stamp(b, 3);
    if (ok && !bad) own_dests(s, Cm, b.peers, b.gidx, sh, rg);
    if (rg.tid == 0) {
      skip = (!ok || bad) ? 1u : 0u;
      fail = ok ? 0u : 1u;
    }
    named_arrive(3, kThreads);
    stamp(b, 15);
    if (ok) {
      recv_tables_body<true>(s, Cm, rt, b.info, cta, sh, b, rg);
      if (!solo && cta == bk && rg.tid < 32) book_recv(s, f, Cm, rg.tid);
      stamp(b, 4);
      // receive metadata while the token role's stores drain, then the
      // private rows that arrived before the layout was known
      recv_rows_body(s, rt, b.rows, b.sources, b.ret_slot, grouped_of(b.region, s), b.dirty, b.send_list,
                     &f->send_cnt, cta, ncta, rg, pd);
    }
    stamp(b, 7);
  }
  __syncthreads();  // stores issued, receive tables and rows built
  if (fail) {
    if (cta == bk) publish_err(f, b.info, s.local_experts);
    return;
  }
  stamp(b, 5);
  if (!solo) signal_counts(s, b.peers, 0, step, sh);
  // the private rows other ranks stored here, once this CTA has signalled
  // (waiting for them before it would make the ranks wait on each other)
  recv_private_rows(s, rt, b.region, step, timeout_ns, cta * (kThreads >> 5) + (threadIdx.x >> 5),
                    ncta * (kThreads >> 5), threadIdx.x & 31);
  stamp(b, 6);
  if (cta == bk) {
    if (!solo) wait_tokens(f, b.info, s.local_experts, timeout_ns);
    else publish_err(f, b.info, s.local_experts);
  }
  stamp(b, 8);
}

// Combine send + reduce in one cooperative launch.
template <int ELEM>
__global__ void __launch_bounds__(kThreads, 1)
k_combine_fused(txb_moe_shape s, txb_moe_bufs b, const uint8_t* __restrict__ out, int64_t ld,
                const float* __restrict__ w, int64_t n, void* dst, int out_bf16, uint64_t timeout_ns) {
  __shared__ Shared sh;
  // Nothing is read before the programmatic dependency resolves, not even
  // the step's weights: a weights upload enqueued between the dispatch and
  // this kernel was observed racing with an early read (an intermittent
  // bf16 mismatch in test_dsv3_decode_device_mode, profiles/r02/README.md).
  grid_dep_wait();  // the producing dispatch (or expert) kernel has completed
  Flags* f = flags_of(b.region, s);
  stamp(b, 9);
  // Large batches with per-token completion (two half-size CTAs per SM):
  // even CTAs return rows, odd CTAs reduce tokens as their rows land, so
  // the reduce runs during the returns instead of after them.
  const int ncta = gridDim.x;
  const bool roles = tok_mode(s) && blockDim.x < kThreads && ncta >= 2;
  const bool sender = !roles || (blockIdx.x & 1) == 0;
  const int sidx = roles ? (int)blockIdx.x >> 1 : (int)blockIdx.x, nsend = roles ? (ncta + 1) >> 1 : ncta;
  const int ridx = roles ? (int)blockIdx.x >> 1 : (int)blockIdx.x, nred = roles ? ncta >> 1 : ncta;
  if (sender) {
    combine_send_rows(s, f, out, ld, b.peers, b.sources, b.ret_slot, b.send_list, sidx, nsend, sh);
  } else {
    for (int q = threadIdx.x; q < s.ranks; q += blockDim.x) sh.cnt[q] = 0;
    __syncthreads();
  }
  stamp(b, 10);
  signal_counts(s, b.peers, 1, 0, sh);
  __syncthreads();
  stamp(b, 11);
  if (!roles || !sender)
    combine_reduce<ELEM>(s, f, comb_of(b.region, s), out, ld, b.pos, b.gidx, w, n, dst, out_bf16, timeout_ns,
                         ridx, nred, sh, b.prof, b.region);
  stamp(b, 12);
  end_of_step(f, ncta);
  stamp(b, 13);
}

// -------------------------------------------------------------- k_barrier

// All-rank device barrier (submit_barrier with one imm per peer,
// engine.py:599-619): publish my epoch into every peer's slot, then
// acquire-wait until every peer's epoch has reached mine.
__global__ void k_barrier(txb_moe_shape s, txb_moe_bufs b, uint64_t timeout_ns) {
  Flags* f = flags_of(b.region, s);
  __shared__ uint64_t ep;
  __shared__ uint32_t fail;
  if (threadIdx.x == 0) {
    ep = f->bar_epoch + 1;
    f->bar_epoch = ep;
    fail = 0;
  }
  __syncthreads();
  const int N = s.ranks;
  for (int q = threadIdx.x; q < N; q += blockDim.x) st_release_sys(&flags_of(b.peers[q], s)->bar[s.me], ep);
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

static int check(const txb_moe_shape* s, const txb_moe_bufs* b) {
  if (!s || !b) {
    set_error("null shape or buffers");
    return TXB_ERR_PROTOCOL;
  }
  if (s->payload_bytes <= 0 || s->region_bytes == 0) {
    set_error("shape not planned (call txb_moe_plan)");
    return TXB_ERR_PROTOCOL;
  }
  if (!b->region || !b->peers) {
    set_error("buffers not wired (region / peer table missing)");
    return TXB_ERR_REGION;
  }
  return TXB_OK;
}

// dynamic shared memory: [layout | recv scratch][route matrix copy], with
// the route-count phase (before the matrix is loaded) overlapping both
static size_t smem_main(const txb_moe_shape* s, bool route) {
  size_t m = cmat_offset(*s) + smem_cmat(s->ranks, s->experts);
  if (route) {
    const size_t q = smem_route(s->experts, kThreads / 32);
    if (q > m) m = q;
  }
  return m;
}

// Raise a kernel's dynamic shared-memory limit once per (kernel, device);
// cudaFuncSetAttribute on every launch costs microseconds of host time.
template <typename K>
static int set_smem(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return TXB_OK;
  struct Entry {
    const void* fn;
    int dev;
    size_t smem;
  };
  static thread_local Entry seen[64];
  static thread_local int nseen = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < nseen; ++i)
    if (seen[i].fn == (const void*)kernel && seen[i].dev == dev && seen[i].smem >= smem) return TXB_OK;
  TXB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nseen < 64) seen[nseen++] = Entry{(const void*)kernel, dev, smem};
  return TXB_OK;
}

// Launch helper; `coop` requests a cooperative launch (all CTAs resident).

// `pdl` marks the launch as a programmatic dependent of the previous kernel
// on the stream: its CTAs may be scheduled while that kernel drains, and
// block in griddepcontrol.wait until it has completed.
template <typename... KArgs, typename... Args>
static int launch_ex(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, bool coop,
                     bool pdl, Args... args) {
  if (int rc = set_smem(kernel, smem)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  }
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  TXB_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
  return TXB_OK;
}

template <typename... KArgs, typename... Args>
static int launch(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, bool coop,
                  Args... args) {
  return launch_ex(kernel, grid, block, smem, st, coop, false, args...);
}

// Largest cooperative grid for a kernel (one wave).
template <typename K>
static int coop_grid(K kernel, int dev, size_t smem, int want, int block = kThreads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
  const int cap = (per_sm > 0 ? per_sm : 1) * sm_count(dev);
  if (want > cap) want = cap;
  return want < 1 ? 1 : want;
}

template <int SRC, int ELEM>
static cudaError_t preload_src_elem() {
  cudaError_t e = cudaSuccess;
  for (cudaError_t r : {touch(k_dispatch_roles<SRC, ELEM, true>), touch(k_dispatch_roles<SRC, ELEM, false>),
                        touch(k_dispatch_fused<SRC, ELEM, true>), touch(k_dispatch_fused<SRC, ELEM, false>),
                        touch(k_dispatch<SRC, ELEM>)})
    if (r != cudaSuccess) e = r;
  return e;
}

unsigned int check_failures_moe() {
#ifdef TXB_CHECKED
  return read_check_fail();
#else
  return 0;
#endif
}

cudaError_t preload_moe() {
  cudaError_t e = cudaSuccess;
  for (cudaError_t r : {preload_src_elem<TXB_SRC_ROWS, 1>(), preload_src_elem<TXB_SRC_F32, 1>(),
                        preload_src_elem<TXB_SRC_F32, 2>(), preload_src_elem<TXB_SRC_F32, 4>(),
                        preload_src_elem<TXB_SRC_BF16, 1>(), preload_src_elem<TXB_SRC_BF16, 2>(),
                        preload_src_elem<TXB_SRC_BF16, 4>(), touch(k_combine_fused<1>), touch(k_combine_fused<2>),
                        touch(k_combine_fused<4>), touch(k_comb_recv<1>), touch(k_comb_recv<2>), touch(k_comb_recv<4>),
                        touch(k_route), touch(k_recv), touch(k_comb_send), touch(k_barrier)})
    if (r != cudaSuccess) e = r;
  return e;
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
  if ((int64_t)s->ranks * s->experts > 16384) {
    set_error("ranks*experts %lld above the supported 16384", (long long)s->ranks * s->experts);
    return TXB_ERR_PROTOCOL;
  }
  if (s->me < 0 || s->me >= s->ranks) { set_error("rank %d outside 0..%d", s->me, s->ranks - 1); return TXB_ERR_PROTOCOL; }
  // PrivateBufferConfig.validate (moe.py:98-102)
  if (s->priv_tokens < 0 || s->priv_tokens > s->max_tokens) {
    set_error("private buffer of %d tokens outside 0..%d", s->priv_tokens, s->max_tokens);
    return TXB_ERR_PROTOCOL;
  }
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
  off = align_up(off + 2ull * N * s->experts * 8, 4096);
  s->off_grouped = off;
  off = align_up(off + (uint64_t)s->grouped_rows * s->payload_bytes, 4096);
  s->off_comb = off;
  off = align_up(off + (uint64_t)s->comb_rows * s->comb_bytes, 256);
  // per-token completion words + origin token index per grouped row
  off = align_up(off + 2ull * (uint64_t)T * 8 + (uint64_t)s->grouped_rows * 4, 4096);
  // speculative private slabs [2][N][priv_tokens] rows + origin token index
  s->off_priv = off;
  const uint64_t npriv = 2ull * (uint64_t)N * (uint64_t)s->priv_tokens;
  off = align_up(off + npriv * (uint64_t)s->payload_bytes + npriv * 4, 4096);
  s->region_bytes = off;
  return TXB_OK;
}

int txb_moe_route(const txb_moe_shape* s, const txb_moe_bufs* b, const int64_t* routes, int64_t n, void* stream) {
  if (int rc = check(s, b)) return rc;
  if (n < 0 || n > s->max_tokens) {
    set_error("%lld tokens exceed the %d-token limit", (long long)n, s->max_tokens);
    return TXB_ERR_PROTOCOL;
  }
  TXB_ON_DEVICE(s->device);
  const size_t smem = smem_route(s->experts, kRouteThreads / 32);
  return launch(k_route, 1, kRouteThreads, smem, (cudaStream_t)stream, false, *s, *b, routes, n);
}

#define TXB_SWITCH_SRC_ELEM(KIND, ELEMSZ, MACRO)         \
  do {                                                   \
    if ((KIND) == TXB_SRC_ROWS) {                        \
      MACRO(TXB_SRC_ROWS, 1);                            \
    } else if ((KIND) == TXB_SRC_F32) {                  \
      if ((ELEMSZ) == 1) MACRO(TXB_SRC_F32, 1);          \
      else if ((ELEMSZ) == 2) MACRO(TXB_SRC_F32, 2);     \
      else MACRO(TXB_SRC_F32, 4);                        \
    } else if ((KIND) == TXB_SRC_BF16) {                 \
      if ((ELEMSZ) == 1) MACRO(TXB_SRC_BF16, 1);         \
      else if ((ELEMSZ) == 2) MACRO(TXB_SRC_BF16, 2);    \
      else MACRO(TXB_SRC_BF16, 4);                       \
    } else {                                             \
      set_error("unknown source kind %d", (KIND));       \
      return TXB_ERR_PROTOCOL;                           \
    }                                                    \
  } while (0)

int txb_moe_dispatch(const txb_moe_shape* s, const txb_moe_bufs* b, const void* x, int src_kind, int64_t n,
                     const int64_t* routes, uint64_t timeout_ns, int grid, void* stream) {
  if (int rc = check(s, b)) return rc;
  TXB_ON_DEVICE(s->device);
  if (grid <= 0) {
    const int64_t g = n < 1 ? 1 : n;
    grid = (int)(g < 4 * sm_count(s->device) ? g : 4 * sm_count(s->device));
  }
  const size_t smem = smem_main(s, false);
  cudaStream_t st = (cudaStream_t)stream;
#define TXB_D(SRC, ELEM) \
  return launch(k_dispatch<SRC, ELEM>, grid, kThreads, smem, st, false, *s, *b, x, n, routes, timeout_ns)
  TXB_SWITCH_SRC_ELEM(src_kind, s->elem_size, TXB_D);
#undef TXB_D
  return TXB_OK;
}

int txb_moe_dispatch_recv(const txb_moe_shape* s, const txb_moe_bufs* b, uint64_t timeout_ns, void* stream) {
  if (int rc = check(s, b)) return rc;
  TXB_ON_DEVICE(s->device);
  const size_t smem = smem_main(s, false);
  const int64_t wpb = kThreads / 32;
  int grid = (int)((s->grouped_rows + wpb - 1) / wpb);
  if (grid > sm_count(s->device)) grid = sm_count(s->device);
  if (grid < 1) grid = 1;
  return launch(k_recv, grid, kThreads, smem, (cudaStream_t)stream, false, *s, *b, timeout_ns);
}

int txb_moe_combine_send(const txb_moe_shape* s, const txb_moe_bufs* b, const void* outputs, int64_t ld, int grid,
                         void* stream) {
  if (int rc = check(s, b)) return rc;
  TXB_ON_DEVICE(s->device);
  if (grid <= 0) {
    const int64_t want = (s->grouped_rows + (kThreads / 32) - 1) / (kThreads / 32);
    const int cap = 2 * sm_count(s->device);
    grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  }
  return launch(k_comb_send, grid, kThreads, 0, (cudaStream_t)stream, false, *s, *b, (const uint8_t*)outputs, ld);
}

int txb_moe_combine_recv(const txb_moe_shape* s, const txb_moe_bufs* b, const void* outputs, int64_t ld,
                         const float* weights, int64_t n, void* out, int out_bf16, uint64_t timeout_ns,
                         void* stream) {
  if (int rc = check(s, b)) return rc;
  TXB_ON_DEVICE(s->device);
  const int grid = (int)(n < 1 ? 1 : (n < 2 * sm_count(s->device) ? n : 2 * sm_count(s->device)));
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* o = (const uint8_t*)outputs;
  switch (s->comb_elem_size) {
    case 1: return launch(k_comb_recv<1>, grid, kThreads, 0, st, false, *s, *b, o, ld, weights, n, out, out_bf16, timeout_ns);
    case 2: return launch(k_comb_recv<2>, grid, kThreads, 0, st, false, *s, *b, o, ld, weights, n, out, out_bf16, timeout_ns);
    default: return launch(k_comb_recv<4>, grid, kThreads, 0, st, false, *s, *b, o, ld, weights, n, out, out_bf16, timeout_ns);
  }
}

int txb_moe_dispatch_fused(const txb_moe_shape* s, const txb_moe_bufs* b, const void* x, int src_kind, int64_t n,
                           const int64_t* routes, uint64_t timeout_ns, void* stream) {
  if (int rc = check(s, b)) return rc;
  if (n < 0 || n > s->max_tokens) {
    set_error("%lld tokens exceed the %d-token limit", (long long)n, s->max_tokens);
    return TXB_ERR_PROTOCOL;
  }
  if (!b->cta_hist || !b->cta_bad) {
    set_error("fused dispatch needs the per-CTA scratch (cta_hist / cta_bad)");
    return TXB_ERR_REGION;
  }
  TXB_ON_DEVICE(s->device);
  const size_t smem = smem_main(s, true);
  cudaStream_t st = (cudaStream_t)stream;
  const int sms = sm_count(s->device);
  // decode specialisation: one token per CTA, row vectorisable in registers
  const int64_t srcb = src_kind == TXB_SRC_F32 ? 4 : 2;
  const int epc = src_kind == TXB_SRC_ROWS ? 16 : 16 / s->elem_size;
  const int64_t nchunk = src_kind == TXB_SRC_ROWS ? s->payload_bytes / 16 : s->hidden / epc;
  bool vec;
  if (src_kind == TXB_SRC_ROWS)
    vec = (s->payload_bytes % 16 == 0) && ((uintptr_t)x % 16 == 0);
  else {
    const int64_t salign = epc * srcb >= 16 ? 16 : epc * srcb;
    vec = ((int64_t)s->hidden * s->elem_size % 16 == 0) && (s->payload_bytes % 16 == 0) &&
          ((uintptr_t)x % salign == 0) && ((int64_t)s->hidden * srcb % salign == 0);
  }
  const bool decode = n >= 1 && n <= sms && s->topk <= kMaxOwn && vec && nchunk <= 2 * kThreads;
  // two warp roles when the token fits the token role's registers
  const bool roles = decode && nchunk <= 2 * (kThreads - kRouteRole);
  const int want = (int)(n < 1 ? 1 : (n < sms ? n : sms));
  // decode: the route ids of the whole batch are staged after the histogram
  const size_t rv_end = (size_t)(s->experts + n * s->topk) * 4 + 16;
  const size_t smem_d = smem > rv_end ? smem : rv_end;
  const size_t solo_end = solo_recv_offset(*s, n) + smem_recv(s->ranks, s->local_experts);
  const size_t smem_r = s->ranks == 1 && solo_end > smem_d ? solo_end : smem_d;
#define TXB_F(SRC, ELEM)                                                                            \
  do {                                                                                              \
    if (roles) {                                                                                    \
      auto kr = s->ranks == 1 ? k_dispatch_roles<SRC, ELEM, true> : k_dispatch_roles<SRC, ELEM, false>; \
      if (int rc = set_smem(kr, smem_r)) return rc;                                                 \
      if (coop_grid(kr, s->device, smem_r, want) == want)                                           \
        return launch(kr, want, kThreads, smem_r, st, true, *s, *b, x, n, routes, timeout_ns);      \
    }                                                                                               \
    if (decode) {                                                                                   \
      auto kd = k_dispatch_fused<SRC, ELEM, true>;                                                  \
      if (int rc = set_smem(kd, smem_d)) return rc;                                                 \
      if (coop_grid(kd, s->device, smem_d, want) == want)                                           \
        return launch(kd, want, kThreads, smem_d, st, true, *s, *b, x, n, routes, timeout_ns);      \
    }                                                                                               \
    /* + the destination pointer table of dispatch_tokens_flat (<= 64 KiB) */                      \
    auto kg = k_dispatch_fused<SRC, ELEM, false>;                                                   \
    const int64_t per = (n + want - 1) / want * s->topk;                                            \
    size_t smem_g = flat_offset(*s) + (size_t)per * sizeof(uint8_t*);                               \
    if (per * (int64_t)sizeof(uint8_t*) > 64 * 1024) smem_g = smem;                                 \
    if (smem_g < smem) smem_g = smem;                                                               \
    if (int rc = set_smem(kg, smem_g)) return rc;                                                   \
    const int grid = coop_grid(kg, s->device, smem_g, want);                                        \
    return launch(kg, grid, kThreads, smem_g, st, true, *s, *b, x, n, routes, timeout_ns);          \
  } while (0)
  TXB_SWITCH_SRC_ELEM(src_kind, s->elem_size, TXB_F);
#undef TXB_F
  return TXB_OK;
}

int txb_moe_combine_fused(const txb_moe_shape* s, const txb_moe_bufs* b, const void* outputs, int64_t ld,
                          const float* weights, int64_t n, void* out, int out_bf16, uint64_t timeout_ns,
                          void* stream) {
  if (int rc = check(s, b)) return rc;
  TXB_ON_DEVICE(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* o = (const uint8_t*)outputs;
  const int sms = sm_count(s->device);
#define TXB_C(ELEM)                                                                                   \
  do {                                                                                                \
    /* large batches: half-size CTAs, two per SM, so one CTA's row loads */                           \
    /* overlap the other's arithmetic and stores (tokens are reduced one per */                       \
    /* CTA pass); decode keeps one 512-thread CTA per token */                                        \
    const int blk = n > sms ? kThreads / 2 : kThreads;                                                \
    const int grid = coop_grid(k_combine_fused<ELEM>, s->device, 0, blk == kThreads ? sms : 2 * sms, blk); \
    /* one rank: no cross-CTA waits, so no co-residency requirement; launched */                      \
    /* as a programmatic dependent so its CTAs land while the dispatch drains */                      \
    const bool solo = s->ranks == 1;                                                                  \
    static const bool no_pdl = getenv("TXB_NO_PDL") != nullptr;                                       \
    return launch_ex(k_combine_fused<ELEM>, grid, blk, 0, st, !solo, !no_pdl, *s, *b, o, ld, weights, \
                     n, out, out_bf16, timeout_ns);                                                   \
  } while (0)
  switch (s->comb_elem_size) {
    case 1: TXB_C(1);
    case 2: TXB_C(2);
    default: TXB_C(4);
  }
#undef TXB_C
}

int txb_moe_barrier(const txb_moe_shape* s, const txb_moe_bufs* b, uint64_t timeout_ns, void* stream) {
  if (int rc = check(s, b)) return rc;
  TXB_ON_DEVICE(s->device);
  return launch(k_barrier, 1, 128, 0, (cudaStream_t)stream, false, *s, *b, timeout_ns);
}

int txb_moe_status(const txb_moe_shape* s, void* region, uint32_t* err, uint64_t* counters, int64_t ncounters) {
  if (!s || !region) {
    set_error("null shape or region");
    return TXB_ERR_PROTOCOL;
  }
  TXB_ON_DEVICE(s->device);
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
    uint64_t buf[10 + 9 * TXB_MAX_RANKS];
    int k = 0;
    buf[k++] = h.step;
    buf[k++] = h.tok_ctr;
    buf[k++] = h.tok_target;
    buf[k++] = h.comb_ctr;
    buf[k++] = h.comb_target;
    buf[k++] = h.priv_ctr[0];
    buf[k++] = h.priv_ctr[1];
    buf[k++] = h.priv_target[0];
    buf[k++] = h.priv_target[1];
    buf[k++] = h.priv_step;
    for (int p = 0; p < 2; ++p)
      for (int q = 0; q < N; ++q) buf[k++] = h.route_tag[p][q];
    const uint64_t* lanes[7] = {h.done, h.tok_src, h.tok_src_t, h.comb_src, h.comb_src_t, h.priv_src, h.priv_src_t};
    for (int l = 0; l < 7; ++l)
      for (int q = 0; q < N; ++q) buf[k++] = lanes[l][q];
    for (int i = 0; i < k && i < ncounters; ++i) counters[i] = buf[i];
  }
  return TXB_OK;
}

}  // extern "C"
