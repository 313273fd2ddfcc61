/*
 * txb200 -- C ABI of the B200-native WriteImm/ImmCounter MoE dispatch/combine
 * path (libtxb200.so, sm_100a).
 *
 * The reference (railtx, /root/reference/pkg/src/railtx) is pure Python and
 * has no FFI of its own; its seam is the Python API of railtx.moe /
 * railtx.engine.  Each entry point below replaces one piece of that API and
 * cites the reference it stands in for.  The Python mirror of the reference
 * interface (paper_2510_27656_b200/moe.py, engine.py) binds these through
 * ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Plain pointers and sizes only; device pointers are CUDA device
 *     addresses, `stream` is a cudaStream_t passed as void*.
 *   - Every call returns an int status: TXB_OK, or a negative error class
 *     mirroring the reference exception taxonomy (errors.py:4-25).
 *     txb_last_error() returns the calling thread's last message.
 *   - Hot-path calls never allocate and never synchronise the stream.
 *   - Device-side failures (route validation, counter timeouts, capacity)
 *     are latched into the rank's error word (TXB_EV_* bits) and read back
 *     with txb_moe_status() at the next host sync point.
 */
#ifndef TXB200_H
#define TXB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TXB_OK 0
#define TXB_ERR_PROTOCOL (-1) /* railtx.errors.ProtocolError  (errors.py:20) */
#define TXB_ERR_TRANSFER (-2) /* railtx.errors.TransferError  (errors.py:16) */
#define TXB_ERR_REGION (-3)   /* railtx.errors.RegionError    (errors.py:12) */
#define TXB_ERR_CUDA (-4)     /* CUDA runtime failure (RailtxError)        */

#define TXB_MAX_RANKS 128
#define TXB_MAX_CTAS 1024 /* cooperative grid bound for the per-CTA scratch */
#define TXB_IPC_HANDLE_BYTES 64

/* Device error-word bits (latched per rank). */
#define TXB_EV_ROUTE_RANGE 0x1u     /* expert index out of range (moe.py:150-151) */
#define TXB_EV_ROUTE_DUP 0x2u       /* duplicate expert in a token (moe.py:152-154) */
#define TXB_EV_WAIT_ROUTE 0x4u      /* timed out waiting for route rows            */
#define TXB_EV_WAIT_TOKEN 0x8u      /* timed out waiting for token writes          */
#define TXB_EV_WAIT_BARRIER 0x10u   /* timed out waiting for peers' step barrier   */
#define TXB_EV_WAIT_COMBINE 0x20u   /* timed out waiting for combine writes        */
#define TXB_EV_CAPACITY 0x40u       /* destination needs more slots than capacity  */
#define TXB_EV_WAIT_IMM 0x80u       /* txb_imm_wait timeout (engine primitive)     */
#define TXB_EV_WAIT_PRIV 0x100u     /* timed out waiting for speculative private rows */

/* Row encodings (RoutingSpec.elem_size, moe.py:40-50; 2 = bf16 extension). */
#define TXB_ELEM_FP8 1
#define TXB_ELEM_BF16 2
#define TXB_ELEM_F32 4

/* Source kinds for txb_moe_dispatch / txb_encode_rows. */
#define TXB_SRC_ROWS 0 /* pre-encoded wire rows u8[n, P] (dispatch_send payload)  */
#define TXB_SRC_F32 1  /* f32 values [n, hidden]: encoded inside the kernel       */
#define TXB_SRC_BF16 2 /* bf16 values [n, hidden]: encoded inside the kernel      */

/*
 * Static shape of one expert-parallel mesh (RoutingSpec, moe.py:36-89) plus
 * the byte layout of each rank's symmetric region.  txb_moe_plan() fills
 * the derived fields; the struct is passed by pointer to every call.
 */
typedef struct txb_moe_shape {
  /* RoutingSpec */
  int32_t ranks, experts, max_tokens, topk, hidden, elem_size, scales;
  /* combine wire format: elem size of the rows combine_send carries */
  int32_t comb_elem_size, comb_scales;
  int32_t me;     /* this rank */
  int32_t device; /* CUDA device of this rank's region and stream */
  int32_t single_device; /* 1 when every rank of the mesh lives on this device:
                            completion fences drop from .sys to .gpu scope */
  int32_t priv_tokens;   /* speculative private rows per source (PrivateBufferConfig.tokens,
                            moe.py:92-102; 0..max_tokens): a source stores the first
                            priv_tokens rows of its slab for a peer into that peer's private
                            slab before the route exchange completes (moe.py:556-582) */
  /* derived by txb_moe_plan */
  int32_t local_experts;
  int64_t payload_bytes;  /* dispatch row bytes  = hidden*elem + 4*scales */
  int64_t comb_bytes;     /* combine row bytes                            */
  int64_t capacity;       /* N*T*max(R, L) (moe.py:80-83)                 */
  int64_t grouped_rows;   /* allocated grouped rows (tight bound + padding) */
  int64_t comb_rows;      /* T*R */
  uint64_t off_flags, off_route, off_grouped, off_comb, off_priv, region_bytes;
} txb_moe_shape;

/* ------------------------------------------------------------ runtime */

const char* txb_last_error(void);
int txb_version(void);
int txb_device_count(int* out);

/* Region registration (stands in for TransferEngine.reg_mr/dereg_mr,
 * engine.py:314-350; MrDesc = the IPC handle, wire.py:64-87). */
int txb_alloc(int device, uint64_t bytes, void** out_ptr);
int txb_free(int device, void* ptr);
int txb_memset(int device, void* ptr, int value, uint64_t bytes, void* stream);
int txb_ipc_export(int device, void* ptr, uint8_t* out_handle /*[64]*/);
int txb_ipc_import(int device, const uint8_t* handle /*[64]*/, void** out_ptr);
int txb_ipc_close(int device, void* ptr);
int txb_enable_peer(int device, int peer_device);
/* A dedicated non-blocking stream for an engine's copies (never one of the
 * framework's pooled streams, which user code may also be handed: a copy
 * kernel waiting on a device clock must not sit in front of the compute
 * that advances it). */
int txb_stream_create(int device, void** out_stream);
/* Load every kernel of the library on `device` now (cudaFuncGetAttributes)
 * instead of at its first launch: under lazy module loading a first launch
 * did not complete while a persistent kernel was polling on the device.
 * Idempotent; TransferEngine calls it when it binds a device. */
int txb_preload(int device);
/* Checked build (make checked -> libtxb200_checked.so, -DTXB_CHECKED): *out =
 * 0x80000000 | bit 0 set when a device-side bounds check has failed since
 * load (device synchronised first).  The release build writes 0. */
int txb_check_failures(int device, uint32_t* out);
int txb_stream_destroy(int device, void* stream);
/* Device address of page-locked host memory (cudaHostAlloc / pinned torch
 * tensors).  The kernels read inputs from and write results to such host
 * buffers in place over PCIe (zero-copy), the way the reference's dispatch
 * and combine take host arrays (moe.py:470-497, 814-866).  Fails with
 * TXB_ERR_REGION for pageable memory. */
int txb_host_device_ptr(void* host_ptr, void** out_device_ptr);

/* ------------------------------------------------------- MoE hot path */

/* Per-rank device buffers (all device pointers).  `region` is the rank's
 * symmetric allocation (txb_moe_shape.region_bytes, laid out by
 * txb_moe_plan); `peers` is a device array of `ranks` region base addresses
 * as seen from this rank (own region at index `me`). */
typedef struct txb_moe_bufs {
  void* region;
  void* const* peers;
  int32_t* rank_scratch; /* [max_tokens*topk] stable rank of each copy in its expert */
  int64_t* pos;          /* [max_tokens*topk] send slot of copy j of token t (moe.py:510-520) */
  int32_t* gidx;         /* [max_tokens*topk] grouped row of copies served by this rank, else -1 */
  int64_t* rows;         /* [grouped_rows] GroupedTokens.rows (moe.py:280) */
  int64_t* sources;      /* [grouped_rows] GroupedTokens.sources (moe.py:281) */
  int32_t* ret_slot;     /* [grouped_rows] combine return slot on the source */
  int64_t* info;         /* [2L+3] group_sizes, group_starts, padded_total, recv_total, error word */
  uint8_t* dirty;        /* [grouped_rows] 1 = row may hold data (zeroed when it becomes padding) */
  uint32_t* cta_hist;    /* [TXB_MAX_CTAS][experts] per-CTA counts of the segmented route phase */
  uint32_t* cta_bad;     /* [TXB_MAX_CTAS] per-CTA route validation bits */
  int32_t* send_list;    /* [grouped_rows] grouped rows whose source is another rank */
  uint64_t* prof;        /* optional [grid][32] %globaltimer phase stamps, grid = the launch's CTA
                            count (<= TXB_MAX_CTAS; NULL = off) */
} txb_moe_bufs;

/* Validate a RoutingSpec (moe.py:52-70) and fill the derived fields. */
int txb_moe_plan(txb_moe_shape* s);

/* ---- fused path (one GPU per rank; cooperative launches) ---------------
 * dispatch_fused = MoeRank.dispatch_send + dispatch_recv (moe.py:470-735):
 * count the routes (_stage, moe.py:499-523; _check_routes 142-155), scatter
 * the own count row to every peer with the route immediate (538-553), wait
 * for all rows, derive the layout (compute_layout 200-225), store every
 * token copy -- encoded on the fly for TXB_SRC_F32/BF16 (encode_tokens
 * 231-246) -- straight into its final grouped row on the owner (the recv
 * slab + pack_rows regroup of 556-722 in one peer store), release-add the
 * row counts on the owners' token counters, build rows/sources/padding and
 * wait for the expected token rows.  routes: i64 [n, R] device (railtx's dtype). */
int txb_moe_dispatch_fused(const txb_moe_shape* s, const txb_moe_bufs* b, const void* x, int src_kind,
                           int64_t n, const int64_t* routes, uint64_t timeout_ns, void* stream);
/* combine_fused = combine_send + combine_recv (moe.py:739-833): every valid
 * grouped row of `outputs` (row stride ld bytes, comb_bytes wide) returns to
 * its source at the originating send slot, counts are release-added, then
 * after the expected rows arrived out[t] = sum_j w[t,j] * row(t,j) in fp32,
 * j ascending, no FMA (kernels.weighted_combine, kernels.py:206-242);
 * out_bf16 selects bf16 RNE output (kernels.bf16_encode, kernels.py:144-150).
 * The last CTA (ticket) advances the local step counter; the end-of-step
 * barrier (moe.dbar) is published by the NEXT dispatch's route phase, next to
 * its count row, so the combine's tail carries no remote store. */
int txb_moe_combine_fused(const txb_moe_shape* s, const txb_moe_bufs* b, const void* outputs, int64_t ld,
                          const float* weights, int64_t n, void* out, int out_bf16, uint64_t timeout_ns,
                          void* stream);

/* ---- split path (same semantics, one phase per kernel; used when several
 * ranks share one GPU and for batches above the fused limit) ------------- */
int txb_moe_route(const txb_moe_shape* s, const txb_moe_bufs* b, const int64_t* routes, int64_t n,
                  void* stream);
int txb_moe_dispatch(const txb_moe_shape* s, const txb_moe_bufs* b, const void* x, int src_kind, int64_t n,
                     const int64_t* routes, uint64_t timeout_ns, int grid, void* stream);
int txb_moe_dispatch_recv(const txb_moe_shape* s, const txb_moe_bufs* b, uint64_t timeout_ns, void* stream);
int txb_moe_combine_send(const txb_moe_shape* s, const txb_moe_bufs* b, const void* outputs, int64_t ld,
                         int grid, void* stream);
int txb_moe_combine_recv(const txb_moe_shape* s, const txb_moe_bufs* b, const void* outputs, int64_t ld,
                         const float* weights, int64_t n, void* out, int out_bf16, uint64_t timeout_ns,
                         void* stream);

/* Device-side all-rank barrier over the mesh (engine submit_barrier,
 * engine.py:599-619): each rank release-stores its epoch into every peer,
 * then acquire-waits for every peer's epoch.  Used to align step starts. */
int txb_moe_barrier(const txb_moe_shape* s, const txb_moe_bufs* b, uint64_t timeout_ns, void* stream);

/* Read the rank's latched error word and counters (synchronous, on a
 * private non-blocking stream; for the host's ProtocolError diagnostics,
 * moe.py:869-899).  counters receives [step, tok_ctr, tok_target, comb_ctr,
 * comb_target, priv_ctr[0], priv_ctr[1], priv_target[0], priv_target[1],
 * priv_step] (10 words), then route_tag[2][N], then seven [N] lanes: done,
 * tok_src, tok_src_target, comb_src, comb_src_target, priv_src,
 * priv_src_target (rows received from / expected of each source rank);
 * 10 + 9N words in all.  NULL skips. */
int txb_moe_status(const txb_moe_shape* s, void* region, uint32_t* err, uint64_t* counters,
                   int64_t ncounters);

/* ------------------------------------------- engine primitives (phase 2) */

/* ImmCounter table (ImmCounterTable, engine.py:138-205), keyed by the full
 * u32 imm: keys u64[TXB_IMM_SLOTS] (0 = empty, else imm + 1) followed by
 * counts u64[TXB_IMM_SLOTS], open addressing.  The owner and every sender
 * claim an imm's slot with a system-scope CAS on the owner's table
 * (txb_imm_slot), so they agree on its counter whoever arrives first; the
 * host keeps `consumed` per imm so a value can be re-armed. */
#define TXB_IMM_SLOTS 131072
#define TXB_MAX_JOBS 64 /* writes per txb_copy_jobs launch (a scatter's peer slices) */

/* One paged write (submit_paged_writes, engine.py:438-466; a single write is
 * one page).  Page i: src_base + src_offset + src_idx[i]*src_stride ->
 * dst_base + dst_offset + dst_idx[i]*dst_stride, page_len bytes (wire.py
 * Pages:100-112).  idx arrays are device i64 (NULL = identity).  imm_ctr:
 * the destination's ImmCounter slot (peer-mapped) or NULL; incremented once,
 * after the whole payload is visible.  ticket: a zeroed device u32 used for
 * last-CTA detection (operations sharing a ticket must be stream-ordered). */
typedef struct txb_pages {
  const void* src_base;
  int64_t src_offset, src_stride;
  const int64_t* src_idx;
  void* dst_base;
  int64_t dst_offset, dst_stride;
  const int64_t* dst_idx;
  int64_t npages, page_len;
  uint64_t* imm_ctr;
  uint32_t* ticket;
  int32_t use_tma;       /* 1: TMA bulk copies (16-byte aligned pages), 0: vector copies */
  int32_t single_device; /* 1: every party on this device (.gpu-scope fences) */
} txb_pages;

int txb_imm_table_slots(void);
/* Slot of `imm` in an ImmCounter table (own or peer-mapped): insert = 1
 * claims it if absent (TXB_ERR_TRANSFER when the table is full), 0 looks it
 * up (*out_slot = -1 when absent).  Synchronous, on a private stream; the
 * caller caches the slot. */
int txb_imm_slot(uint64_t* table, uint32_t imm, int insert, int64_t* out_slot);
/* Current values of n (<= 64) device words, e.g. ImmCounter receipt
 * counters (ImmCounterTable.received_total, engine.py:197-205): one
 * device-to-host copy each on a private non-blocking stream, so a poll never
 * waits behind kernels spinning on other streams. */
int txb_read_u64(const uint64_t* const* ptrs, int n, uint64_t* out);
/* Move the pages and release one increment on *imm_ctr (engine.py:480-508, 759-782). */
int txb_copy_pages(const txb_pages* job, int grid, void* stream);
/* 1..TXB_MAX_JOBS writes in ONE launch (submit_scatter's per-peer slices,
 * engine.py:563-597): each job completes on its own, one increment on its
 * imm_ctr after its whole payload is visible.  Jobs are passed by value
 * (host array). */
int txb_copy_jobs(const txb_pages* jobs, int njobs, int grid, void* stream);

/* Persistent paged stream: the KV-cache layer-by-layer transfer
 * (PrefillerNode._on_progress, kvcache.py:477-507) with the LayerClock
 * (kvcache.py:317-334) on the device.  Step k (0-based) moves pages
 * [k*pages_per_step, (k+1)*pages_per_step) of src_idx/dst_idx (page numbers,
 * page_len bytes each) once *clock >= clock_base + k + 1, and releases one
 * increment on *imm_ctr when the step is complete.  tickets: zeroed u32
 * [nsteps] (device). */
typedef struct txb_stream_job {
  const void* src;
  void* dst;
  int64_t page_len;
  const int64_t* src_idx;
  const int64_t* dst_idx;
  int64_t pages_per_step;
  int32_t nsteps;
  int32_t use_tma;
  const uint64_t* clock;
  uint64_t clock_base;
  uint64_t* imm_ctr;
  uint32_t* tickets;
  uint64_t timeout_ns;
  uint32_t* err;
  int32_t single_device;
  int32_t pad;
} txb_stream_job;
int txb_kv_stream(const txb_stream_job* job, int grid, void* stream);
/* Device layer clock: write / wait on a u64 word in stream order through
 * the GPU front end (cuStreamWriteValue64 / cuStreamWaitValue64 GEQ), no SM
 * and no host thread; a one-thread kernel stands in where 64-bit stream
 * memory operations are unavailable (wait: TXB_EV_WAIT_IMM in *err on
 * timeout, err may be NULL). */
int txb_stream_write_value64(uint64_t* addr, uint64_t value, void* stream);
int txb_stream_wait_value64(const uint64_t* addr, uint64_t value, uint64_t timeout_ns, uint32_t* err, void* stream);
/* Zero-length writes carrying an immediate: +value on each of n counters
 * (ctrs: device array of peer-mapped counter pointers) (submit_barrier). */
int txb_imm_add(uint64_t* const* ctrs, int n, uint64_t value, int single_device, void* stream);
/* Block `stream` until *ctr >= threshold (device-side ImmFlag wait); on
 * timeout sets TXB_EV_WAIT_IMM in *err (may be NULL). */
int txb_imm_wait(const uint64_t* ctr, uint64_t threshold, uint64_t timeout_ns, uint32_t* err, void* stream);
/* Diagnostics: one %globaltimer sample (ns) written to *out on `stream`,
 * the clock the kernels' phase stamps (txb_moe_bufs.prof) use. */
int txb_globaltimer(uint64_t* out, void* stream);
/* Per-tensor fp8 narrowing of bf16 words (weights.prepare, weights.py:383-387):
 * out = e4m3(x / f32(amax/448)) bytes followed by the f32 scale (n + 4 bytes). */
int txb_fp8_quantize_tensor(const uint16_t* x, int64_t n, uint32_t* amax_scratch, uint8_t* out, void* stream);

/* ----------------------------------- codecs (kernels.py registry "cuda") */

/* encode_tokens (moe.py:231-246): values (f32 or bf16 [n, hidden]) ->
 * wire rows u8[n, hidden*elem + 4*scales]. */
int txb_encode_rows(const void* values, int src_kind, int64_t n, int32_t hidden,
                    int32_t elem_size, int32_t scales, void* out, void* stream);
/* decode_tokens (moe.py:249-262): wire rows -> f32 [n, hidden]. */
int txb_decode_rows(const void* rows, int64_t n, int32_t hidden, int32_t elem_size,
                    int32_t scales, float* out, void* stream);
/* kernels.pack_rows (kernels.py:184-203): out[k] = src[rows[k]]. */
int txb_pack_rows(const void* src, int64_t width, const int64_t* rows, int64_t k, void* out,
                  void* stream);
/* kernels.weighted_combine (kernels.py:206-242). */
int txb_weighted_combine(const float* y, int64_t hidden, const int64_t* pos, const float* w,
                         int64_t n, int32_t topk, float* out, void* stream);
/* kernels.fp8_encode / fp8_decode / bf16_encode elementwise. */
int txb_fp8_encode(const float* x, int64_t n, uint8_t* out, void* stream);
int txb_fp8_decode(const uint8_t* b, int64_t n, float* out, void* stream);
int txb_bf16_encode(const float* x, int64_t n, uint16_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TXB200_H */
