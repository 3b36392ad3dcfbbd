/*
 * ss_b200.h — C ABI of the B200-native Symbiosis base executor ("splitserve" hot path).
 *
 * The reference computes one executor batch inline in Python:
 *   BaseExecutor._compute_batch   pkg/src/splitserve/executor.py:191-231
 *     concat_rows                 pkg/src/splitserve/tensor_ops.py:145-146
 *     affine_forward              pkg/src/splitserve/tensor_ops.py:71-78     (PASS_FORWARD = 0)
 *     affine_backward_input       pkg/src/splitserve/tensor_ops.py:81-89     (PASS_BACKWARD = 1)
 *     matmul (bias nullified)     pkg/src/splitserve/executor.py:221-222     (PASS_NOISE_EFFECT = 2)
 *     split_rows                  pkg/src/splitserve/tensor_ops.py:149-156
 * and applies each client's adapter client-side afterwards:
 *   apply_adapter                 pkg/src/splitserve/adapters.py:127-145  (LoRA + IA3, forward)
 *   lora_backward (grad_x term)   pkg/src/splitserve/adapters.py:26-41    (backward)
 *   ClientModel._layer_backward   pkg/src/splitserve/client.py:286-305    (IA3 g = dy * l)
 *
 * This library replaces that inline compute with one call per dispatch: ss_compute_batch()
 * runs gather -> (LoRA shrink) -> fused base GEMM + adapter epilogue -> per-segment scatter
 * on a CUDA stream. No C++ exception crosses this boundary; every entry point returns an
 * int status (SS_OK or a negative SS_E* code) and ss_last_error() gives the message.
 *
 * All activation pointers are DEVICE pointers owned by the caller (client exchange buffers).
 * Weight / adapter uploads accept host or device pointers (SS_MEM_DEVICE).
 */
#ifndef SS_B200_H
#define SS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SS_API __attribute__((visibility("default")))
#else
#define SS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------- */
#define SS_OK 0
#define SS_E_ARG (-1)       /* bad argument (null ctx, bad pass, bad dims) */
#define SS_E_CUDA (-2)      /* CUDA runtime / driver failure */
#define SS_E_NOLAYER (-3)   /* unknown (block, role) — reference: "unknown layer" executor.py:172-174 */
#define SS_E_NOMEM (-4)
#define SS_E_UNSUPPORTED (-5)
#define SS_E_PROTOCOL (-6)  /* LSV1 stream corrupt (bad magic / version): connection-level rejection */

/* per-segment status written to seg_status[i] (0 = computed) */
#define SS_SEG_OK 0
#define SS_SEG_BAD_WIDTH 1  /* reference: "row width ... does not match layer" executor.py:208-211 */
#define SS_SEG_BAD_PTR 2
#define SS_SEG_NO_ADAPTER 3 /* SS_SEGF_ADAPTER set but no adapter registered for this layer */

/* passes — same values as protocol.py:40-42 */
#define SS_PASS_FORWARD 0
#define SS_PASS_BACKWARD 1
#define SS_PASS_NOISE_EFFECT 2

/* memory / dtype flags for uploads */
#define SS_MEM_DEVICE (1u << 0) /* pointer is device memory (else host) */
#define SS_DT_BF16 (1u << 1)    /* element type bf16 (else f32) */

/* adapter kinds (bit mask) — adapters.py:44-115 */
#define SS_ADAPTER_LORA 1u
#define SS_ADAPTER_IA3 2u

/* segment flags */
#define SS_SEGF_SRC_BF16 (1u << 0)  /* src rows are bf16 (else f32) */
#define SS_SEGF_DST_BF16 (1u << 1)  /* dst rows are bf16 (else f32) */
#define SS_SEGF_BASE_BF16 (1u << 2) /* dst_base rows are bf16 (else f32) */
#define SS_SEGF_ADAPTER (1u << 3)   /* apply this client's registered adapter for the layer; on
                                       SS_PASS_NOISE_EFFECT: the noise effect of the adapted layer,
                                       (n.W + s n.A.B) * l, bias-free (privacy.py:1-12 blinding
                                       with an executor-fused adapter) */
#define SS_SEGF_PINNED (1u << 4)    /* ss_compute_batch_host: the caller has verified that src / dst /
                                       dst_base are page-locked host memory (skips the per-pointer
                                       query of the zero-copy path) */
/* Summation class of a segment's rows (see decode_rows below). Without either flag the class
 * follows the segment's own row count; a caller that splits one request into several segments
 * (the library's host pipelines do) sets the class of the whole request on every piece, so the
 * pieces give the same bits as the request would in one piece. */
#define SS_SEGF_CLASS_DECODE (1u << 5)   /* force the decode class (split-K order; segments of
                                            at most 16 rows, ignored on longer ones) */
#define SS_SEGF_CLASS_PREFILL (1u << 6)  /* force the single-chain class */

/* One request (envelope) of a batch, in batch order. Rows are concatenated in array order
 * exactly like concat_rows(); row r of segment i is batch row off_i + r, off_i = sum_{j<i} rows_j
 * over the segments whose status is SS_SEG_OK (split_rows, tensor_ops.py:149-156). */
typedef struct ss_seg {
  uint32_t client_id;
  uint32_t rows;     /* token_count */
  uint32_t width;    /* payload width as sent; must equal d_in (fwd/noise) or d_out (bwd) */
  uint32_t flags;    /* SS_SEGF_* */
  const void* src;   /* device, [rows, src_ld] */
  int64_t src_ld;    /* elements */
  void* dst;         /* device, [rows, dst_ld]; may alias src (in-place exchange buffer) */
  int64_t dst_ld;
  void* dst_base;    /* optional pre-IA3 output (IA3 fine-tune clients need y_base,
                        client.py:241-242, 293), forward and noise passes; NULL if not wanted */
  int64_t base_ld;
} ss_seg;

typedef struct ss_ctx ss_ctx;

/* Create a context on CUDA device `device`. tp_rank / tp_size describe this process's
 * tensor-parallel position (metadata; sharding is expressed through the shards loaded). */
SS_API int ss_ctx_create(int device, int tp_rank, int tp_size, ss_ctx** out);
SS_API int ss_ctx_destroy(ss_ctx* ctx);
SS_API const char* ss_last_error(const ss_ctx* ctx);
/* Library version / build string, usable without a GPU. */
SS_API const char* ss_version(void);

/* Load one frozen affine layer (AffineParams, tensor_ops.py:39-68): weight [d_in, d_out]
 * row-major with row stride w_ld elements, optional bias [d_out]. Stored as bf16. */
SS_API int ss_load_layer(ss_ctx* ctx, int block, int role, int d_in, int d_out, const void* weight,
                  int64_t w_ld, const void* bias, uint32_t flags);
SS_API int ss_unload_layer(ss_ctx* ctx, int block, int role);

/* Register / refresh a client's adapter for one layer. LoRA: A [d_in, rank], B [rank, d_out],
 * scale = alpha / rank (lora_forward adapters.py:19-23). IA3: l [d_out] (adapters.py:142-144).
 * kind is a mask of SS_ADAPTER_*; pointers of kinds not in the mask may be NULL.
 * Refreshing with the same rank re-packs in place (call after every optimizer step). */
SS_API int ss_set_adapter(ss_ctx* ctx, uint32_t client_id, int block, int role, uint32_t kind, int rank,
                   float scale, const void* A, const void* B, const void* l, uint32_t flags);
SS_API int ss_clear_adapter(ss_ctx* ctx, uint32_t client_id, int block, int role);
/* Drop every adapter of a client (deregister). */
SS_API int ss_clear_client(ss_ctx* ctx, uint32_t client_id);

/* Compute one batch for layer (block, role) and pass. `stream` is a cudaStream_t (NULL =
 * legacy default stream). Asynchronous: results are visible after the stream reaches this
 * point. seg_status[n_seg] receives per-segment status; rejected segments are not written.
 * A context's dispatches share one device workspace: a dispatch on a different stream than the
 * context's previous one is ordered after it (stream wait on its completion event). */
SS_API int ss_compute_batch(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg,
                     const ss_seg* segs, void* stream, int32_t* seg_status);

/* Same dispatch over HOST buffers (the reference's clients hold numpy activations, and the
 * LocalChannel reply lands in the client's SharedBuffer, transport.py:28-49, 73-98): src / dst /
 * dst_base are host pointers (page-locked for full PCIe speed). The batch is split into row
 * sub-batches; the H2D copy of sub-batch j+1, the kernels of j and the D2H copy of j-1 overlap
 * on the library's copy streams and a 4-slot device staging ring. Rows are independent and the
 * kernels never mix rows (tensor_ops.py:1-8), so the results are bitwise those of
 * ss_compute_batch on device copies. A dispatch of at most `zero_copy_bytes` payload bytes
 * (option, default 4 MiB: decode-size batches) over page-locked buffers makes no copies: the
 * kernels read the request rows and write the reply rows in host memory directly (UVA), one
 * launch sequence instead of two memcpy calls per segment. Synchronous: the replies are in the
 * host buffers when it returns. All segments must share one src dtype and one dst dtype. */
SS_API int ss_compute_batch_host(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg,
                                 const ss_seg* segs, void* stream, int32_t* seg_status);

/* ---- LSV1 wire frames ---------------------------------------------------------------------
 * The reference's byte-stream channel frames every tensor (protocol.py:6-25: 30-byte
 * little-endian header "LSV1", u16 version 1, u32 client_id, u64 request_id, u16 block, u8 role,
 * u8 pass, u32 token_count, u32 width, then token_count*width f32), decoding and re-encoding
 * payloads on the host (protocol.py:96-153, transport.py:104-275). ss_serve_frames serves a run
 * of request frames as received from a stream WITHOUT a host-side decode:
 *   - frames are parsed in place; each one goes through the executor's intake checks in order
 *     (unknown pass, non-increasing request_id per client, unknown layer: executor.py:162-178);
 *   - the run of frames is copied to the GPU as raw bytes in one transfer; the f32 payloads
 *     (behind 30-byte headers, so not 4-byte aligned) are decoded THERE into bf16 operand rows;
 *   - valid frames are grouped by (block, role, pass) in arrival order, one fused dispatch per
 *     group (FIFO inside it, executor.py:247-300), with the client's registered adapter fused;
 *   - the reply stream is encoded on the GPU — per frame in request order a complete LSV1 frame:
 *     the header echoing the request's ids and pass (executor.py:295-300) and the f32 payload,
 *     or a PASS_ERROR (255) frame with the reference's UTF-8 message (protocol.py:86-89) — and
 *     returned to `out` in one transfer.
 * *consumed = bytes of the whole frames parsed (a trailing partial frame stays for the next
 * call, like try_decode). Bad magic / version: SS_E_PROTOCOL, nothing served. If out_cap is
 * too small: SS_E_NOMEM with *out_len = the bytes needed, nothing served. */
SS_API int ss_serve_frames(ss_ctx* ctx, const uint8_t* in, size_t in_len, size_t* consumed,
                           uint8_t* out, size_t out_cap, size_t* out_len, void* stream);

/* ---- prebuilt dispatch plans ------------------------------------------------------------
 * For clients whose exchange buffers do not move (DeviceChannel after its first grow), the
 * routing tables of a dispatch (what ss_compute_batch rebuilds on every call: validation,
 * M-tiles, LoRA chunk lists, tensor maps) are built once into plan-owned device memory;
 * ss_plan_launch then only launches the kernels — a few microseconds of host time, and
 * capturable in a CUDA graph. Same semantics and bitwise the same results as
 * ss_compute_batch on the same segments. A plan rebuilds itself transparently when the
 * context's workspace grew or an adapter it references moved (rank change, clear, layer
 * reload); it fails (SS_E_ARG) if that changed a segment's status. Plans must be destroyed
 * before their context. */
typedef struct ss_plan ss_plan;
SS_API int ss_plan_create(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg,
                          const ss_seg* segs, int32_t* seg_status, ss_plan** out);
SS_API int ss_plan_launch(ss_plan* plan, void* stream);
SS_API int ss_plan_destroy(ss_plan* plan);

/* ---- adapter weight gradients (the client-side half of a fine-tune step) -----------------
 * The reference computes these in numpy on the client after every executor backward reply:
 *   ClientModel._layer_backward   pkg/src/splitserve/client.py:286-305
 *     IA3  grad_l += sum_rows(dy * y_base)                    client.py:291-293
 *     LoRA lora_backward(x_saved, g, A, B, alpha, rank)       adapters.py:26-41
 *          grad_a = s * x^T . (g . B^T),  grad_b = s * (x . A)^T . g,  s = alpha / rank
 *     accumulated into the grads dict (client.py _accumulate).
 * ss_adapter_grads computes them on the GPU for every listed client of one layer, using the
 * adapter registered with ss_set_adapter (its A, B, l). Activations are DEVICE pointers:
 * x [rows, d_in] and dy [rows, d_out] bf16 with 16-byte aligned rows for LoRA (TMA-loaded);
 * dy / y_base bf16 or f32 for IA3. Gradients are f32 device buffers, row-major like the
 * reference's arrays: grad_a [d_in, rank], grad_b [rank, d_out], grad_l [d_out]. Output
 * buffers of different segments must not overlap. A client with both LoRA and IA3 on one
 * layer is rejected (SS_SEG_UNSUPPORTED): a reference AdapterState has one method. */
#define SS_GRADF_ACCUMULATE (1u << 0) /* += into the gradient buffers (else overwrite) */
#define SS_GRADF_X_BF16 (1u << 1)
#define SS_GRADF_DY_BF16 (1u << 2)
#define SS_GRADF_BASE_BF16 (1u << 3)
#define SS_SEG_UNSUPPORTED 5

typedef struct ss_grad_seg {
  uint32_t client_id;
  uint32_t rows;
  uint32_t flags;        /* SS_GRADF_* */
  uint32_t reserved;
  const void* x;         /* LoRA: the layer's forward input (client-saved), [rows, x_ld] */
  int64_t x_ld;
  const void* dy;        /* grad of the layer output, [rows, dy_ld] */
  int64_t dy_ld;
  const void* y_base;    /* IA3: the pre-IA3 forward output, [rows, base_ld] */
  int64_t base_ld;
  float* grad_a;         /* LoRA [d_in, rank] */
  float* grad_b;         /* LoRA [rank, d_out] */
  float* grad_l;         /* IA3  [d_out] */
} ss_grad_seg;

SS_API int ss_adapter_grads(ss_ctx* ctx, int block, int role, int n_seg, const ss_grad_seg* segs,
                            void* stream, int32_t* seg_status);

/* Dims of a loaded layer (SS_E_NOLAYER if absent); device of a context. */
SS_API int ss_layer_dims(ss_ctx* ctx, int block, int role, int* d_in, int* d_out);
SS_API int ss_ctx_device(const ss_ctx* ctx);

/* ---- native scheduler: batch formation + dispatch off the Python interpreter --------------
 * The reference's executor forms batches in a scheduler thread: submit() validates and queues
 * an envelope per (block, role, pass) (executor.py:162-178), _loop/_pick_ready pick a ripe
 * queue under the BatchPolicy (executor.py:235-283: nolockstep = one request per dispatch;
 * lockstep = wait until every registered client -- every backward sender for backward --
 * has a request queued; opportunistic = dispatch when the queue holds max_batch_tokens, or
 * when its oldest member has waited min(wait_cap, wait_per_token * smallest member's tokens);
 * the noise pass is never batched), _dispatch computes it and replies (executor.py:285-300).
 * ss_sched_* runs exactly that loop on a native thread over DEVICE-resident requests: a client
 * thread's ss_sched_request() is one call that queues the request and blocks (without the
 * Python GIL: ctypes releases it) until the batch holding it has been launched, then makes the
 * client's stream wait for that batch's completion; the scheduler thread makes its stream wait
 * for each request's `ready` event, runs ss_compute_batch, and records one completion event per
 * batch. Validation mirrors submit(): unknown pass, non-increasing request_id per client,
 * unknown layer complete immediately with a request status (the width check is the batch's
 * per-segment status). Results are bitwise those of ss_compute_batch on the same batch. */
#define SS_SCHED_NOLOCKSTEP 0
#define SS_SCHED_LOCKSTEP 1
#define SS_SCHED_OPPORTUNISTIC 2
/* request status: SS_SEG_* (0 = computed) or */
#define SS_REQ_BAD_PASS 16    /* "unknown pass {pass}" executor.py:163-165 */
#define SS_REQ_BAD_ID 17      /* "request_id {id} not increasing (last {aux})" executor.py:166-171 */
#define SS_REQ_NO_LAYER 18    /* "unknown layer {layer}" executor.py:172-174 */
#define SS_REQ_FAILED 19      /* the batch's dispatch failed (ss_sched_last_error) */
typedef struct ss_sched_policy {
  int32_t mode;               /* SS_SCHED_* */
  int32_t reserved;
  double wait_per_token;      /* seconds */
  double wait_cap;            /* seconds */
  int64_t max_batch_tokens;
} ss_sched_policy;
typedef struct ss_request {
  uint32_t client_id;
  uint32_t pass_kind;
  int32_t block;
  int32_t role;
  uint64_t request_id;
  ss_seg seg;                 /* rows, width, flags, src / dst / dst_base (device); client_id unused */
  void* ready;                /* cudaEvent_t recorded after the payload was written, or NULL */
} ss_request;
typedef struct ss_sched_rec { /* one per request of a dispatched batch */
  uint64_t dispatch;          /* dispatch sequence number (requests of one batch share it) */
  int32_t block, role, pass_kind, rows;
  double wait_s;              /* queued -> batch picked */
} ss_sched_rec;
typedef struct ss_sched ss_sched;
SS_API int ss_sched_create(ss_ctx* ctx, const ss_sched_policy* policy, void* stream, ss_sched** out);
/* stops the thread after the queued requests are dispatched (drain != 0) or failed (drain == 0) */
SS_API int ss_sched_destroy(ss_sched* s, int drain);
SS_API int ss_sched_set_policy(ss_sched* s, const ss_sched_policy* policy);
SS_API int ss_sched_register(ss_sched* s, uint32_t client_id, int sends_backward);
SS_API int ss_sched_deregister(ss_sched* s, uint32_t client_id);
/* queue a request; notify != 0: its completion is also reported by ss_sched_next_done */
SS_API int ss_sched_submit(ss_sched* s, const ss_request* req, int notify, uint64_t* ticket);
/* block until `ticket` completed (timeout_us < 0: forever); on completion make `wait_stream`
 * wait for its batch (if not NULL; a client on the legacy default stream passes cudaStreamLegacy,
 * since NULL means "no stream"). Returns SS_OK, or SS_E_ARG (unknown ticket) / 1 (timeout). */
SS_API int ss_sched_wait(ss_sched* s, uint64_t ticket, void* wait_stream, int64_t timeout_us,
                         int32_t* status, int64_t* aux);
/* ss_sched_submit + ss_sched_wait in one call */
SS_API int ss_sched_request(ss_sched* s, const ss_request* req, void* wait_stream, int64_t timeout_us,
                            int32_t* status, int64_t* aux);
/* next completed notify-ticket in completion order (1 = timeout, nothing completed) */
SS_API int ss_sched_next_done(ss_sched* s, void* wait_stream, int64_t timeout_us, uint64_t* ticket,
                              int32_t* status, int64_t* aux);
/* move up to `cap` dispatch records out of the scheduler's log; *n = records returned */
SS_API int ss_sched_log(ss_sched* s, ss_sched_rec* out, int cap, int* n);
SS_API int64_t ss_sched_queued(ss_sched* s);
SS_API const char* ss_sched_last_error(ss_sched* s);

/* ---- cross-process device hand-off (CUDA IPC) ---------------------------------------------
 * The paper's co-located mode shares a pre-allocated CUDA exchange tensor between the client
 * process and the executor process (share_memory_() / rebuild_cuda_tensor());
 * the reference package's process mode (harness.py:243-260 _process_worker, :367-394
 * _run_processes) otherwise serialises every payload through host memory and a socket
 * (RemoteChannel / ExecutorServer, transport.py:104-275). With these calls a client process
 * exports its request / reply / y_base buffers once per grow (SharedBuffer's grow-only rule,
 * transport.py:28-49) and the executor process maps them; the segments of ss_compute_batch
 * then point straight into the client's memory (a client on another GPU: peer memory over
 * NVLink). Stream ordering between the processes uses interprocess events: the client records
 * one after writing a request, the executor's stream waits on it; the executor records its
 * own after the reply, the client's stream waits on that. No ss_ctx needed; errors of these
 * calls are reported by ss_ipc_last_error() (per thread). */
typedef struct ss_ipc_mem {
  uint8_t handle[64];   /* cudaIpcMemHandle_t of the allocation that holds the buffer */
  uint64_t offset;      /* byte offset of the buffer inside that allocation */
  uint64_t bytes;
  int32_t device;       /* CUDA device of the exporting process's allocation */
  uint32_t reserved;
} ss_ipc_mem;
typedef struct ss_ipc_evt {
  uint8_t handle[64];   /* cudaIpcEventHandle_t */
} ss_ipc_evt;
SS_API const char* ss_ipc_last_error(void);
/* client side: export any cudaMalloc'd range (e.g. a torch tensor's storage), or allocate a
 * dedicated exchange buffer and export it */
SS_API int ss_ipc_export(const void* dptr, uint64_t bytes, ss_ipc_mem* out);
SS_API int ss_ipc_alloc(int device, uint64_t bytes, void** dptr, ss_ipc_mem* out);
SS_API int ss_ipc_free(void* dptr);
/* executor side: map an exported buffer (one mapping per allocation per process, reference
 * counted: opening the same handle twice returns pointers into one mapping); close unmaps the
 * last reference. The caller must have ordered any work touching the buffer before close. */
SS_API int ss_ipc_open(int device, const ss_ipc_mem* mem, void** dptr);
SS_API int ss_ipc_close(void* dptr);
/* interprocess events (cudaEventInterprocess | cudaEventDisableTiming) */
SS_API int ss_ipc_event_create(int device, void** event, ss_ipc_evt* out);
SS_API int ss_ipc_event_open(int device, const ss_ipc_evt* h, void** event);
SS_API int ss_ipc_event_record(void* event, void* stream);
SS_API int ss_ipc_event_wait(void* stream, void* event);
SS_API int ss_ipc_event_sync(void* event);
SS_API int ss_ipc_event_destroy(void* event);

/* Device bytes held: weights (+bias), adapter packs, transient workspace high-water mark. */
SS_API int ss_memory_stats(const ss_ctx* ctx, int64_t* weight_bytes, int64_t* adapter_bytes,
                    int64_t* workspace_bytes);

/* Number of kernels launched by this context since creation (evidence / bench counter). */
SS_API int64_t ss_kernel_launches(const ss_ctx* ctx);

/* Monotonic counter that moves whenever the context frees or moves a device buffer that
 * launched kernels reference (workspace growth, LoRA pack growth, adapter rank / kind / scale
 * change, layer unload). Kernels captured into a CUDA graph bake those addresses: a graph
 * captured at epoch E must not be replayed once ss_ctx_epoch() != E (re-capture instead;
 * GpuBaseExecutor.capture does this automatically). Plans rebuild themselves on launch. */
SS_API uint64_t ss_ctx_epoch(const ss_ctx* ctx);

/* In-stream kernel timing (bench evidence): while enabled, every launch of kind
 * SS_KERNEL_{GATHER,SHRINK,GEMM} is bracketed by CUDA events on its own stream, and its
 * algorithmic FLOPs / bytes are accumulated. ss_profile_read synchronizes the recorded events
 * and returns totals since the last ss_profile(ctx, 1). */
#define SS_KERNEL_GATHER 0
#define SS_KERNEL_SHRINK 1
#define SS_KERNEL_GEMM 2
#define SS_KERNEL_GRAD 3   /* K6 + K7 (+ their K3 shrinks) of ss_adapter_grads */
SS_API int ss_profile(ss_ctx* ctx, int enable);
SS_API int ss_profile_read(ss_ctx* ctx, int kernel, double* total_ms, int64_t* launches,
                           double* flops, double* bytes);

/* Numerics class of a request (a property of the request alone, so batching stays invisible):
 *   decode_rows (16)    segments of at most this many rows (0..16; layers with K % 64 == 0) are
 *                       "decode class": their rows reduce K as C = ceil(K / (64 * decode_chunk_kb))
 *                       fixed contiguous chunks summed left to right in chunk order (split-K
 *                       kernel K1d + fixup), then their own LoRA chain; every other row reduces K
 *                       as one chain. 0: no decode class (every row single-chain).
 *   decode_chunk_kb (20) 64-deep k-blocks per chunk of the decode class's order (1..48)
 *   host_convert (1)    ss_compute_batch_host: pageable f32 request rows are converted to bf16 by
 *                       host threads into a page-locked ring, one DMA per sub-batch (results
 *                       unchanged: the same rounding as the device gather; not for backward
 *                       IA3 rows)
 *   host_threads (0)    threads of that conversion (0: min(16, hardware threads))
 *   decode_lora_piece (24) rank chunks (16 rows, hi and lo counted) per LoRA piece of a decode tile:
 *                       pieces are whole segments, each one chain and one unit per column tile
 *                       (results unchanged: a row's LoRA chain is its own segment's)
 *   decode_prologue (1) decode-only dispatch with decode-class LoRA rows: their shrink and the
 *                       row gather in one launch (else a side-stream shrink beside the gather;
 *                       results unchanged)
 *   group_m_longk (0)   M-grouped raster group size of dispatches with K >= longk (0: group_m)
 *   longk (8192)        the K from which group_m_longk applies
 *   tail_split (1)      CTA-pair 256 x 512 dispatches whose last wave is under half full: the last
 *                       (partial + one full) wave of tiles runs as 256 x 256 tiles in a second,
 *                       programmatically launched kernel (results unchanged)
 *   decode_fixup_fused (0) decode class: the ordered chunk fold + epilogue run inside the GEMM
 *                       launch (each CTA once its groups are done, behind per-tile completion
 *                       counters) instead of a separate fixup launch (bitwise the same fold;
 *                       measured 9.26 vs 8.69 ms per 13B decode step: the fixup launch folds with
 *                       far more threads in flight)
 *   decode_split (0)    decode-only dispatch with a side-stream shrink: the decode-class GEMM's
 *                       chunk groups launch behind the gather, beside the shrink; its LoRA groups
 *                       after the join (results unchanged; measured 9.84 vs 9.29 ms per 13B decode step)
 *   grad_fused (0)      ss_adapter_grads: LoRA shrinks + token contractions in one launch, client
 *                       by client (x / g re-read from L2); 0: two launches (bitwise the same)
 *   grad_fused_lag (2)  clients between a client's shrinks and its contractions (fused path)
 *   decode_trace (0)    testing: device address of an int64 buffer [4 x SMs] the decode-class
 *                       kernel fills with {start ns, end ns, first unit, end unit} per CTA
 * Tuning / testing knobs (none changes results: every kernel choice gives bitwise the same rows).
 *   group_m (16)        M-tiles per raster group of the persistent GEMM
 *   raster (0)          0 M-grouped, 1 N-grouped (W columns held in L2), -1 fewer modelled bytes
 *   group_n, l2_budget_mb (0, 48)  N-group width (0: as many W columns as fit the budget)
 *   l2_hints (1)        L2 evict_last on the operand a raster group re-reads, evict_first on outputs
 *   gemm_2cta (-1)      CTA-pair kernel: -1 by dispatch size, 1 / 0 forced
 *   pair_n (0)          CTA-pair tile width 256 (double-buffered TMEM) or 512 (12 warps); 0 auto
 *   side_shrink (1)     a LoRA shrink that reads no packed rows runs on a side stream beside the gather
 *   lora_overlap (0)    the weight-streaming kernel runs beside that shrink and spins on its
 *                       completion counter only before its LoRA k-blocks (when both fit the SMs).
 *                       Opt-in: only safe when no other work on the GPU can keep the shrink's
 *                       CTAs from being scheduled (the executor owns the GPU); ignored under
 *                       tools that serialise launches (CUDA_INJECTION64_PATH, i.e. ncu /
 *                       compute-sanitizer, or CUDA_LAUNCH_BLOCKING=1)
 *   cluster4 (0)        256x256 pair tiles as 4-CTA clusters sharing B by multicast (measured
 *                       35 % slower in the step: off)
 *   tile_n (0)          force the single-CTA tile width 64 / 128 / 256 (0 auto)
 *   direct_tiles (1)    TMA-load whole tiles of bf16 segments in place (else gather everything)
 *   tma_store (1)       bf16 outputs through swizzled smem + TMA bulk stores
 *   stream_gemm (1)     weight-streaming kernel for dispatches of <= 64 rows (K % 64 == 0)
 *   a_rows64 (1)        64-row A box for such dispatches in the single-CTA kernel
 *   shrink_mode (0)     LoRA shrink: 0 auto, 1 one CTA per slab, 2 one CTA per (slab, K chunk)
 *   shrink_kb_chunk     k-blocks (of 64) per fixed K chunk of the shrink
 *   lora_hilo (2)       LoRA intermediate s*x.A as a hi / lo bf16 pair read against the same B rows
 *                       (fp32-output precision): 0 never, 1 f32-destination segments, 2 all
 *   ia3_lo (1)          IA3 backward operand g = dy*l as hi + lo with a second K pass over lo:
 *                       0 never, 1 f32-destination segments, 2 all IA3 backward segments
 *   pdl (0)             programmatic dependent launch between a dispatch's kernels (no gain measured)
 *   wide_decode (1)     dispatches of <= 64 rows whose 64-wide tiles would need more than one wave
 *                       but whose 128-wide tiles fit one run the single-CTA kernel with 128-wide tiles
 *   stream_pdl (1)      the weight-streaming GEMM is launched with programmatic dependent launch
 *                       behind the gather: its first W stages stream before griddepcontrol.wait
 *   zc_cache (1)        zero-copy host dispatches that recur with the same segment array reuse their
 *                       built routing tables (invalidated by workspace growth, adapter moves, any
 *                       option change)
 *   zero_copy_bytes (4 MiB)  ss_compute_batch_host dispatches up to this size: no copies (UVA)
 *   force_remote (0)    testing: route every segment as if it lived on a peer GPU
 *   pipeline_rows, pipeline_bytes  sub-batch size of ss_compute_batch_host */
SS_API int ss_set_option(ss_ctx* ctx, const char* key, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* SS_B200_H */
