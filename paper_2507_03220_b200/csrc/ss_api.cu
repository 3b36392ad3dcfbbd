// Host side of the C ABI declared in include/ss_b200.h.
//
// Owns: bf16 copies of the frozen layers (+ f32 bias), per-layer LoRA packs (A^T and B rows of
// every registered client, 16-row aligned), IA3 vectors, and a grow-only transient workspace
// (the concatenated operand X, the block-diagonal LoRA operand, routing tables). Everything
// the reference keeps per request (executor.py:191-231) is rebuilt per dispatch; nothing
// survives a dispatch except weights and adapters (statelessness, executor.py:1-9).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ss_b200.h"
#include "kernels.cuh"
#include "decode.cuh"
#include "grads.cuh"
#include "frames.cuh"

using namespace ss;

namespace {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int kStagingSlots = 16;

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct AdapterSlot {
  uint32_t kind = 0;
  int rank = 0, rank_pad = 0, pack_row = -1;
  float scale = 0.f;
  float* ia3 = nullptr;  // device [d_out]
};

struct Layer {
  int block = 0, role = 0, d_in = 0, d_out = 0;
  __nv_bfloat16* W = nullptr;
  int64_t ldw = 0;
  float* bias = nullptr;
  CUtensorMap tm_w_fwd, tm_w_bwd, tm_w_bwd2, tm_w_bwd64;  // bwd box rows 256 / 128 / 64
  CUtensorMap tm_w_fwd_s, tm_w_bwd_s;                      // weight-streaming kernel
  CUtensorMap tm_w_dec;                                    // split-K decode kernel (K1d): {64, 64} boxes
  // LoRA packs: rows = rank index of every registered client (16-aligned blocks)
  __nv_bfloat16* at_pack = nullptr;  // [cap, ld_at]  (A^T: rank rows x d_in)
  __nv_bfloat16* b_pack = nullptr;   // [cap, ld_b]   (B:   rank rows x d_out)
  int64_t ld_at = 0, ld_b = 0;
  int pack_rows = 0, pack_cap = 0;
  CUtensorMap tm_at, tm_b;
  CUtensorMap tm_at64, tm_b64;   // same packs, {64, 64-row} boxes (decode-class LoRA stages)
  std::map<uint32_t, AdapterSlot> adapters;
};

struct ProfRec {
  cudaEvent_t a, b;
  int kind;
  double flops, bytes;
};

struct Staging {
  void* host = nullptr;     // pinned
  void* dev = nullptr;      // device copy of the tables
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
};

}  // namespace

namespace { struct ZcPlan; }
// Host worker threads for the host side of a dispatch (f32 -> bf16 payload conversion into
// page-locked staging, ss_compute_batch_host): run(T, fn) runs fn(0 .. T-1) over the workers and
// the calling thread and returns when every task is done.
class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void run(int tasks, const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      tasks_ = tasks;
      next_.store(0);
      pending_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (int t; (t = next_.fetch_add(1)) < tasks_;) (*fn_)(t);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> l(m_);
      cv_.wait(l, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      l.unlock();
      work();
      l.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int tasks_ = 0, pending_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct ss_ctx {
  int device = 0, tp_rank = 0, tp_size = 1, num_sms = 148;
  // Every entry point that reads or changes the context holds this (re-entrant: entry points
  // call each other): the native scheduler thread (ss_sched_*) dispatches while client threads
  // refresh adapters, and pack growth frees what a concurrent table build would read.
  std::recursive_mutex mu;
  std::string err;
  PFN_encodeTiled_t encode = nullptr;
  std::map<std::pair<int, int>, Layer> layers;
  std::map<uint32_t, uint64_t> last_request_id;  // LSV1 intake (executor.py:164-169)
  // LSV1 serving: device copies of the request / reply streams, decoded operand, f32 replies
  char* fr_in = nullptr;
  char* fr_out = nullptr;
  char* fr_x = nullptr;
  char* fr_o = nullptr;
  size_t fr_in_cap = 0, fr_out_cap = 0, fr_x_cap = 0, fr_o_cap = 0;
  // workspace
  __nv_bfloat16* X = nullptr;
  size_t x_cap = 0;
  __nv_bfloat16* X_lo = nullptr;   // lo halves of IA3-backward operands (SEGF_IA3_LO)
  size_t xlo_cap = 0;
  __nv_bfloat16* a_lora = nullptr;
  size_t al_cap = 0;
  int32_t* row_seg = nullptr;
  size_t rs_cap = 0;
  size_t ws_high = 0;
  Staging staging[kStagingSlots];
  int slot = 0;
  cudaStream_t upload = nullptr;
  // host-buffer dispatches (ss_compute_batch_host): copy streams + a device staging ring
  cudaStream_t h2d = nullptr, d2h = nullptr;
  // side stream for a LoRA shrink that does not depend on the gather (fork / join events)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int side_shrink = 1;
  // 0 by default: the overlapped streaming GEMM spins on a counter the side-stream shrink
  // writes, which is only safe when nothing else can keep the shrink's CTAs off the SMs (the
  // executor owns the GPU). Opt in with ss_set_option("lora_overlap", 1).
  int lora_overlap = 0;
  int serial_launches = 0;       // a tool serialises kernel launches (ncu, sanitizer): no overlap
  int stream_pdl = 1;
  int wide_decode = 1;           // decode-size dispatches: 128-wide single-CTA tiles when they fit one wave
  // segments of <= decode_rows rows reduce K in the decode class's split-K order (K1d, decode.cuh)
  int decode_rows = 16;
  int decode_chunk_kb = 20;          // 64-deep k-blocks per K chunk of the decode class (numerics!)
  long long* decode_trace = nullptr; // testing: K1d per-CTA timings (device buffer, 4 x int64 per CTA)
  int* sync_ctr = nullptr;       // [2] shrink-done counter + GEMM ticket (zero between dispatches)
  struct HostSlot {
    void* in = nullptr;
    void* out = nullptr;
    void* base = nullptr;
    size_t in_cap = 0, out_cap = 0, base_cap = 0;
    cudaEvent_t ev_in = nullptr, ev_comp = nullptr, ev_out = nullptr;
    bool used = false;
  } hslot[4];
  // pageable f32 request rows (numpy clients): converted to bf16 on the host by `pool` into a
  // page-locked ring, then one DMA per sub-batch (half the PCIe bytes, no driver staging)
  struct HostConv {
    uint16_t* buf = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool used = false;
  } hconv[4];
  int host_convert = 1;
  int host_threads = 0;            // 0: min(16, hardware threads)
  std::unique_ptr<HostPool> pool;
  int64_t pipeline_bytes = 24 << 20;  // target bytes of the wider side per sub-batch
  int pipeline_rows = 4096;
  cudaEvent_t upload_done = nullptr, compute_done = nullptr;
  cudaStream_t last_stream = nullptr;   // stream of the previous dispatch (cross-stream ordering)
  bool done_captured = false;           // compute_done was last recorded inside a graph capture
  bool any_compute = false;
  int64_t launches = 0;
  int group_m = 16;
  int group_m_longk = 0;     // > 0: group_m of dispatches with K >= longk (0: group_m)
  int longk = 8192;
  // GEMM tile raster: 0 M-grouped (group_m M-tiles per group), 1 N-grouped (W columns of a group
  // held in L2 while A streams), -1 auto: the order with fewer estimated DRAM bytes, where an
  // N group is as many W column tiles as fit `l2_budget_mb`. group_n > 0 forces the group width.
  int raster = 0;
  int group_n = 0;
  // whole-dispatch device slices + per-sub-batch events of the aliased host dispatch
  void* ha_in = nullptr;
  void* ha_out = nullptr;
  void* ha_base = nullptr;
  size_t ha_in_cap = 0, ha_out_cap = 0, ha_base_cap = 0;
  std::vector<cudaEvent_t> chunk_ev;
  uint64_t peers_enabled = 0;  // peer GPUs whose memory this context's kernels may touch
  int64_t zero_copy_bytes = 4 << 20;  // host dispatches up to this many payload bytes: zero-copy
  int force_remote = 0;      // testing: route every segment as if it lived on a peer GPU
  int cluster4 = 0;          // 256 x 256 pair tiles as clusters of two pairs sharing B (multicast)
  int pdl = 0;               // programmatic dependent launch between a dispatch's kernels (measured: no gain)
  int stream_gemm = 1;       // weight-streaming kernel for those dispatches (K % 64 == 0)
  int a_rows64 = 1;          // 64-row A box for single-tile dispatches of <= 64 rows
  int l2_budget_mb = 48;
  // 1: L2 evict_last on the operand a raster group re-reads (A rows in M order, W columns in N
  // order) and evict_first on the outputs (written once, never re-read by this launch)
  int l2_hints = 1;
  // -1 auto: CTA-pair kernel whenever the dispatch has at least half an SM-pair wave of
  // 256 x 256 tiles, else the single-CTA kernel with 256/128/64-wide tiles. (Round-1 v1 used the
  // single-CTA kernel for K > 8192; with the current epilogue the pair wins there too: 13B step
  // 699 vs 713 ms, profiles/r01_gemm_variants.md.) 1 / 0 force one kernel.
  int gemm_2cta = -1;
  int direct_tiles = 1;  // 1: TMA-load whole tiles of bf16 segments in place (no gather)
  int force_tbn = 0;     // testing: force the single-CTA tile width (64 / 128 / 256)
  int tma_store = 1;     // 1: bf16 outputs leave through swizzled smem + TMA bulk stores
  // CTA-pair tile width: 256 (double-buffered TMEM) or 512 (one accumulator, 12 warps; 25 %
  // fewer operand bytes per FLOP: less L2 traffic, less power, higher clock on the power-capped
  // part: 13B step 784-789 -> 767-770 ms); 0 = 512 when the dispatch has >= 2 waves of 256x512
  // pair tiles, else 256
  int pair_n = 0;
  int shrink_kb_chunk = SHRINK_KB_CHUNK;  // K-split of the LoRA shrink (k-blocks of 64 per chunk)
  int shrink_mode = 0;   // 0 auto, 1 one CTA per slab (all chunks), 2 one CTA per (slab, chunk)
  int* grad_sync = nullptr;       // fused adapter-gradient kernel: ticket + per-client counters
  size_t grad_sync_cap = 0;
  int grad_fused = 0;             // ss_adapter_grads: K3 + K6 in one launch (grads.cuh; measured slower)
  int grad_fused_lag = 2;         // clients between a client's shrinks and its contractions
  int* dec_claim = nullptr;       // K1d group tickets: [0..1] main launch, [2..3] LoRA launch
  float* dshr_part = nullptr;     // decode shrink: fp32 chunk partials
  size_t dshr_part_cap = 0;
  int* dshr_ticket = nullptr;     // decode shrink: per-item arrival counters (zero between launches)
  size_t dshr_ticket_cap = 0;
  int decode_lora_piece = DEC_LP_CHUNKS;   // max 16-row rank chunks per decode LoRA piece (tuning)
  int tail_split = 1;               // CTA-pair 512 dispatches: an under-half-full last wave runs as 256-wide tiles (second launch)
  int decode_fixup_fused = 0;       // decode class: chunk fold + epilogue inside K1d (whole CTA after its groups), no fixup launch (measured slower)
  int* dec_fx = nullptr;            // [0] fixup-unit ticket, then per (tile, n tile, half) group counters
  size_t dec_fx_cap = 0;
  int decode_prologue = 1;          // decode-only dispatch: decode shrink + gather in one launch
  int decode_split = 0;           // K1d chunk groups beside the side-stream shrink, LoRA groups after (slower)
  float* dec_part = nullptr;      // K1d: fp32 chunk partials of the decode tiles
  size_t dec_part_cap = 0;
  // LoRA intermediate s*x.A as a hi / lo bf16 pair (ShrinkItem::hilo): 0 never, 1 segments with
  // f32 destinations, 2 every segment. A per-segment property, so batching stays invisible.
  int lora_hilo = 2;
  // IA3 backward operand g = dy*l as hi + lo with a second K pass over lo (SEGF_IA3_LO):
  // 0 never, 1 segments with f32 destinations (default; bf16 outputs round far coarser than
  // the operand), 2 every IA3 backward segment
  int ia3_lo = 1;
  int64_t weight_bytes = 0, adapter_bytes = 0;
  // Plans (ss_plan_*) cache routing tables that embed workspace and adapter pointers; these
  // counters tell a plan to rebuild itself after the workspace grew or an adapter moved.
  uint64_t ws_epoch = 0, ad_epoch = 0;
  // bumped whenever ANY device buffer a launched kernel may reference is freed or replaced
  // (workspace incl. the shrink partials, packs, IA3 vectors): a CUDA graph captured before
  // must not be replayed (ss_ctx_epoch; GpuBaseExecutor.capture re-captures)
  uint64_t free_epoch = 0;
  uint64_t zc_swept = 0;         // ws + ad + opt epoch at the last stale-entry sweep of zc_cache
  // zero-copy host dispatches that recur (decode: clients reuse their buffers every step) reuse
  // their routing tables: keyed by the segment array's bytes, valid while the epochs, the
  // options and the reply slot are unchanged (see ss_compute_batch_host)
  std::map<uint64_t, ZcPlan*> zc_cache;
  int zc_cache_on = 1;
  uint64_t opt_epoch = 0;        // bumped by every ss_set_option: cached tables depend on options
  // in-stream profiling
  bool profiling = false;
  std::vector<ProfRec> prof;       // pending event pairs
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[4] = {0, 0, 0, 0}, prof_flops[4] = {0, 0, 0, 0}, prof_bytes[4] = {0, 0, 0, 0};
  int64_t prof_n[4] = {0, 0, 0, 0};
  // adapter-gradient workspace: s*x.A and s*g.B^T per segment (Qx, Qg)
  __nv_bfloat16* qx = nullptr;   // [s*x.A ; s*g.B^T]
  size_t qx_cap = 0;
  char* ia3_part = nullptr;       // IA3 grad_l chunk sums
  size_t ia3_part_cap = 0;
  float* shrink_part = nullptr;   // K-split shrink: fp32 chunk partials
  size_t shrink_part_cap = 0;
  int* shrink_ticket = nullptr;   // per shrink item arrival counters (zero between launches)
  size_t shrink_ticket_cap = 0;
};

namespace {

int fail(ss_ctx* c, int code, const char* fmt, ...) {
  if (c) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, SS_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                   \
  } while (0)

int encode_2d(ss_ctx* ctx, CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
              uint64_t ld_elems, uint32_t box_cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, SS_E_CUDA, "cuTensorMapEncodeTiled failed (%d) cols=%llu rows=%llu ld=%llu",
                (int)r, (unsigned long long)cols, (unsigned long long)rows,
                (unsigned long long)ld_elems);
  return SS_OK;
}

// K-major operand [rows, cols] (row stride ld_elems, cols a multiple of 64 within ld) viewed as
// {64 k, rows, cols / 64 chunks}: one box of {64, box_rows, box_chunks} loads several 64-wide
// K chunks of box_rows rows in a single TMA operation, chunk c landing box_rows * 128 B after
// chunk c - 1 (the 128B-swizzled K-major layout of each chunk is unchanged).
int encode_kchunks(ss_ctx* ctx, CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                   uint64_t ld_elems, uint32_t box_rows, uint32_t box_chunks) {
  cuuint64_t dims[3] = {64, rows, (cols + 63) / 64};
  cuuint64_t strides[2] = {ld_elems * 2, 128};
  cuuint32_t box[3] = {64, box_rows, box_chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, SS_E_CUDA, "cuTensorMapEncodeTiled (3-D) failed (%d) cols=%llu rows=%llu ld=%llu",
                (int)r, (unsigned long long)cols, (unsigned long long)rows, (unsigned long long)ld_elems);
  return SS_OK;
}

// Copy a [rows, cols] matrix (host/device, f32/bf16, row stride src_ld) into a bf16 device
// destination, optionally transposed. Synchronous with respect to the source buffer.
int upload_bf16(ss_ctx* ctx, const void* src, uint32_t flags, int rows, int cols, int64_t src_ld,
                __nv_bfloat16* dst, int64_t dst_ld, bool transpose) {
  const bool src_bf16 = flags & SS_DT_BF16;
  const size_t esz = src_bf16 ? 2 : 4;
  const void* dsrc = src;
  void* tmp = nullptr;
  if (!(flags & SS_MEM_DEVICE)) {
    const size_t bytes = (size_t)rows * src_ld * esz;
    CK(cudaMallocAsync(&tmp, std::max<size_t>(bytes, 16), ctx->upload));
    CK(cudaMemcpyAsync(tmp, src, bytes, cudaMemcpyHostToDevice, ctx->upload));
    dsrc = tmp;
  }
  const int64_t total = (int64_t)rows * cols;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (total > 0) {
    if (transpose)
      transpose_to_bf16_kernel<<<grid, 256, 0, ctx->upload>>>(dsrc, src_bf16, src_ld, dst, dst_ld,
                                                              rows, cols);
    else
      copy_to_bf16_kernel<<<grid, 256, 0, ctx->upload>>>(dsrc, src_bf16, src_ld, dst, dst_ld, rows,
                                                         cols);
    CK(cudaGetLastError());
  }
  if (tmp) CK(cudaFreeAsync(tmp, ctx->upload));
  CK(cudaStreamSynchronize(ctx->upload));
  return SS_OK;
}

int upload_f32(ss_ctx* ctx, const void* src, uint32_t flags, int n, float* dst) {
  const bool src_bf16 = flags & SS_DT_BF16;
  const size_t bytes = (size_t)n * (src_bf16 ? 2 : 4);
  if (!(flags & SS_MEM_DEVICE) && !src_bf16) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->upload));
  } else {
    const void* dsrc = src;
    void* tmp = nullptr;
    if (!(flags & SS_MEM_DEVICE)) {
      CK(cudaMallocAsync(&tmp, std::max<size_t>(bytes, 16), ctx->upload));
      CK(cudaMemcpyAsync(tmp, src, bytes, cudaMemcpyHostToDevice, ctx->upload));
      dsrc = tmp;
    }
    copy_to_f32_kernel<<<std::max(1, std::min((n + 255) / 256, 1024)), 256, 0, ctx->upload>>>(
        dsrc, src_bf16, dst, n);
    CK(cudaGetLastError());
    if (tmp) CK(cudaFreeAsync(tmp, ctx->upload));
  }
  CK(cudaStreamSynchronize(ctx->upload));
  return SS_OK;
}

// Uploads must not overwrite packs that an in-flight dispatch still reads.
int upload_begin(ss_ctx* ctx) {
  if (ctx->any_compute) CK(cudaStreamWaitEvent(ctx->upload, ctx->compute_done, 0));
  return SS_OK;
}
int upload_end(ss_ctx* ctx) {
  CK(cudaEventRecord(ctx->upload_done, ctx->upload));
  return SS_OK;
}

int grow_packs(ss_ctx* ctx, Layer& L, int need_rows) {
  if (need_rows <= L.pack_cap) return SS_OK;
  int cap = std::max(64, L.pack_cap);
  while (cap < need_rows) cap *= 2;
  __nv_bfloat16 *at = nullptr, *b = nullptr;
  CK(cudaMalloc(&at, (size_t)cap * L.ld_at * 2));
  CK(cudaMalloc(&b, (size_t)cap * L.ld_b * 2));
  CK(cudaMemsetAsync(at, 0, (size_t)cap * L.ld_at * 2, ctx->upload));
  CK(cudaMemsetAsync(b, 0, (size_t)cap * L.ld_b * 2, ctx->upload));
  if (L.pack_rows > 0) {
    CK(cudaMemcpyAsync(at, L.at_pack, (size_t)L.pack_rows * L.ld_at * 2, cudaMemcpyDeviceToDevice,
                       ctx->upload));
    CK(cudaMemcpyAsync(b, L.b_pack, (size_t)L.pack_rows * L.ld_b * 2, cudaMemcpyDeviceToDevice,
                       ctx->upload));
  }
  CK(cudaStreamSynchronize(ctx->upload));
  if (L.at_pack) {
    CK(cudaFree(L.at_pack));
    CK(cudaFree(L.b_pack));
    ctx->free_epoch++;
    ctx->adapter_bytes -= (int64_t)L.pack_cap * (L.ld_at + L.ld_b) * 2;
  }
  L.at_pack = at;
  L.b_pack = b;
  L.pack_cap = cap;
  ctx->adapter_bytes += (int64_t)cap * (L.ld_at + L.ld_b) * 2;
  int rc = encode_2d(ctx, &L.tm_at, L.at_pack, L.d_in, cap, L.ld_at, 64, LORA_CHUNK);
  if (rc) return rc;
  if ((rc = encode_2d(ctx, &L.tm_at64, L.at_pack, L.d_in, cap, L.ld_at, 64, 64))) return rc;
  if ((rc = encode_2d(ctx, &L.tm_b64, L.b_pack, L.d_out, cap, L.ld_b, 64, 64))) return rc;
  return encode_2d(ctx, &L.tm_b, L.b_pack, L.d_out, cap, L.ld_b, 64, LORA_CHUNK);
}

// Grow-only device workspace. `plan_visible`: prebuilt plans embed this buffer's address (X,
// LoRA operand, row_seg), so growing it must tell them to rebuild.
template <typename T>
int ensure_dev(ss_ctx* ctx, T*& ptr, size_t& cap, size_t bytes, bool plan_visible = true) {
  if (bytes <= cap) return SS_OK;
  if (plan_visible) ctx->ws_epoch++;
  size_t n = std::max(bytes, cap + cap / 2);
  n = round_up((int64_t)n, 1 << 20);
  if (ptr) {
    CK(cudaFree(ptr));
    ctx->free_epoch++;
  }
  ptr = nullptr;
  cap = 0;
  CK(cudaMalloc(reinterpret_cast<void**>(&ptr), n));
  cap = n;
  return SS_OK;
}

// True when `p` is device memory of another GPU (a client on a peer GPU, reached over NVLink):
// such segments are read by the gather kernel and written by plain stores (UVA peer access),
// never through TMA tensor maps.
bool is_remote(ss_ctx* ctx, const void* p) {
  if (!p) return false;
  if (ctx->force_remote) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // pinned host memory (UVA-mapped): the kernels read / write it over PCIe with plain loads and
  // stores (the zero-copy path of small host dispatches)
  if (a.type == cudaMemoryTypeHost) return true;
  if (a.type != cudaMemoryTypeDevice || a.device == ctx->device) return false;
  if (a.device >= 0 && a.device < 64 && !(ctx->peers_enabled >> a.device & 1)) {
    // first segment from this peer: map its memory into this GPU's address space (NVLink)
    cudaSetDevice(ctx->device);
    const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
    if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) ctx->peers_enabled |= 1ull << a.device;
    cudaGetLastError();
  }
  return true;
}

bool aligned16(const void* p, int64_t ld, size_t esz) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * (int64_t)esz) % 16 == 0);
}

cudaEvent_t pool_event(ss_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Bracket one launch: returns the index of the record (or -1 when not profiling).
bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

int prof_begin(ss_ctx* ctx, cudaStream_t st, int kind, double flops, double bytes) {
  if (!ctx->profiling || capturing(st)) return -1;
  ProfRec r{pool_event(ctx), pool_event(ctx), kind, flops, bytes};
  cudaEventRecord(r.a, st);
  ctx->prof.push_back(r);
  return (int)ctx->prof.size() - 1;
}
void prof_end(ss_ctx* ctx, cudaStream_t st, int idx) {
  if (idx >= 0) cudaEventRecord(ctx->prof[idx].b, st);
}
void prof_drain(ss_ctx* ctx) {
  for (auto& r : ctx->prof) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    ctx->prof_ms[r.kind] += ms;
    ctx->prof_flops[r.kind] += r.flops;
    ctx->prof_bytes[r.kind] += r.bytes;
    ctx->prof_n[r.kind] += 1;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->prof.clear();
}

// Workspace of a K-split shrink launch over `n_items` slabs (kernels.cuh, SHRINK_KB_CHUNK).
// Tickets must be zero when a launch starts: fresh ones are cleared, the kernel resets its own.
int ensure_shrink_ws(ss_ctx* ctx, size_t n_items, int max_chunks, int part_ld) {
  int rc = ensure_dev(ctx, ctx->shrink_part, ctx->shrink_part_cap,
                      std::max<size_t>(1, n_items * (size_t)max_chunks * BM * part_ld) * sizeof(float), false);
  if (rc) return rc;
  if (ctx->shrink_ticket_cap < n_items * sizeof(int)) {
    rc = ensure_dev(ctx, ctx->shrink_ticket, ctx->shrink_ticket_cap, n_items * sizeof(int), false);
    if (rc) return rc;
    CK(cudaMemset(ctx->shrink_ticket, 0, ctx->shrink_ticket_cap));
  }
  return SS_OK;
}

// Next pinned-host + device staging slot for a dispatch's routing tables (ring of
// kStagingSlots; a slot is reused only after the dispatch that last used it has copied it).
int acquire_staging(ss_ctx* ctx, size_t total, Staging*& out) {
  Staging& st = ctx->staging[ctx->slot];
  ctx->slot = (ctx->slot + 1) % kStagingSlots;
  if (st.pending) CK(cudaEventSynchronize(st.done));
  if (st.cap < total) {
    if (st.host) CK(cudaFreeHost(st.host));
    if (st.dev) CK(cudaFree(st.dev));
    st.host = nullptr;
    st.dev = nullptr;
    st.cap = 0;
    const size_t cap = round_up((int64_t)std::max(total, (size_t)1 << 16), 1 << 16);
    CK(cudaMallocHost(&st.host, cap));
    CK(cudaMalloc(&st.dev, cap));
    st.cap = cap;
  }
  out = &st;
  return SS_OK;
}

// Everything ss_compute_batch derives from the segment list alone: validation (per-segment
// status), the M-tile list (direct / packed), LoRA rank-chunk lists and shrink items, TMA-store
// ops, tensor maps — serialised into one blob of device tables — plus the launch shapes.
struct Built {
  int pass_kind = 0, block = 0, role = 0, K = 0, N = 0;
  int64_t M = 0, MX = 0, lora_ld = 64, al_rows = 0, ldx = 0;
  bool any_lora = false, pair = false, a_rows64 = false, stream = false;
  bool shrink_indep = false;   // the shrink reads no packed rows: it may run beside the gather
  bool any_lo = false;         // some segment is SEGF_IA3_LO (X_lo written, tiles run two passes)
  int tbn = BN, pn = 256, num_m = 0, n_piece = 0, n_items = 0, part_ld = 16, shrink_chunks_ = 1;
  int kb_chunk = SHRINK_KB_CHUNK;
  size_t off_tm = 0, off_seg = 0, off_tile = 0, off_piece = 0, off_ch = 0, off_st = 0, off_it = 0;
  // decode-class part (K1d): tiles, LoRA runs, X / X_lo tensor maps, cluster size
  size_t off_dt = 0;
  size_t off_dcb = 0, off_lp = 0, off_ls = 0, off_di = 0;   // K1d work groups, LoRA pieces / stages, decode shrink items
  int n_ditems = 0, dec_rank_max = 0, dec_rows_max = 0;
  int dec_S = 0;
  int n_dec = 0, dec_C = 0, dec_kbc = 0, dec_chunk_groups = 0, dec_groups = 0;
  int32_t dec_amap = 0, dec_alo = 0;
  int64_t Mp = 0;                      // single-chain rows (M - decode-class rows)
  double dec_flops = 0, dec_bytes = 0;
  std::vector<char> blob;
  std::vector<int32_t> status;
  double gather_bytes = 0, shrink_flops = 0, shrink_bytes = 0, gemm_flops = 0, gemm_bytes = 0;
  uint64_t ws_epoch = 0, ad_epoch = 0;
};

// A cached zero-copy dispatch: its built tables and row-copy ops in plan-owned device memory.
struct ZcPlan {
  int pass_kind = 0, block = 0, role = 0;
  std::vector<ss_seg> segs;
  std::vector<int32_t> status;
  Built b;
  uint64_t opt_epoch = 0;
  void* out = nullptr;
  void* base = nullptr;
  char* dev = nullptr;
  size_t ops_off = 0;
  int n_ops = 0;
  int64_t copy_rows = 0;
};

static void zc_cache_clear(ss_ctx* ctx) {
  if (ctx->zc_cache.empty()) return;
  cudaDeviceSynchronize();   // (host dispatches synchronise on return: nothing still reads them)
  for (auto& kv : ctx->zc_cache) {
    cudaFree(kv.second->dev);
    delete kv.second;
  }
  ctx->zc_cache.clear();
}

static uint64_t zc_key(int pass_kind, int block, int role, int n_seg, const ss_seg* segs) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  const int hdr[4] = {pass_kind, block, role, n_seg};
  mix(hdr, sizeof(hdr));
  mix(segs, sizeof(ss_seg) * (size_t)n_seg);
  return h;
}

// `local_buffers`: every pointer is a staging slice this context allocated on its own device
// (host pipelines), so the per-pointer peer-GPU query is skipped.
// `src_remote`: the caller already established that every source is pinned host memory read
// with plain loads (the zero-copy host dispatch; its destinations are local slots): no query.
int build_batch(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg, const ss_seg* segs,
                int32_t* seg_status, Built& B, bool local_buffers = false, bool src_remote = false) {
  if (pass_kind < 0 || pass_kind > 2) return fail(ctx, SS_E_ARG, "unknown pass %d", pass_kind);
  if (n_seg < 0 || (n_seg > 0 && (!segs || !seg_status)))
    return fail(ctx, SS_E_ARG, "bad segment array");
  auto lit = ctx->layers.find({block, role});
  if (lit == ctx->layers.end())
    return fail(ctx, SS_E_NOLAYER, "unknown layer (%d, %d)", block, role);
  Layer& L = lit->second;
  const bool bwd = pass_kind == SS_PASS_BACKWARD;
  const int K = bwd ? L.d_out : L.d_in;
  const int N = bwd ? L.d_in : L.d_out;
  B = Built();
  B.pass_kind = pass_kind;
  B.block = block;
  B.role = role;
  B.K = K;
  B.N = N;

  // ---- validate + build device segment records (batch order == envelope order)
  std::vector<DevSeg> ds;
  std::vector<const ss_seg*> src_of;
  std::vector<char> dec_of;       // decode class (K1d split-K order), see decode_rows
  ds.reserve(n_seg);
  int64_t M = 0, Md = 0;
  const bool dec_ok = K % 64 == 0 && ctx->decode_rows > 0;
  bool any_lora = false;
  for (int i = 0; i < n_seg; ++i) {
    const ss_seg& s = segs[i];
    seg_status[i] = SS_SEG_OK;
    if ((int)s.width != K) { seg_status[i] = SS_SEG_BAD_WIDTH; continue; }
    if (s.rows == 0) continue;
    if (!s.src || !s.dst || s.src_ld < K || s.dst_ld < N) { seg_status[i] = SS_SEG_BAD_PTR; continue; }
    DevSeg d{};
    d.xrow0 = -1;
    d.rows = (int32_t)s.rows;
    d.src = s.src;
    d.src_ld = s.src_ld;
    d.dst = s.dst;
    d.dst_ld = s.dst_ld;
    d.pack_row = -1;
    int f = 0;
    if (s.flags & SS_SEGF_SRC_BF16) f |= SEGF_SRC_BF16;
    if (s.flags & SS_SEGF_DST_BF16) f |= SEGF_DST_BF16;
    if (aligned16(s.src, s.src_ld, (s.flags & SS_SEGF_SRC_BF16) ? 2 : 4)) f |= SEGF_SRC_VEC;
    if (aligned16(s.dst, s.dst_ld, (s.flags & SS_SEGF_DST_BF16) ? 2 : 4)) f |= SEGF_DST_VEC;
    if (src_remote) f |= SEGF_REMOTE_SRC;
    if (!local_buffers || ctx->force_remote) {
      if (is_remote(ctx, s.src)) f |= SEGF_REMOTE_SRC;
      if (is_remote(ctx, s.dst) || (s.dst_base && is_remote(ctx, s.dst_base))) f |= SEGF_REMOTE_DST;
    }
    // NOISE with the adapter flag = the noise effect of the ADAPTED layer, (n.W + s n.A.B) * l
    // (bias-free): what a client with an executor-fused adapter subtracts to unblind its reply
    if (s.flags & SS_SEGF_ADAPTER) {
      auto a = L.adapters.find(s.client_id);
      if (a == L.adapters.end()) { seg_status[i] = SS_SEG_NO_ADAPTER; continue; }
      const AdapterSlot& as = a->second;
      if (as.kind & SS_ADAPTER_LORA) {
        f |= SEGF_LORA;
        d.pack_row = as.pack_row;
        d.rank_pad = as.rank_pad;
        d.lora_scale = as.scale;
        any_lora = true;
      }
      if (as.kind & SS_ADAPTER_IA3) {
        f |= SEGF_IA3;
        d.ia3 = as.ia3;
        if (bwd && (ctx->ia3_lo == 2 || (ctx->ia3_lo == 1 && !(s.flags & SS_SEGF_DST_BF16)))) {
          f |= SEGF_IA3_LO;
          B.any_lo = true;
        }
      }
    }
    if (s.dst_base && pass_kind != SS_PASS_BACKWARD) {
      if (s.base_ld < N) { seg_status[i] = SS_SEG_BAD_PTR; continue; }
      f |= SEGF_WANT_BASE;
      if (s.flags & SS_SEGF_BASE_BF16) f |= SEGF_BASE_BF16;
      if (aligned16(s.dst_base, s.base_ld, (s.flags & SS_SEGF_BASE_BF16) ? 2 : 4)) f |= SEGF_BASE_VEC;
      d.dst_base = s.dst_base;
      d.base_ld = s.base_ld;
    }
    d.flags = f;
    ds.push_back(d);
    src_of.push_back(&s);
    const bool dec = dec_ok && (int)s.rows <= DEC_SHR_MAXROWS &&
                     ((s.flags & SS_SEGF_CLASS_DECODE) ||
                      (!(s.flags & SS_SEGF_CLASS_PREFILL) && (int)s.rows <= ctx->decode_rows));
    dec_of.push_back(dec ? 1 : 0);
    M += s.rows;
    if (dec) Md += s.rows;
  }
  B.status.assign(seg_status, seg_status + n_seg);
  // A reply written over request rows (the reference's SharedBuffer hand-off, transport.py:
  // 76-97, reuses one buffer for both) must not be read in place: a tile's epilogue would
  // overwrite rows other tiles still stream. Such segments are gathered into the operand first
  // (the gather completes before the GEMM starts), like the reference's concat_rows copy.
  {
    struct Range { uintptr_t a, b; };
    auto span = [](const void* p, int64_t rows, int64_t ld, int64_t width, size_t esz) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(p);
      return Range{a, a + (uintptr_t)(((rows - 1) * ld + width) * (int64_t)esz)};
    };
    std::vector<Range> outs;
    for (const DevSeg& d : ds) {
      outs.push_back(span(d.dst, d.rows, d.dst_ld, N, (d.flags & SEGF_DST_BF16) ? 2 : 4));
      if (d.flags & SEGF_WANT_BASE)
        outs.push_back(span(d.dst_base, d.rows, d.base_ld, N, (d.flags & SEGF_BASE_BF16) ? 2 : 4));
    }
    for (DevSeg& d : ds) {
      const Range in = span(d.src, d.rows, d.src_ld, K, (d.flags & SEGF_SRC_BF16) ? 2 : 4);
      for (const Range& o : outs)
        if (in.a < o.b && o.a < in.b) { d.flags |= SEGF_SRC_ALIASED; break; }
    }
  }
  if (M == 0) return SS_OK;
  if (M > (int64_t)1 << 30) return fail(ctx, SS_E_ARG, "batch too large (%lld rows)", (long long)M);
  CK(cudaSetDevice(ctx->device));

  // ---- M-tiles: segment-aligned direct tiles for whole tiles of bf16 rows, the rest packed
  // Kernel / tile choice depends only on the layer shape and the dispatch size, never on which
  // segments are present; every choice reduces K in the same order (bitwise-equal rows).
  // Decode-class rows (dec_of) are packed after every other row into 64-row tiles of whole
  // segments for the split-K kernel; the choices below see the single-chain rows Mp only.
  const int64_t Mp = M - Md;
  const int n256 = (N + BN - 1) / BN;
  const bool pair = ctx->gemm_2cta < 0 ? (((Mp + BM2 - 1) / BM2) * n256 >= ctx->num_sms / 2)
                                       : ctx->gemm_2cta != 0;
  const int TM = pair ? BM2 : BM;
  int tbn = BN;
  if (!pair) {
    const int64_t m128 = (Mp + BM - 1) / BM;
    if (m128 * n256 < ctx->num_sms) tbn = (m128 * ((N + 127) / 128) >= ctx->num_sms) ? 128 : 64;
    if (ctx->force_tbn) tbn = ctx->force_tbn;
  }
  std::vector<TileDesc> tiles;
  std::vector<int32_t> piece_seg;          // packed pieces in X order
  std::vector<int32_t> direct_src;         // segment of each direct tensor map (map = 1 + i)
  int64_t MX = 0;
  for (size_t j = 0; j < ds.size(); ++j) {
    DevSeg& d = ds[j];
    if (dec_of[j]) continue;
    const bool direct_ok = ctx->direct_tiles && (d.flags & SEGF_SRC_BF16) && (d.flags & SEGF_SRC_VEC) &&
                           !(d.flags & (SEGF_REMOTE_SRC | SEGF_SRC_ALIASED)) &&
                           !(bwd && (d.flags & SEGF_IA3)) && (d.src_ld * 2) % 16 == 0;
    const int nd = direct_ok ? (d.rows / TM) * TM : 0;
    if (nd > 0) {
      const int amap = 1 + (int)direct_src.size();
      direct_src.push_back((int32_t)j);
      for (int r = 0; r < nd; r += TM)
        tiles.push_back(TileDesc{amap, r, (int32_t)j, TM, 0, 0, 0, 0, -1});
    }
    if (d.rows > nd) {
      d.xrow0 = (int32_t)MX;
      d.xlocal0 = nd;
      piece_seg.push_back((int32_t)j);
      MX += d.rows - nd;
    }
  }
  for (int64_t x = 0; x < MX; x += TM)
    tiles.push_back(TileDesc{0, (int32_t)x, -1, (int32_t)std::min<int64_t>(TM, MX - x), 0, 0, 0, 0, -1});
  const int num_m = (int)tiles.size();
  const int64_t MXp = MX;
  // decode tiles: whole decode-class segments, in batch order, <= DEC_ROWS rows per tile
  std::vector<DecTile> dtiles;
  std::vector<int32_t> dtile_of(ds.size(), -1);
  for (size_t j = 0; j < ds.size(); ++j) {
    if (!dec_of[j]) continue;
    DevSeg& d = ds[j];
    if (dtiles.empty() || dtiles.back().rows + d.rows > DEC_ROWS) {
      DecTile t{};
      t.arow = (int32_t)MX;
      dtiles.push_back(t);
    }
    DecTile& t = dtiles.back();
    d.xrow0 = (int32_t)MX;
    d.xlocal0 = 0;
    piece_seg.push_back((int32_t)j);
    MX += d.rows;
    t.rows += d.rows;
    if (d.flags & SEGF_IA3_LO) t.lo = 1;
    dtile_of[j] = (int32_t)dtiles.size() - 1;
  }
  const int dec_kbc = ctx->decode_chunk_kb;
  const int dec_C = dtiles.empty() ? 0 : (K / BK + dec_kbc - 1) / dec_kbc;

  // ---- LoRA: per tile rank-chunk lists (block-diagonal over the tile's segments) + shrink items
  std::vector<int32_t> chunks;
  std::vector<int2> lpieces;      // decode tiles' LoRA pieces {first stage, stage count}
  std::vector<DecShrinkItem> ditems;   // decode-class segments' LoRA shrink (dec_shrink_kernel)
  std::vector<int4> lstages;      // decode LoRA stages {pack row, 16-row chunks, A_lora hi col, lo col | -1}
  int lp_chunks = 0;
  std::vector<ShrinkItem> items;
  int max_cols = 0;
  if (any_lora) {
    size_t pi = 0;  // packed-piece cursor
    for (int mt = 0; mt < num_m; ++mt) {
      TileDesc& td = tiles[mt];
      td.chunk_begin = (int32_t)chunks.size();
      auto add_piece = [&](int sj, int amap, int arow, int p0, int nrows) {
        const DevSeg& d = ds[sj];
        if (!(d.flags & SEGF_LORA)) return;
        const int col = (int)(chunks.size() - td.chunk_begin) * LORA_CHUNK;
        // hi / lo halves of s*x.A (ShrinkItem::hilo): the expand reads the same B rows twice
        const int hilo = ctx->lora_hilo == 2 || (ctx->lora_hilo == 1 && !(d.flags & SEGF_DST_BF16));
        for (int rep = 0; rep <= hilo; ++rep)
          for (int q = 0; q < d.rank_pad / LORA_CHUNK; ++q) chunks.push_back(d.pack_row + q * LORA_CHUNK);
        for (int r = 0; r < nrows; r += BM)
          items.push_back(ShrinkItem{sj, amap, arow + r, std::min(BM, nrows - r), mt * TM + p0 + r, col, 0, 0,
                                     r == 0 ? 1 : 0, mt * TM, TM, p0, p0 + nrows, hilo, 0, 0});
      };
      if (td.seg >= 0) {
        add_piece(td.seg, td.amap, td.arow, 0, td.rows);
      } else {
        const int64_t x0 = td.arow, x1 = x0 + td.rows;
        while (pi < piece_seg.size() &&
               ds[piece_seg[pi]].xrow0 + (ds[piece_seg[pi]].rows - ds[piece_seg[pi]].xlocal0) <= x0)
          ++pi;
        for (size_t k = pi; k < piece_seg.size(); ++k) {
          const DevSeg& d = ds[piece_seg[k]];
          const int64_t p0 = std::max<int64_t>(x0, d.xrow0);
          const int64_t p1 = std::min<int64_t>(x1, d.xrow0 + (d.rows - d.xlocal0));
          if (p0 >= x1) break;
          if (p1 > p0) add_piece(piece_seg[k], 0, (int)p0, (int)(p0 - x0), (int)(p1 - p0));
        }
      }
      td.chunk_count = (int32_t)chunks.size() - td.chunk_begin;
      max_cols = std::max(max_cols, td.chunk_count * LORA_CHUNK);
    }
    // decode tiles: the tile's rank chunks, block-diagonal over its segments, cut into pieces of
    // whole segments of <= decode_lora_piece chunks (one LoRA chain each, see decode.cuh)
    for (size_t t = 0; t < dtiles.size(); ++t) {
      DecTile& dt = dtiles[t];
      dt.al_row = (int32_t)((int64_t)num_m * TM + (int64_t)t * DEC_ROWS);
      dt.chunk_begin = (int32_t)chunks.size();
      dt.lp_begin = (int32_t)lpieces.size();
      for (size_t j = 0; j < ds.size(); ++j) {
        if (dtile_of[j] != (int32_t)t || !(ds[j].flags & SEGF_LORA)) continue;
        DevSeg& d = ds[j];
        const int col = (int)(chunks.size() - dt.chunk_begin) * LORA_CHUNK;
        const int hilo = ctx->lora_hilo == 2 || (ctx->lora_hilo == 1 && !(d.flags & SEGF_DST_BF16));
        const int nch = (1 + hilo) * (d.rank_pad / LORA_CHUNK);
        if (dt.lp_count == 0 || lp_chunks + nch > ctx->decode_lora_piece) {
          lpieces.push_back(make_int2((int)lstages.size(), 0));
          dt.lp_count++;
          lp_chunks = 0;
        }
        lp_chunks += nch;
        // one stage per 64-row slice of the rank block: its B rows once, hi then lo columns
        for (int r0 = 0; r0 < d.rank_pad; r0 += 64) {
          lstages.push_back(make_int4(d.pack_row + r0, std::min(4, (d.rank_pad - r0) / LORA_CHUNK), col + r0,
                                      hilo ? col + d.rank_pad + r0 : -1));
          lpieces.back().y++;
        }
        d.dec_piece = dt.lp_count - 1;
        for (int rep = 0; rep <= hilo; ++rep)
          for (int q = 0; q < d.rank_pad / LORA_CHUNK; ++q) chunks.push_back(d.pack_row + q * LORA_CHUNK);
        // its LoRA intermediate: the decode-class shrink (CUDA cores, decode.cuh); the source
        // rows are resolved once X is allocated (below)
        DecShrinkItem di{};
        di.seg = (int32_t)j;
        di.rows = d.rows;
        di.hilo = hilo;
        di.col = col;
        di.tile_row0 = dt.al_row;
        di.p0 = d.xrow0 - dt.arow;
        ditems.push_back(di);
      }
      dt.chunk_count = (int32_t)chunks.size() - dt.chunk_begin;
      max_cols = std::max(max_cols, dt.chunk_count * LORA_CHUNK);
    }
    if (chunks.empty()) chunks.push_back(0);
  }
  const int64_t lora_ld = std::max<int64_t>(64, round_up(max_cols, 64));

  // ---- workspace
  const int64_t ldx = round_up(K, 64);
  const int64_t mx_pad = round_up(std::max<int64_t>(MX, 1), TM);
  int rc = ensure_dev(ctx, ctx->X, ctx->x_cap, (size_t)mx_pad * ldx * 2);
  if (rc) return rc;
  if (B.any_lo && (rc = ensure_dev(ctx, ctx->X_lo, ctx->xlo_cap, (size_t)mx_pad * ldx * 2))) return rc;
  rc = ensure_dev(ctx, ctx->row_seg, ctx->rs_cap, (size_t)mx_pad * 4);
  if (rc) return rc;
  const int64_t al_rows = (int64_t)num_m * TM + (int64_t)dtiles.size() * DEC_ROWS;
  if (any_lora) {
    rc = ensure_dev(ctx, ctx->a_lora, ctx->al_cap, (size_t)al_rows * lora_ld * 2);
    if (rc) return rc;
  }
  ctx->ws_high = std::max(ctx->ws_high, ctx->x_cap + ctx->al_cap + ctx->rs_cap + ctx->qx_cap);

  // ---- tensor maps: [0] = X, [1 + i] = direct source i (box {64, 128} rows), then the
  // destination maps of TMA-stored segments: one over the whole segment (direct tiles) and one
  // over its packed tail only (so a packed tile's store can never touch the segment's head rows)
  std::vector<CUtensorMap> tmaps(1 + direct_src.size());
  rc = encode_2d(ctx, &tmaps[0], ctx->X, K, std::max<int64_t>(MX, 1), ldx, 64, BM);
  if (rc) return rc;
  for (size_t i = 0; i < direct_src.size(); ++i) {
    const DevSeg& d = ds[direct_src[i]];
    rc = encode_2d(ctx, &tmaps[1 + i], d.src, K, d.rows, d.src_ld, 64, BM);
    if (rc) return rc;
  }
  int32_t lo_map = -1;
  if (B.any_lo) {
    // X_lo map (same geometry as X) for every packed tile holding an SEGF_IA3_LO piece
    lo_map = (int32_t)tmaps.size();
    tmaps.emplace_back();
    rc = encode_2d(ctx, &tmaps.back(), ctx->X_lo, K, std::max<int64_t>(MX, 1), ldx, 64, BM);
    if (rc) return rc;
    for (TileDesc& td : tiles) {
      if (td.seg >= 0) continue;
      const int64_t x0 = td.arow, x1 = x0 + td.rows;
      for (int32_t sj : piece_seg) {
        const DevSeg& d = ds[sj];
        const int64_t p0 = d.xrow0, p1 = d.xrow0 + (d.rows - d.xlocal0);
        if ((d.flags & SEGF_IA3_LO) && p0 < x1 && x0 < p1) { td.amap_lo = lo_map; break; }
      }
    }
  }
  std::vector<int32_t> dmap_full(ds.size(), -1), dmap_tail(ds.size(), -1);
  for (size_t j = 0; j < ds.size(); ++j) {
    DevSeg& d = ds[j];
    if (!ctx->tma_store || !(d.flags & SEGF_DST_BF16) || !(d.flags & SEGF_DST_VEC) ||
        (d.flags & SEGF_REMOTE_DST))
      continue;
    d.flags |= SEGF_TMA_STORE;
    const bool has_direct = d.xrow0 < 0 || d.xlocal0 > 0;
    if (has_direct) {
      dmap_full[j] = (int32_t)tmaps.size();
      tmaps.emplace_back();
      rc = encode_2d(ctx, &tmaps.back(), d.dst, N, d.rows, d.dst_ld, 64, BM);
      if (rc) return rc;
    }
    if (d.xrow0 >= 0) {
      dmap_tail[j] = (int32_t)tmaps.size();
      tmaps.emplace_back();
      rc = encode_2d(ctx, &tmaps.back(), static_cast<const char*>(d.dst) + (int64_t)d.xlocal0 * d.dst_ld * 2, N,
                     d.rows - d.xlocal0, d.dst_ld, 64, BM);
      if (rc) return rc;
    }
  }
  std::vector<int2> stores;
  {
    size_t pi = 0;
    for (TileDesc& td : tiles) {
      td.store_begin = (int32_t)stores.size();
      if (td.seg >= 0) {
        if (dmap_full[td.seg] >= 0) stores.push_back(make_int2(dmap_full[td.seg], td.arow));
      } else {
        const int64_t x0 = td.arow, x1 = x0 + td.rows;
        while (pi < piece_seg.size() &&
               ds[piece_seg[pi]].xrow0 + (ds[piece_seg[pi]].rows - ds[piece_seg[pi]].xlocal0) <= x0)
          ++pi;
        for (size_t k = pi; k < piece_seg.size(); ++k) {
          const DevSeg& d = ds[piece_seg[k]];
          if (d.xrow0 >= x1) break;
          // only pieces that start at or before the tile's first row (non-negative box
          // coordinate); the kernel stores rows of later-starting pieces directly
          if (dmap_tail[piece_seg[k]] >= 0 && d.xrow0 <= x0)
            stores.push_back(make_int2(dmap_tail[piece_seg[k]], (int32_t)(x0 - d.xrow0)));
        }
      }
      td.store_count = (int32_t)stores.size() - td.store_begin;
    }
  }

  // ---- weight-streaming dispatch (one packed tile of <= 64 rows): the GEMM reads A through a
  // 64-row box (MMA rows 64-127 are never stored); with `stream_gemm` (K a multiple of 64) the
  // streaming kernel moves 4 k-blocks of A and of W per TMA operation instead
  if (ctx->a_rows64 && !pair && num_m == 1 && direct_src.empty() && MXp <= 64 && !B.any_lo) {
    tiles[0].amap = (int32_t)tmaps.size();
    tmaps.emplace_back();
    // At these sizes a tile's time is set by its K/16-long chain of dependent UMMAs, not by its
    // bytes (profiles/r01_l2_and_decode.md): when 64-wide tiles would need more than one wave
    // and 128-wide ones fit in one, the single-CTA kernel's 128-wide tiles finish in one chain
    const bool one_wave_128 = ctx->wide_decode && (N + 63) / 64 > ctx->num_sms && (N + 127) / 128 <= ctx->num_sms;
    if (one_wave_128 && !ctx->force_tbn) {
      rc = encode_2d(ctx, &tmaps.back(), ctx->X, K, MX, ldx, 64, 64);
      tbn = 128;
    } else if (ctx->stream_gemm && K % 64 == 0 && !ctx->force_tbn) {
      rc = encode_kchunks(ctx, &tmaps.back(), ctx->X, K, MX, ldx, 64, 4);
      B.stream = true;
      tbn = 64;
    } else {
      rc = encode_2d(ctx, &tmaps.back(), ctx->X, K, MX, ldx, 64, 64);
    }
    if (rc) return rc;
    B.a_rows64 = true;
  }

  // ---- decode tiles read X (and X_lo) as {64 k, 64 rows, 2 k-chunks} boxes
  if (!dtiles.empty()) {
    B.dec_amap = (int32_t)tmaps.size();
    tmaps.emplace_back();
    if ((rc = encode_2d(ctx, &tmaps.back(), ctx->X, K, MX, ldx, 64, DEC_ROWS))) return rc;
    B.dec_alo = B.dec_amap;
    for (const DecTile& t : dtiles) {
      if (!t.lo) continue;
      B.dec_alo = (int32_t)tmaps.size();
      tmaps.emplace_back();
      if ((rc = encode_2d(ctx, &tmaps.back(), ctx->X_lo, K, MX, ldx, 64, DEC_ROWS))) return rc;
      break;
    }
  }

  // ---- short LoRA pieces of the packed operand (decode rows): the shrink reads them straight
  // from the client's rows through a 16-row box over the segment (so it no longer waits for the
  // gather and can run beside it), or, for sources TMA cannot read in place, through a 16-row
  // box over the packed operand instead of 128 rows of neighbouring clients' rows
  if (any_lora && MX > 0) {
    int32_t small_map = -1, small_lo_map = -1;
    std::vector<int32_t> seg_map(ds.size(), -1);
    // shrinks of IA3-backward rows with the lo pass read g = hi + lo like the GEMM does
    for (ShrinkItem& it : items)
      if (it.amap == 0 && (ds[it.seg].flags & SEGF_IA3_LO)) it.amap_lo = lo_map;
    for (ShrinkItem& it : items) {
      if (it.amap != 0 || it.rows > 16) continue;
      const DevSeg& d = ds[it.seg];
      // (backward + IA3: the shrink must read g = dy*l, which only the packed operand holds)
      const bool in_place = (d.flags & SEGF_SRC_BF16) && (d.flags & SEGF_SRC_VEC) &&
                            !(d.flags & (SEGF_REMOTE_SRC | SEGF_SRC_ALIASED)) &&
                            !(bwd && (d.flags & SEGF_IA3)) && (d.src_ld * 2) % 16 == 0;
      if (in_place) {
        if (seg_map[it.seg] < 0) {
          seg_map[it.seg] = (int32_t)tmaps.size();
          tmaps.emplace_back();
          rc = encode_2d(ctx, &tmaps.back(), d.src, K, d.rows, d.src_ld, 64, 16);
          if (rc) return rc;
        }
        it.arow = it.arow - d.xrow0 + d.xlocal0;       // X row -> segment row
        it.amap = seg_map[it.seg];
      } else {
        if (small_map < 0) {
          small_map = (int32_t)tmaps.size();
          tmaps.emplace_back();
          rc = encode_2d(ctx, &tmaps.back(), ctx->X, K, MX, ldx, 64, 16);
          if (rc) return rc;
        }
        it.amap = small_map;
        if (d.flags & SEGF_IA3_LO) {
          if (small_lo_map < 0) {
            small_lo_map = (int32_t)tmaps.size();
            tmaps.emplace_back();
            if ((rc = encode_2d(ctx, &tmaps.back(), ctx->X_lo, K, MX, ldx, 64, 16))) return rc;
          }
          it.amap_lo = small_lo_map;
        }
      }
      it.a_rows = 16;
    }
    // the shrink depends on the gather only if some item reads the packed operand
    B.shrink_indep = true;
    for (const ShrinkItem& it : items)
      if (it.amap == 0 || it.amap == small_map) B.shrink_indep = false;
    // decode-class shrink items: the client's rows in place (bf16 or f32, device or page-locked
    // host), or the packed rows where only they hold the operand (backward IA3: g = dy*l)
    for (DecShrinkItem& di : ditems) {
      const DevSeg& d = ds[di.seg];
      const bool in_place = !(d.flags & (SEGF_REMOTE_SRC | SEGF_SRC_ALIASED)) && !(bwd && (d.flags & SEGF_IA3));
      if (in_place) {
        di.src = d.src;
        di.ld = d.src_ld;
        di.kind = (d.flags & SEGF_SRC_BF16) ? 0 : 1;
        di.src_lo = nullptr;
      } else {
        di.src = ctx->X + (int64_t)d.xrow0 * ldx;
        di.ld = ldx;
        di.kind = 0;
        di.src_lo = (d.flags & SEGF_IA3_LO) ? ctx->X_lo + (int64_t)d.xrow0 * ldx : nullptr;
        B.shrink_indep = false;
      }
    }
  }

  // ---- serialise the device tables
  const size_t off_tm = 0;
  // ---- K1d work groups {mt, kind << 8 | g, slot, first n tile}: every chunk group (groups of
  // DEC_G column tiles of one chunk), then every LoRA-piece group (DEC_G_LORA column tiles)
  std::vector<int4> dgroups;
  if (!dtiles.empty()) {
    const int n_n = (N + DEC_TN - 1) / DEC_TN;
    for (size_t m = 0; m < dtiles.size(); ++m)
      for (int rep = 0; rep <= dtiles[m].lo; ++rep)
        for (int c = 0; c < dec_C; ++c)
          for (int n = 0; n < n_n; n += DEC_G)
            dgroups.push_back(make_int4((int)m, std::min(DEC_G, n_n - n), rep * dec_C + c, n));
    B.dec_chunk_groups = (int)dgroups.size();
    for (size_t m = 0; m < dtiles.size(); ++m)
      for (int q = 0; q < dtiles[m].lp_count; ++q)
        for (int n = 0; n < n_n; n += DEC_G_LORA)
          dgroups.push_back(make_int4((int)m, (1 << 8) | std::min(DEC_G_LORA, n_n - n), 2 * dec_C + q, n));
    B.dec_groups = (int)dgroups.size();
  }
  const size_t off_seg = round_up(tmaps.size() * sizeof(CUtensorMap), 256);
  const size_t off_tile = off_seg + round_up(ds.size() * sizeof(DevSeg), 256);
  const size_t off_piece = off_tile + round_up(tiles.size() * sizeof(TileDesc), 256);
  const size_t off_ch = off_piece + round_up(std::max<size_t>(1, piece_seg.size()) * 4, 256);
  const size_t off_st = off_ch + round_up(std::max<size_t>(1, chunks.size()) * 4, 256);
  const size_t off_it = off_st + round_up(std::max<size_t>(1, stores.size()) * sizeof(int2), 256);
  const size_t off_dt = off_it + round_up(std::max<size_t>(1, items.size()) * sizeof(ShrinkItem), 256);
  const size_t off_dcb = off_dt + round_up(std::max<size_t>(1, dtiles.size()) * sizeof(DecTile), 256);
  const size_t off_lp = off_dcb + round_up(std::max<size_t>(1, dgroups.size()) * sizeof(int4), 256);
  const size_t off_ls = off_lp + round_up(std::max<size_t>(1, lpieces.size()) * sizeof(int2), 256);
  const size_t off_di = off_ls + round_up(std::max<size_t>(1, lstages.size()) * sizeof(int4), 256);
  const size_t total = off_di + round_up(std::max<size_t>(1, ditems.size()) * sizeof(DecShrinkItem), 256);
  B.blob.assign(total, 0);
  char* h = B.blob.data();
  memcpy(h + off_tm, tmaps.data(), tmaps.size() * sizeof(CUtensorMap));
  memcpy(h + off_seg, ds.data(), ds.size() * sizeof(DevSeg));
  memcpy(h + off_tile, tiles.data(), tiles.size() * sizeof(TileDesc));
  if (!piece_seg.empty()) memcpy(h + off_piece, piece_seg.data(), piece_seg.size() * 4);
  if (!stores.empty()) memcpy(h + off_st, stores.data(), stores.size() * sizeof(int2));
  if (any_lora) {
    memcpy(h + off_ch, chunks.data(), chunks.size() * 4);
    memcpy(h + off_it, items.data(), items.size() * sizeof(ShrinkItem));
  }
  if (!dtiles.empty()) {
    memcpy(h + off_dt, dtiles.data(), dtiles.size() * sizeof(DecTile));
    memcpy(h + off_dcb, dgroups.data(), dgroups.size() * sizeof(int4));
    if (!lpieces.empty()) memcpy(h + off_lp, lpieces.data(), lpieces.size() * sizeof(int2));
    if (!lstages.empty()) memcpy(h + off_ls, lstages.data(), lstages.size() * sizeof(int4));
    if (!ditems.empty()) memcpy(h + off_di, ditems.data(), ditems.size() * sizeof(DecShrinkItem));
  }
  B.off_di = off_di;
  B.n_ditems = (int)ditems.size();
  for (const DecShrinkItem& di : ditems) {
    B.dec_rank_max = std::max(B.dec_rank_max, (int)ds[di.seg].rank_pad);
    B.dec_rows_max = std::max(B.dec_rows_max, (int)di.rows);
  }
  if (!ditems.empty()) {
    const size_t pbytes = ditems.size() * (size_t)dec_C * DEC_SHR_MAXROWS * 256 * sizeof(float);
    if ((rc = ensure_dev(ctx, ctx->dshr_part, ctx->dshr_part_cap, pbytes))) return rc;
    if (ctx->dshr_ticket_cap < ditems.size() * sizeof(int)) {
      if ((rc = ensure_dev(ctx, ctx->dshr_ticket, ctx->dshr_ticket_cap, ditems.size() * sizeof(int)))) return rc;
      CK(cudaMemset(ctx->dshr_ticket, 0, ctx->dshr_ticket_cap));
    }
    for (const DecShrinkItem& di : ditems) {
      const double r = ds[di.seg].rank_pad;
      B.shrink_flops += 2.0 * di.rows * r * K;
      B.shrink_bytes += r * K * 2.0 + (double)di.rows * K * (di.kind ? 4 : 2) + DEC_ROWS * r * 2 * (1 + di.hilo);
    }
  }
  B.off_lp = off_lp;
  B.off_ls = off_ls;
  B.dec_S = 2 * dec_C + 1;
  for (const DecTile& t : dtiles) B.dec_S = std::max(B.dec_S, 2 * dec_C + t.lp_count);
  B.off_tm = off_tm; B.off_seg = off_seg; B.off_tile = off_tile; B.off_piece = off_piece;
  B.off_ch = off_ch; B.off_st = off_st; B.off_it = off_it; B.off_dt = off_dt; B.off_dcb = off_dcb;
  B.n_dec = (int)dtiles.size();
  B.dec_C = dec_C;
  B.dec_kbc = dec_kbc;
  if (!dtiles.empty()) {
    const int64_t tiles_dec = (int64_t)dtiles.size() * ((N + DEC_TN - 1) / DEC_TN);
    if ((rc = ensure_dev(ctx, ctx->dec_part, ctx->dec_part_cap,
                         (size_t)tiles_dec * B.dec_S * DEC_PART * sizeof(float)))) return rc;
    // in-kernel fixup: ticket + per (tile, half) counters, all zero between launches
    const size_t fx_bytes = (size_t)(1 + 2 * tiles_dec) * sizeof(int);
    if (ctx->dec_fx_cap < fx_bytes) {
      if ((rc = ensure_dev(ctx, ctx->dec_fx, ctx->dec_fx_cap, fx_bytes))) return rc;
      CK(cudaMemset(ctx->dec_fx, 0, ctx->dec_fx_cap));
    }
  }
  B.Mp = Mp;
  B.M = M; B.MX = MX; B.lora_ld = lora_ld; B.al_rows = al_rows; B.ldx = ldx;
  B.any_lora = any_lora; B.pair = pair; B.tbn = tbn;   // (B.any_lo set during validation)
  B.pn = ctx->pair_n ? ctx->pair_n
                     : (((M + BM2 - 1) / BM2) * ((N + 511) / 512) >= (int64_t)ctx->num_sms ? 512 : 256);
  B.num_m = num_m; B.n_piece = (int)piece_seg.size(); B.n_items = (int)items.size();
  if (any_lora) {
    for (const ShrinkItem& it : items) B.part_ld = std::max(B.part_ld, ds[it.seg].rank_pad);
    B.shrink_chunks_ = shrink_chunks(K, ctx->shrink_kb_chunk);
    B.kb_chunk = ctx->shrink_kb_chunk;
    int rc2 = ensure_shrink_ws(ctx, items.size(), B.shrink_chunks_, B.part_ld);
    if (rc2) return rc2;
  }
  // algorithmic work for the in-stream profiler
  for (size_t k = 0; k < piece_seg.size(); ++k) {
    const DevSeg& d = ds[piece_seg[k]];
    B.gather_bytes += (double)(d.rows - d.xlocal0) * K * ((d.flags & SEGF_SRC_BF16) ? 2 : 4);
  }
  B.gather_bytes += (double)MX * K * 2 + MX * 4.0;
  for (const ShrinkItem& it : items) {
    const DevSeg& d = ds[it.seg];
    B.shrink_flops += 2.0 * it.rows * d.rank_pad * K;
    B.shrink_bytes += (double)it.rows * K * 2 + (double)d.rank_pad * K * 2 + (double)it.rows * d.rank_pad * 2;
  }
  // base GEMM + each LoRA segment's own rank (the block-diagonal zeros of neighbouring
  // segments are not counted); bytes: A rows, W, outputs
  B.gemm_flops = 2.0 * (double)Mp * N * K;
  B.gemm_bytes = Mp ? (double)Mp * K * 2 + (double)K * N * 2 : 0.0;
  B.dec_flops = 2.0 * (double)Md * N * K;
  B.dec_bytes = Md ? (double)Md * K * 2 + (double)K * N * 2 : 0.0;
  for (size_t j = 0; j < ds.size(); ++j) {
    const DevSeg& d = ds[j];
    double& fl = dec_of[j] ? B.dec_flops : B.gemm_flops;
    double& by = dec_of[j] ? B.dec_bytes : B.gemm_bytes;
    by += (double)d.rows * N * ((d.flags & SEGF_DST_BF16) ? 2 : 4);
    if (d.flags & SEGF_WANT_BASE) by += (double)d.rows * N * ((d.flags & SEGF_BASE_BF16) ? 2 : 4);
    if (d.flags & SEGF_LORA) fl += 2.0 * d.rows * d.rank_pad * N;
  }
  B.ws_epoch = ctx->ws_epoch;
  B.ad_epoch = ctx->ad_epoch;
  return SS_OK;
}

// Kernel launch with programmatic stream serialization (ctx->pdl): the kernel may start its
// prologue while the previous kernel on the stream drains; it waits (griddepcontrol.wait) before
// touching global data. Captured into graphs as programmatic edges.
template <typename... KArgs, typename... Args>
cudaError_t launch_kp(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(const ss_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args... args) {
  return launch_kp(ctx->pdl && !ctx->profiling, kernel, grid, block, smem, st, args...);
}

// One workspace per context (X, the LoRA operand, shrink / decode partials, tickets): work issued
// on a different stream than the context's previous work waits for it (not while capturing a
// graph: the captured sequence is ordered on its own stream and follows a synchronised run; and
// not on an event last recorded inside a capture, which cannot be waited on outside it).
int order_after_previous(ss_ctx* ctx, cudaStream_t stream) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(stream, &cs));
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  if (ctx->any_compute && stream != ctx->last_stream && !capturing && !ctx->done_captured)
    CK(cudaStreamWaitEvent(stream, ctx->compute_done, 0));
  ctx->last_stream = stream;
  ctx->done_captured = capturing;
  return SS_OK;
}

// Launch the kernels of a built batch whose tables are at device address `dv` (stream-ordered
// after whatever copied them there).
int launch_batch(ss_ctx* ctx, const Built& B, char* dv, cudaStream_t stream) {
  auto lit = ctx->layers.find({B.block, B.role});
  if (lit == ctx->layers.end()) return fail(ctx, SS_E_NOLAYER, "unknown layer (%d, %d)", B.block, B.role);
  Layer& L = lit->second;
  CK(cudaSetDevice(ctx->device));
  const int pass_kind = B.pass_kind;
  const bool bwd = pass_kind == SS_PASS_BACKWARD;
  const int K = B.K, N = B.N;
  const int64_t MX = B.MX, lora_ld = B.lora_ld, al_rows = B.al_rows, ldx = B.ldx;
  const bool any_lora = B.any_lora, pair = B.pair;
  const int tbn = B.tbn, num_m = B.num_m;
  int rc = SS_OK;
  const CUtensorMap* d_tmaps = reinterpret_cast<const CUtensorMap*>(dv + B.off_tm);
  if ((rc = order_after_previous(ctx, stream))) return rc;
  const DevSeg* d_segs = reinterpret_cast<const DevSeg*>(dv + B.off_seg);
  // ---- K4 gather of the packed rows
  auto gather_params = [&](GatherParams& gp, int& grid) {
    gp.MX = (int)MX;
    gp.K = K;
    gp.ldx = (int)ldx;
    gp.n_piece = B.n_piece;
    gp.ia3_in_prologue = bwd ? 1 : 0;
    gp.segs = d_segs;
    gp.piece_seg = reinterpret_cast<const int32_t*>(dv + B.off_piece);
    gp.X = ctx->X;
    gp.row_seg = ctx->row_seg;
    gp.X_lo = B.any_lo ? ctx->X_lo : nullptr;
    // several warps per row when the dispatch has too few rows to fill the GPU
    gp.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>((K / 8 + 127) / 128, ((int64_t)ctx->num_sms * 16 + MX - 1) / MX));
    grid = (int)std::min<int64_t>((MX * gp.nsplit + 7) / 8, (int64_t)ctx->num_sms * 8);
  };
  auto launch_gather = [&]() -> int {
    GatherParams gp;
    int grid = 0;
    gather_params(gp, grid);
    const int pi = prof_begin(ctx, stream, SS_KERNEL_GATHER, 0.0, B.gather_bytes);
    CK(launch_k(ctx, gather_rows_kernel, grid, 256, 0, stream, gp));
    prof_end(ctx, stream, pi);
    CK(cudaGetLastError());
    ctx->launches++;
    return SS_OK;
  };

  CUtensorMap tmAL = L.tm_w_fwd;  // (unused without LoRA)
  // one CTA per slab walking every K chunk when there are enough slabs to fill the GPU and the
  // ranks fit the register sums; else one CTA per (slab, chunk). Same sums either way.
  const bool whole = B.shrink_chunks_ == 1 ||
                     (B.part_ld <= 64 && (ctx->shrink_mode == 1 || (ctx->shrink_mode == 0 && B.n_items >= ctx->num_sms)));
  const int shrink_ctas = any_lora ? B.n_items * (whole ? 1 : B.shrink_chunks_) : 0;
  // decode-only dispatch whose LoRA shrink is all decode-class items reading rows in place: the
  // shrink and the gather share one launch (no side stream, the GEMM keeps its PDL edge)
  const bool prologue = ctx->decode_prologue && any_lora && MX > 0 && num_m == 0 && B.n_items == 0 &&
                        B.n_ditems > 0 && B.shrink_indep && !ctx->profiling && !ctx->decode_split;
  const bool side = !prologue && any_lora && MX > 0 && B.shrink_indep && ctx->side_shrink && !ctx->profiling;
  // Overlap (streaming kernel): the GEMM does not wait for the side-stream shrink; its producer
  // waits on the shrink's completion counter right before the LoRA stages. Only when the
  // shrink's CTAs (2 per SM) and the GEMM's fit on the GPU together, so neither can starve.
  const int gemm_ctas = (int)std::min<int64_t>((int64_t)num_m * ((N + 63) / 64), ctx->num_sms);
  const bool overlap = side && B.stream && ctx->lora_overlap && gemm_ctas + (shrink_ctas + 1) / 2 <= ctx->num_sms;
  // decode-only dispatch with a side-stream shrink: the decode GEMM's chunk groups run beside the
  // shrink (their own launch, right behind the gather); the LoRA groups after the join
  const bool dec_split = side && !overlap && ctx->decode_split && B.num_m == 0 && B.dec_groups > B.dec_chunk_groups;
  auto dec_shrink_params = [&](DecShrinkParams& dsp) {
    dsp.K = K;
    dsp.kbc = B.dec_kbc;
    dsp.C = B.dec_C;
    dsp.lora_ld = (int)lora_ld;
    dsp.segs = d_segs;
    dsp.items = reinterpret_cast<const DecShrinkItem*>(dv + B.off_di);
    dsp.pack = bwd ? L.b_pack : L.at_pack;
    dsp.pack_ld = bwd ? L.ld_b : L.ld_at;
    dsp.a_lora = ctx->a_lora;
    dsp.part = ctx->dshr_part;
    dsp.ticket = ctx->dshr_ticket;
  };
  auto launch_shrink = [&](cudaStream_t st) -> int {
    // the streaming kernel (<= 64 rows) reads the LoRA operand through a 64-row box too
    rc = encode_2d(ctx, &tmAL, ctx->a_lora, lora_ld, al_rows, lora_ld, 64, B.stream ? 64 : BM);
    if (rc) return rc;
    // ---- K3 shrink into the zeroed block-diagonal operand
    // (no memset: the shrink's first slab of each piece writes the block-diagonal zeros)
    ShrinkParams sp;
    sp.K = K;
    sp.lora_ld = (int)lora_ld;
    sp.segs = d_segs;
    sp.items = reinterpret_cast<const ShrinkItem*>(dv + B.off_it);
    sp.tmaps = d_tmaps;
    sp.a_lora = ctx->a_lora;
    sp.part = ctx->shrink_part;
    sp.part_ld = B.part_ld;
    sp.max_chunks = B.shrink_chunks_;
    sp.kb_chunk = B.kb_chunk;
    sp.ticket = ctx->shrink_ticket;
    const int pi = prof_begin(ctx, st, SS_KERNEL_SHRINK, B.shrink_flops, B.shrink_bytes);
    sp.K2 = K;
    sp.done_ctr = overlap ? ctx->sync_ctr : nullptr;
    if (B.n_items > 0) {
      CK(launch_k(ctx, lora_shrink_kernel, dim3(B.n_items, whole ? 1 : B.shrink_chunks_), GEMM_THREADS, SHRINK_SMEM,
                  st, bwd ? L.tm_b : L.tm_at, bwd ? L.tm_b : L.tm_at, sp));
      ctx->launches++;
    }
    if (B.n_ditems > 0) {
      DecShrinkParams dsp;
      dec_shrink_params(dsp);
      const int rmax = std::max(16, B.dec_rank_max);
      const dim3 g(B.n_ditems, B.dec_C, (rmax + 31) / 32);
      const size_t smem = (size_t)DEC_SHR_MAXROWS * B.dec_kbc * 64 * sizeof(float);
      if (B.dec_rows_max <= 4) CK(launch_k(ctx, dec_shrink_kernel<4>, g, DEC_SHR_THREADS, smem, st, dsp));
      else CK(launch_k(ctx, dec_shrink_kernel<DEC_SHR_MAXROWS>, g, DEC_SHR_THREADS, smem, st, dsp));
      ctx->launches++;
    }
    prof_end(ctx, st, pi);
    CK(cudaGetLastError());
    return SS_OK;
  };
  // The shrink reads the client rows in place (no packed rows) -> it runs on the side stream
  // beside the gather: fork after everything queued so far (the previous dispatch's GEMM reads
  // the LoRA operand the shrink rewrites), join before the GEMM.
  if (side) {
    CK(cudaEventRecord(ctx->ev_fork, stream));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    if ((rc = launch_shrink(ctx->side))) return rc;
    CK(cudaEventRecord(ctx->ev_join, ctx->side));
    if ((rc = launch_gather())) return rc;
    if (!overlap && !dec_split) CK(cudaStreamWaitEvent(stream, ctx->ev_join, 0));
  } else if (prologue) {
    // decode-only dispatch: shrink + gather in one launch (dec_prologue_kernel)
    rc = encode_2d(ctx, &tmAL, ctx->a_lora, lora_ld, al_rows, lora_ld, 64, B.stream ? 64 : BM);
    if (rc) return rc;
    DecShrinkParams dsp;
    dec_shrink_params(dsp);
    GatherParams gp;
    int ggrid = 0;
    gather_params(gp, ggrid);
    const int sy = B.dec_C, sz = (std::max(16, B.dec_rank_max) + 31) / 32;
    const int n_shr = B.n_ditems * sy * sz;
    const size_t smem = (size_t)DEC_SHR_MAXROWS * B.dec_kbc * 64 * sizeof(float);
    const int pi = prof_begin(ctx, stream, SS_KERNEL_SHRINK, B.shrink_flops, B.shrink_bytes + B.gather_bytes);
    if (B.dec_rows_max <= 4)
      CK(launch_k(ctx, dec_prologue_kernel<4>, n_shr + ggrid, DEC_SHR_THREADS, smem, stream, dsp, gp, n_shr, sy, sz));
    else
      CK(launch_k(ctx, dec_prologue_kernel<DEC_SHR_MAXROWS>, n_shr + ggrid, DEC_SHR_THREADS, smem, stream, dsp, gp,
                  n_shr, sy, sz));
    prof_end(ctx, stream, pi);
    CK(cudaGetLastError());
    ctx->launches++;
  } else {
    if (MX > 0 && (rc = launch_gather())) return rc;
    if (any_lora && (rc = launch_shrink(stream))) return rc;
  }

  // ---- K1 / K2 / K5 fused GEMM
  GemmParams gpm;
  gpm.N = N;
  gpm.K = K;
  gpm.num_m_tiles = num_m;
  const int pn = B.pn;                      // CTA-pair tile width (256 or 512)
  gpm.num_n_tiles = pair ? (N + pn - 1) / pn : (N + tbn - 1) / tbn;
  // long-K dispatches: a raster group's A rows (group_m x 256 rows x K) must stay in L2 while W
  // streams past; at K = 13824 sixteen pair M-tiles are 113 MB
  gpm.group_m = (ctx->group_m_longk > 0 && K >= ctx->longk) ? ctx->group_m_longk : ctx->group_m;
  gpm.group_n = 0;
  {
    // DRAM bytes of the two raster orders (A = the dispatch rows, W = the layer; outputs equal)
    const int tn = pair ? pn : tbn;
    const double a_bytes = (double)B.M * K * 2, w_bytes = (double)K * N * 2;
    const int nn = gpm.num_n_tiles;
    int h = ctx->group_n > 0 ? ctx->group_n
                             : (int)std::max<int64_t>(1, ((int64_t)ctx->l2_budget_mb << 20) / ((int64_t)tn * K * 2));
    h = std::min(h, nn);
    const double t_m = a_bytes + w_bytes * ((num_m + ctx->group_m - 1) / ctx->group_m);
    const double t_n = w_bytes + a_bytes * ((nn + h - 1) / h);
    if (ctx->raster == 1 || (ctx->raster < 0 && t_n < t_m)) gpm.group_n = h;
  }
  gpm.hint_a = (ctx->l2_hints && gpm.group_n == 0) ? 2 : 0;
  gpm.hint_b = (ctx->l2_hints && gpm.group_n > 0) ? 2 : 0;
  gpm.hint_out = ctx->l2_hints ? 1 : 0;
  gpm.a_bytes = B.a_rows64 ? A_STAGE_BYTES / 2 : A_STAGE_BYTES;
  gpm.lora_ready = overlap ? ctx->sync_ctr : nullptr;
  gpm.lora_expect = overlap ? shrink_ctas : 0;
  // the streaming GEMM starts behind the kernel before it (gather, or the main-stream shrink)
  // and streams its first W stages meanwhile; not across the side-stream join event
  const bool early = B.stream && ctx->stream_pdl && !ctx->profiling && MX > 0 && !(side && !overlap);
  gpm.pdl_early = early ? 1 : 0;
  gpm.has_bias = (pass_kind == SS_PASS_FORWARD && L.bias) ? 1 : 0;
  gpm.any_lora = any_lora ? 1 : 0;
  gpm.ia3_in_epilogue = (pass_kind != SS_PASS_BACKWARD) ? 1 : 0;
  gpm.bias = L.bias;
  gpm.segs = d_segs;
  gpm.row_seg = ctx->row_seg;
  gpm.tiles = reinterpret_cast<const TileDesc*>(dv + B.off_tile);
  gpm.chunks = reinterpret_cast<const int32_t*>(dv + B.off_ch);
  gpm.tmaps = d_tmaps;
  gpm.stores = reinterpret_cast<const int2*>(dv + B.off_st);
  const int ntiles = gpm.num_m_tiles * gpm.num_n_tiles;
  const int grid = pair ? 2 * std::min(ntiles, ctx->num_sms / 2) : std::min(ntiles, ctx->num_sms);
  const CUtensorMap& tmBP = any_lora ? (bwd ? L.tm_at : L.tm_b) : L.tm_w_fwd;
  const int pg = num_m > 0 ? prof_begin(ctx, stream, SS_KERNEL_GEMM, B.gemm_flops, B.gemm_bytes) : -1;
  if (num_m == 0) {
    // only decode-class rows: no single-chain GEMM
  } else if (B.stream) {
    if (bwd)
      CK(launch_kp(early || (ctx->pdl && !ctx->profiling), seg_gemm_stream_kernel<true>, grid, GEMM_THREADS,
                   STREAM_SMEM, stream, L.tm_w_bwd_s, tmAL, tmBP, gpm));
    else
      CK(launch_kp(early || (ctx->pdl && !ctx->profiling), seg_gemm_stream_kernel<false>, grid, GEMM_THREADS,
                   STREAM_SMEM, stream, L.tm_w_fwd_s, tmAL, tmBP, gpm));
  } else if (pair && pn == 256 && ctx->cluster4 && num_m >= 2 && !B.any_lo) {
    const int ng = (int)std::min<int64_t>((int64_t)((num_m + 1) / 2) * gpm.num_n_tiles, ctx->num_sms / 4);
    if (bwd)
      CK(launch_k(ctx, seg_gemm4_kernel<true>, 4 * ng, GEMM_THREADS, GEMM4_SMEM, stream, L.tm_w_bwd64, tmAL, tmBP, gpm));
    else
      CK(launch_k(ctx, seg_gemm4_kernel<false>, 4 * ng, GEMM_THREADS, GEMM4_SMEM, stream, L.tm_w_fwd, tmAL, tmBP, gpm));
  } else if (pair && pn == 512) {
    // Tail split: when the last wave of 512-wide tiles is under half full (T = W x P + r, r < P/2
    // clusters), the last r + P raster tiles run as 2 (r + P) 256-wide tiles in a second launch
    // that fills the SMs the first one frees: W + 1/2 wave times instead of W + 1 (the two
    // kernels give every output element the same bits, tests/test_gpu_parity.py).
    const int P = grid / 2;
    const int T = ntiles;
    const int r = T % P;
    // (N a multiple of 512: no 256-wide half starts past the last column)
    const bool split = ctx->tail_split && r > 0 && 2 * r < P && T > 2 * P && N % 512 == 0;
    GemmParams g1 = gpm;
    if (split) g1.tiles_total = T - (r + P);
    if (bwd)
      CK(launch_k(ctx, seg_gemm2_kernel<true, 512>, grid, PairCfg<512>::THREADS, GEMM2W_SMEM, stream, L.tm_w_bwd2, tmAL, tmBP, g1));
    else
      CK(launch_k(ctx, seg_gemm2_kernel<false, 512>, grid, PairCfg<512>::THREADS, GEMM2W_SMEM, stream, L.tm_w_fwd, tmAL, tmBP, g1));
    if (split) {
      GemmParams g2 = gpm;
      g2.tail_from = T - (r + P);
      g2.tail_nn = gpm.num_n_tiles;
      g2.tiles_total = 2 * (r + P);
      g2.wait_at_end = 1;
      const int grid2 = 2 * std::min(g2.tiles_total, ctx->num_sms / 2);
      const bool tpdl = !ctx->profiling;
      if (bwd)
        CK(launch_kp(tpdl, seg_gemm2_kernel<true, 256>, grid2, GEMM_THREADS, GEMM2_SMEM, stream, L.tm_w_bwd2, tmAL, tmBP, g2));
      else
        CK(launch_kp(tpdl, seg_gemm2_kernel<false, 256>, grid2, GEMM_THREADS, GEMM2_SMEM, stream, L.tm_w_fwd, tmAL, tmBP, g2));
      ctx->launches++;
    }
  } else if (pair) {
    if (bwd)
      CK(launch_k(ctx, seg_gemm2_kernel<true, 256>, grid, GEMM_THREADS, GEMM2_SMEM, stream, L.tm_w_bwd2, tmAL, tmBP, gpm));
    else
      CK(launch_k(ctx, seg_gemm2_kernel<false, 256>, grid, GEMM_THREADS, GEMM2_SMEM, stream, L.tm_w_fwd, tmAL, tmBP, gpm));
  } else if (tbn == 256) {
    if (bwd) CK(launch_k(ctx, seg_gemm_kernel<true, 256>, grid, GEMM_THREADS, TileCfg<256>::SMEM, stream, L.tm_w_bwd, tmAL, tmBP, gpm));
    else CK(launch_k(ctx, seg_gemm_kernel<false, 256>, grid, GEMM_THREADS, TileCfg<256>::SMEM, stream, L.tm_w_fwd, tmAL, tmBP, gpm));
  } else if (tbn == 128) {
    if (bwd) CK(launch_k(ctx, seg_gemm_kernel<true, 128>, grid, GEMM_THREADS, TileCfg<128>::SMEM, stream, L.tm_w_bwd2, tmAL, tmBP, gpm));
    else CK(launch_k(ctx, seg_gemm_kernel<false, 128>, grid, GEMM_THREADS, TileCfg<128>::SMEM, stream, L.tm_w_fwd, tmAL, tmBP, gpm));
  } else {
    if (bwd) CK(launch_k(ctx, seg_gemm_kernel<true, 64>, grid, GEMM_THREADS, TileCfg<64>::SMEM, stream, L.tm_w_bwd64, tmAL, tmBP, gpm));
    else CK(launch_k(ctx, seg_gemm_kernel<false, 64>, grid, GEMM_THREADS, TileCfg<64>::SMEM, stream, L.tm_w_fwd, tmAL, tmBP, gpm));
  }
  if (num_m > 0) {
    prof_end(ctx, stream, pg);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  if (overlap) CK(cudaStreamWaitEvent(stream, ctx->ev_join, 0));   // join the side stream
  // ---- K1d: decode-class rows, persistent split-K (dec_C chunks + a LoRA chain per tile) + fixup
  if (B.n_dec > 0) {
    CUtensorMap tmALd = L.tm_w_fwd;   // (unused without LoRA)
    if (any_lora && (rc = encode_2d(ctx, &tmALd, ctx->a_lora, lora_ld, al_rows, lora_ld, 64, DEC_ROWS))) return rc;
    DecParams dp;
    dp.N = N;
    dp.K = K;
    dp.C = B.dec_C;
    dp.kbc = B.dec_kbc;
    dp.n_m = B.n_dec;
    dp.n_n = (N + DEC_TN - 1) / DEC_TN;
    dp.S = B.dec_S;
    dp.has_bias = gpm.has_bias;
    dp.ia3_in_epilogue = gpm.ia3_in_epilogue;
    dp.bias = L.bias;
    dp.segs = d_segs;
    dp.row_seg = ctx->row_seg;
    dp.tiles = reinterpret_cast<const DecTile*>(dv + B.off_dt);
    dp.chunks = gpm.chunks;
    dp.groups = reinterpret_cast<const int4*>(dv + B.off_dcb);
    dp.lpieces = reinterpret_cast<const int2*>(dv + B.off_lp);
    dp.lstages = reinterpret_cast<const int4*>(dv + B.off_ls);
    dp.tmaps = d_tmaps;
    dp.amap = B.dec_amap;
    dp.alo_map = B.dec_alo;
    dp.part = ctx->dec_part;
    dp.trace = ctx->decode_trace;
    // streams its first W stages behind the kernel before it when that is the gather or the
    // main-stream shrink of this dispatch (PDL edge; not across an event join)
    const bool dec_early = ctx->stream_pdl && !ctx->profiling && MX > 0 && (!side || dec_split) && num_m == 0;
    const bool dpdl = (ctx->pdl || dec_early) && !ctx->profiling;
    const int pd = prof_begin(ctx, stream, SS_KERNEL_GEMM, B.dec_flops, B.dec_bytes);
    const CUtensorMap& tmBP64 = any_lora ? (bwd ? L.tm_at64 : L.tm_b64) : L.tm_w_fwd;
    auto launch_dec = [&](int g0, int g1, int* claim, bool early, bool pdl) -> int {
      dp.g_begin = g0;
      dp.g_end = g1;
      dp.claim = claim;
      dp.pdl_early = early ? 1 : 0;
      const int dgrid = std::min(g1 - g0, ctx->num_sms);
      if (bwd) CK(launch_kp(pdl, seg_gemm_dec_kernel<true>, dgrid, GEMM_THREADS, DEC_SMEM, stream, L.tm_w_dec, tmALd, tmBP, tmBP64, dp));
      else CK(launch_kp(pdl, seg_gemm_dec_kernel<false>, dgrid, GEMM_THREADS, DEC_SMEM, stream, L.tm_w_dec, tmALd, tmBP, tmBP64, dp));
      ctx->launches++;
      return SS_OK;
    };
    const bool fx_fused = ctx->decode_fixup_fused && !dec_split;
    dp.fx_claim = fx_fused ? ctx->dec_fx : nullptr;
    dp.fx_cnt = fx_fused ? ctx->dec_fx + 1 : nullptr;
    if (dec_split) {
      if ((rc = launch_dec(0, B.dec_chunk_groups, ctx->dec_claim, dec_early, dpdl))) return rc;
      CK(cudaStreamWaitEvent(stream, ctx->ev_join, 0));   // the shrink's A_lora
      if ((rc = launch_dec(B.dec_chunk_groups, B.dec_groups, ctx->dec_claim + 2, false, false))) return rc;
    } else {
      if ((rc = launch_dec(0, B.dec_groups, ctx->dec_claim, dec_early, dpdl))) return rc;
    }
    if (!fx_fused) {
      CK(launch_kp(dpdl, dec_fixup_kernel, dp.n_n * dp.n_m * (DEC_ROWS / DEC_FIX_ROWS), DEC_FIX_THREADS, 0, stream, dp));
      ctx->launches += 1;
    }
    prof_end(ctx, stream, pd);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(ctx->compute_done, stream));
  ctx->any_compute = true;
  return SS_OK;
}


// Row-block copy between host and device; a plain 1-D copy when both sides are dense (the 2-D
// engine path is measurably slower for host-to-device on this part).
cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                      size_t rows, cudaMemcpyKind kind, cudaStream_t st) {
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, kind, st);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, st);
}

struct KernelAttrs {
  bool done = false;
};
KernelAttrs g_attrs;

int set_kernel_attrs(ss_ctx* ctx) {
  if (g_attrs.done) return SS_OK;
  CK(cudaFuncSetAttribute(seg_gemm_kernel<false, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          TileCfg<256>::SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_kernel<true, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          TileCfg<256>::SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_kernel<false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          TileCfg<128>::SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_kernel<true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          TileCfg<128>::SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_kernel<false, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          TileCfg<64>::SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_kernel<true, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          TileCfg<64>::SMEM));
  CK(cudaFuncSetAttribute(seg_gemm2_kernel<false, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          GEMM2_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm2_kernel<true, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          GEMM2_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm2_kernel<false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          GEMM2W_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm2_kernel<true, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          GEMM2W_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm4_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM4_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm4_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM4_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_stream_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          STREAM_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_stream_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          STREAM_SMEM));
  CK(cudaFuncSetAttribute(lora_shrink_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          SHRINK_SMEM));
  CK(cudaFuncSetAttribute(seg_gemm_dec_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DEC_SMEM));
  CK(cudaFuncSetAttribute(dec_shrink_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          DEC_SHR_MAXROWS * DEC_MAX_KBC * 64 * (int)sizeof(float)));
  CK(cudaFuncSetAttribute(dec_shrink_kernel<DEC_SHR_MAXROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          DEC_SHR_MAXROWS * DEC_MAX_KBC * 64 * (int)sizeof(float)));
  CK(cudaFuncSetAttribute(dec_prologue_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          DEC_SHR_MAXROWS * DEC_MAX_KBC * 64 * (int)sizeof(float)));
  CK(cudaFuncSetAttribute(dec_prologue_kernel<DEC_SHR_MAXROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          DEC_SHR_MAXROWS * DEC_MAX_KBC * 64 * (int)sizeof(float)));
  CK(cudaFuncSetAttribute(seg_gemm_dec_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DEC_SMEM));
  CK(cudaFuncSetAttribute(lora_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GRAD_SMEM));
  CK(cudaFuncSetAttribute(lora_grad_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GRAD_FUSED_SMEM));
  g_attrs.done = true;
  return SS_OK;
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

const char* ss_version(void) {
  return "ss_b200 1.0 (sm_100a tcgen05/TMEM/TMA segmented executor; CTA-pair 256x512 / 256x256, single-CTA 128x{256,128,64}, weight-streaming 128x64)";
}

const char* ss_last_error(const ss_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int ss_ctx_create(int device, int tp_rank, int tp_size, ss_ctx** out) {
  if (!out) return SS_E_ARG;
  *out = nullptr;
  ss_ctx* ctx = new ss_ctx();
  ctx->device = device;
  ctx->tp_rank = tp_rank;
  ctx->tp_size = tp_size;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return SS_E_CUDA;
  }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (major != 10) {
    delete ctx;
    return SS_E_UNSUPPORTED;  // sm_100a only
  }
  // The GEMM / shrink overlap needs both kernels resident at once; tools that serialise kernel
  // launches (ncu, compute-sanitizer, CUDA_LAUNCH_BLOCKING) would leave the GEMM waiting.
  {
    const char* inj = getenv("CUDA_INJECTION64_PATH");
    const char* blk = getenv("CUDA_LAUNCH_BLOCKING");
    if ((inj && *inj) || (blk && *blk == '1')) ctx->serial_launches = 1;
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn) {
    delete ctx;
    return SS_E_CUDA;
  }
  ctx->encode = reinterpret_cast<PFN_encodeTiled_t>(fn);
  if (cudaStreamCreateWithFlags(&ctx->upload, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->upload_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->compute_done, cudaEventDisableTiming) != cudaSuccess) {
    delete ctx;
    return SS_E_CUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&ctx->sync_ctr, 2 * sizeof(int)) != cudaSuccess ||
      cudaMemset(ctx->sync_ctr, 0, 2 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&ctx->dec_claim, 4 * sizeof(int)) != cudaSuccess ||
      cudaMemset(ctx->dec_claim, 0, 4 * sizeof(int)) != cudaSuccess) {
    delete ctx;
    return SS_E_CUDA;
  }
  for (auto& hs : ctx->hslot) {
    if (cudaEventCreateWithFlags(&hs.ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&hs.ev_comp, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&hs.ev_out, cudaEventDisableTiming) != cudaSuccess) {
      delete ctx;
      return SS_E_CUDA;
    }
  }
  for (auto& s : ctx->staging) {
    if (cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) {
      delete ctx;
      return SS_E_CUDA;
    }
  }
  if (set_kernel_attrs(ctx) != SS_OK) {
    delete ctx;
    return SS_E_CUDA;
  }
  cudaEventRecord(ctx->upload_done, ctx->upload);
  *out = ctx;
  return SS_OK;
}

int ss_ctx_destroy(ss_ctx* ctx) {
  if (!ctx) return SS_E_ARG;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  zc_cache_clear(ctx);
  for (auto& kv : ctx->layers) {
    Layer& L = kv.second;
    cudaFree(L.W);
    cudaFree(L.bias);
    cudaFree(L.at_pack);
    cudaFree(L.b_pack);
    for (auto& a : L.adapters) cudaFree(a.second.ia3);
  }
  cudaFree(ctx->X);
  cudaFree(ctx->X_lo);
  cudaFree(ctx->ha_in);
  cudaFree(ctx->ha_out);
  cudaFree(ctx->ha_base);
  for (cudaEvent_t e : ctx->chunk_ev) cudaEventDestroy(e);
  cudaFree(ctx->a_lora);
  cudaFree(ctx->row_seg);
  cudaFree(ctx->qx);
  cudaFree(ctx->ia3_part);
  cudaFree(ctx->shrink_part);
  cudaFree(ctx->shrink_ticket);
  cudaFree(ctx->dec_part);
  cudaFree(ctx->dec_fx);
  cudaFree(ctx->dec_claim);
  cudaFree(ctx->dshr_part);
  cudaFree(ctx->dshr_ticket);
  cudaFree(ctx->grad_sync);
  cudaFree(ctx->fr_in);
  cudaFree(ctx->fr_out);
  cudaFree(ctx->fr_x);
  cudaFree(ctx->fr_o);
  for (auto& s : ctx->staging) {
    cudaFreeHost(s.host);
    cudaFree(s.dev);
    cudaEventDestroy(s.done);
  }
  cudaEventDestroy(ctx->upload_done);
  cudaEventDestroy(ctx->compute_done);
  cudaStreamDestroy(ctx->upload);
  for (auto& hs : ctx->hslot) {
    cudaFree(hs.in);
    cudaFree(hs.out);
    cudaFree(hs.base);
    cudaEventDestroy(hs.ev_in);
    cudaEventDestroy(hs.ev_comp);
    cudaEventDestroy(hs.ev_out);
  }
  for (auto& hc : ctx->hconv) {
    if (hc.ev) cudaEventSynchronize(hc.ev);
    cudaFreeHost(hc.buf);
    if (hc.ev) cudaEventDestroy(hc.ev);
  }
  ctx->pool.reset();
  cudaStreamDestroy(ctx->h2d);
  cudaStreamDestroy(ctx->d2h);
  cudaStreamDestroy(ctx->side);
  cudaFree(ctx->sync_ctr);
  cudaEventDestroy(ctx->ev_fork);
  cudaEventDestroy(ctx->ev_join);
  delete ctx;
  return SS_OK;
}

int ss_set_option(ss_ctx* ctx, const char* key, int64_t value) {
  if (!ctx || !key) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  ctx->opt_epoch++;   // options shape the built tables: cached dispatches rebuild
  if (!strcmp(key, "zc_cache")) {
    ctx->zc_cache_on = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "ia3_lo")) {
    if (value < 0 || value > 2) return fail(ctx, SS_E_ARG, "ia3_lo must be 0, 1 or 2");
    ctx->ia3_lo = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "lora_hilo")) {
    if (value < 0 || value > 2) return fail(ctx, SS_E_ARG, "lora_hilo must be 0, 1 or 2");
    ctx->lora_hilo = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "shrink_mode")) {
    if (value < 0 || value > 2) return fail(ctx, SS_E_ARG, "shrink_mode must be 0 (auto), 1 (whole) or 2 (split)");
    ctx->shrink_mode = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "shrink_kb_chunk")) {
    if (value < 1) return fail(ctx, SS_E_ARG, "shrink_kb_chunk must be >= 1");
    ctx->shrink_kb_chunk = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "pipeline_rows")) {
    if (value < 1) return fail(ctx, SS_E_ARG, "pipeline_rows must be >= 1");
    ctx->pipeline_rows = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "pipeline_bytes")) {
    if (value < 1) return fail(ctx, SS_E_ARG, "pipeline_bytes must be >= 1");
    ctx->pipeline_bytes = value;
    return SS_OK;
  }
  if (!strcmp(key, "pair_n")) {
    if (value != 0 && value != 256 && value != 512)
      return fail(ctx, SS_E_ARG, "pair_n must be 0 (auto), 256 or 512");
    ctx->pair_n = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "tma_store")) {
    ctx->tma_store = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "tile_n")) {
    if (value != 0 && value != 64 && value != 128 && value != 256)
      return fail(ctx, SS_E_ARG, "tile_n must be 0 (auto), 64, 128 or 256");
    ctx->force_tbn = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "direct_tiles")) {
    ctx->direct_tiles = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "gemm_2cta")) {
    ctx->gemm_2cta = value < 0 ? -1 : (value ? 1 : 0);
    return SS_OK;
  }
  if (!strcmp(key, "raster")) {
    ctx->raster = value < 0 ? -1 : (value ? 1 : 0);
    return SS_OK;
  }
  if (!strcmp(key, "group_n")) {
    if (value < 0) return fail(ctx, SS_E_ARG, "group_n must be >= 0");
    ctx->group_n = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "l2_budget_mb")) {
    if (value < 1) return fail(ctx, SS_E_ARG, "l2_budget_mb must be >= 1");
    ctx->l2_budget_mb = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "zero_copy_bytes")) {
    if (value < 0) return fail(ctx, SS_E_ARG, "zero_copy_bytes must be >= 0");
    ctx->zero_copy_bytes = value;
    return SS_OK;
  }
  if (!strcmp(key, "force_remote")) {
    ctx->force_remote = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "decode_rows")) {
    if (value < 0 || value > DEC_SHR_MAXROWS) return fail(ctx, SS_E_ARG, "decode_rows must be 0..%d", DEC_SHR_MAXROWS);
    ctx->decode_rows = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "host_convert")) {
    ctx->host_convert = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "host_threads")) {
    if (value < 0 || value > 256) return fail(ctx, SS_E_ARG, "host_threads must be 0..256");
    ctx->host_threads = (int)value;
    ctx->pool.reset();
    return SS_OK;
  }
  if (!strcmp(key, "decode_lora_piece")) {
    if (value < 1 || value > 1024) return fail(ctx, SS_E_ARG, "decode_lora_piece must be 1..1024");
    ctx->decode_lora_piece = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "tail_split")) {
    ctx->tail_split = value ? 1 : 0;
    ctx->opt_epoch++;
    return SS_OK;
  }
  if (!strcmp(key, "decode_fixup_fused")) {
    ctx->decode_fixup_fused = value ? 1 : 0;
    ctx->opt_epoch++;
    return SS_OK;
  }
  if (!strcmp(key, "decode_prologue")) {
    ctx->decode_prologue = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "decode_split")) {
    ctx->decode_split = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "grad_fused")) {
    ctx->grad_fused = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "grad_fused_lag")) {
    if (value < 0) return fail(ctx, SS_E_ARG, "grad_fused_lag must be >= 0");
    ctx->grad_fused_lag = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "decode_trace")) {
    ctx->decode_trace = reinterpret_cast<long long*>(static_cast<intptr_t>(value));
    return SS_OK;
  }
  if (!strcmp(key, "decode_chunk_kb")) {
    if (value < 1 || value > DEC_MAX_KBC) return fail(ctx, SS_E_ARG, "decode_chunk_kb must be 1..%d", DEC_MAX_KBC);
    ctx->decode_chunk_kb = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "wide_decode")) {
    ctx->wide_decode = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "stream_pdl")) {
    ctx->stream_pdl = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "lora_overlap")) {
    ctx->lora_overlap = (value && !ctx->serial_launches) ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "side_shrink")) {
    ctx->side_shrink = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "cluster4")) {
    ctx->cluster4 = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "pdl")) {
    ctx->pdl = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "stream_gemm")) {
    ctx->stream_gemm = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "a_rows64")) {
    ctx->a_rows64 = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "l2_hints")) {
    ctx->l2_hints = value ? 1 : 0;
    return SS_OK;
  }
  if (!strcmp(key, "group_m_longk")) {
    if (value < 0) return fail(ctx, SS_E_ARG, "group_m_longk must be >= 0");
    ctx->group_m_longk = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "longk")) {
    if (value < 1) return fail(ctx, SS_E_ARG, "longk must be >= 1");
    ctx->longk = (int)value;
    return SS_OK;
  }
  if (!strcmp(key, "group_m")) {
    if (value < 1) return fail(ctx, SS_E_ARG, "group_m must be >= 1");
    ctx->group_m = (int)value;
    return SS_OK;
  }
  return fail(ctx, SS_E_ARG, "unknown option %s", key);
}

int ss_load_layer(ss_ctx* ctx, int block, int role, int d_in, int d_out, const void* weight,
                  int64_t w_ld, const void* bias, uint32_t flags) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  if (d_in <= 0 || d_out <= 0 || !weight || w_ld < d_out)
    return fail(ctx, SS_E_ARG, "bad layer dims d_in=%d d_out=%d ld=%lld", d_in, d_out,
                (long long)w_ld);
  CK(cudaSetDevice(ctx->device));
  ss_unload_layer(ctx, block, role);
  Layer L;
  L.block = block;
  L.role = role;
  L.d_in = d_in;
  L.d_out = d_out;
  L.ldw = round_up(d_out, 64);
  L.ld_at = round_up(d_in, 64);
  L.ld_b = round_up(d_out, 64);
  CK(cudaMalloc(&L.W, (size_t)d_in * L.ldw * 2));
  CK(cudaMemsetAsync(L.W, 0, (size_t)d_in * L.ldw * 2, ctx->upload));
  int rc = upload_bf16(ctx, weight, flags, d_in, d_out, w_ld, L.W, L.ldw, false);
  if (rc) { cudaFree(L.W); return rc; }
  if (bias) {
    CK(cudaMalloc(&L.bias, (size_t)round_up(d_out, 64) * 4));
    CK(cudaMemsetAsync(L.bias, 0, (size_t)round_up(d_out, 64) * 4, ctx->upload));
    rc = upload_f32(ctx, bias, flags, d_out, L.bias);
    if (rc) return rc;
  }
  rc = encode_2d(ctx, &L.tm_w_fwd, L.W, d_out, d_in, L.ldw, 64, BK);
  if (rc) return rc;
  rc = encode_2d(ctx, &L.tm_w_bwd, L.W, d_out, d_in, L.ldw, 64, BN);
  if (rc) return rc;
  rc = encode_2d(ctx, &L.tm_w_bwd2, L.W, d_out, d_in, L.ldw, 64, BN / 2);
  if (rc) return rc;
  rc = encode_2d(ctx, &L.tm_w_bwd64, L.W, d_out, d_in, L.ldw, 64, 64);
  if (rc) return rc;
  // weight-streaming kernel: forward box {64 n, 256 k}; backward 4 K-chunks of 64 rows at once
  rc = encode_2d(ctx, &L.tm_w_fwd_s, L.W, d_out, d_in, L.ldw, 64, SK);
  if (rc) return rc;
  rc = encode_kchunks(ctx, &L.tm_w_bwd_s, L.W, L.ldw, d_in, L.ldw, 64, 4);
  if (rc) return rc;
  // split-K decode kernel: {64, 64} boxes of W (forward {64 n, 64 k}, backward {64 k, 64 n})
  rc = encode_2d(ctx, &L.tm_w_dec, L.W, d_out, d_in, L.ldw, 64, 64);
  if (rc) return rc;
  ctx->weight_bytes += (int64_t)d_in * L.ldw * 2 + (bias ? round_up(d_out, 64) * 4 : 0);
  ctx->layers[{block, role}] = L;
  return SS_OK;
}

int ss_unload_layer(ss_ctx* ctx, int block, int role) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  auto it = ctx->layers.find({block, role});
  if (it == ctx->layers.end()) return SS_E_NOLAYER;
  cudaDeviceSynchronize();
  Layer& L = it->second;
  ctx->weight_bytes -= (int64_t)L.d_in * L.ldw * 2 + (L.bias ? round_up(L.d_out, 64) * 4 : 0);
  cudaFree(L.W);
  cudaFree(L.bias);
  if (L.at_pack) ctx->adapter_bytes -= (int64_t)L.pack_cap * (L.ld_at + L.ld_b) * 2;
  cudaFree(L.at_pack);
  cudaFree(L.b_pack);
  for (auto& a : L.adapters) {
    if (a.second.ia3) ctx->adapter_bytes -= (int64_t)L.d_out * 4;
    cudaFree(a.second.ia3);
  }
  ctx->layers.erase(it);
  ctx->ad_epoch++;
  return SS_OK;
}

int ss_set_adapter(ss_ctx* ctx, uint32_t client_id, int block, int role, uint32_t kind, int rank,
                   float scale, const void* A, const void* B, const void* l, uint32_t flags) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  auto it = ctx->layers.find({block, role});
  if (it == ctx->layers.end())
    return fail(ctx, SS_E_NOLAYER, "unknown layer (%d, %d)", block, role);
  Layer& L = it->second;
  if (kind == 0 || (kind & ~(SS_ADAPTER_LORA | SS_ADAPTER_IA3)))
    return fail(ctx, SS_E_ARG, "bad adapter kind %u", kind);
  if ((kind & SS_ADAPTER_LORA) && (rank <= 0 || rank > SHRINK_MAXN || !A || !B))
    return fail(ctx, SS_E_ARG, "LoRA needs 1 <= rank <= %d and A, B (rank=%d)", SHRINK_MAXN, rank);
  if ((kind & SS_ADAPTER_IA3) && !l) return fail(ctx, SS_E_ARG, "IA3 needs l");
  CK(cudaSetDevice(ctx->device));
  int rc = upload_begin(ctx);
  if (rc) return rc;
  AdapterSlot& s = L.adapters[client_id];
  // cached tables (plans, zero-copy entries, graphs) bake the kind's segment flags and the
  // LoRA scale: any change of either invalidates them like a move does
  if (s.kind != kind || ((kind & SS_ADAPTER_LORA) && s.scale != scale)) ctx->ad_epoch++;
  if (kind & SS_ADAPTER_LORA) {
    const int rp = (int)round_up(rank, LORA_CHUNK);
    if (s.pack_row < 0 || s.rank_pad != rp) {
      // new block at the end of the packs (old block, if any, is abandoned: zero cost to
      // correctness since no segment references it any more)
      rc = grow_packs(ctx, L, L.pack_rows + rp);
      if (rc) return rc;
      s.pack_row = L.pack_rows;
      ctx->ad_epoch++;
      s.rank_pad = rp;
      L.pack_rows += rp;
    }
    s.rank = rank;
    s.scale = scale;
    // zero the padding rows, then A^T rows [pack_row, pack_row + rank) and B rows
    CK(cudaMemsetAsync(L.at_pack + (int64_t)s.pack_row * L.ld_at, 0, (size_t)rp * L.ld_at * 2,
                       ctx->upload));
    CK(cudaMemsetAsync(L.b_pack + (int64_t)s.pack_row * L.ld_b, 0, (size_t)rp * L.ld_b * 2,
                       ctx->upload));
    rc = upload_bf16(ctx, A, flags, L.d_in, rank, rank, L.at_pack + (int64_t)s.pack_row * L.ld_at,
                     L.ld_at, /*transpose=*/true);
    if (rc) return rc;
    rc = upload_bf16(ctx, B, flags, rank, L.d_out, L.d_out,
                     L.b_pack + (int64_t)s.pack_row * L.ld_b, L.ld_b, false);
    if (rc) return rc;
  }
  if (kind & SS_ADAPTER_IA3) {
    if (!s.ia3) {
      ctx->ad_epoch++;
      CK(cudaMalloc(&s.ia3, (size_t)round_up(L.d_out, 64) * 4));
      CK(cudaMemsetAsync(s.ia3, 0, (size_t)round_up(L.d_out, 64) * 4, ctx->upload));
      ctx->adapter_bytes += (int64_t)L.d_out * 4;
    }
    rc = upload_f32(ctx, l, flags, L.d_out, s.ia3);
    if (rc) return rc;
  }
  s.kind = kind;
  return upload_end(ctx);
}

int ss_clear_adapter(ss_ctx* ctx, uint32_t client_id, int block, int role) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  auto it = ctx->layers.find({block, role});
  if (it == ctx->layers.end()) return SS_E_NOLAYER;
  auto a = it->second.adapters.find(client_id);
  if (a == it->second.adapters.end()) return SS_OK;
  if (a->second.ia3) {
    cudaDeviceSynchronize();
    cudaFree(a->second.ia3);
    ctx->adapter_bytes -= (int64_t)it->second.d_out * 4;
  }
  it->second.adapters.erase(a);
  ctx->ad_epoch++;
  return SS_OK;
}

int ss_clear_client(ss_ctx* ctx, uint32_t client_id) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  for (auto& kv : ctx->layers) ss_clear_adapter(ctx, client_id, kv.first.first, kv.first.second);
  return SS_OK;
}

int ss_memory_stats(const ss_ctx* ctx, int64_t* w, int64_t* a, int64_t* ws) {
  if (!ctx) return SS_E_ARG;
  if (w) *w = ctx->weight_bytes;
  if (a) *a = ctx->adapter_bytes;
  if (ws) *ws = (int64_t)ctx->ws_high;
  return SS_OK;
}

int64_t ss_kernel_launches(const ss_ctx* ctx) { return ctx ? ctx->launches : -1; }

int ss_layer_dims(ss_ctx* ctx, int block, int role, int* d_in, int* d_out) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  auto it = ctx->layers.find({block, role});
  if (it == ctx->layers.end()) return SS_E_NOLAYER;
  if (d_in) *d_in = it->second.d_in;
  if (d_out) *d_out = it->second.d_out;
  return SS_OK;
}

int ss_ctx_device(const ss_ctx* ctx) { return ctx ? ctx->device : -1; }

uint64_t ss_ctx_epoch(const ss_ctx* ctx) {
  return ctx ? ctx->ws_epoch + ctx->ad_epoch + ctx->free_epoch : 0;
}

int ss_profile(ss_ctx* ctx, int enable) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  prof_drain(ctx);
  for (int k = 0; k < 4; ++k) {
    ctx->prof_ms[k] = ctx->prof_flops[k] = ctx->prof_bytes[k] = 0;
    ctx->prof_n[k] = 0;
  }
  ctx->profiling = enable != 0;
  return SS_OK;
}

int ss_profile_read(ss_ctx* ctx, int kernel, double* total_ms, int64_t* launches, double* flops,
                    double* bytes) {
  if (!ctx || kernel < 0 || kernel > 3) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  prof_drain(ctx);
  if (total_ms) *total_ms = ctx->prof_ms[kernel];
  if (launches) *launches = ctx->prof_n[kernel];
  if (flops) *flops = ctx->prof_flops[kernel];
  if (bytes) *bytes = ctx->prof_bytes[kernel];
  return SS_OK;
}

int ss_compute_batch(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg, const ss_seg* segs,
                     void* stream_, int32_t* seg_status) {
  if (!ctx) return SS_E_ARG;
  Built b;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  int rc = build_batch(ctx, pass_kind, block, role, n_seg, segs, seg_status, b);
  if (rc || b.M == 0) return rc;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  // routing tables -> pinned staging slot -> device (one async copy)
  Staging* stp = nullptr;
  if ((rc = acquire_staging(ctx, b.blob.size(), stp))) return rc;
  memcpy(stp->host, b.blob.data(), b.blob.size());
  // adapters uploaded on the side stream must be complete before this dispatch reads them
  CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
  CK(cudaMemcpyAsync(stp->dev, stp->host, b.blob.size(), cudaMemcpyHostToDevice, stream));
  CK(cudaEventRecord(stp->done, stream));
  stp->pending = true;
  return launch_batch(ctx, b, static_cast<char*>(stp->dev), stream);
}

// ---- prebuilt dispatch plans --------------------------------------------------------------
struct ss_plan {
  ss_ctx* ctx = nullptr;
  int pass_kind = 0, block = 0, role = 0;
  std::vector<ss_seg> segs;
  Built b;
  char* dev = nullptr;
  size_t dev_cap = 0;
};

static int plan_build(ss_plan* p, int32_t* seg_status) {
  ss_ctx* ctx = p->ctx;
  std::vector<int32_t> st(std::max<size_t>(1, p->segs.size()));
  int rc = build_batch(ctx, p->pass_kind, p->block, p->role, (int)p->segs.size(), p->segs.data(),
                       seg_status ? seg_status : st.data(), p->b);
  if (rc) return rc;
  if (p->b.M == 0) return SS_OK;
  if (p->dev) CK(cudaDeviceSynchronize());  // rebuild: no launch of this plan may still read p->dev
  if (p->dev_cap < p->b.blob.size()) {
    if (p->dev) CK(cudaFree(p->dev));
    p->dev = nullptr;
    p->dev_cap = 0;
    CK(cudaMalloc(&p->dev, p->b.blob.size()));
    p->dev_cap = p->b.blob.size();
  }
  CK(cudaMemcpy(p->dev, p->b.blob.data(), p->b.blob.size(), cudaMemcpyHostToDevice));
  return SS_OK;
}

int ss_plan_create(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg, const ss_seg* segs,
                   int32_t* seg_status, ss_plan** out) {
  if (!ctx || !out) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  *out = nullptr;
  if (n_seg < 0 || (n_seg > 0 && (!segs || !seg_status))) return fail(ctx, SS_E_ARG, "bad segment array");
  CK(cudaSetDevice(ctx->device));
  ss_plan* p = new ss_plan();
  p->ctx = ctx;
  p->pass_kind = pass_kind;
  p->block = block;
  p->role = role;
  p->segs.assign(segs, segs + n_seg);
  int rc = plan_build(p, seg_status);
  if (rc) {
    ss_plan_destroy(p);
    return rc;
  }
  *out = p;
  return SS_OK;
}

int ss_plan_launch(ss_plan* p, void* stream_) {
  if (!p) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(p->ctx->mu);
  ss_ctx* ctx = p->ctx;
  if (p->b.ws_epoch != ctx->ws_epoch || p->b.ad_epoch != ctx->ad_epoch) {
    // workspace grew or an adapter moved since the tables were built: rebuild them (a plan's
    // segments were validated at creation; a status change now is reported as an error)
    std::vector<int32_t> st(std::max<size_t>(1, p->segs.size()));
    std::vector<int32_t> st0(std::max<size_t>(1, p->segs.size()));
    for (size_t i = 0; i < p->segs.size(); ++i) st0[i] = p->b.status[i];
    int rc = plan_build(p, st.data());
    if (rc) return rc;
    for (size_t i = 0; i < p->segs.size(); ++i)
      if (st[i] != st0[i]) return fail(ctx, SS_E_ARG, "plan segment %zu status changed to %d", i, st[i]);
  }
  if (p->b.M == 0) return SS_OK;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  // (under CUDA-graph capture the adapter uploads must already be complete: the capture
  // cannot wait on an event recorded outside it)
  if (!capturing(stream)) CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
  return launch_batch(ctx, p->b, p->dev, stream);
}

int ss_plan_destroy(ss_plan* p) {
  if (!p) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(p->ctx->mu);
  if (p->dev) {
    cudaDeviceSynchronize();
    cudaFree(p->dev);
  }
  delete p;
  return SS_OK;
}

int ss_adapter_grads(ss_ctx* ctx, int block, int role, int n_seg, const ss_grad_seg* segs,
                     void* stream_, int32_t* seg_status) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  if (n_seg < 0 || (n_seg > 0 && (!segs || !seg_status))) return fail(ctx, SS_E_ARG, "bad segment array");
  auto lit = ctx->layers.find({block, role});
  if (lit == ctx->layers.end()) return fail(ctx, SS_E_NOLAYER, "unknown layer (%d, %d)", block, role);
  Layer& L = lit->second;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int d_in = L.d_in, d_out = L.d_out;

  // ---- validate; split into LoRA and IA3 work
  std::vector<DevSeg> sh;           // shrink records (pack_row, rank_pad, scale)
  std::vector<LoraGradSeg> lg;
  std::vector<const ss_grad_seg*> lsrc;
  std::vector<Ia3GradSeg> ig;
  int64_t qrows = 0;
  int qld = 64;
  for (int i = 0; i < n_seg; ++i) {
    const ss_grad_seg& s = segs[i];
    seg_status[i] = SS_SEG_OK;
    auto a = L.adapters.find(s.client_id);
    if (a == L.adapters.end()) { seg_status[i] = SS_SEG_NO_ADAPTER; continue; }
    const AdapterSlot& as = a->second;
    if ((as.kind & SS_ADAPTER_LORA) && (as.kind & SS_ADAPTER_IA3)) { seg_status[i] = SS_SEG_UNSUPPORTED; continue; }
    if (s.rows == 0) continue;
    if (!s.dy || s.dy_ld < d_out) { seg_status[i] = SS_SEG_BAD_PTR; continue; }
    const bool acc = s.flags & SS_GRADF_ACCUMULATE;
    if (as.kind & SS_ADAPTER_LORA) {
      if (!s.x || s.x_ld < d_in || !s.grad_a || !s.grad_b || !(s.flags & SS_GRADF_X_BF16) ||
          !(s.flags & SS_GRADF_DY_BF16) || !aligned16(s.x, s.x_ld, 2) || !aligned16(s.dy, s.dy_ld, 2)) {
        seg_status[i] = SS_SEG_BAD_PTR;
        continue;
      }
      DevSeg d{};
      d.rows = (int32_t)s.rows;
      d.pack_row = as.pack_row;
      d.rank_pad = as.rank_pad;
      d.lora_scale = as.scale;
      sh.push_back(d);
      LoraGradSeg g{};
      g.rows = (int32_t)s.rows;
      g.qrow0 = (int32_t)qrows;
      g.rank = as.rank;
      g.npad = (int32_t)round_up(as.rank, 64);
      g.accumulate = acc ? 1 : 0;
      g.dA = s.grad_a;
      g.dB = s.grad_b;
      lg.push_back(g);
      lsrc.push_back(&s);
      qrows += round_up(s.rows, 64);
      qld = std::max(qld, g.npad);
    } else {
      if (!s.y_base || s.base_ld < d_out || !s.grad_l) { seg_status[i] = SS_SEG_BAD_PTR; continue; }
      Ia3GradSeg g{};
      g.rows = (int32_t)s.rows;
      const bool dbf = s.flags & SS_GRADF_DY_BF16, bbf = s.flags & SS_GRADF_BASE_BF16;
      g.flags = (dbf ? 1 : 0) | (bbf ? 2 : 0) |
                ((aligned16(s.dy, s.dy_ld, dbf ? 2 : 4) && aligned16(s.y_base, s.base_ld, bbf ? 2 : 4)) ? 4 : 0) |
                (acc ? 8 : 0);
      g.dy = s.dy;
      g.dy_ld = s.dy_ld;
      g.yb = s.y_base;
      g.yb_ld = s.base_ld;
      g.dl = s.grad_l;
      ig.push_back(g);
    }
  }
  if (lg.empty() && ig.empty()) return SS_OK;
  CK(cudaSetDevice(ctx->device));

  // ---- LoRA tables: tensor maps [4j + 0/1] = x / g with box {64, 128} (shrink, K-major A),
  // [4j + 2/3] = x / g with box {64, 64} (grad kernel, MN-major A); shrink and grad items
  std::vector<CUtensorMap> tmaps(std::max<size_t>(1, 4 * lg.size()));
  std::vector<ShrinkItem> sitems;   // x items (pack 0 = A^T rows, K = d_in), then g items (pack 1 = B rows, K = d_out)
  std::vector<LoraGradItem> gitems;
  int rc = SS_OK;
  for (size_t j = 0; j < lg.size(); ++j) {
    const ss_grad_seg& s = *lsrc[j];
    if ((rc = encode_2d(ctx, &tmaps[4 * j + 0], s.x, d_in, s.rows, s.x_ld, 64, BM))) return rc;
    if ((rc = encode_2d(ctx, &tmaps[4 * j + 1], s.dy, d_out, s.rows, s.dy_ld, 64, BM))) return rc;
    if ((rc = encode_2d(ctx, &tmaps[4 * j + 2], s.x, d_in, s.rows, s.x_ld, 64, 64))) return rc;
    if ((rc = encode_2d(ctx, &tmaps[4 * j + 3], s.dy, d_out, s.rows, s.dy_ld, 64, 64))) return rc;
    lg[j].xmap = (int32_t)(4 * j + 2);
    lg[j].gmap = (int32_t)(4 * j + 3);
    for (int r = 0; r < (int)s.rows; r += BM) {
      const int n = std::min<int>(BM, s.rows - r);
      sitems.push_back(ShrinkItem{(int32_t)j, (int32_t)(4 * j + 0), r, n, lg[j].qrow0 + r, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0});
      sitems.push_back(ShrinkItem{(int32_t)j, (int32_t)(4 * j + 1), r, n, (int32_t)qrows + lg[j].qrow0 + r, 0, 1, 0, 0,
                                  0, 0, 0, 0, 0, 0, 0});
    }
  }
  // token contractions in reverse client order: the shrink (items in client order) read the last
  // clients' x / g most recently, so their second read is the likeliest to hit L2 (two-launch
  // path); the fused path walks `work` instead
  std::vector<int32_t> g_first(lg.size() + 1, 0);
  for (size_t jj = lg.size(); jj-- > 0;) {
    const int32_t j = (int32_t)jj;
    g_first[j] = (int32_t)gitems.size();
    for (int m = 0; m < d_in; m += BM) gitems.push_back(LoraGradItem{j, 0, m, 0});
    for (int m = 0; m < d_out; m += BM) gitems.push_back(LoraGradItem{j, 1, m, 0});
  }
  // fused K3 + K6 (grads.cuh lora_grad_fused_kernel): shrink items of client j, then the
  // contractions of client j - lag; whole-mode shrinks only (rank_pad <= 64)
  int max_rank_pad = 0;
  for (const DevSeg& d : sh) max_rank_pad = std::max(max_rank_pad, d.rank_pad);
  const bool fused = ctx->grad_fused && !lg.empty() && max_rank_pad <= 64;
  std::vector<int2> work;
  std::vector<int32_t> need(std::max<size_t>(1, lg.size()), 0);
  if (fused) {
    for (size_t i = 0; i < sitems.size(); ++i) need[sitems[i].seg]++;
    const int lag = ctx->grad_fused_lag;
    size_t si = 0;
    auto contractions = [&](int32_t j) {
      const int32_t g0 = g_first[j], g1 = g0 + (d_in + BM - 1) / BM + (d_out + BM - 1) / BM;
      for (int32_t q = g0; q < g1; ++q) work.push_back(make_int2(1, q));
    };
    for (size_t j = 0; j < lg.size(); ++j) {
      for (; si < sitems.size() && sitems[si].seg == (int32_t)j; ++si) work.push_back(make_int2(0, (int)si));
      if ((int)j >= lag) contractions((int32_t)(j - lag));
    }
    for (int j = std::max<int>(0, (int)lg.size() - lag); j < (int)lg.size(); ++j) contractions(j);
  }
  std::vector<Ia3PartItem> pitems;
  std::vector<Ia3FinItem> fitems;
  for (size_t j = 0; j < ig.size(); ++j)
    for (int c = 0; c < d_out; c += IA3_COLS) {
      const int nch = (ig[j].rows + IA3_ROWS - 1) / IA3_ROWS;
      fitems.push_back(Ia3FinItem{(int32_t)j, c, (int32_t)pitems.size(), nch});
      for (int k = 0; k < nch; ++k)
        pitems.push_back(Ia3PartItem{(int32_t)j, c, k * IA3_ROWS, (int32_t)pitems.size()});
    }

  auto sz = [](size_t n, size_t e) { return round_up((int64_t)std::max<size_t>(1, n) * e, 256); };
  const size_t o_tm = 0;
  const size_t o_sh = o_tm + sz(tmaps.size(), sizeof(CUtensorMap));
  const size_t o_lg = o_sh + sz(sh.size(), sizeof(DevSeg));
  const size_t o_ix = o_lg + sz(lg.size(), sizeof(LoraGradSeg));
  const size_t o_gi = o_ix + sz(sitems.size(), sizeof(ShrinkItem));
  const size_t o_is = o_gi + sz(gitems.size(), sizeof(LoraGradItem));
  const size_t o_ii = o_is + sz(ig.size(), sizeof(Ia3GradSeg));
  const size_t o_if = o_ii + sz(pitems.size(), sizeof(Ia3PartItem));
  const size_t o_wk = o_if + sz(fitems.size(), sizeof(Ia3FinItem));
  const size_t o_nd = o_wk + sz(work.size(), sizeof(int2));
  const size_t total = o_nd + sz(need.size(), sizeof(int32_t));
  Staging* stp = nullptr;
  if ((rc = acquire_staging(ctx, total, stp))) return rc;
  char* h = static_cast<char*>(stp->host);
  memcpy(h + o_tm, tmaps.data(), tmaps.size() * sizeof(CUtensorMap));
  if (!lg.empty()) {
    memcpy(h + o_sh, sh.data(), sh.size() * sizeof(DevSeg));
    memcpy(h + o_lg, lg.data(), lg.size() * sizeof(LoraGradSeg));
    memcpy(h + o_ix, sitems.data(), sitems.size() * sizeof(ShrinkItem));
    memcpy(h + o_gi, gitems.data(), gitems.size() * sizeof(LoraGradItem));
  }
  if (fused) {
    memcpy(h + o_wk, work.data(), work.size() * sizeof(int2));
    memcpy(h + o_nd, need.data(), need.size() * sizeof(int32_t));
  }
  if (!ig.empty()) {
    memcpy(h + o_is, ig.data(), ig.size() * sizeof(Ia3GradSeg));
    memcpy(h + o_ii, pitems.data(), pitems.size() * sizeof(Ia3PartItem));
    memcpy(h + o_if, fitems.data(), fitems.size() * sizeof(Ia3FinItem));
  }
  if ((rc = order_after_previous(ctx, stream))) return rc;   // (shared shrink partials / tickets)
  CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
  CK(cudaMemcpyAsync(stp->dev, stp->host, total, cudaMemcpyHostToDevice, stream));
  CK(cudaEventRecord(stp->done, stream));
  stp->pending = true;
  char* dv = static_cast<char*>(stp->dev);

  if (!lg.empty()) {
    const size_t qbytes = (size_t)2 * qrows * qld * 2;
    if ((rc = ensure_dev(ctx, ctx->qx, ctx->qx_cap, qbytes, false))) return rc;
    ctx->ws_high = std::max(ctx->ws_high, ctx->x_cap + ctx->al_cap + ctx->rs_cap + ctx->qx_cap);
    CK(cudaMemsetAsync(ctx->qx, 0, qbytes, stream));
    double fl = 0, by = 0;
    for (size_t j = 0; j < lg.size(); ++j) {
      const double t = lg[j].rows, r = lg[j].rank;
      fl += 2.0 * 2.0 * t * r * (d_in + d_out);  // two shrinks + two token contractions
      by += t * (d_in + d_out) * 2.0 + r * (d_in + d_out) * (4.0 + 2.0);
    }
    const int pi = prof_begin(ctx, stream, SS_KERNEL_GRAD, fl, by);
    // K3 (one launch for both shrinks): Q[0, qrows) = s * x.A (pack A^T rows, K = d_in),
    // Q[qrows, 2 qrows) = s * g.B^T (pack B rows, K = d_out); then K6 token contractions
    ShrinkParams sp;
    sp.lora_ld = qld;
    sp.segs = reinterpret_cast<const DevSeg*>(dv + o_sh);
    sp.tmaps = reinterpret_cast<const CUtensorMap*>(dv + o_tm);
    sp.K = d_in;
    sp.K2 = d_out;
    sp.a_lora = ctx->qx;
    int part_ld = 16;
    for (const DevSeg& d : sh) part_ld = std::max(part_ld, d.rank_pad);
    const int max_chunks = std::max(shrink_chunks(d_in, ctx->shrink_kb_chunk), shrink_chunks(d_out, ctx->shrink_kb_chunk));
    sp.kb_chunk = ctx->shrink_kb_chunk;
    if ((rc = ensure_shrink_ws(ctx, sitems.size(), max_chunks, part_ld))) return rc;
    sp.part = ctx->shrink_part;
    sp.part_ld = part_ld;
    sp.max_chunks = max_chunks;
    sp.ticket = ctx->shrink_ticket;
    CUtensorMap tmQ;
    if ((rc = encode_2d(ctx, &tmQ, ctx->qx, qld, 2 * qrows, qld, 64, 64))) return rc;
    LoraGradParams gp;
    gp.d_in = d_in;
    gp.d_out = d_out;
    gp.qrows = (int)qrows;
    gp.segs = reinterpret_cast<const LoraGradSeg*>(dv + o_lg);
    gp.tmaps = reinterpret_cast<const CUtensorMap*>(dv + o_tm);
    // (one launch each over all clients: the shrink has only t/128 x 2 CTAs per client, so
    // splitting the clients into L2-sized groups starves the GPU — measured 2.3x slower)
    sp.items = reinterpret_cast<const ShrinkItem*>(dv + o_ix);
    gp.items = reinterpret_cast<const LoraGradItem*>(dv + o_gi);
    if (fused) {
      // one launch; the ticket and per-client counters are zeroed in stream order first
      const size_t sync_bytes = (1 + lg.size()) * sizeof(int);
      if ((rc = ensure_dev(ctx, ctx->grad_sync, ctx->grad_sync_cap, sync_bytes, false))) return rc;
      CK(cudaMemsetAsync(ctx->grad_sync, 0, sync_bytes, stream));
      GradFusedParams fp;
      fp.work = reinterpret_cast<const int2*>(dv + o_wk);
      fp.queue = ctx->grad_sync;
      fp.done = ctx->grad_sync + 1;
      fp.need = reinterpret_cast<const int32_t*>(dv + o_nd);
      lora_grad_fused_kernel<<<(int)work.size(), GEMM_THREADS, GRAD_FUSED_SMEM, stream>>>(L.tm_at, L.tm_b, tmQ, sp, gp, fp);
      CK(cudaGetLastError());
      ctx->launches += 1;
    } else {
      const bool whole = max_chunks == 1 ||
                         (part_ld <= 64 && (ctx->shrink_mode == 1 || (ctx->shrink_mode == 0 && (int)sitems.size() >= ctx->num_sms)));
      lora_shrink_kernel<<<dim3((unsigned)sitems.size(), whole ? 1 : max_chunks), GEMM_THREADS, SHRINK_SMEM, stream>>>(
          L.tm_at, L.tm_b, sp);
      CK(cudaGetLastError());
      lora_grad_kernel<<<(int)gitems.size(), GEMM_THREADS, GRAD_SMEM, stream>>>(tmQ, gp);
      CK(cudaGetLastError());
      ctx->launches += 2;
    }
    prof_end(ctx, stream, pi);
  }
  if (!ig.empty()) {
    double by = 0;
    for (const Ia3GradSeg& g : ig) by += (double)g.rows * d_out * (((g.flags & 1) ? 2 : 4) + ((g.flags & 2) ? 2 : 4)) + d_out * 4.0;
    const int pi = prof_begin(ctx, stream, SS_KERNEL_GRAD, 2.0 * by / 4, by);
    float* part = nullptr;
    if ((rc = ensure_dev(ctx, ctx->ia3_part, ctx->ia3_part_cap, pitems.size() * IA3_COLS * sizeof(float), false))) return rc;
    part = reinterpret_cast<float*>(ctx->ia3_part);
    Ia3PartParams pp;
    pp.d_out = d_out;
    pp.segs = reinterpret_cast<const Ia3GradSeg*>(dv + o_is);
    pp.items = reinterpret_cast<const Ia3PartItem*>(dv + o_ii);
    pp.part = part;
    ia3_grad_partial_kernel<<<(int)pitems.size(), 256, 0, stream>>>(pp);
    CK(cudaGetLastError());
    Ia3FinParams fp;
    fp.d_out = d_out;
    fp.segs = pp.segs;
    fp.items = reinterpret_cast<const Ia3FinItem*>(dv + o_if);
    fp.part = part;
    ia3_grad_finalize_kernel<<<(int)fitems.size(), 256, 0, stream>>>(fp);
    CK(cudaGetLastError());
    prof_end(ctx, stream, pi);
    ctx->launches += 2;
  }
  CK(cudaEventRecord(ctx->compute_done, stream));
  ctx->any_compute = true;
  return SS_OK;
}

}  // extern "C"

namespace {
struct HostPiece { int seg; int64_t r0, r1; };

// f32 -> bf16 on the host: round to nearest even, NaN -> 0x7FFF, the conversion the gather kernel
// applies to f32 request rows (cvt.rn.bf16), so converting on the host gives the same bits.

// One row of f32_to_bf16_rn, branch-free so the compiler vectorises it (AVX2 where present).
#define SS_CVT_BODY                                                                     \
  for (int64_t k = 0; k < K; ++k) {                                                     \
    uint32_t u;                                                                         \
    memcpy(&u, src + k, 4);                                                             \
    const uint32_t r = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;                          \
    dst[k] = (uint16_t)(((u & 0x7fffffffu) > 0x7f800000u) ? 0x7fffu : r);               \
  }
__attribute__((target("avx2"))) void cvt_row_avx2(const float* __restrict src, uint16_t* __restrict dst, int64_t K) {
  SS_CVT_BODY
}
void cvt_row_base(const float* __restrict src, uint16_t* __restrict dst, int64_t K) { SS_CVT_BODY }
#undef SS_CVT_BODY
inline void cvt_row(const float* src, uint16_t* dst, int64_t K) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) cvt_row_avx2(src, dst, K);
  else cvt_row_base(src, dst, K);
}

// True when `p` is ordinary pageable host memory (not device, not page-locked / registered).
bool pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// The host conversion pool and page-locked ring slots of at least `bytes` each.
int ensure_host_conv(ss_ctx* ctx, size_t bytes) {
  if (!ctx->pool) {
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int n = ctx->host_threads > 0 ? ctx->host_threads : std::min(16, hw);
    ctx->pool.reset(new HostPool(std::max(0, n - 1)));   // + the calling thread
  }
  for (auto& hc : ctx->hconv) {
    if (!hc.ev) CK(cudaEventCreateWithFlags(&hc.ev, cudaEventDisableTiming));
    if (hc.cap < bytes) {
      if (hc.used) CK(cudaEventSynchronize(hc.ev));
      CK(cudaFreeHost(hc.buf));
      hc.buf = nullptr;
      hc.cap = 0;
      CK(cudaHostAlloc(reinterpret_cast<void**>(&hc.buf), bytes, cudaHostAllocDefault));
      hc.cap = bytes;
      hc.used = false;
    }
  }
  return SS_OK;
}

// The numerics class of a whole request (decode_rows), for the pieces a host pipeline splits it
// into: a piece must reduce K the way the request would in one piece.
uint32_t class_flag(const ss_ctx* ctx, int K, const ss_seg& s) {
  if (s.flags & (SS_SEGF_CLASS_DECODE | SS_SEGF_CLASS_PREFILL)) return 0;
  return (K % 64 == 0 && ctx->decode_rows > 0 && (int)s.rows <= ctx->decode_rows) ? SS_SEGF_CLASS_DECODE
                                                                                   : SS_SEGF_CLASS_PREFILL;
}

// Host dispatch whose replies overwrite request rows of later sub-batches (see
// ss_compute_batch_host): every sub-batch gets its own slice of dispatch-sized device buffers
// (so the H2D stream never waits for compute), and the D2H of sub-batch j is issued right after
// the H2D of sub-batch wait_for[j] was enqueued, waiting for it.
int host_dispatch_aliased(ss_ctx* ctx, int pass_kind, int block, int role, const ss_seg* segs,
                          int32_t* seg_status, cudaStream_t stream, int K, int N, size_t esz_in,
                          size_t esz_out, size_t esz_base, int64_t rows_total,
                          const std::vector<std::vector<HostPiece>>& chunks, const std::vector<int>& wait_for) {
  int rc = SS_OK;
  bool any_base = false;
  for (const auto& ch : chunks)
    for (const HostPiece& p : ch) any_base |= segs[p.seg].dst_base && pass_kind != SS_PASS_BACKWARD;
  if ((rc = ensure_dev(ctx, ctx->ha_in, ctx->ha_in_cap, (size_t)rows_total * K * esz_in, false))) return rc;
  if ((rc = ensure_dev(ctx, ctx->ha_out, ctx->ha_out_cap, (size_t)rows_total * N * esz_out, false))) return rc;
  if (any_base && (rc = ensure_dev(ctx, ctx->ha_base, ctx->ha_base_cap, (size_t)rows_total * N * esz_base, false)))
    return rc;
  ctx->ws_high = std::max(ctx->ws_high, ctx->x_cap + ctx->al_cap + ctx->rs_cap + ctx->qx_cap + ctx->ha_in_cap +
                                            ctx->ha_out_cap + ctx->ha_base_cap);
  while (ctx->chunk_ev.size() < 2 * chunks.size()) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->chunk_ev.push_back(e);
  }
  // the previous host dispatch drained its D2H before returning; the device path may still be
  // reading an older dispatch's slices: order after everything queued on `stream`
  CK(cudaEventRecord(ctx->chunk_ev[0], stream));
  CK(cudaStreamWaitEvent(ctx->h2d, ctx->chunk_ev[0], 0));
  std::vector<int64_t> row0(chunks.size() + 1, 0);
  for (size_t j = 0; j < chunks.size(); ++j) {
    int64_t n = 0;
    for (const HostPiece& p : chunks[j]) n += p.r1 - p.r0;
    row0[j + 1] = row0[j] + n;
  }
  std::vector<char> issued(chunks.size(), 0);
  auto issue_d2h = [&](size_t j) -> int {
    cudaEvent_t comp = ctx->chunk_ev[2 * j + 1];
    CK(cudaStreamWaitEvent(ctx->d2h, comp, 0));
    if (wait_for[j] >= 0) CK(cudaStreamWaitEvent(ctx->d2h, ctx->chunk_ev[2 * wait_for[j]], 0));
    int64_t pos = row0[j];
    for (const HostPiece& p : chunks[j]) {
      const ss_seg& s = segs[p.seg];
      const int64_t n = p.r1 - p.r0;
      if (seg_status[p.seg] == SS_SEG_OK) {
        CK(copy_rows(static_cast<char*>(s.dst) + p.r0 * s.dst_ld * esz_out, (size_t)s.dst_ld * esz_out,
                     static_cast<const char*>(ctx->ha_out) + pos * N * esz_out, (size_t)N * esz_out,
                     (size_t)N * esz_out, (size_t)n, cudaMemcpyDeviceToHost, ctx->d2h));
        if (s.dst_base && pass_kind != SS_PASS_BACKWARD)
          CK(copy_rows(static_cast<char*>(s.dst_base) + p.r0 * s.base_ld * esz_base, (size_t)s.base_ld * esz_base,
                       static_cast<const char*>(ctx->ha_base) + pos * N * esz_base, (size_t)N * esz_base,
                       (size_t)N * esz_base, (size_t)n, cudaMemcpyDeviceToHost, ctx->d2h));
      }
      pos += n;
    }
    issued[j] = 1;
    return SS_OK;
  };
  std::vector<ss_seg> cs;
  std::vector<int32_t> cst;
  for (size_t k = 0; k < chunks.size(); ++k) {
    cs.clear();
    int64_t pos = row0[k];
    for (const HostPiece& p : chunks[k]) {
      const ss_seg& s = segs[p.seg];
      const int64_t n = p.r1 - p.r0;
      char* din = static_cast<char*>(ctx->ha_in) + pos * K * esz_in;
      CK(copy_rows(din, (size_t)K * esz_in, static_cast<const char*>(s.src) + p.r0 * s.src_ld * esz_in,
                   (size_t)s.src_ld * esz_in, (size_t)K * esz_in, (size_t)n, cudaMemcpyHostToDevice, ctx->h2d));
      ss_seg d = s;
      d.rows = (uint32_t)n;
      d.flags |= class_flag(ctx, K, s);   // a piece keeps its request's numerics class
      d.src = din;
      d.src_ld = K;
      d.dst = static_cast<char*>(ctx->ha_out) + pos * N * esz_out;
      d.dst_ld = N;
      if (s.dst_base && pass_kind != SS_PASS_BACKWARD) {
        d.dst_base = static_cast<char*>(ctx->ha_base) + pos * N * esz_base;
        d.base_ld = N;
      } else {
        d.dst_base = nullptr;
        d.base_ld = 0;
      }
      cs.push_back(d);
      pos += n;
    }
    cst.assign(cs.size(), 0);
    Built b;
    if ((rc = build_batch(ctx, pass_kind, block, role, (int)cs.size(), cs.data(), cst.data(), b, true))) return rc;
    for (size_t q = 0; q < cs.size(); ++q)
      if (cst[q] != SS_SEG_OK) seg_status[chunks[k][q].seg] = cst[q];
    Staging* stp = nullptr;
    if (b.M > 0) {
      if ((rc = acquire_staging(ctx, b.blob.size(), stp))) return rc;
      memcpy(stp->host, b.blob.data(), b.blob.size());
      CK(cudaMemcpyAsync(stp->dev, stp->host, b.blob.size(), cudaMemcpyHostToDevice, ctx->h2d));
    }
    CK(cudaEventRecord(ctx->chunk_ev[2 * k], ctx->h2d));
    CK(cudaStreamWaitEvent(stream, ctx->chunk_ev[2 * k], 0));
    if (b.M > 0) {
      CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
      if ((rc = launch_batch(ctx, b, static_cast<char*>(stp->dev), stream))) return rc;
      // the staging slot may be reused only after these kernels read their tables
      CK(cudaEventRecord(stp->done, stream));
      stp->pending = true;
    }
    CK(cudaEventRecord(ctx->chunk_ev[2 * k + 1], stream));
    for (size_t j = 0; j <= k; ++j)
      if (!issued[j] && wait_for[j] <= (int)k && (rc = issue_d2h(j))) return rc;
  }
  for (size_t j = 0; j < chunks.size(); ++j)
    if (!issued[j] && (rc = issue_d2h(j))) return rc;
  CK(cudaStreamSynchronize(ctx->d2h));
  return SS_OK;
}
}  // namespace

extern "C" {

// ---- host-buffer dispatch ---------------------------------------------------------------
int ss_compute_batch_host(ss_ctx* ctx, int pass_kind, int block, int role, int n_seg, const ss_seg* segs,
                          void* stream_, int32_t* seg_status) {
  if (!ctx) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  if (pass_kind < 0 || pass_kind > 2) return fail(ctx, SS_E_ARG, "unknown pass %d", pass_kind);
  if (n_seg < 0 || (n_seg > 0 && (!segs || !seg_status))) return fail(ctx, SS_E_ARG, "bad segment array");
  auto lit = ctx->layers.find({block, role});
  if (lit == ctx->layers.end()) return fail(ctx, SS_E_NOLAYER, "unknown layer (%d, %d)", block, role);
  const Layer& L = lit->second;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const bool bwd = pass_kind == SS_PASS_BACKWARD;
  const int K = bwd ? L.d_out : L.d_in;
  const int N = bwd ? L.d_in : L.d_out;
  CK(cudaSetDevice(ctx->device));

  // ---- validate (the same per-segment checks as build_batch, so statuses agree)
  std::vector<int> good;
  int64_t rows_total = 0;
  size_t esz_in = 2, esz_out = 2, esz_base = 2;
  bool any_base = false;
  for (int i = 0; i < n_seg; ++i) {
    const ss_seg& s = segs[i];
    seg_status[i] = SS_SEG_OK;
    if ((int)s.width != K) { seg_status[i] = SS_SEG_BAD_WIDTH; continue; }
    if (s.rows == 0) continue;
    if (!s.src || !s.dst || s.src_ld < K || s.dst_ld < N) { seg_status[i] = SS_SEG_BAD_PTR; continue; }
    if ((s.flags & SS_SEGF_ADAPTER) && L.adapters.find(s.client_id) == L.adapters.end()) { seg_status[i] = SS_SEG_NO_ADAPTER; continue; }
    if (s.dst_base && pass_kind != SS_PASS_BACKWARD && s.base_ld < N) { seg_status[i] = SS_SEG_BAD_PTR; continue; }
    good.push_back(i);
    rows_total += s.rows;
  }
  if (good.empty()) return SS_OK;
  // one dtype per side for the staging ring (the kernels take bf16 / f32 per segment, but the
  // ring's slot sizes are per dispatch)
  esz_in = (segs[good[0]].flags & SS_SEGF_SRC_BF16) ? 2 : 4;
  esz_out = (segs[good[0]].flags & SS_SEGF_DST_BF16) ? 2 : 4;
  for (int i : good) {
    const ss_seg& s = segs[i];
    if (((s.flags & SS_SEGF_SRC_BF16) ? 2u : 4u) != esz_in || ((s.flags & SS_SEGF_DST_BF16) ? 2u : 4u) != esz_out)
      return fail(ctx, SS_E_ARG, "host dispatch: all segments must share src / dst dtypes");
    if (s.dst_base && pass_kind != SS_PASS_BACKWARD) {
      any_base = true;
      esz_base = (s.flags & SS_SEGF_BASE_BF16) ? 2 : 4;
    }
  }

  // ---- small dispatches (decode: a few rows per client): no copies at all. The kernels read the
  // request rows from pinned host memory (gather, UVA) and the epilogue stores the reply rows
  // straight into it: one launch sequence and one synchronisation instead of two memcpy calls
  // per segment, whose API cost dominates a dispatch of tens of two-row segments.
  // Small dispatch of pageable f32 request rows (numpy decode clients): the host threads convert
  // them into a page-locked slot (bf16), and the dispatch goes on as a zero-copy one over those
  // rows (the same bits as the device gather's conversion).
  std::vector<ss_seg> conv_segs;
  if (ctx->host_convert && esz_in == 4 &&
      (double)rows_total * (K * 2 + N * esz_out) <= (double)ctx->zero_copy_bytes) {
    // (only when every row converts and the replies can be written in place: then the dispatch
    // surely takes the zero-copy path below)
    bool eligible = true;
    for (int i : good) {
      const ss_seg& s = segs[i];
      if ((s.flags & SS_SEGF_PINNED) || !pageable(s.src) || pageable(s.dst) || (s.dst_base && pageable(s.dst_base))) {
        eligible = false;
        break;
      }
      if (bwd && (s.flags & SS_SEGF_ADAPTER)) {
        auto ad = L.adapters.find(s.client_id);
        if (ad != L.adapters.end() && (ad->second.kind & SS_ADAPTER_IA3)) { eligible = false; break; }
      }
    }
    if (eligible) {
      std::vector<char> f32(n_seg, 0);   // (none here; kept for the row layout below)
      int64_t bytes = 0;
      for (int i : good) bytes += (int64_t)segs[i].rows * K * 2;
      int rc0 = ensure_host_conv(ctx, (size_t)std::max<int64_t>(bytes, 1 << 20));
      if (rc0) return rc0;
      auto& hc = ctx->hconv[0];
      if (hc.used) CK(cudaEventSynchronize(hc.ev));
      conv_segs.assign(segs, segs + n_seg);
      std::vector<int64_t> off(n_seg, 0);
      int64_t o = 0;
      for (int i : good) {
        off[i] = o;
        o += (int64_t)segs[i].rows * K * (f32[i] ? 4 : 2);
      }
      char* ring = reinterpret_cast<char*>(hc.buf);
      ctx->pool->run((int)good.size(), [&](int t) {
        const int i = good[t];
        const ss_seg& s = segs[i];
        for (int64_t r = 0; r < (int64_t)s.rows; ++r) {
          const float* src = static_cast<const float*>(s.src) + r * s.src_ld;
          char* dst = ring + off[i] + r * K * (f32[i] ? 4 : 2);
          if (f32[i]) memcpy(dst, src, (size_t)K * 4);
          else cvt_row(src, reinterpret_cast<uint16_t*>(dst), K);
        }
      });
      for (int i : good) {
        ss_seg& d = conv_segs[i];
        d.src = ring + off[i];
        d.src_ld = K;
        d.flags |= SS_SEGF_SRC_BF16 | SS_SEGF_PINNED;   // (dst / dst_base checked above)
      }
      segs = conv_segs.data();
      esz_in = 2;
    }
  }
  bool zero_copy = (double)rows_total * (K * esz_in + N * esz_out) <= (double)ctx->zero_copy_bytes;
  for (size_t q = 0; zero_copy && q < good.size(); ++q) {
    // only pinned (UVA-mapped) or device memory can be touched by the kernels directly
    const ss_seg& sg = segs[good[q]];
    if (sg.flags & SS_SEGF_PINNED) continue;   // verified by the caller
    for (const void* ptr : {sg.src, static_cast<const void*>(sg.dst), static_cast<const void*>(sg.dst_base)}) {
      if (!ptr) continue;
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess ||
          (a.type != cudaMemoryTypeHost && a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)) {
        cudaGetLastError();
        zero_copy = false;
        break;
      }
    }
  }
  if (zero_copy) {
    // request rows are gathered from host memory by the kernels (UVA); replies land in a device
    // slot and one row-copy kernel writes them to the host rows (coalesced), so the dispatch
    // makes no memcpy calls at all
    auto& hs = ctx->hslot[0];
    const size_t out_need = (size_t)rows_total * N * esz_out, base_need = any_base ? (size_t)rows_total * N * esz_base : 0;
    if (hs.used) CK(cudaEventSynchronize(hs.ev_out));
    int rc = SS_OK;
    if (hs.out_cap < out_need && (rc = ensure_dev(ctx, reinterpret_cast<char*&>(hs.out), hs.out_cap, out_need, false))) return rc;
    if (hs.base_cap < base_need && (rc = ensure_dev(ctx, reinterpret_cast<char*&>(hs.base), hs.base_cap, base_need, false))) return rc;
    const uint64_t key = ctx->zc_cache_on ? zc_key(pass_kind, block, role, n_seg, segs) : 0;
    if (ctx->zc_cache_on && ctx->zc_swept != ctx->ws_epoch + ctx->ad_epoch + ctx->opt_epoch) {
      // an epoch moved since the last sweep: entries built before can never hit again, free
      // them now (every earlier host dispatch synchronised on return: nothing reads them)
      for (auto it = ctx->zc_cache.begin(); it != ctx->zc_cache.end();) {
        ZcPlan* z = it->second;
        if (z->b.ws_epoch != ctx->ws_epoch || z->b.ad_epoch != ctx->ad_epoch || z->opt_epoch != ctx->opt_epoch) {
          cudaFree(z->dev);
          delete z;
          it = ctx->zc_cache.erase(it);
        } else {
          ++it;
        }
      }
      ctx->zc_swept = ctx->ws_epoch + ctx->ad_epoch + ctx->opt_epoch;
    }
    if (ctx->zc_cache_on) {
      auto it = ctx->zc_cache.find(key);
      ZcPlan* z = it == ctx->zc_cache.end() ? nullptr : it->second;
      if (z && z->pass_kind == pass_kind && z->block == block && z->role == role && z->segs.size() == (size_t)n_seg &&
          !memcmp(z->segs.data(), segs, sizeof(ss_seg) * (size_t)n_seg) && z->b.ws_epoch == ctx->ws_epoch &&
          z->b.ad_epoch == ctx->ad_epoch && z->opt_epoch == ctx->opt_epoch && z->out == hs.out &&
          z->base == hs.base) {
        // the same dispatch as before (same buffers, rows, clients): launch its tables as built
        for (int i = 0; i < n_seg; ++i) seg_status[i] = z->status[i];
        CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
        if ((rc = launch_batch(ctx, z->b, z->dev, stream))) return rc;
        copy_rows_kernel<<<(int)std::min<int64_t>((z->copy_rows + 7) / 8, (int64_t)ctx->num_sms * 8), 256, 0, stream>>>(
            reinterpret_cast<const RowCopy*>(z->dev + z->ops_off), z->n_ops, (int)z->copy_rows);
        CK(cudaGetLastError());
        ctx->launches++;
        CK(cudaStreamSynchronize(stream));
        return SS_OK;
      }
    }
    std::vector<ss_seg> cs;
    std::vector<RowCopy> ops;
    std::vector<int> op_seg;    // index into cs of each row copy
    int64_t pos = 0;
    for (int i : good) {
      ss_seg d = segs[i];
      d.dst = static_cast<char*>(hs.out) + pos * N * esz_out;
      d.dst_ld = N;
      ops.push_back(RowCopy{static_cast<const char*>(d.dst), static_cast<char*>(segs[i].dst), (int64_t)N * (int64_t)esz_out,
                            segs[i].dst_ld * (int64_t)esz_out, (int32_t)segs[i].rows, (int32_t)(N * esz_out)});
      op_seg.push_back((int)cs.size());
      if (segs[i].dst_base && pass_kind != SS_PASS_BACKWARD) {
        d.dst_base = static_cast<char*>(hs.base) + pos * N * esz_base;
        d.base_ld = N;
        ops.push_back(RowCopy{static_cast<const char*>(d.dst_base), static_cast<char*>(segs[i].dst_base),
                              (int64_t)N * (int64_t)esz_base, segs[i].base_ld * (int64_t)esz_base,
                              (int32_t)segs[i].rows, (int32_t)(N * esz_base)});
        op_seg.push_back((int)cs.size());
      }
      cs.push_back(d);
      pos += segs[i].rows;
    }
    std::vector<int32_t> cst(cs.size(), 0);
    Built b;
    if ((rc = build_batch(ctx, pass_kind, block, role, (int)cs.size(), cs.data(), cst.data(), b, true, true)))
      return rc;
    for (size_t q = 0; q < cs.size(); ++q)
      if (cst[q] != SS_SEG_OK) seg_status[good[q]] = cst[q];
    if (b.M == 0) return SS_OK;
    {
      // rejected segments are not written: drop their row copies (their slot rows are stale)
      size_t k = 0;
      for (size_t o = 0; o < ops.size(); ++o)
        if (cst[op_seg[o]] == SS_SEG_OK && ops[o].rows > 0) ops[k++] = ops[o];
      ops.resize(k);
    }
    if (ops.empty()) return SS_OK;
    const size_t ops_off = round_up((int64_t)b.blob.size(), 256);
    Staging* stp = nullptr;
    if ((rc = acquire_staging(ctx, ops_off + ops.size() * sizeof(RowCopy), stp))) return rc;
    memcpy(stp->host, b.blob.data(), b.blob.size());
    memcpy(static_cast<char*>(stp->host) + ops_off, ops.data(), ops.size() * sizeof(RowCopy));
    CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
    CK(cudaMemcpyAsync(stp->dev, stp->host, ops_off + ops.size() * sizeof(RowCopy), cudaMemcpyHostToDevice, stream));
    if ((rc = launch_batch(ctx, b, static_cast<char*>(stp->dev), stream))) return rc;
    int64_t copy_rows = 0;
    for (const RowCopy& o : ops) copy_rows += o.rows;
    copy_rows_kernel<<<(int)std::min<int64_t>((copy_rows + 7) / 8, (int64_t)ctx->num_sms * 8), 256, 0, stream>>>(
        reinterpret_cast<const RowCopy*>(static_cast<char*>(stp->dev) + ops_off), (int)ops.size(), (int)copy_rows);
    CK(cudaGetLastError());
    ctx->launches++;
    CK(cudaEventRecord(stp->done, stream));
    stp->pending = true;
    if (ctx->zc_cache_on) {
      // keep this dispatch's tables for its next occurrence (a copy of the staged bytes)
      if (ctx->zc_cache.size() >= 4096) zc_cache_clear(ctx);
      ZcPlan* z = new ZcPlan();
      const size_t total = ops_off + ops.size() * sizeof(RowCopy);
      if (cudaMalloc(&z->dev, total) != cudaSuccess) {
        cudaGetLastError();
        delete z;
      } else {
        CK(cudaMemcpyAsync(z->dev, stp->dev, total, cudaMemcpyDeviceToDevice, stream));
        z->pass_kind = pass_kind;
        z->block = block;
        z->role = role;
        z->segs.assign(segs, segs + n_seg);
        z->status.assign(seg_status, seg_status + n_seg);
        z->opt_epoch = ctx->opt_epoch;
        z->b = std::move(b);
        z->b.blob.clear();
        z->b.blob.shrink_to_fit();
        z->out = hs.out;
        z->base = hs.base;
        z->ops_off = ops_off;
        z->n_ops = (int)ops.size();
        z->copy_rows = copy_rows;
        auto it = ctx->zc_cache.find(key);
        if (it != ctx->zc_cache.end()) {
          cudaFree(it->second->dev);   // (stale: an epoch or the slot changed)
          delete it->second;
        }
        ctx->zc_cache[key] = z;
      }
    }
    CK(cudaStreamSynchronize(stream));   // replies are in the caller's host buffers on return
    return SS_OK;
  }

  // ---- sub-batches of whole rows: the H2D of j+1, the kernels of j and the D2H of j-1 overlap
  const int64_t wide = std::max<int64_t>(K * esz_in, N * esz_out);
  const int64_t target = std::max<int64_t>(64, std::min<int64_t>(ctx->pipeline_rows, ctx->pipeline_bytes / wide));
  // Chunk sizes ramp up (t/8, t/4, t/2, t, ...) and back down at the end, so the pipeline
  // fills and drains in a fraction of one full sub-batch: with the synchronous reference API
  // the first H2D and the last D2H of every dispatch cannot overlap anything.
  std::vector<int64_t> sizes;
  {
    const int64_t t8 = std::max<int64_t>(64, target / 8);
    const int64_t ramp[3] = {t8, std::max<int64_t>(t8, target / 4), std::max<int64_t>(t8, target / 2)};
    int64_t left = rows_total;
    std::vector<int64_t> head, tail;
    for (int k = 0; k < 3 && left > 0; ++k) {
      const int64_t a = std::min(left, ramp[k]);
      head.push_back(a);
      left -= a;
      if (left <= 0) break;
      const int64_t b = std::min(left, ramp[k]);
      tail.push_back(b);
      left -= b;
    }
    sizes = head;
    while (left > 0) {
      const int64_t a = std::min(left, target);
      sizes.push_back(a);
      left -= a;
    }
    sizes.insert(sizes.end(), tail.rbegin(), tail.rend());
  }
  using Piece = HostPiece;
  std::vector<std::vector<Piece>> chunks(1);
  size_t ci = 0;
  int64_t cur = 0;
  for (int i : good) {
    const int64_t t = segs[i].rows;
    int64_t r = 0;
    while (r < t) {
      const int64_t take = std::min(t - r, sizes[ci] - cur);
      chunks.back().push_back(Piece{i, r, r + take});
      cur += take;
      r += take;
      if (cur >= sizes[ci]) {
        chunks.emplace_back();
        cur = 0;
        ci = std::min(ci + 1, sizes.size() - 1);
      }
    }
  }
  if (chunks.back().empty()) chunks.pop_back();
  int rc = SS_OK;
  // In-place hand-off (the reference's SharedBuffer reuses one buffer for request and reply,
  // transport.py:76-97): the D2H of sub-batch j may land on host rows a LATER sub-batch has
  // not uploaded yet. wait_for[j] = the last later sub-batch whose H2D source bytes intersect
  // sub-batch j's reply bytes; with any such hazard every sub-batch gets its own device slice
  // (no ring reuse, so no wait cycle) and D2H j waits for that H2D.
  std::vector<int> wait_for(chunks.size(), -1);
  {
    struct Range { uintptr_t a, b; };
    auto rows_span = [](const void* p, int64_t r0, int64_t r1, int64_t ld, int64_t width, size_t esz) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(p) + (uintptr_t)(r0 * ld * (int64_t)esz);
      return Range{a, a + (uintptr_t)(((r1 - r0 - 1) * ld + width) * (int64_t)esz)};
    };
    std::vector<std::vector<Range>> in_r(chunks.size()), out_r(chunks.size());
    for (size_t j = 0; j < chunks.size(); ++j)
      for (const Piece& p : chunks[j]) {
        const ss_seg& sg = segs[p.seg];
        in_r[j].push_back(rows_span(sg.src, p.r0, p.r1, sg.src_ld, K, esz_in));
        out_r[j].push_back(rows_span(sg.dst, p.r0, p.r1, sg.dst_ld, N, esz_out));
        if (sg.dst_base && pass_kind != SS_PASS_BACKWARD)
          out_r[j].push_back(rows_span(sg.dst_base, p.r0, p.r1, sg.base_ld, N, esz_base));
      }
    for (size_t j = 0; j < chunks.size(); ++j)
      for (size_t k = chunks.size() - 1; k > j && wait_for[j] < 0; --k)
        for (const Range& o : out_r[j]) {
          bool hit = false;
          for (const Range& i : in_r[k])
            if (i.a < o.b && o.a < i.b) { hit = true; break; }
          if (hit) { wait_for[j] = (int)k; break; }
        }
  }
  const bool aliased = std::any_of(wait_for.begin(), wait_for.end(), [](int k) { return k >= 0; });
  if (aliased)
    return host_dispatch_aliased(ctx, pass_kind, block, role, segs, seg_status, stream, K, N, esz_in, esz_out,
                                 esz_base, rows_total, chunks, wait_for);
  // Pageable f32 request rows (the reference's numpy payloads): the host pool converts each
  // sub-batch to bf16 into a page-locked ring slot, one DMA moves it (half the PCIe bytes of f32,
  // no driver bounce copies), and the kernels see bf16 rows — the same bits the gather's own
  // f32 -> bf16 conversion would give. Not for backward IA3 rows (the gather scales dy by l in
  // f32 before rounding) or page-locked / device sources (DMA-able as they are).
  // Backward IA3 rows stay f32 (copied, not converted, by the same threads into the same ring).
  bool conv = ctx->host_convert && esz_in == 4;
  std::vector<char> keep_f32(n_seg, 0);
  for (size_t q = 0; conv && q < good.size(); ++q) {
    const ss_seg& s = segs[good[q]];
    if ((s.flags & SS_SEGF_PINNED) || !pageable(s.src)) conv = false;
    if (bwd && (s.flags & SS_SEGF_ADAPTER)) {
      auto ad = L.adapters.find(s.client_id);
      if (ad != L.adapters.end() && (ad->second.kind & SS_ADAPTER_IA3)) keep_f32[good[q]] = 1;
    }
  }
  // request row bytes per value in the device slot / the ring (bf16 where converted)
  auto esz_of = [&](int seg) -> size_t { return conv && !keep_f32[seg] ? 2 : esz_in; };
  if (conv && (rc = ensure_host_conv(ctx, (size_t)target * K * 4))) return rc;
  const size_t in_need = (size_t)target * K * esz_in, out_need = (size_t)target * N * esz_out;
  const size_t base_need = any_base ? (size_t)target * N * esz_base : 0;
  for (auto& hs : ctx->hslot) {
    if (hs.in_cap < in_need || hs.out_cap < out_need || hs.base_cap < base_need) {
      if (hs.used) CK(cudaEventSynchronize(hs.ev_out));
      if (hs.in_cap < in_need && (rc = ensure_dev(ctx, reinterpret_cast<char*&>(hs.in), hs.in_cap, in_need, false))) return rc;
      if (hs.out_cap < out_need && (rc = ensure_dev(ctx, reinterpret_cast<char*&>(hs.out), hs.out_cap, out_need, false))) return rc;
      if (hs.base_cap < base_need && (rc = ensure_dev(ctx, reinterpret_cast<char*&>(hs.base), hs.base_cap, base_need, false))) return rc;
    }
  }
  ctx->ws_high = std::max(ctx->ws_high, ctx->x_cap + ctx->al_cap + ctx->rs_cap + ctx->qx_cap +
                                            4 * (ctx->hslot[0].in_cap + ctx->hslot[0].out_cap + ctx->hslot[0].base_cap));

  std::vector<ss_seg> cs;
  std::vector<int32_t> cst;
  for (size_t j = 0; j < chunks.size(); ++j) {
    auto& hs = ctx->hslot[j % 4];
    const auto& ch = chunks[j];
    // H2D: the slot's previous kernels must have consumed its input buffer
    if (hs.used) CK(cudaStreamWaitEvent(ctx->h2d, hs.ev_comp, 0));
    int64_t pos = 0;
    cs.clear();
    if (conv) {
      // this sub-batch's rows, converted (or, backward IA3 rows, copied) by the pool into ring
      // slot j % 4 (once its previous DMA has read it), then one copy
      auto& hc = ctx->hconv[j % 4];
      if (hc.used) CK(cudaEventSynchronize(hc.ev));
      std::vector<int64_t> row0(ch.size() + 1, 0), byte0(ch.size() + 1, 0);
      for (size_t q = 0; q < ch.size(); ++q) {
        row0[q + 1] = row0[q] + (ch[q].r1 - ch[q].r0);
        byte0[q + 1] = byte0[q] + (ch[q].r1 - ch[q].r0) * K * (int64_t)esz_of(ch[q].seg);
      }
      const int64_t nrows = row0.back();
      constexpr int64_t kRowsPerTask = 16;
      const int tasks = (int)((nrows + kRowsPerTask - 1) / kRowsPerTask);
      char* ring = reinterpret_cast<char*>(hc.buf);
      ctx->pool->run(tasks, [&](int t) {
        const int64_t a0 = t * kRowsPerTask, a1 = std::min(nrows, a0 + kRowsPerTask);
        size_t q = std::upper_bound(row0.begin(), row0.end(), a0) - row0.begin() - 1;
        for (int64_t r = a0; r < a1; ++r) {
          while (r >= row0[q + 1]) ++q;
          const ss_seg& s = segs[ch[q].seg];
          const float* src = static_cast<const float*>(s.src) + (ch[q].r0 + (r - row0[q])) * s.src_ld;
          const size_t e = esz_of(ch[q].seg);
          char* dst = ring + byte0[q] + (r - row0[q]) * K * (int64_t)e;
          if (e == 2) cvt_row(src, reinterpret_cast<uint16_t*>(dst), K);
          else memcpy(dst, src, (size_t)K * 4);
        }
      });
      CK(cudaMemcpyAsync(hs.in, hc.buf, (size_t)byte0.back(), cudaMemcpyHostToDevice, ctx->h2d));
      CK(cudaEventRecord(hc.ev, ctx->h2d));
      hc.used = true;
    }
    int64_t in_off = 0;   // bytes into the device slot
    for (const Piece& p : ch) {
      const ss_seg& s = segs[p.seg];
      const int64_t n = p.r1 - p.r0;
      char* din = static_cast<char*>(hs.in) + in_off;
      in_off += n * K * (int64_t)esz_of(p.seg);
      if (!conv)
        CK(copy_rows(din, (size_t)K * esz_in, static_cast<const char*>(s.src) + p.r0 * s.src_ld * esz_in,
                     (size_t)s.src_ld * esz_in, (size_t)K * esz_in, (size_t)n, cudaMemcpyHostToDevice, ctx->h2d));
      ss_seg d = s;
      d.rows = (uint32_t)n;
      d.flags |= class_flag(ctx, K, s);   // a piece keeps its request's numerics class
      if (esz_of(p.seg) == 2) d.flags |= SS_SEGF_SRC_BF16;
      d.src = din;
      d.src_ld = K;
      d.dst = static_cast<char*>(hs.out) + pos * N * esz_out;
      d.dst_ld = N;
      if (s.dst_base && pass_kind != SS_PASS_BACKWARD) {
        d.dst_base = static_cast<char*>(hs.base) + pos * N * esz_base;
        d.base_ld = N;
      } else {
        d.dst_base = nullptr;
        d.base_ld = 0;
      }
      cs.push_back(d);
      pos += n;
    }
    // routing tables of this sub-batch: built on the host, copied on the SAME copy stream right
    // after its payload (a table copy queued on the compute stream would wait behind later
    // sub-batches' payload copies in the host-to-device engine)
    cst.assign(cs.size(), 0);
    Built b;
    if ((rc = build_batch(ctx, pass_kind, block, role, (int)cs.size(), cs.data(), cst.data(), b, true))) return rc;
    for (size_t k = 0; k < cs.size(); ++k)
      if (cst[k] != SS_SEG_OK) seg_status[ch[k].seg] = cst[k];
    Staging* stp = nullptr;
    if (b.M > 0) {
      if ((rc = acquire_staging(ctx, b.blob.size(), stp))) return rc;
      memcpy(stp->host, b.blob.data(), b.blob.size());
      CK(cudaMemcpyAsync(stp->dev, stp->host, b.blob.size(), cudaMemcpyHostToDevice, ctx->h2d));
      CK(cudaEventRecord(stp->done, ctx->h2d));
      stp->pending = true;
    }
    CK(cudaEventRecord(hs.ev_in, ctx->h2d));
    // kernels: after the input landed and the slot's previous outputs were drained
    CK(cudaStreamWaitEvent(stream, hs.ev_in, 0));
    if (hs.used) CK(cudaStreamWaitEvent(stream, hs.ev_out, 0));
    if (b.M > 0) {
      CK(cudaStreamWaitEvent(stream, ctx->upload_done, 0));
      if ((rc = launch_batch(ctx, b, static_cast<char*>(stp->dev), stream))) return rc;
    }
    CK(cudaEventRecord(hs.ev_comp, stream));
    // D2H
    CK(cudaStreamWaitEvent(ctx->d2h, hs.ev_comp, 0));
    pos = 0;
    for (const Piece& p : ch) {
      const ss_seg& s = segs[p.seg];
      const int64_t n = p.r1 - p.r0;
      if (seg_status[p.seg] == SS_SEG_OK) {
        CK(copy_rows(static_cast<char*>(s.dst) + p.r0 * s.dst_ld * esz_out, (size_t)s.dst_ld * esz_out,
                     static_cast<const char*>(hs.out) + pos * N * esz_out, (size_t)N * esz_out,
                     (size_t)N * esz_out, (size_t)n, cudaMemcpyDeviceToHost, ctx->d2h));
        if (s.dst_base && pass_kind != SS_PASS_BACKWARD)
          CK(copy_rows(static_cast<char*>(s.dst_base) + p.r0 * s.base_ld * esz_base,
                       (size_t)s.base_ld * esz_base, static_cast<const char*>(hs.base) + pos * N * esz_base,
                       (size_t)N * esz_base, (size_t)N * esz_base, (size_t)n, cudaMemcpyDeviceToHost, ctx->d2h));
      }
      pos += n;
    }
    CK(cudaEventRecord(hs.ev_out, ctx->d2h));
    hs.used = true;
  }
  // results are in the caller's host buffers when this returns (serve_* is synchronous)
  CK(cudaStreamSynchronize(ctx->d2h));
  return SS_OK;
}

}  // extern "C"

// ---- LSV1 frames ------------------------------------------------------------------------
namespace {
constexpr size_t kHdr = 30;
const char* kRoleNames[7] = {"Q", "K", "V", "O", "FF_UP", "FF_DOWN", "LM_HEAD"};

struct Frame {
  size_t off = 0;          // offset of the header in `in`
  uint32_t client = 0;
  uint64_t rid = 0;
  uint16_t block = 0;
  uint8_t role = 0, pass = 0;
  uint32_t t = 0, w = 0;
  std::string err;         // non-empty: reply is a PASS_ERROR frame with this message
  uint32_t out_w = 0;      // reply width (compute frames)
  size_t out_off = 0;      // offset of the reply frame in `out`
};

template <typename T>
T rd(const uint8_t* p) {
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}
template <typename T>
void wr(uint8_t* p, T v) {
  memcpy(p, &v, sizeof(T));
}

// repr of the reference's LayerAddress (config.py:27-33), as executor messages print it
std::string addr_repr(int block, int role) {
  char buf[96];
  if (role >= 0 && role < 7)
    snprintf(buf, sizeof buf, "LayerAddress(block=%d, role=<Role.%s: %d>)", block, kRoleNames[role], role);
  else
    snprintf(buf, sizeof buf, "LayerAddress(block=%d, role=%d)", block, role);
  return buf;
}

void write_header(uint8_t* p, const Frame& f, uint8_t pass, uint32_t t, uint32_t w) {
  memcpy(p, "LSV1", 4);
  wr<uint16_t>(p + 4, 1);
  wr<uint32_t>(p + 6, f.client);
  wr<uint64_t>(p + 10, f.rid);
  wr<uint16_t>(p + 18, f.block);
  wr<uint8_t>(p + 20, f.role);
  wr<uint8_t>(p + 21, pass);
  wr<uint32_t>(p + 22, t);
  wr<uint32_t>(p + 26, w);
}
}  // namespace

extern "C" int ss_serve_frames(ss_ctx* ctx, const uint8_t* in, size_t in_len, size_t* consumed,
                               uint8_t* out, size_t out_cap, size_t* out_len, void* stream_) {
  if (!ctx || (!in && in_len) || !consumed || !out_len) return SS_E_ARG;
  std::lock_guard<std::recursive_mutex> guard_(ctx->mu);
  *consumed = 0;
  *out_len = 0;
  // ---- parse whole frames (try_decode, protocol.py:125-153)
  std::vector<Frame> fr;
  size_t pos = 0;
  while (true) {
    const size_t left = in_len - pos;
    if (left < kHdr) {
      if (left >= 4 && memcmp(in + pos, "LSV1", 4) != 0) return fail(ctx, SS_E_PROTOCOL, "bad magic");
      break;
    }
    const uint8_t* p = in + pos;
    if (memcmp(p, "LSV1", 4) != 0) return fail(ctx, SS_E_PROTOCOL, "bad magic");
    const uint16_t version = rd<uint16_t>(p + 4);
    if (version != 1) return fail(ctx, SS_E_PROTOCOL, "unsupported protocol version %u", version);
    Frame f;
    f.off = pos;
    f.client = rd<uint32_t>(p + 6);
    f.rid = rd<uint64_t>(p + 10);
    f.block = rd<uint16_t>(p + 18);
    f.role = rd<uint8_t>(p + 20);
    f.pass = rd<uint8_t>(p + 21);
    f.t = rd<uint32_t>(p + 22);
    f.w = rd<uint32_t>(p + 26);
    const size_t size = f.pass == 255 ? (size_t)f.t : (size_t)4 * f.t * f.w;
    if (left < kHdr + size) break;
    fr.push_back(f);
    pos += kHdr + size;
  }
  // ---- intake checks in arrival order (BaseExecutor.submit, executor.py:162-178), on a copy of
  // the request-id table: nothing is committed unless the frames are actually served
  std::map<uint32_t, uint64_t> rids = ctx->last_request_id;
  for (Frame& f : fr) {
    char msg[160];
    if (f.pass > 2) {
      snprintf(msg, sizeof msg, "unknown pass %u", f.pass);
      f.err = msg;
      continue;
    }
    auto it = rids.find(f.client);
    if (it != rids.end() && f.rid <= it->second) {
      snprintf(msg, sizeof msg, "request_id %llu not increasing (last %llu)", (unsigned long long)f.rid,
               (unsigned long long)it->second);
      f.err = msg;
      continue;
    }
    rids[f.client] = f.rid;
    auto lit = ctx->layers.find({(int)f.block, (int)f.role});
    if (lit == ctx->layers.end()) {
      f.err = "unknown layer " + addr_repr(f.block, f.role);
      continue;
    }
    const Layer& L = lit->second;
    const uint32_t expected = f.pass == SS_PASS_BACKWARD ? L.d_out : L.d_in;
    // _compute_batch's width check (executor.py:208-211)
    if (f.w != expected) {
      snprintf(msg, sizeof msg, "row width %u does not match layer %s expected %u", f.w,
               addr_repr(f.block, f.role).c_str(), expected);
      f.err = msg;
      continue;
    }
    f.out_w = f.pass == SS_PASS_BACKWARD ? L.d_in : L.d_out;
  }
  // ---- reply layout (request order) and capacity
  size_t need = 0;
  for (Frame& f : fr) {
    f.out_off = need;
    need += kHdr + (f.err.empty() ? (size_t)4 * f.t * f.out_w : f.err.size());
  }
  if (need > out_cap) {
    *out_len = need;
    return fail(ctx, SS_E_NOMEM, "reply buffer too small: need %zu bytes", need);
  }
  ctx->last_request_id.swap(rids);
  *consumed = pos;
  *out_len = need;
  if (fr.empty()) return SS_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);

  // ---- device-side frame table: decoded-operand and reply-row offsets, reply headers, messages
  std::vector<FrameDesc> fd(fr.size());
  std::string msgs;
  int64_t x_elems = 0, o_elems = 0, max_vals = 1;
  for (size_t i = 0; i < fr.size(); ++i) {
    const Frame& f = fr[i];
    FrameDesc& d = fd[i];
    memset(&d, 0, sizeof d);
    d.in_off = (int64_t)(f.off + kHdr);
    d.out_off = (int64_t)f.out_off;
    if (f.err.empty()) {
      write_header(d.hdr, f, f.pass, f.t, f.out_w);
      d.t = (int32_t)f.t;
      d.w = (int32_t)f.w;
      d.out_w = (int32_t)f.out_w;
      d.x_off = x_elems;
      d.o_off = o_elems;
      x_elems += round_up((int64_t)f.t * f.w, 8);          // 16-byte aligned operand rows
      o_elems += round_up((int64_t)f.t * f.out_w, 4);
      max_vals = std::max<int64_t>(max_vals, (int64_t)f.t * std::max(f.w, f.out_w));
    } else {
      write_header(d.hdr, f, 255, (uint32_t)f.err.size(), 0);
      d.is_err = 1;
      d.msg_off = (int32_t)msgs.size();
      d.msg_len = (int32_t)f.err.size();
      msgs += f.err;
    }
  }
  int rc = SS_OK;
  if ((rc = ensure_dev(ctx, ctx->fr_in, ctx->fr_in_cap, round_up(in_len, 256) + 256, false))) return rc;
  if ((rc = ensure_dev(ctx, ctx->fr_out, ctx->fr_out_cap, round_up(need, 256) + 256, false))) return rc;
  if ((rc = ensure_dev(ctx, ctx->fr_x, ctx->fr_x_cap, (size_t)std::max<int64_t>(x_elems, 8) * 2, false))) return rc;
  if ((rc = ensure_dev(ctx, ctx->fr_o, ctx->fr_o_cap, (size_t)std::max<int64_t>(o_elems, 4) * 4, false))) return rc;
  const size_t t_bytes = round_up(fd.size() * sizeof(FrameDesc), 256);
  const size_t total = t_bytes + round_up(std::max<size_t>(1, msgs.size()), 256);
  Staging* stp = nullptr;
  if ((rc = acquire_staging(ctx, total, stp))) return rc;
  memcpy(stp->host, fd.data(), fd.size() * sizeof(FrameDesc));
  if (!msgs.empty()) memcpy(static_cast<char*>(stp->host) + t_bytes, msgs.data(), msgs.size());
  // raw request bytes and the frame table in, on the copy stream
  CK(cudaMemcpyAsync(ctx->fr_in, in, in_len, cudaMemcpyHostToDevice, ctx->h2d));
  CK(cudaMemcpyAsync(stp->dev, stp->host, total, cudaMemcpyHostToDevice, ctx->h2d));
  CK(cudaEventRecord(stp->done, ctx->h2d));
  stp->pending = true;
  CK(cudaStreamWaitEvent(stream, stp->done, 0));
  const FrameDesc* dfd = reinterpret_cast<const FrameDesc*>(stp->dev);
  const uint8_t* dmsg = static_cast<const uint8_t*>(stp->dev) + t_bytes;
  const int gx = (int)std::min<int64_t>((max_vals + 511) / 512, 4 * ctx->num_sms);
  for (size_t f0 = 0; f0 < fd.size(); f0 += 65535) {
    const unsigned gy = (unsigned)std::min<size_t>(65535, fd.size() - f0);
    frame_decode_kernel<<<dim3(gx, gy), 256, 0, stream>>>(reinterpret_cast<const uint8_t*>(ctx->fr_in), dfd + f0,
                                                          reinterpret_cast<__nv_bfloat16*>(ctx->fr_x));
    CK(cudaGetLastError());
    ctx->launches++;
  }
  // ---- one fused dispatch per (block, role, pass) group, FIFO within the group
  std::vector<char> done(fr.size(), 0);
  for (size_t i = 0; i < fr.size(); ++i) {
    if (done[i] || !fr[i].err.empty()) continue;
    const Layer& L = ctx->layers.find({(int)fr[i].block, (int)fr[i].role})->second;
    std::vector<ss_seg> segs;
    std::vector<int> grp;
    for (size_t j = i; j < fr.size(); ++j) {
      const Frame& f = fr[j];
      if (done[j] || !f.err.empty() || f.block != fr[i].block || f.role != fr[i].role || f.pass != fr[i].pass) continue;
      done[j] = 1;
      grp.push_back((int)j);
      ss_seg s{};
      s.client_id = f.client;
      s.rows = f.t;
      s.width = f.w;
      s.flags = SS_SEGF_SRC_BF16 | (L.adapters.count(f.client) ? SS_SEGF_ADAPTER : 0);  // f32 reply rows
      s.src = reinterpret_cast<__nv_bfloat16*>(ctx->fr_x) + fd[j].x_off;
      s.src_ld = f.w;
      s.dst = reinterpret_cast<float*>(ctx->fr_o) + fd[j].o_off;
      s.dst_ld = f.out_w;
      segs.push_back(s);
    }
    std::vector<int32_t> st(segs.size(), 0);
    if ((rc = ss_compute_batch(ctx, fr[i].pass, fr[i].block, fr[i].role, (int)segs.size(), segs.data(), stream,
                               st.data())))
      return rc;
    for (size_t k = 0; k < segs.size(); ++k)
      if (st[k] != SS_SEG_OK) return fail(ctx, SS_E_ARG, "frame %d rejected after validation (status %d)", grp[k], st[k]);
  }
  // ---- reply stream encoded on the device, one copy back
  for (size_t f0 = 0; f0 < fd.size(); f0 += 65535) {
    const unsigned gy = (unsigned)std::min<size_t>(65535, fd.size() - f0);
    frame_encode_kernel<<<dim3(gx, gy), 256, 0, stream>>>(reinterpret_cast<uint8_t*>(ctx->fr_out), dfd + f0,
                                                          reinterpret_cast<const float*>(ctx->fr_o), dmsg);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  CK(cudaMemcpyAsync(out, ctx->fr_out, need, cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  return SS_OK;
}
