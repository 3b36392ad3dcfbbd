// Adapter weight-gradient kernels: the client-side half of a fine-tune
// step that the reference computes in numpy after every executor backward reply.
//
//   K6 lora_grad_kernel : grad_b = s * (x.A)^T . g and grad_a = s * x^T . (g.B^T)
//                         (lora_backward, reference adapters.py:26-41). The two shrinks
//                         s*x.A and s*g.B^T run first on lora_shrink_kernel (K3, one launch
//                         for both) into per-segment blocks of one Q buffer; this kernel then contracts over the TOKEN axis:
//                         D[128 rows of d_in | d_out, npad] = Src^T . Q, with Src = x (grad_a)
//                         or g (grad_b) loaded MN-major straight from the client's rows.
//   K7 ia3_grad_*       : grad_l = sum_rows dy * y_base (ClientModel._layer_backward,
//                         reference client.py:291-293), a deterministic two-phase column
//                         reduction (128-row chunk sums, then chunk-ordered totals).
//
// Both are HBM-bound (each reads the client's saved activations once; LoRA: 2*r FLOP per
// byte of x / g per contraction), so they run 2 CTAs per SM.
#pragma once
#include "kernels.cuh"

namespace ss {

struct LoraGradSeg {
  int32_t rows;       // tokens t
  int32_t qrow0;      // first row of this segment's block in Qx / Qg (64-aligned, zero-padded)
  int32_t rank;
  int32_t npad;       // UMMA N: rank rounded up to 64 (<= 256)
  int32_t accumulate; // 1: += into grad_a / grad_b (client.py _accumulate), 0: overwrite
  int32_t xmap;       // tensor map (box {64, 64}) over x  [t, d_in]
  int32_t gmap;       // tensor map (box {64, 64}) over g  [t, d_out]
  int32_t pad_;
  float* dA;          // [d_in, rank]  row-major f32
  float* dB;          // [rank, d_out] row-major f32
};

struct LoraGradItem {
  int32_t seg;
  int32_t which;      // 0: grad_a (M over d_in, Src = x, Q = s*g.B^T); 1: grad_b (M over d_out, Src = g, Q = s*x.A)
  int32_t m0;         // first output row of d_in / d_out
  int32_t pad_;
};

struct LoraGradParams {
  int d_in, d_out;
  int qrows;          // rows of the s*x.A half of Q; the s*g.B^T half follows
  const LoraGradSeg* segs;
  const LoraGradItem* items;
  const CUtensorMap* tmaps;
};

constexpr int GRAD_SMEM = 110 * 1024;
constexpr int GRAD_MAX_STAGES = 8;
constexpr int GRAD_CHUNK_BYTES = 64 * 64 * 2;  // one {64 MN, 64 K} SW128 box = 8 KB

__device__ __forceinline__ void lora_grad_body(const CUtensorMap& tmQ,  // [s*x.A ; s*g.B^T] [2*qrows, qld] bf16
                                               const LoraGradParams& p, const int item) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const LoraGradItem it = p.items[item];
  const LoraGradSeg sg = p.segs[it.seg];
  const int npad = sg.npad;
  const int nq = npad / 64;
  const CUtensorMap* tmSrc = p.tmaps + (it.which ? sg.gmap : sg.xmap);
  const int qrow = sg.qrow0 + (it.which ? 0 : p.qrows);
  const int b_bytes = nq * GRAD_CHUNK_BYTES;
  const int stage_bytes = A_STAGE_BYTES + b_bytes;
  const int NST = min(GRAD_MAX_STAGES, (GRAD_SMEM - 2048) / stage_bytes);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty_bar = full_bar + GRAD_MAX_STAGES;
  uint64_t* tfull = empty_bar + GRAD_MAX_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  uint8_t* stage0 = smem + 1024;

  if (warp == 0 && lane == 0) {
    tensormap_acquire(tmSrc);
    tma_prefetch_desc(tmSrc);
    tma_prefetch_desc(&tmQ);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = (sg.rows + 63) / 64;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        mbar_expect_tx(&full_bar[s], stage_bytes);
        uint8_t* a = stage0 + s * stage_bytes;
        // A = Src^T: two MN chunks of 64 output rows x 64 tokens (rows past t are zero-filled)
        tma_load_2d(a, tmSrc, &full_bar[s], it.m0, kb * 64);
        tma_load_2d(a + GRAD_CHUNK_BYTES, tmSrc, &full_bar[s], it.m0 + 64, kb * 64);
        for (int q = 0; q < nq; ++q)
          tma_load_2d(a + A_STAGE_BYTES + q * GRAD_CHUNK_BYTES, &tmQ, &full_bar[s], q * 64,
                      qrow + kb * 64);
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(BM, (uint32_t)npad, true, true);
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full_bar[s], ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a_addr = smem_u32(stage0 + s * stage_bytes);
        const uint32_t b_addr = a_addr + A_STAGE_BYTES;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_bf16_ss(tmem_base, make_sdesc_sw128(a_addr + k * (UK * 128), GRAD_CHUNK_BYTES, 1024),
                      make_sdesc_sw128(b_addr + k * (UK * 128), GRAD_CHUNK_BYTES, 1024), idesc,
                      (kb | k) != 0);
        mma_commit(&empty_bar[s]);
      }
      __syncwarp();
      if (++s == NST) { s = 0; ph ^= 1; }
    }
    if (lane == 0) mma_commit(tfull);
    __syncwarp();
  } else if (warp >= 4) {
    const uint32_t ew = warp - 4;
    const int m = it.m0 + ew * 32 + lane;  // output row (of d_in for grad_a, of d_out for grad_b)
    const int mdim = it.which ? p.d_out : p.d_in;
    const bool ok = m < mdim && nkb > 0;
    mbar_wait(tfull, 0);
    tc_fence_after();
    for (int c = 0; c < npad / 16; ++c) {
      if (c * 16 >= sg.rank) break;
      uint32_t r[16];
      tmem_ld_32x32b_x16(tmem_base + c * 16 + ((ew * 32u) << 16), r);
      tmem_wait_ld();
      if (!ok) continue;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = c * 16 + j;
        if (col < sg.rank) {
          // grad_a[m, col] (row-major [d_in, r]); grad_b[col, m] (row-major [r, d_out]: a warp
          // writes 32 consecutive floats per column)
          float* o = it.which ? sg.dB + (int64_t)col * p.d_out + m : sg.dA + (int64_t)m * sg.rank + col;
          const float v = __uint_as_float(r[j]);
          *o = sg.accumulate ? *o + v : v;
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 256);
  }
}

__global__ void __launch_bounds__(GEMM_THREADS, 2)
    lora_grad_kernel(const __grid_constant__ CUtensorMap tmQ, const LoraGradParams p) {
  lora_grad_body(tmQ, p, (int)blockIdx.x);
}

// K3 + K6 in one launch, client by client. Two launches (every shrink, then every token
// contraction) read each client's x and g twice from HBM: by the time the contractions run, the
// shrinks have streamed every other client's activations through L2. Here a CTA takes the next
// entry of a work list (atomic ticket, so entries start in list order) that interleaves the
// shrink items of client j with the contraction items of client j - lag; a contraction waits
// until its client's shrink items have all finished (Q complete), which are earlier entries,
// already running on started CTAs, so the wait always ends (no co-residency assumption) and
// the client's x / g are still in L2 when the contraction re-reads them. Per-item code is the
// two kernels' own, so every output is bitwise that of the two-launch path.
constexpr int GRAD_FUSED_SMEM = SHRINK_SMEM > GRAD_SMEM ? SHRINK_SMEM : GRAD_SMEM;

struct GradFusedParams {
  const int2* work;   // {0: shrink item | 1: contraction item, index}
  int* queue;         // ticket (zero before the launch)
  int* done;          // [clients] finished shrink items (zero before the launch)
  const int* need;    // [clients] shrink items per client
};

__global__ void __launch_bounds__(GEMM_THREADS, 2)
    lora_grad_fused_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmP2,
                           const __grid_constant__ CUtensorMap tmQ, const ShrinkParams sp,
                           const LoraGradParams gp, const GradFusedParams fp) {
  __shared__ int s_entry;
  if (threadIdx.x == 0) s_entry = atomicAdd(fp.queue, 1);
  __syncthreads();
  const int2 w = fp.work[s_entry];
  if (w.x == 0) {
    lora_shrink_body(tmP, tmP2, sp, w.y, 0, 1);
    __threadfence();   // this CTA's Q rows before the arrival
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(fp.done + sp.items[w.y].seg, 1);
  } else {
    const int seg = gp.items[w.y].seg;
    if (threadIdx.x == 0) {
      while (ld_acquire_gpu(fp.done + seg) < fp.need[seg]) __nanosleep(64);
      fence_proxy_async_global();   // Q (generic-proxy stores) before this CTA's TMA reads
    }
    __syncthreads();
    lora_grad_body(tmQ, gp, w.y);
  }
}

// ---------------------------------------------------------------------------- K7 IA3 grad
struct Ia3GradSeg {
  int32_t rows;
  int32_t flags;        // bit0 dy bf16, bit1 y_base bf16, bit2 both 16-byte aligned rows, bit3 accumulate
  const void* dy;
  int64_t dy_ld;
  const void* yb;
  int64_t yb_ld;
  float* dl;            // [d_out]
};

__device__ __forceinline__ void load8(const void* base, int64_t off, bool bf, bool vec, int ncols,
                                      float (&v)[8]) {
  if (vec && ncols == 8) {
    if (bf) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + off));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      }
    } else {
      const float4* f4 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off);
      const float4 a = __ldg(f4), b = __ldg(f4 + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = i < ncols ? (bf ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[off + i])
                             : reinterpret_cast<const float*>(base)[off + i])
                       : 0.f;
  }
}

// Two deterministic phases, balanced over the SMs: K7a = one 256-thread block per (segment,
// 256 columns, 128-row chunk) — lane group cg owns 8 columns, warp rg takes every 8th row of the
// chunk — writes the chunk's column sums (fixed-order warp partials) to a workspace; K7b adds the
// chunk sums of each (segment, column) in chunk order into grad_l. No atomics: the result does
// not depend on scheduling (or on which other clients share the call).
constexpr int IA3_ROWS = 128;
constexpr int IA3_COLS = 256;

struct Ia3PartItem {
  int32_t seg;
  int32_t c0;           // first of 256 columns
  int32_t r0;           // first row of the 128-row chunk
  int32_t part;         // workspace row of this item's 256 partial sums
};
struct Ia3FinItem {
  int32_t seg;
  int32_t c0;
  int32_t part0;        // workspace row of chunk 0; chunks follow consecutively
  int32_t nchunk;
};
struct Ia3PartParams {
  int d_out;
  const Ia3GradSeg* segs;
  const Ia3PartItem* items;
  float* part;          // [n_items, 256]
};
struct Ia3FinParams {
  int d_out;
  const Ia3GradSeg* segs;
  const Ia3FinItem* items;
  const float* part;
};

__global__ void __launch_bounds__(256) ia3_grad_partial_kernel(const Ia3PartParams p) {
  __shared__ float sm[8][IA3_COLS + 1];
  const Ia3PartItem it = p.items[blockIdx.x];
  const Ia3GradSeg sg = p.segs[it.seg];
  const int cg = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int c = it.c0 + cg * 8;
  const int ncols = max(0, min(8, p.d_out - c));
  const bool dbf = sg.flags & 1, bbf = sg.flags & 2, vec = sg.flags & 4;
  const int r1 = min(sg.rows, it.r0 + IA3_ROWS);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (ncols > 0) {
#pragma unroll 4
    for (int r = it.r0 + rg; r < r1; r += 8) {
      float a[8], b[8];
      load8(sg.dy, (int64_t)r * sg.dy_ld + c, dbf, vec, ncols, a);
      load8(sg.yb, (int64_t)r * sg.yb_ld + c, bbf, vec, ncols, b);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(a[i], b[i], acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sm[rg][cg * 8 + i] = acc[i];
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) s += sm[g][threadIdx.x];
  p.part[(int64_t)it.part * IA3_COLS + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ia3_grad_finalize_kernel(const Ia3FinParams p) {
  const Ia3FinItem it = p.items[blockIdx.x];
  const int col = it.c0 + threadIdx.x;
  if (col >= p.d_out) return;
  const Ia3GradSeg sg = p.segs[it.seg];
  float s = 0.f;
  for (int k = 0; k < it.nchunk; ++k) s += p.part[(int64_t)(it.part0 + k) * IA3_COLS + threadIdx.x];
  float* o = sg.dl + col;
  *o = (sg.flags & 8) ? *o + s : s;
}

}  // namespace ss
