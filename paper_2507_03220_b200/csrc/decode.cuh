// K1d: split-K GEMM for decode-class segments (SURVEY §8a affine_forward /
// affine_backward_input / noise matmul + the fused adapter epilogue, for requests of a few rows).
//
// Why a separate kernel and a separate summation order. A decode dispatch streams W (HBM-bound in
// principle), but every output column of the single-chain kernels is K/16 dependent UMMAs
// accumulating into one TMEM accumulator, and at decode sizes that chain, not HBM, sets the time
// (DESIGN.md "Decode"). Only a shorter chain helps, and a shorter chain is a different fp32
// summation order. Rows of a decode-class segment (its own row count <= decode_rows, a property
// of the request alone) therefore use their own fixed order, independent of the dispatch:
//
//   K is cut into C = ceil(K / (64 * kbc)) contiguous chunks of kbc 64-deep k-blocks (kbc =
//   decode_chunk_kb, a per-context constant); chunk c is one UMMA chain in K order. Backward
//   segments with the IA3 lo operand (SEGF_IA3_LO) add C more chains over the lo halves. The
//   LoRA expand of a row is one chain over its own rank block: per 64-row slice, the hi columns,
//   then the lo columns (fp32-tier hi / lo pair). y = fold(p_0 ..
//   p_{C-1}, [lo_0 .. lo_{C-1}], [p_lora]) left to right, then bias / y_base / IA3.
//
// A row's bits depend only on its segment's class, K and its own values (foreign rows of the
// block-diagonal LoRA operand contribute exact zeros, and so do the lo chains of rows without a
// lo half). The tile's LoRA operand is block-diagonal over its segments and is cut into pieces of
// whole segments (shorter chains, spread over CTAs); a row reads the piece holding its block,
// whose chain over the other segments' columns adds exact zeros. So batched == solo holds for decode-class rows exactly as for the single-chain kernels
// (tests/test_gpu_decode.py).
//
// Work. A unit is (64-row decode tile m, chunk c, 64-column tile n). Consecutive units of one
// chunk form host-built groups of g <= DEC_G = 4 n tiles (LoRA pieces: DEC_G_LORA), which the
// CTAs of a persistent grid claim through an atomic ticket (a CTA that starts late does fewer): one UMMA of N = 64 g covers the group (a chain of
// kbc * 4 UMMAs per group instead of K / 16), and each stage carries one k-block of A (8 KB, read
// once per group) beside the group's W boxes (32 KB). W is streamed with L2 evict_first; each
// unit's fp32 partial goes to the workspace with evict_last, so it is still in L2 for the fixup; no CTA waits on another: the fixed-order sum, bias / y_base / IA3 and the stores run
// in dec_fixup_kernel, launched behind the GEMM with programmatic dependent launch.
//
// The UMMA is M = 128: the A box holds 64 rows; MMA rows 64-127 read the W boxes that follow it in
// the stage and their outputs are never read.
#pragma once
#include "kernels.cuh"

namespace ss {

constexpr int DEC_ROWS = 64;                            // packed rows per decode tile
constexpr int DEC_TN = 64;                              // output columns per unit
constexpr int DEC_G = 4;                                // n tiles interleaved per group
constexpr int DEC_MAX_KBC = 48;                         // k-blocks per chunk (option bound: decode shrink smem)
constexpr int DEC_KB_BYTES = DEC_ROWS * 128;            // one k-block of A (64 rows x 64 k): 8 KB
constexpr int DEC_WBOX = 64 * 128;                      // one {64 n, 64 k} W box: 8 KB
// stage (40 KB). Chunk units: one k-block, the A box (8 KB) + the group's W boxes (<= 32 KB).
// LoRA units (groups of <= DEC_G_LORA n tiles): one <= 64-row slice of a segment's rank block,
// its A_lora hi and lo columns (16 KB) + the group's pack boxes of those rows (<= 24 KB, read
// once for hi and lo)
constexpr int DEC_G_LORA = 3;
constexpr int DEC_STAGE = DEC_KB_BYTES + DEC_G * DEC_WBOX;
constexpr int DEC_STAGES = 5;
__host__ __device__ constexpr int dec_b_off(int kind) { return kind ? 2 * DEC_KB_BYTES : DEC_KB_BYTES; }
constexpr int DEC_LP_CHUNKS = 24;                       // max LoRA chunks per piece (unless one segment has more)
constexpr int DEC_PART = DEC_ROWS * DEC_TN;             // fp32 values per unit partial (16 KB)
constexpr int DEC_GQ = 8;                               // claimed-group ring depth
constexpr int DEC_SMEM = DEC_STAGES * DEC_STAGE + 1024 + 512;

struct DecTile {
  int32_t arow;          // first packed (X) row
  int32_t rows;          // valid rows (<= DEC_ROWS), whole segments
  int32_t al_row;        // first row of the tile's block-diagonal LoRA operand
  int32_t lo;            // 1: some row is SEGF_IA3_LO -> C lo chains over X_lo
  int32_t chunk_begin;   // LoRA rank chunks (pack rows) of the tile in `chunks`
  int32_t chunk_count;   // 0: no LoRA for this tile
  int32_t unit_begin;    // first unit of the tile
  int32_t lp_begin;      // the tile's LoRA pieces in `lpieces`
  int32_t lp_count;
  int32_t pad_[3];
};

struct DecParams {
  int N, K;
  int C;                 // K chunks
  int kbc;               // k-blocks per chunk
  int n_m, n_n;          // decode tiles, 64-column tiles
  int S;                 // partial slots per (m, n): 2C + max pieces (hi chunks, lo chunks, LoRA pieces)
  int has_bias, ia3_in_epilogue;
  const float* bias;
  const DevSeg* segs;
  const int32_t* row_seg;
  const DecTile* tiles;
  const int32_t* chunks;
  const int2* lpieces;        // LoRA pieces: {first entry in `lstages`, stage count}
  const int4* lstages;        // LoRA stages: {pack row, 16-row chunks (<= 4), A_lora hi col, lo col | -1}
  const int4* groups;         // work groups {mt, kind << 8 | g, c, nt0}: chunk groups, then LoRA groups
  int g_begin, g_end;         // this launch's groups
  int* claim;                 // [2] group ticket + exiting-CTA count (zero between launches: the
                              // last CTA to exit resets both)
  const CUtensorMap* tmaps;
  int amap, alo_map;     // X / X_lo as {64 k, 64 rows, kbc k-blocks} boxes
  float* part;           // [(m * n_n + n) * S + slot][DEC_ROWS][DEC_TN] fp32 partials
  long long* trace;      // testing: per CTA {start ns, end ns, groups run, units run} (nullptr: off)
  int pdl_early;         // launched behind the gather / shrink: the producer streams its first W
                         // stages before griddepcontrol.wait (every other role waits on its loads)
  // In-kernel fixup (nullptr: the separate dec_fixup_kernel runs behind the GEMM). fx_cnt counts,
  // per (m, n tile, 32-row half), the groups whose partials are stored (release by the epilogue
  // warp of that half; self-resetting); the CTA's otherwise idle warps claim fixup units through
  // fx_claim[0] in unit order and fold a unit once its count is complete.
  int* fx_cnt;
  int* fx_claim;
};

__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A group of units one CTA runs back to back: kind 0 a chunk (slot c; the lo chains have slots
// C + c), kind 1 LoRA piece c - 2C (slot c); g consecutive n tiles starting at nt0. Groups are
// host-built and claimed dynamically (atomic ticket), so a CTA that starts late (its SM busy with
// the side-stream shrink) simply runs fewer of them.
struct DecGroup {
  int mt, kind, c, nt0, g;
};

__device__ __forceinline__ DecGroup dec_group(const DecParams& p, int id) {
  const int4 v = p.groups[id];
  DecGroup gr;
  gr.mt = v.x;
  gr.kind = v.y >> 8;
  gr.g = v.y & 0xff;
  gr.c = v.z;
  gr.nt0 = v.w;
  return gr;
}

__device__ __forceinline__ void dec_store8(const float (&v)[8], int ncols, char* dst, bool bf, bool vec) {
  if (ncols == 8 && vec) {
    if (bf) {
      *reinterpret_cast<uint4*>(dst) = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                                                  pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
    } else {
      float4* o = reinterpret_cast<float4*>(dst);
      o[0] = make_float4(v[0], v[1], v[2], v[3]);
      o[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < ncols) {
        if (bf) reinterpret_cast<__nv_bfloat16*>(dst)[j] = __float2bfloat16_rn(v[j]);
        else reinterpret_cast<float*>(dst)[j] = v[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------- decode shrink
// The LoRA intermediate s*x.A (forward) / s*g.B^T (backward) of decode-class segments (<= 16
// rows), on CUDA cores: at a few rows the tensor-core shrink is a chain of K/16 UMMAs per CTA for
// M = 2, and its time is that chain plus a split-K tail. Order (part of the decode class's
// numerics): K in the class's chunks (kbc k-blocks, as the GEMM); within a chunk, lane l of a
// warp owns k = 8 l + 256 i (ascending i, the 8 products in order), then an xor-shuffle tree over
// the 32 lanes (grid: item x chunk x 32-row rank group; a warp takes 4 rank rows); chunks added in order by the item's last CTA, times alpha / r, rounded to bf16
// (hi) and, for hi / lo segments, bf16(v - hi) (lo) into the tile's block-diagonal LoRA operand;
// the tile's other rows get zeros in this segment's columns.
struct DecShrinkItem {
  int32_t seg;          // DevSeg (pack_row, rank_pad, lora_scale)
  int32_t rows;         // <= 16
  int32_t kind;         // 0: bf16 rows at src, 1: f32 rows at src (rounded to bf16 on load)
  int32_t hilo;         // 1: write the lo half too
  const void* src;      // first row (the client's rows in place, or the packed X rows)
  int64_t ld;           // elements
  const __nv_bfloat16* src_lo;   // non-null: + X_lo rows (backward IA3 lo operand), ld `ld`
  int32_t col;          // first column of the segment's rank block
  int32_t tile_row0;    // A_lora row of its decode tile's first row
  int32_t p0;           // the segment's first row within the tile
};

struct DecShrinkParams {
  int K, kbc, C;
  int lora_ld;
  const DevSeg* segs;
  const DecShrinkItem* items;
  const __nv_bfloat16* pack;     // [R, K] K-major pack rows (A^T forward, B backward)
  int64_t pack_ld;
  __nv_bfloat16* a_lora;
  float* part;                   // [items][C][16][256] fp32 chunk partials
  int* ticket;                   // [items] (zero between launches; the last CTA resets)
};

constexpr int DEC_SHR_THREADS = 256;
constexpr int DEC_SHR_MAXROWS = 16;

// Block (bx, by, bz) of a (items, C, gz) grid: the kernel below, or a share of a combined
// launch with the gather (dec_prologue_kernel).
template <int MAXR>   // rows per item bound (4 or DEC_SHR_MAXROWS): the accumulators' registers
__device__ __forceinline__ void dec_shrink_body(const DecShrinkParams& p, const int bx, const int by, const int bz,
                                                const int gz) {
  extern __shared__ float xs[];   // [rows][kbc * 64] bf16-rounded x of this chunk
  __shared__ int last;
  const DecShrinkItem it = p.items[bx];
  const DevSeg sg = p.segs[it.seg];
  const int R = sg.rank_pad, rows = it.rows;
  const int c = by;
  const int kc = p.kbc * 64;
  const int k0 = c * kc, kn = min(p.K - k0, kc);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // x rows of the chunk -> shared memory (as the GEMM's bf16 operand would hold them)
  // (8 consecutive values per thread and load: 16-byte bf16 / 2 x 16-byte f32 vectors when the
  // rows are 16-byte aligned, all of a thread's loads issued before its shared-memory stores)
  const bool vec = it.kind == 0 ? ((reinterpret_cast<uintptr_t>(it.src) | (uintptr_t)(it.ld * 2)) & 15) == 0
                                : ((reinterpret_cast<uintptr_t>(it.src) | (uintptr_t)(it.ld * 4)) & 15) == 0;
  // this CTA: rank rows [32 z, 32 z + 32); warp w: 4 of them, every load of a 4 x 1024-k block
  // issued before its FMAs (the kernel is load-latency bound at these sizes); the first block's
  // loads go out before the x rows are even read
  const int q0 = bz * 32 + warp * 4;
  const __nv_bfloat16* prow = p.pack + (int64_t)(sg.pack_row + q0) * p.pack_ld + k0;
  uint4 raw[4][4];
  auto load_block = [&](int kb) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int k = kb + v * 256 + lane * 8;
        raw[i][v] = (q0 + i < R && k < kn) ? __ldg(reinterpret_cast<const uint4*>(prow + (int64_t)i * p.pack_ld + k))
                                           : make_uint4(0, 0, 0, 0);
      }
  };
  load_block(0);
  const int n8 = rows * (kn / 8);
  for (int i = tid; i < n8; i += DEC_SHR_THREADS) {
    const int r = i / (kn / 8), k = (i - r * (kn / 8)) * 8;
    const int64_t off = (int64_t)r * it.ld + k0 + k;
    float v[8];
    if (vec && it.kind == 0) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(it.src) + off));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
      }
    } else if (vec) {
      const float4* f4 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(it.src) + off);
      const float4 a = __ldg(f4), b = __ldg(f4 + 1);
      const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(__float2bfloat16_rn(f[j]));
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = it.kind == 0 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(it.src)[off + j])
                            : __bfloat162float(__float2bfloat16_rn(reinterpret_cast<const float*>(it.src)[off + j]));
    }
    if (it.src_lo) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += __bfloat162float(it.src_lo[off + j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) xs[r * kc + k + j] = v[j];
  }
  __syncthreads();
  float* part = p.part + ((int64_t)bx * p.C + c) * DEC_SHR_MAXROWS * 256;
  float acc[4][MAXR];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int r = 0; r < MAXR; ++r) acc[i][r] = 0.f;
  for (int kb = 0; kb < kn; kb += 4 * 256) {
    if (kb > 0) load_block(kb);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int k = kb + v * 256 + lane * 8;
      if (k >= kn) break;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[i][v]);
        float w[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(h[j]);
          w[2 * j] = f.x;
          w[2 * j + 1] = f.y;
        }
#pragma unroll
        for (int r = 0; r < MAXR; ++r) {
          if (r < rows) {
            const float4 xa = *reinterpret_cast<const float4*>(xs + r * kc + k);
            const float4 xb = *reinterpret_cast<const float4*>(xs + r * kc + k + 4);
            float a = acc[i][r];
            a = fmaf(xa.x, w[0], a); a = fmaf(xa.y, w[1], a); a = fmaf(xa.z, w[2], a); a = fmaf(xa.w, w[3], a);
            a = fmaf(xb.x, w[4], a); a = fmaf(xb.y, w[5], a); a = fmaf(xb.z, w[6], a); a = fmaf(xb.w, w[7], a);
            acc[i][r] = a;
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      if (r < rows) {
        float v = acc[i][r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && q0 + i < R) part[r * 256 + q0 + i] = v;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(p.ticket + bx, 1) == p.C * gz - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float* base = p.part + (int64_t)bx * p.C * DEC_SHR_MAXROWS * 256;
  const int nh = it.hilo ? 2 : 1;
  // the tile's other rows: zeros in this segment's columns
  for (int i = tid; i < (DEC_ROWS - rows) * R; i += DEC_SHR_THREADS) {
    const int k = i / R, q = i - k * R;
    const int tr = k < it.p0 ? k : k + rows;
    __nv_bfloat16* out = p.a_lora + (int64_t)(it.tile_row0 + tr) * p.lora_ld + it.col + q;
    out[0] = __float2bfloat16_rn(0.f);
    if (nh == 2) out[R] = __float2bfloat16_rn(0.f);
  }
  // the segment's rows: chunk partials in chunk order, x alpha / r, hi (and lo) bf16
  for (int i = tid; i < rows * R; i += DEC_SHR_THREADS) {
    const int r = i / R, q = i - r * R;
    float v = 0.f;
    for (int cc = 0; cc < p.C; ++cc) v += __ldcg(base + (int64_t)cc * DEC_SHR_MAXROWS * 256 + r * 256 + q);
    v *= sg.lora_scale;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    __nv_bfloat16* out = p.a_lora + (int64_t)(it.tile_row0 + it.p0 + r) * p.lora_ld + it.col + q;
    out[0] = hi;
    if (nh == 2) out[R] = __float2bfloat16_rn(v - __bfloat162float(hi));
  }
  if (tid == 0) p.ticket[bx] = 0;   // ready for the next launch
}

template <int MAXR>
__global__ void __launch_bounds__(DEC_SHR_THREADS)
    dec_shrink_kernel(const DecShrinkParams p) {
  pdl_wait();
  pdl_trigger();
  dec_shrink_body<MAXR>(p, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)gridDim.z);
}

// A decode-only dispatch's prologue in ONE launch: blocks [0, n_shr) run the decode-class LoRA
// shrink (items x C x gz), the rest gather the rows into X. The two are independent (the shrink
// reads the client rows in place), so they run side by side as with a side-stream shrink, but
// the GEMM behind them keeps its programmatic edge (it streams W before griddepcontrol.wait).
template <int MAXR>
__global__ void __launch_bounds__(DEC_SHR_THREADS)
    dec_prologue_kernel(const DecShrinkParams sp, const GatherParams gp, const int n_shr, const int sy,
                        const int sz) {
  pdl_wait();
  pdl_trigger();
  const int b = (int)blockIdx.x;
  if (b < n_shr) {
    const int bz = b % sz, by = (b / sz) % sy, bx = b / (sz * sy);
    dec_shrink_body<MAXR>(sp, bx, by, bz, sz);
  } else {
    gather_rows_body(gp, b - n_shr, (int)gridDim.x - n_shr);
  }
}

__device__ __forceinline__ void st_f4_evict_last(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

// K1d fixup: y = fold(p_0 .. p_{C-1}, [lo_0 .. lo_{C-1}], [p_lora]) left to right, then bias /
// y_base / IA3 / dst, for every valid row of every decode tile. Launched behind the GEMM (PDL: the
// grid is resident early and waits on griddepcontrol.wait, which covers the GEMM's partial
// stores). One CTA per 32 rows x 64 columns of a tile; a thread owns one row x 8 columns and
// issues the loads of 8 partials at a time before adding them (the sum order is fixed, the loads
// are not serialised).
constexpr int DEC_FIX_ROWS = 32;
constexpr int DEC_FIX_THREADS = DEC_FIX_ROWS * (DEC_TN / 8);   // 256

__device__ __forceinline__ void dec_fixup_unit(const DecParams& p, const int unit, const int t) {
  const int q = unit % (DEC_ROWS / DEC_FIX_ROWS);
  const int tile = unit / (DEC_ROWS / DEC_FIX_ROWS);   // mt * n_n + nt
  const int mt = tile / p.n_n, nt = tile - mt * p.n_n;
  const int row = q * DEC_FIX_ROWS + t / (DEC_TN / 8);
  const int col = (t % (DEC_TN / 8)) * 8;
  const DecTile td = p.tiles[mt];
  const int n = nt * DEC_TN + col;
  if (row >= td.rows || n >= p.N) return;
  const float4* src = reinterpret_cast<const float4*>(p.part + (int64_t)tile * p.S * DEC_PART +
                                                      (int64_t)row * DEC_TN + col);
  constexpr int P4 = DEC_PART / 4;
  const int xrow = td.arow + row;
  const DevSeg sg = p.segs[p.row_seg[xrow]];
  // slots in fold order: hi chunks 0..C-1, lo chunks C..2C-1 (lo tiles only), then the LoRA
  // piece holding this row's rank block (every other piece is exact zeros for this row)
  const int nhl = td.lo ? 2 * p.C : p.C;
  const int nslots = nhl + ((sg.flags & SEGF_LORA) && td.lp_count > 0 ? 1 : 0);
  float v[8];
  for (int i0 = 0; i0 < nslots; i0 += 8) {
    float4 buf[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i0 + i < nslots) {
        const int slot = i0 + i < nhl ? i0 + i : 2 * p.C + sg.dec_piece;
        const float4* s = src + (int64_t)slot * P4;
        buf[i][0] = __ldcg(s);
        buf[i][1] = __ldcg(s + 1);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i0 + i < nslots) {
        const float w[8] = {buf[i][0].x, buf[i][0].y, buf[i][0].z, buf[i][0].w,
                            buf[i][1].x, buf[i][1].y, buf[i][1].z, buf[i][1].w};
        if (i0 + i == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = w[j];
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] += w[j];
        }
      }
    }
  }
  const int ncols = min(8, p.N - n);
  const int64_t r_local = xrow - sg.xrow0 + sg.xlocal0;
  const bool bf = sg.flags & SEGF_DST_BF16, bbf = sg.flags & SEGF_BASE_BF16;
  if (p.has_bias) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < ncols) v[j] += __ldg(p.bias + n + j);
  }
  if (sg.flags & SEGF_WANT_BASE)
    dec_store8(v, ncols, reinterpret_cast<char*>(sg.dst_base) + (r_local * sg.base_ld + n) * (bbf ? 2 : 4), bbf,
               sg.flags & SEGF_BASE_VEC);
  if (p.ia3_in_epilogue && (sg.flags & SEGF_IA3)) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < ncols) v[j] *= __ldg(sg.ia3 + n + j);
  }
  dec_store8(v, ncols, reinterpret_cast<char*>(sg.dst) + (r_local * sg.dst_ld + n) * (bf ? 2 : 4), bf,
             sg.flags & SEGF_DST_VEC);
}

template <bool kBwd>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    seg_gemm_dec_kernel(const __grid_constant__ CUtensorMap tmB,   // W: {64 n, 64 k} fwd / {64 k, 64 n} bwd
                        const __grid_constant__ CUtensorMap tmAL,  // A_lora, box {64, 64 rows}
                        const __grid_constant__ CUtensorMap tmBP,  // pack [R, N] (MN-major B), box {64, 16}
                        const __grid_constant__ CUtensorMap tmBP64,  // same pack, box {64, 64}
                        const DecParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + DEC_STAGES * DEC_STAGE);
  uint64_t* empty_bar = full_bar + DEC_STAGES;
  uint64_t* tfull_bar = empty_bar + DEC_STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;           // [2]
  uint64_t* qfull_bar = tempty_bar + 2;           // [DEC_GQ] claimed-group ring
  uint64_t* qempty_bar = qfull_bar + DEC_GQ;      // [DEC_GQ]
  int* q_id = reinterpret_cast<int*>(qempty_bar + DEC_GQ);   // [DEC_GQ]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_id + DEC_GQ);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const int nkb = p.K / BK;
  long long t_start = 0;
  if (p.trace && threadIdx.x == 0) t_start = globaltimer_ns();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmAL);
    tma_prefetch_desc(&tmBP);
    tma_prefetch_desc(&tmBP64);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2);   // warps 4 and 5 (TMEM lanes 0-63) read the accumulators
    }
    for (int q = 0; q < DEC_GQ; ++q) {
      mbar_init(&qfull_bar[q], 1);
      mbar_init(&qempty_bar[q], 3);   // the MMA warp and epilogue warps 4, 5
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * DEC_G * DEC_TN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!p.pdl_early) pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int pre = 0;      // stages whose W was issued before griddepcontrol.wait (A still to load)
      const CUtensorMap* tmA = p.tmaps + p.amap;
      const CUtensorMap* tmAlo = p.tmaps + p.alo_map;
      tensormap_acquire(tmA);
      if (p.alo_map != p.amap) tensormap_acquire(tmAlo);
      const uint64_t pol_w = policy_evict_first();   // W streams once; keep L2 for the partials
      int qi = 0;
      uint32_t qph = 0;
      int n_groups = 0, n_units = 0;
      // claim the next group and hand its id to the MMA / epilogue warps (-1: no more)
      auto claim = [&]() {
        const int t = atomicAdd(p.claim, 1) + p.g_begin;
        const int id = t < p.g_end ? t : -1;
        mbar_wait(&qempty_bar[qi], qph ^ 1);
        q_id[qi] = id;
        mbar_arrive(&qfull_bar[qi]);
        if (++qi == DEC_GQ) { qi = 0; qph ^= 1; }
        return id;
      };
      int id = claim();
      DecGroup gr;
      if (p.pdl_early) {
        // the first group's first stages: W (no dependency on the previous kernels) now, A (the
        // gathered rows) after griddepcontrol.wait
        if (id >= 0) {
          gr = dec_group(p, id);
          if (gr.kind == 0) {
            const int cc = gr.c >= p.C ? gr.c - p.C : gr.c;
            pre = min(DEC_STAGES, min(nkb, (cc + 1) * p.kbc) - cc * p.kbc);
            for (int st = 0; st < pre; ++st) {
              const int kb = cc * p.kbc + st;
              mbar_expect_tx(&full_bar[st], DEC_KB_BYTES + gr.g * DEC_WBOX);
              uint8_t* b = smem + st * DEC_STAGE + dec_b_off(0);
              for (int j = 0; j < gr.g; ++j) {
                const int n0 = (gr.nt0 + j) * DEC_TN;
                if (kBwd) tma_load_2d_hint(b + j * DEC_WBOX, &tmB, &full_bar[st], kb * BK, n0, pol_w);
                else tma_load_2d_hint(b + j * DEC_WBOX, &tmB, &full_bar[st], n0, kb * BK, pol_w);
              }
            }
          }
        }
        pdl_wait();
      }
      for (; id >= 0; id = claim()) {
        gr = dec_group(p, id);
        ++n_groups;
        n_units += gr.g;
        const DecTile td = p.tiles[gr.mt];
        if (gr.kind == 0) {
          const bool lo = gr.c >= p.C;
          const int cc = lo ? gr.c - p.C : gr.c;
          const int kb0 = cc * p.kbc, kb1 = min(nkb, kb0 + p.kbc);
          for (int kb = kb0; kb < kb1; ++kb) {
            if (pre > 0) {
              // W of this stage is already in flight (ring slot kb - kb0 of the first pass)
              tma_load_2d(smem + s * DEC_STAGE, lo ? tmAlo : tmA, &full_bar[s], kb * BK, td.arow);
              --pre;
              if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
              continue;
            }
            mbar_wait(&empty_bar[s], ph ^ 1);
            mbar_expect_tx(&full_bar[s], DEC_KB_BYTES + gr.g * DEC_WBOX);
            uint8_t* a = smem + s * DEC_STAGE;
            uint8_t* b = a + dec_b_off(0);
            tma_load_2d(a, lo ? tmAlo : tmA, &full_bar[s], kb * BK, td.arow);
            for (int j = 0; j < gr.g; ++j) {
              const int n0 = (gr.nt0 + j) * DEC_TN;
              if (kBwd) tma_load_2d_hint(b + j * DEC_WBOX, &tmB, &full_bar[s], kb * BK, n0, pol_w);
              else tma_load_2d_hint(b + j * DEC_WBOX, &tmB, &full_bar[s], n0, kb * BK, pol_w);
            }
            if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
          }
        } else {
          const int2 lp = p.lpieces[td.lp_begin + gr.c - 2 * p.C];
          for (int e = lp.x; e < lp.x + lp.y; ++e) {
            const int4 ls = p.lstages[e];
            const bool lo_box = ls.w >= 0 && ls.w + ls.y * LORA_CHUNK > ls.z + 64;   // lo outside the hi box
            mbar_wait(&empty_bar[s], ph ^ 1);
            mbar_expect_tx(&full_bar[s], (lo_box ? 2 : 1) * DEC_KB_BYTES + gr.g * ls.y * LORA_CHUNK_BYTES);
            uint8_t* a = smem + s * DEC_STAGE;
            uint8_t* b = a + dec_b_off(1);
            tma_load_2d(a, &tmAL, &full_bar[s], ls.z, td.al_row);
            if (lo_box) tma_load_2d(a + DEC_KB_BYTES, &tmAL, &full_bar[s], ls.w, td.al_row);
            for (int j = 0; j < gr.g; ++j) {
              const int n0 = (gr.nt0 + j) * DEC_TN;
              if (ls.y == 4) {
                tma_load_2d(b + j * DEC_WBOX, &tmBP64, &full_bar[s], n0, ls.x);
              } else {
                for (int q = 0; q < ls.y; ++q)
                  tma_load_2d(b + j * DEC_WBOX + q * LORA_CHUNK_BYTES, &tmBP, &full_bar[s], n0, ls.x + q * LORA_CHUNK);
              }
            }
            if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
      if (p.trace) {
        p.trace[4 * blockIdx.x + 2] = n_groups;
        p.trace[4 * blockIdx.x + 3] = n_units;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    int qi = 0;
    uint32_t qph = 0;
    for (;;) {
      mbar_wait(&qfull_bar[qi], qph);
      const int id = q_id[qi];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty_bar[qi]);
      if (++qi == DEC_GQ) { qi = 0; qph ^= 1; }
      if (id < 0) break;
      const DecGroup gr = dec_group(p, id);
      const DecTile td = p.tiles[gr.mt];
      mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + acc * (DEC_G * DEC_TN);
      // one UMMA covers the group's g n tiles (N = 64 g): their W boxes / pack boxes sit 8 KB /
      // 2 KB apart (the MN-major LBO; backward: consecutive K-major row blocks)
      const uint32_t idesc_base = make_idesc_bf16(BM, DEC_TN * gr.g, false, !kBwd);
      const uint32_t idesc_lora = make_idesc_bf16(BM, DEC_TN * gr.g, false, true);
      int nst, e0 = 0;
      if (gr.kind == 0) {
        const int cc = gr.c >= p.C ? gr.c - p.C : gr.c;
        nst = min(nkb, (cc + 1) * p.kbc) - cc * p.kbc;
      } else {
        const int2 lp = p.lpieces[td.lp_begin + gr.c - 2 * p.C];
        e0 = lp.x;
        nst = lp.y;
      }
      for (int st = 0; st < nst; ++st) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(smem + s * DEC_STAGE);
          const uint32_t b_addr = a_addr + dec_b_off(gr.kind);
          if (gr.kind == 0) {
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
              const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
              const uint64_t bd = kBwd ? make_sdesc_sw128(b_addr + k * 32, 16, 1024)
                                       : make_sdesc_sw128(b_addr + k * (UK * 128), DEC_WBOX, 1024);
              mma_bf16_ss(d0, ad, bd, idesc_base, (st != 0 || k != 0) ? 1u : 0u);
            }
          } else {
            // this slice's hi columns, then its lo columns, against the same pack rows
            const int4 ls = p.lstages[e0 + st];
            const bool lo_box = ls.w >= 0 && ls.w + ls.y * LORA_CHUNK > ls.z + 64;
            const uint32_t lo_addr = lo_box ? a_addr + DEC_KB_BYTES : a_addr + (ls.w - ls.z) * 2;
            for (int h = 0; h < (ls.w >= 0 ? 2 : 1); ++h) {
              for (int q = 0; q < ls.y; ++q) {
                const uint64_t ad = make_sdesc_sw128((h ? lo_addr : a_addr) + q * 32, 16, 1024);
                const uint64_t bd = make_sdesc_sw128(b_addr + q * LORA_CHUNK_BYTES, DEC_WBOX, 1024);
                mma_bf16_ss(d0, ad, bd, idesc_lora, (st | h | q) != 0 ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty_bar[s]);
        }
        __syncwarp();
        if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
      }
      if (lane == 0) mma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  } else if (warp == 4 || warp == 5) {
    // ------------------------------------------------------------ unit partials -> workspace
    // TMEM lane = tile row (warps 4 and 5 own lanes 0-63); layout [row][col], 256 B per row;
    // stored with L2 evict_last so the fixup finds them in L2 behind the streamed W
    const int row = (int)((warp - 4) * 32 + lane);
    const uint64_t pol = policy_evict_last();
    int acc = 0;
    uint32_t acc_ph = 0;
    int row_mt = -1, row_rows = 0, row_piece = -1;   // this row's tile / LoRA piece (-1: none)
    int qi = 0;
    uint32_t qph = 0;
    for (;;) {
      mbar_wait(&qfull_bar[qi], qph);
      const int id = q_id[qi];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty_bar[qi]);
      if (++qi == DEC_GQ) { qi = 0; qph ^= 1; }
      if (id < 0) break;
      const DecGroup gr = dec_group(p, id);
      if (gr.mt != row_mt) {
        row_mt = gr.mt;
        const DecTile td = p.tiles[gr.mt];
        row_rows = td.rows;
        row_piece = -1;
        if (row < td.rows && td.lp_count > 0) {
          const DevSeg& sg = p.segs[p.row_seg[td.arow + row]];
          if (sg.flags & SEGF_LORA) row_piece = sg.dec_piece;
        }
      }
      // a LoRA piece stores only the rows whose rank block it holds (the fixup reads no other)
      const bool ok = row < row_rows && (gr.kind == 0 || row_piece == gr.c - 2 * p.C);
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      for (int j = 0; j < gr.g; ++j) {
        float4* dst = reinterpret_cast<float4*>(
            p.part + ((int64_t)(gr.mt * p.n_n + gr.nt0 + j) * p.S + gr.c) * DEC_PART + (int64_t)row * DEC_TN);
#pragma unroll
        for (int h = 0; h < DEC_TN / 32; ++h) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + acc * (DEC_G * DEC_TN) + j * DEC_TN + h * 32 + (((warp - 4) * 32u) << 16), r);
          tmem_wait_ld();
          if (ok) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              st_f4_evict_last(dst + h * 8 + q,
                               make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                           __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])),
                               pol);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (p.fx_cnt) {
        __threadfence();   // this lane's partial stores before the count (release)
        __syncwarp();
        if (lane == 0)
          for (int j = 0; j < gr.g; ++j)
            atomicAdd(p.fx_cnt + (int64_t)(gr.mt * p.n_n + gr.nt0 + j) * 2 + (warp - 4), 1);
      }
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  }
  if (p.fx_cnt) {
    // ------------------------------------------------------------ in-kernel fixup (whole CTA)
    // Once this CTA's groups are done, its 256 threads claim fixup units (the fixup kernel's
    // blocks: 32 rows x 64 columns of one tile, thread t = the fixup kernel's thread t, the same
    // fold bit for bit) in unit order and fold each once its tile half has counted every group.
    int* unit_slot = reinterpret_cast<int*>(tmem_slot + 1);   // smem broadcast of the claimed unit
    const int n_units = p.n_m * p.n_n * (DEC_ROWS / DEC_FIX_ROWS);
    pdl_wait();   // the destinations may alias rows the kernels before this one read
    for (;;) {
      __syncthreads();   // everyone has read the previous slot
      if (threadIdx.x == 0) {
        int u = atomicAdd(p.fx_claim, 1);
        if (u < n_units) {
          const int q = u % (DEC_ROWS / DEC_FIX_ROWS), tile = u / (DEC_ROWS / DEC_FIX_ROWS);
          const DecTile td = p.tiles[tile / p.n_n];
          const int want = (1 + (td.lo ? 1 : 0)) * p.C + td.lp_count;
          int* cnt = p.fx_cnt + (int64_t)tile * 2 + q;
          while (ld_acquire_gpu(cnt) < want) __nanosleep(64);
          *cnt = 0;   // every group of this launch has counted: ready for the next launch
        } else {
          u = -1;
        }
        *(volatile int*)unit_slot = u;
      }
      __syncthreads();
      const int u = *(volatile int*)unit_slot;
      if (u < 0) break;
      dec_fixup_unit(p, u, (int)threadIdx.x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (p.trace) {
      p.trace[4 * blockIdx.x] = t_start;
      p.trace[4 * blockIdx.x + 1] = globaltimer_ns();
    }
    // the last CTA out resets the ticket for the next launch (every claim is made by now)
    if (atomicAdd(p.claim + 1, 1) == (int)gridDim.x - 1) {
      p.claim[0] = 0;
      p.claim[1] = 0;
      if (p.fx_claim) p.fx_claim[0] = 0;
      __threadfence();
    }
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * DEC_G * DEC_TN);
  }
}

__global__ void __launch_bounds__(DEC_FIX_THREADS)
    dec_fixup_kernel(const DecParams p) {
  pdl_wait();
  pdl_trigger();
  dec_fixup_unit(p, (int)blockIdx.x, (int)threadIdx.x);
}

}  // namespace ss
