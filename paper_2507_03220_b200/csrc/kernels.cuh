// Device kernels of the segmented base executor (sm_100a).
//
//   K4 gather_rows_kernel  : client segments -> contiguous bf16 operand X (concat_rows,
//                            reference tensor_ops.py:145-146), IA3 prologue for backward
//                            (client.py:291-294), per-row segment index for routing.
//   K3 lora_shrink_kernel  : per segment s*x.A (fwd, adapters.py:23) or s*g.B^T (bwd,
//                            adapters.py:37) on tcgen05, written block-diagonally into a
//                            per-M-tile operand so the expand rides the base GEMM's K loop.
//   K1/K2/K5 seg_gemm_kernel: persistent warp-specialised TMA -> tcgen05 -> TMEM GEMM:
//                            y = x.W + b (affine_forward tensor_ops.py:71-78), dx = g.W^T
//                            (affine_backward_input tensor_ops.py:81-89) or n.W (noise,
//                            executor.py:221-222), LoRA expand as extra K steps into the same
//                            TMEM accumulator, then bias / IA3 epilogue (adapters.py:127-145)
//                            and the per-segment scatter (split_rows tensor_ops.py:149-156)
//                            straight into each client's destination rows.
#pragma once
#include "ptx.cuh"

namespace ss {

// Segment flags (device side).
enum : int32_t {
  SEGF_SRC_BF16 = 1 << 0,
  SEGF_DST_BF16 = 1 << 1,
  SEGF_BASE_BF16 = 1 << 2,
  SEGF_LORA = 1 << 3,
  SEGF_IA3 = 1 << 4,
  SEGF_WANT_BASE = 1 << 5,
  SEGF_SRC_VEC = 1 << 6,   // src rows 16-byte aligned
  SEGF_DST_VEC = 1 << 7,   // dst rows 16-byte aligned
  SEGF_BASE_VEC = 1 << 8,  // base rows 16-byte aligned
  SEGF_TMA_STORE = 1 << 9, // bf16 destination written by TMA bulk stores
  SEGF_REMOTE_SRC = 1 << 10,  // source rows on a peer GPU (gathered with plain loads)
  SEGF_REMOTE_DST = 1 << 11,  // destination on a peer GPU (plain stores over NVLink)
  SEGF_SRC_ALIASED = 1 << 12, // source rows overlap a destination of the dispatch (gathered first)
  SEGF_IA3_LO = 1 << 13,      // backward IA3: g = dy*l also kept as lo = bf16(g - bf16(g)) in X_lo,
                              // and the tile runs a second K pass over it (fp32-output tier)
};

struct DevSeg {
  int32_t xrow0;       // first row of this segment's packed piece in X (-1: none)
  int32_t rows;
  int32_t flags;
  int32_t xlocal0;     // segment-local row index of that first packed row
  const void* src;
  int64_t src_ld;      // elements
  void* dst;
  int64_t dst_ld;
  void* dst_base;      // pre-IA3 output for IA3 fine-tune clients (forward)
  int64_t base_ld;
  const float* ia3;    // IA3 scale vector (length d_out of the layer)
  float lora_scale;    // alpha / r
  int32_t pack_row;    // first row of this client's rank block in the layer's LoRA packs
  int32_t rank_pad;    // rank rounded up to 16
  int32_t dec_piece;   // decode class (decode.cuh): the LoRA piece of its tile holding its rank block
};

constexpr int BM = 128;           // rows per tile == TMEM lanes
constexpr int BN = 256;           // columns per tile (one UMMA N=256)
constexpr int BK = 64;            // K per pipeline stage (one 128-byte swizzle row)
constexpr int UK = 16;            // K per tcgen05.mma for bf16
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 2;       // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int LORA_CHUNK = 16;                   // rank granularity
constexpr int LORA_CHUNK_BYTES = 64 * LORA_CHUNK * 2;  // one {64, 16} box = 2 KB
constexpr int GEMM_THREADS = 256;                // 8 warps
constexpr int GEMM_SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// One M-tile of the dispatch (TM = 128 rows single-CTA, 256 rows CTA pair). A "direct" tile is
// TM rows of one segment, TMA-loaded straight from the client's buffer through that segment's
// tensor map; a "packed" tile covers rows of X (small / f32 / IA3-backward pieces gathered by K4).
struct TileDesc {
  int32_t amap;         // index into GemmParams::tmaps (0 = packed operand X)
  int32_t arow;         // row coordinate of the tile's first row in that tensor map
  int32_t seg;          // direct tile: its segment; packed tile: -1
  int32_t rows;         // valid rows (<= TM)
  int32_t chunk_begin;  // LoRA: first entry in `chunks`
  int32_t chunk_count;  // LoRA: 16-wide rank chunks (block-diagonal over the tile's segments)
  int32_t store_begin;  // TMA-store ops of this tile: entries in GemmParams::stores
  int32_t store_count;
  int32_t amap_lo;      // >= 0: tensor map of X_lo; the tile's K loop runs twice (X, then X_lo)
                        // so IA3-backward rows see g = hi + lo (SEGF_IA3_LO); -1: one pass
};

struct GemmParams {
  int N, K;
  int num_m_tiles, num_n_tiles, group_m;
  int group_n;                      // > 0: N-grouped raster (walk M inside groups of N tiles)
  int hint_a, hint_b, hint_out;     // L2 policy of A loads / W loads / output stores (0 none,
                                    // 1 evict_first, 2 evict_last)
  int a_bytes;                      // bytes one A-operand TMA box delivers (64- or 128-row box)
  // Overlap mode (streaming kernel): the LoRA shrink runs concurrently on another stream; the
  // producer waits until lora_ready[0] == lora_expect (shrink CTAs done) before its first LoRA
  // stage. lora_ready[1] counts the CTAs past that point; the last one re-arms both counters.
  int* lora_ready = nullptr;
  int lora_expect = 0;
  // Streaming kernel launched with programmatic dependent launch behind the gather / shrink:
  // the producer issues the first stages' W loads, then griddepcontrol.wait, then their A loads.
  int pdl_early = 0;
  // CTA-pair tail split: a 512-wide launch stops at raster tile `tiles_total`, and a 256-wide
  // launch behind it (programmatic launch, griddepcontrol.wait only before exiting, so it fills
  // the SMs the 512-wide tiles free and still completes after them) runs the remaining tiles of
  // the 512 raster as two 256-wide halves each: tail_nn = the 512 raster's N tiles (0: off),
  // tail_from = its first tile. tiles_total > 0 overrides num_m_tiles * num_n_tiles.
  int tiles_total = 0;
  int tail_from = 0, tail_nn = 0;
  int wait_at_end = 0;
  int has_bias;
  int any_lora;
  int ia3_in_epilogue;              // forward: scale output columns by IA3
  const float* bias;
  const DevSeg* segs;
  const int32_t* row_seg;           // per packed X row: its segment
  const TileDesc* tiles;            // per M-tile
  const int32_t* chunks;            // pack row of each rank chunk
  const CUtensorMap* tmaps;         // [0] = X, then per-dispatch source / destination maps
  const int2* stores;               // (dst tensor map, row coordinate of tile row 0) per op
};

// Persistent-tile raster. M-grouped (default): groups of `group_m` M-tiles, N walked inside a
// group, so a group's A rows stay in L2 while W streams past (W read once per group).
// N-grouped (`group_n` > 0): groups of `group_n` N-tiles, M walked inside, so a group's W
// columns stay in L2 while A streams (A read once per group) — the cheaper order when W is
// small next to A (Q/K/V/O at prefill sizes fit W in L2 whole).
__device__ __forceinline__ void raster_coords(int t, int num_m, int num_n, int group_m, int group_n, int& mb,
                                              int& nb) {
  if (group_n > 0) {
    const int per_group = group_n * num_m;
    const int g = t / per_group;
    const int first_n = g * group_n;
    const int gsize = min(group_n, num_n - first_n);
    const int r = t % per_group;
    nb = first_n + r % gsize;
    mb = r / gsize;
    return;
  }
  const int per_group = group_m * num_n;
  const int g = t / per_group;
  const int first_m = g * group_m;
  const int gsize = min(group_m, num_m - first_m);
  const int r = t % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}
__device__ __forceinline__ void tile_coords(int t, const GemmParams& p, int& mb, int& nb) {
  if (p.tail_nn > 0) {
    // tail launch: 256-wide halves of the 512 raster's tiles from tail_from on
    raster_coords(p.tail_from + (t >> 1), p.num_m_tiles, p.tail_nn, p.group_m, p.group_n, mb, nb);
    nb = 2 * nb + (t & 1);
    return;
  }
  raster_coords(t, p.num_m_tiles, p.num_n_tiles, p.group_m, p.group_n, mb, nb);
}

__device__ __forceinline__ uint64_t l2_policy(int h) {
  return h == 2 ? policy_evict_last() : policy_evict_first();
}
__device__ __forceinline__ void load_a_or_b(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1, int hint, uint64_t pol) {
  if (hint) tma_load_2d_hint(dst, map, bar, c0, c1, pol);
  else tma_load_2d(dst, map, bar, c0, c1);
}
__device__ __forceinline__ void load_a_or_b_2sm(void* dst, const CUtensorMap* map, uint32_t bar, int32_t c0,
                                                int32_t c1, int hint, uint64_t pol) {
  if (hint) tma_load_2d_2sm_hint(dst, map, bar, c0, c1, pol);
  else tma_load_2d_2sm(dst, map, bar, c0, c1);
}

// Store `ncols` (<= 64) fp32 values of one row to a bf16 / f32 destination with plain global
// stores (16-byte vectors when aligned). Used for f32 destinations, misaligned rows and y_base.
// (All loops over the 64 values are unrolled with compile-time indices so `v` stays in registers.)
__device__ __forceinline__ void store_row_global(const float (&v)[64], int ncols, char* dst, bool bf,
                                                 bool vec) {
  if (ncols == 64 && vec) {
    if (bf) {
      uint4* o = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        o[j] = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                          pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
    } else {
      float4* o = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      if (j < ncols) {
        if (bf) reinterpret_cast<__nv_bfloat16*>(dst)[j] = __float2bfloat16_rn(v[j]);
        else reinterpret_cast<float*>(dst)[j] = v[j];
      }
    }
  }
}

constexpr int EPI_CHUNK = 64;                           // columns per epilogue step
constexpr int EPI_STAGE_BYTES = BM * EPI_CHUNK * 2;     // 16 KB bf16 staging (128 rows x 128 B)
constexpr int EPI_SMEM = 2 * EPI_STAGE_BYTES;           // double-buffered

// Epilogue of one accumulator tile, executed by the 4 epilogue warps (128 threads, thread =
// TMEM lane = row r of this CTA's 128 rows). Per 64-column chunk: tcgen05.ld -> + bias ->
// optional pre-IA3 y_base store -> * IA3 l -> bf16 into a 128B-swizzled staging tile -> one TMA
// bulk store per destination segment piece of the tile (rows outside a piece are clipped by its
// tensor map, so a tile shared by several clients needs no masking). Rows whose destination is
// f32 or misaligned fall back to direct global stores. Releases the TMEM accumulator (tempty)
// as soon as its last column has been read. `store_row0` = this CTA's first row within the
// tile (0, or 128 for the second CTA of a pair).
// `c_begin`..`c_end` = this warp group's 64-column chunks (a 512-wide pair tile splits them over
// two groups of 4 warps, each with its own staging buffers and named barrier `bar_id`).
template <int TBN>
__device__ __forceinline__ void epilogue_tile(const GemmParams& p, uint32_t tmem_acc, uint32_t ew,
                                              uint32_t lane, const TileDesc& td, int store_row0, int n0,
                                              uint64_t* tfull, uint32_t tfull_ph, uint8_t* stage,
                                              uint32_t tempty_cluster_addr, int c_begin = 0,
                                              int c_end = TBN / EPI_CHUNK, uint32_t bar_id = 1) {
  const int r = store_row0 + ew * 32 + lane;  // row within the tile
  const bool row_ok = r < td.rows;
  const bool leader_thread = ew == 0 && lane == 0;
  DevSeg sg;
  int r_local = 0;
  if (row_ok) {
    if (td.seg >= 0) {
      sg = p.segs[td.seg];
      r_local = td.arow + r;
    } else {
      const int xrow = td.arow + r;
      sg = p.segs[p.row_seg[xrow]];
      r_local = xrow - sg.xrow0 + sg.xlocal0;
    }
  }
  const bool use_ia3 = row_ok && p.ia3_in_epilogue && (sg.flags & SEGF_IA3);
  const bool want_base = row_ok && (sg.flags & SEGF_WANT_BASE);
  // TMA box coordinates must be >= 0: a packed piece that starts inside the tile has no bulk
  // store op (host side) and its rows take the direct-store path.
  const bool tma_row = row_ok && (sg.flags & SEGF_TMA_STORE) && (td.seg >= 0 || sg.xrow0 <= td.arow);
  const int lrow = ew * 32 + lane;            // row within this CTA's staging tile
  if (leader_thread) {
    for (int k = 0; k < td.store_count; ++k) tensormap_acquire(p.tmaps + p.stores[td.store_begin + k].x);
  }
  mbar_wait(tfull, tfull_ph);
  tc_fence_after();
#pragma unroll 1
  for (int c = c_begin; c < c_end; ++c) {
    uint32_t ra[32], rb[32];
    tmem_ld_32x32b_x32(tmem_acc + c * EPI_CHUNK + ((ew * 32u) << 16), ra);
    tmem_ld_32x32b_x32(tmem_acc + c * EPI_CHUNK + 32 + ((ew * 32u) << 16), rb);
    tmem_wait_ld();
    if (c == c_end - 1) {
      // every column of this warp's share is in registers: hand TMEM back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_cluster_addr);
    }
    const int n = n0 + c * EPI_CHUNK;
    const int ncols = max(0, min(EPI_CHUNK, p.N - n));
    float v[64];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = __uint_as_float(ra[j]);
      v[32 + j] = __uint_as_float(rb[j]);
    }
    if (row_ok && ncols > 0) {
      if (p.has_bias) {
        if (ncols == 64) {
          const float4* b4 = reinterpret_cast<const float4*>(p.bias + n);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 bb = __ldg(b4 + j);
            v[4 * j] += bb.x; v[4 * j + 1] += bb.y; v[4 * j + 2] += bb.z; v[4 * j + 3] += bb.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < ncols) v[j] += __ldg(p.bias + n + j);
        }
      }
      if (want_base) {
        const bool bf = sg.flags & SEGF_BASE_BF16;
        char* base = reinterpret_cast<char*>(sg.dst_base) + ((int64_t)r_local * sg.base_ld + n) * (bf ? 2 : 4);
        store_row_global(v, ncols, base, bf, sg.flags & SEGF_BASE_VEC);
      }
      if (use_ia3) {
        if (ncols == 64) {
          const float4* l4 = reinterpret_cast<const float4*>(sg.ia3 + n);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 ll = __ldg(l4 + j);
            v[4 * j] *= ll.x; v[4 * j + 1] *= ll.y; v[4 * j + 2] *= ll.z; v[4 * j + 3] *= ll.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < ncols) v[j] *= __ldg(sg.ia3 + n + j);
        }
      }
      if (!tma_row) {
        const bool bf = sg.flags & SEGF_DST_BF16;
        char* dst = reinterpret_cast<char*>(sg.dst) + ((int64_t)r_local * sg.dst_ld + n) * (bf ? 2 : 4);
        store_row_global(v, ncols, dst, bf, sg.flags & SEGF_DST_VEC);
      }
    }
    if (td.store_count > 0) {
      uint8_t* sb = stage + (c & 1) * EPI_STAGE_BYTES;
      if (leader_thread) bulk_wait_read<1>();      // the store issued 2 chunks ago freed `sb`
      named_bar_sync(bar_id, 128);
      if (tma_row && ncols > 0) {
        uint8_t* rowp = sb + lrow * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(rowp + ((j ^ (lrow & 7)) << 4)) =
              make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                         pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
      }
      fence_async_smem();
      named_bar_sync(bar_id, 128);
      if (leader_thread && ncols > 0) {
        const uint64_t pol = l2_policy(p.hint_out);
        for (int k = 0; k < td.store_count; ++k) {
          const int2 op = p.stores[td.store_begin + k];
          if (p.hint_out) tma_store_2d_hint(p.tmaps + op.x, sb, n, op.y + store_row0, pol);
          else tma_store_2d(p.tmaps + op.x, sb, n, op.y + store_row0);
        }
        bulk_commit();
      }
    }
  }
}

// Epilogue variant for the single (non-double-buffered) 512-column accumulator: a warp reads its
// NCH chunks out of TMEM first — bias, y_base, IA3 applied, bf16 values held in registers —
// and releases the accumulator before any staging / TMA store, so the next tile's MMAs start
// after the TMEM reads instead of after the stores. Same values and stores as epilogue_tile.
template <int NCH, int BUFS>
__device__ __forceinline__ void epilogue_tile_hold(const GemmParams& p, uint32_t tmem_acc, uint32_t ew,
                                                   uint32_t lane, const TileDesc& td, int store_row0, int n0,
                                                   uint64_t* tfull, uint32_t tfull_ph, uint8_t* stage,
                                                   uint32_t tempty_cluster_addr, int c_begin, uint32_t bar_id) {
  const int r = store_row0 + ew * 32 + lane;
  const bool row_ok = r < td.rows;
  const bool leader_thread = ew == 0 && lane == 0;
  DevSeg sg;
  int r_local = 0;
  if (row_ok) {
    if (td.seg >= 0) {
      sg = p.segs[td.seg];
      r_local = td.arow + r;
    } else {
      const int xrow = td.arow + r;
      sg = p.segs[p.row_seg[xrow]];
      r_local = xrow - sg.xrow0 + sg.xlocal0;
    }
  }
  const bool use_ia3 = row_ok && p.ia3_in_epilogue && (sg.flags & SEGF_IA3);
  const bool want_base = row_ok && (sg.flags & SEGF_WANT_BASE);
  const bool tma_row = row_ok && (sg.flags & SEGF_TMA_STORE) && (td.seg >= 0 || sg.xrow0 <= td.arow);
  const int lrow = ew * 32 + lane;
  if (leader_thread) {
    for (int k = 0; k < td.store_count; ++k) tensormap_acquire(p.tmaps + p.stores[td.store_begin + k].x);
  }
  // pull this group's bias / IA3 columns into L1 while the MMAs run, so the drain below (the
  // bubble before the next tile's MMAs) does not wait on L2 for them
#ifndef SS_NO_EPI_PF
  {
    const int nb0 = n0 + c_begin * EPI_CHUNK;
    const int span = min(NCH * EPI_CHUNK, p.N - nb0);      // columns of this group
    if (span > 0 && lane < (span + 31) / 32) {
      if (p.has_bias) prefetch_l1(p.bias + nb0 + lane * 32);
      if (use_ia3) prefetch_l1(sg.ia3 + nb0 + lane * 32);
    }
  }
#endif
  mbar_wait(tfull, tfull_ph);
  tc_fence_after();
  uint32_t hold[NCH][32];                     // bf16x2 of each held chunk
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const int c = c_begin + q;
    uint32_t ra[32], rb[32];
    tmem_ld_32x32b_x32(tmem_acc + c * EPI_CHUNK + ((ew * 32u) << 16), ra);
    tmem_ld_32x32b_x32(tmem_acc + c * EPI_CHUNK + 32 + ((ew * 32u) << 16), rb);
    tmem_wait_ld();
    if (q == NCH - 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_cluster_addr);
    }
    const int n = n0 + c * EPI_CHUNK;
    const int ncols = max(0, min(EPI_CHUNK, p.N - n));
    float v[64];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = __uint_as_float(ra[j]);
      v[32 + j] = __uint_as_float(rb[j]);
    }
    if (row_ok && ncols > 0) {
      if (p.has_bias) {
        if (ncols == 64) {
          const float4* b4 = reinterpret_cast<const float4*>(p.bias + n);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 bb = __ldg(b4 + j);
            v[4 * j] += bb.x; v[4 * j + 1] += bb.y; v[4 * j + 2] += bb.z; v[4 * j + 3] += bb.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < ncols) v[j] += __ldg(p.bias + n + j);
        }
      }
      if (want_base) {
        const bool bf = sg.flags & SEGF_BASE_BF16;
        char* base = reinterpret_cast<char*>(sg.dst_base) + ((int64_t)r_local * sg.base_ld + n) * (bf ? 2 : 4);
        store_row_global(v, ncols, base, bf, sg.flags & SEGF_BASE_VEC);
      }
      if (use_ia3) {
        if (ncols == 64) {
          const float4* l4 = reinterpret_cast<const float4*>(sg.ia3 + n);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 ll = __ldg(l4 + j);
            v[4 * j] *= ll.x; v[4 * j + 1] *= ll.y; v[4 * j + 2] *= ll.z; v[4 * j + 3] *= ll.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < ncols) v[j] *= __ldg(sg.ia3 + n + j);
        }
      }
      if (!tma_row) {
        const bool bf = sg.flags & SEGF_DST_BF16;
        char* dst = reinterpret_cast<char*>(sg.dst) + ((int64_t)r_local * sg.dst_ld + n) * (bf ? 2 : 4);
        store_row_global(v, ncols, dst, bf, sg.flags & SEGF_DST_VEC);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) hold[q][j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
  }
  if (td.store_count == 0) return;
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const int c = c_begin + q;
    const int n = n0 + c * EPI_CHUNK;
    const int ncols = max(0, min(EPI_CHUNK, p.N - n));
    uint8_t* sb = stage + (q % BUFS) * EPI_STAGE_BYTES;
    if (leader_thread) bulk_wait_read<BUFS - 1>();   // the store that last used `sb` has read it
    named_bar_sync(bar_id, 128);
    if (tma_row && ncols > 0) {
      uint8_t* rowp = sb + lrow * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<uint4*>(rowp + ((j ^ (lrow & 7)) << 4)) =
            make_uint4(hold[q][4 * j], hold[q][4 * j + 1], hold[q][4 * j + 2], hold[q][4 * j + 3]);
    }
    fence_async_smem();
    named_bar_sync(bar_id, 128);
    if (leader_thread && ncols > 0) {
      const uint64_t pol = l2_policy(p.hint_out);
      for (int k = 0; k < td.store_count; ++k) {
        const int2 op = p.stores[td.store_begin + k];
        if (p.hint_out) tma_store_2d_hint(p.tmaps + op.x, sb, n, op.y + store_row0, pol);
        else tma_store_2d(p.tmaps + op.x, sb, n, op.y + store_row0);
      }
      bulk_commit();
    }
  }
}

// ============================================================================ K1/K2/K5
// Single-CTA kernel, tile 128 x TBN. TBN < 256 is used when a dispatch has too few 128 x 256
// tiles to fill the SMs (decode-style batches): the per-element K-reduction order does not
// depend on TBN, so every tile width gives bitwise the same rows (batching stays invisible).
template <int TBN>
struct TileCfg {
  static constexpr int B_STAGE = TBN * BK * 2;
#ifndef SS_STAGES64
#define SS_STAGES64 8
#endif
  static constexpr int STAGES_ = TBN == 256 ? 4 : (TBN == 128 ? 6 : SS_STAGES64);
  static constexpr int STAGE = A_STAGE_BYTES + B_STAGE;
  static constexpr int SMEM = STAGES_ * STAGE + EPI_SMEM + 1024 + 256;
};

template <bool kBwd, int TBN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    seg_gemm_kernel(const __grid_constant__ CUtensorMap tmB,   // W  [d_in, d_out] bf16
                    const __grid_constant__ CUtensorMap tmAL,  // A_lora [M, R_w] bf16
                    const __grid_constant__ CUtensorMap tmBP,  // pack [R, N] bf16 (MN-major B)
                    const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smA = smem;
  constexpr int STAGES = TileCfg<TBN>::STAGES_;
  constexpr int B_STAGE_BYTES = TileCfg<TBN>::B_STAGE;
  constexpr int STAGE_BYTES = TileCfg<TBN>::STAGE;
  uint8_t* smB = smem + STAGES * A_STAGE_BYTES;
  uint8_t* epi_stage = smem + STAGES * STAGE_BYTES;  // 2 x 16 KB TMA-store staging
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi_stage + EPI_SMEM);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;   // 2 accumulator buffers
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    if (p.any_lora) {
      tma_prefetch_desc(&tmAL);
      tma_prefetch_desc(&tmBP);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);    // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * TBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  const int num_tiles = p.num_m_tiles * p.num_n_tiles;
  const int nkb = (p.K + BK - 1) / BK;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint64_t pol_a = l2_policy(p.hint_a), pol_b = l2_policy(p.hint_b);
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p, mb, nb);
        const TileDesc td = p.tiles[mb];
        const CUtensorMap* tmA = p.tmaps + td.amap;
        const CUtensorMap* tmA_lo = p.tmaps + (td.amap_lo >= 0 ? td.amap_lo : td.amap);
        const int m0 = mb * BM, n0 = nb * TBN;
        tensormap_acquire(tmA);
        if (td.amap_lo >= 0) tensormap_acquire(tmA_lo);
        const int nkb_t = td.amap_lo >= 0 ? 2 * nkb : nkb;
        for (int kb2 = 0; kb2 < nkb_t; ++kb2) {
          const int kb = kb2 < nkb ? kb2 : kb2 - nkb;
          mbar_wait(&empty_bar[s], ph ^ 1);
          mbar_expect_tx(&full_bar[s], p.a_bytes + B_STAGE_BYTES);
          load_a_or_b(smA + s * A_STAGE_BYTES, kb2 < nkb ? tmA : tmA_lo, &full_bar[s], kb * BK, td.arow, p.hint_a, pol_a);
          uint8_t* b = smB + s * B_STAGE_BYTES;
          if (kBwd) {
            // W viewed K-major: rows = d_in (the GEMM's N), cols = d_out (the GEMM's K).
            load_a_or_b(b, &tmB, &full_bar[s], kb * BK, n0, p.hint_b, pol_b);
          } else {
            // W MN-major: 4 chunks of 64 output columns x 64 K rows.
#pragma unroll
            for (int j = 0; j < TBN / 64; ++j)
              load_a_or_b(b + j * (BK * 128), &tmB, &full_bar[s], n0 + 64 * j, kb * BK, p.hint_b, pol_b);
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (p.any_lora) {
          const int cb = td.chunk_begin;
          const int cc = td.chunk_count;
          for (int ls = 0; ls * 4 < cc; ++ls) {
            const int nq = min(4, cc - ls * 4);
            mbar_wait(&empty_bar[s], ph ^ 1);
            mbar_expect_tx(&full_bar[s], A_STAGE_BYTES + nq * (TBN / 64) * LORA_CHUNK_BYTES);
            tma_load_2d(smA + s * A_STAGE_BYTES, &tmAL, &full_bar[s], ls * BK, m0);
            uint8_t* b = smB + s * B_STAGE_BYTES;
            for (int q = 0; q < nq; ++q) {
              const int prow = p.chunks[cb + ls * 4 + q];
#pragma unroll
              for (int j = 0; j < TBN / 64; ++j)
                tma_load_2d(b + j * (BK * 128) + q * LORA_CHUNK_BYTES, &tmBP, &full_bar[s],
                            n0 + 64 * j, prow);
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_base = make_idesc_bf16(BM, TBN, false, !kBwd);
    constexpr uint32_t idesc_lora = make_idesc_bf16(BM, TBN, false, true);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * TBN;
      const int nkb_t = p.tiles[mb].amap_lo >= 0 ? 2 * nkb : nkb;
      for (int kb = 0; kb < nkb_t; ++kb) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(smA + s * A_STAGE_BYTES);
          const uint32_t b_addr = smem_u32(smB + s * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = kBwd ? make_sdesc_sw128(b_addr + k * 32, 16, 1024)
                                     : make_sdesc_sw128(b_addr + k * (UK * 128), BK * 128, 1024);
            mma_bf16_ss(d_tmem, ad, bd, idesc_base, (kb | k) != 0);
          }
          mma_commit(&empty_bar[s]);
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      if (p.any_lora) {
        const int cc = p.tiles[mb].chunk_count;
        for (int ls = 0; ls * 4 < cc; ++ls) {
          const int nq = min(4, cc - ls * 4);
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(smA + s * A_STAGE_BYTES);
            const uint32_t b_addr = smem_u32(smB + s * B_STAGE_BYTES);
            for (int q = 0; q < nq; ++q) {
              const uint64_t ad = make_sdesc_sw128(a_addr + q * 32, 16, 1024);
              const uint64_t bd = make_sdesc_sw128(b_addr + q * LORA_CHUNK_BYTES, BK * 128, 1024);
              mma_bf16_ss(d_tmem, ad, bd, idesc_lora, 1u);
            }
            mma_commit(&empty_bar[s]);
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (lane == 0) mma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t ew = warp - 4;  // TMEM lane quarter
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);  // own CTA (cluster of 1)
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      const TileDesc td = p.tiles[mb];
      epilogue_tile<TBN>(p, tmem_base + acc * TBN, ew, lane, td, 0, nb * TBN, &tfull_bar[acc], acc_ph,
                         epi_stage, tempty0 + acc * 8);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
    if (ew == 0 && lane == 0) bulk_wait_all();
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * TBN);
  }
}

// ============================================================================ K1/K2/K5, streaming
// Weight-streaming variant of the single-CTA kernel for decode-size dispatches (one packed tile
// of <= 64 rows, 64-wide N tiles): the GEMM only streams W, and a CTA keeps about eight TMA
// operations in flight whatever their size (profiles/r01_l2_and_decode.md: 0.24 us per 64-deep
// k-block at 3..8 stages of 8 KB boxes). So each operation moves 32 KB: one stage is SK = 256
// of K — A as ONE 3-D box {64 k, 64 rows, 4 k-chunks} (chunk c = k-block c's 64 rows, 8 KB apart)
// and W as ONE box {64 n, 256 k} (forward, MN-major) or 3-D {64 k, 64 n, 4 k-chunks}
// (backward, K-major). The MMA of k-block c reads 128 A rows from chunk c: rows 64-127 are the
// next chunk (or the stage's W bytes) — garbage rows whose outputs are never stored. Same MMAs
// in the same K order as the other kernels: bitwise the same rows.
// Overlap mode: wait for the concurrently running LoRA shrink (all its CTAs arrived), then
// make its global writes visible to this thread's TMA loads.
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// (Bounded: the shrink runs on another stream and the GPU does not formally guarantee the two
// kernels run concurrently; if it has not arrived within 2 s, fail loudly instead of hanging.)
__device__ __forceinline__ void spin_until_ready(const GemmParams& p) {
  const uint64_t t0 = global_ns();
  while (ld_acquire_gpu(p.lora_ready) < p.lora_expect) {
    __nanosleep(256);
    if (global_ns() - t0 > 2000000000ull) __trap();
  }
}
__device__ __forceinline__ void wait_lora_ready(const GemmParams& p) {
  spin_until_ready(p);
  fence_proxy_async_global();
}
// Every CTA takes one ticket once it no longer reads the counter; the last one re-arms both
// counters for the next dispatch (after the shrink's last arrival, so none can land late).
__device__ __forceinline__ void lora_ready_ticket(const GemmParams& p) {
  if (atomicAdd(p.lora_ready + 1, 1) == (int)gridDim.x - 1) {
    spin_until_ready(p);
    atomicExch(p.lora_ready, 0);
    atomicExch(p.lora_ready + 1, 0);
  }
}

constexpr int SK = 256;                                  // K per streaming stage
constexpr int S_A_BYTES = 4 * 64 * 128;                  // 32 KB: 4 chunks x 64 rows x 128 B
constexpr int S_B_BYTES = 64 * SK * 2;                   // 32 KB
constexpr int S_STAGE = S_A_BYTES + S_B_BYTES;
constexpr int S_STAGES = 3;
constexpr int STREAM_SMEM = S_STAGES * S_STAGE + EPI_SMEM + 1024 + 256;

template <bool kBwd>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    seg_gemm_stream_kernel(const __grid_constant__ CUtensorMap tmB,   // W stream map (see above)
                           const __grid_constant__ CUtensorMap tmAL,  // A_lora [M, R_w] bf16
                           const __grid_constant__ CUtensorMap tmBP,  // pack [R, N] bf16
                           const GemmParams p) {
  constexpr int TBN = 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* epi_stage = smem + S_STAGES * S_STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi_stage + EPI_SMEM);
  uint64_t* empty_bar = full_bar + S_STAGES;
  uint64_t* tfull_bar = empty_bar + S_STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    if (p.any_lora) {
      tma_prefetch_desc(&tmAL);
      tma_prefetch_desc(&tmBP);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * TBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!p.pdl_early) pdl_wait();   // (else the producer waits, after its first W loads)
  pdl_trigger();

  const int num_tiles = p.num_m_tiles * p.num_n_tiles;
  const int nkb = (p.K + BK - 1) / BK;        // 64-deep k-blocks
  const int nst = (nkb + 3) / 4;              // streaming stages per tile

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint64_t pol_b = l2_policy(p.hint_b);
      bool lora_waited = p.lora_ready == nullptr;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p, mb, nb);
        const TileDesc td = p.tiles[mb];
        const CUtensorMap* tmA = p.tmaps + td.amap;
        const int n0 = nb * TBN;
        tensormap_acquire(tmA);
        int st0 = 0;
        if (p.pdl_early && t == (int)blockIdx.x) {
          // first tile: W of the first stages streams in while the gather finishes (the ring
          // is empty, s == 0); A (the gathered rows) only after griddepcontrol.wait
          const int pre = min(S_STAGES, nst);
          for (int st = 0; st < pre; ++st) {
            mbar_expect_tx(&full_bar[st], S_STAGE);
            uint8_t* b = smem + st * S_STAGE + S_A_BYTES;
            if (kBwd) tma_load_3d(b, &tmB, &full_bar[st], 0, n0, st * 4);
            else load_a_or_b(b, &tmB, &full_bar[st], n0, st * SK, p.hint_b, pol_b);
          }
          pdl_wait();
          for (int st = 0; st < pre; ++st)
            tma_load_3d(smem + st * S_STAGE, tmA, &full_bar[st], 0, td.arow, st * 4);
          st0 = pre;
          s = pre == S_STAGES ? 0 : pre;
          ph = pre == S_STAGES ? 1 : 0;
        }
        for (int st = st0; st < nst; ++st) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          mbar_expect_tx(&full_bar[s], S_STAGE);
          uint8_t* a = smem + s * S_STAGE;
          uint8_t* b = a + S_A_BYTES;
          tma_load_3d(a, tmA, &full_bar[s], 0, td.arow, st * 4);
          if (kBwd) tma_load_3d(b, &tmB, &full_bar[s], 0, n0, st * 4);
          else load_a_or_b(b, &tmB, &full_bar[s], n0, st * SK, p.hint_b, pol_b);
          if (++s == S_STAGES) { s = 0; ph ^= 1; }
        }
        if (p.any_lora) {
          const int cb = td.chunk_begin;
          const int cc = td.chunk_count;
          const int m0 = mb * BM;
          if (!lora_waited && cc > 0) {            // the base K loop ran beside the shrink
            wait_lora_ready(p);
            lora_ready_ticket(p);
            lora_waited = true;
          }
          for (int ls = 0; ls * 4 < cc; ++ls) {
            const int nq = min(4, cc - ls * 4);
            mbar_wait(&empty_bar[s], ph ^ 1);
            mbar_expect_tx(&full_bar[s], A_STAGE_BYTES / 2 + nq * LORA_CHUNK_BYTES);   // 64-row A_lora box
            uint8_t* a = smem + s * S_STAGE;
            uint8_t* b = a + S_A_BYTES;
            tma_load_2d(a, &tmAL, &full_bar[s], ls * BK, m0);
            for (int q = 0; q < nq; ++q)
              tma_load_2d(b + q * LORA_CHUNK_BYTES, &tmBP, &full_bar[s], n0, p.chunks[cb + ls * 4 + q]);
            if (++s == S_STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
      if (!lora_waited) lora_ready_ticket(p);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_base = make_idesc_bf16(BM, TBN, false, !kBwd);
    constexpr uint32_t idesc_lora = make_idesc_bf16(BM, TBN, false, true);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * TBN;
      for (int st = 0; st < nst; ++st) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(smem + s * S_STAGE);
          const uint32_t b_addr = a_addr + S_A_BYTES;
          const int kbs = min(4, nkb - st * 4);
          for (int c = 0; c < kbs; ++c) {
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
              const uint64_t ad = make_sdesc_sw128(a_addr + c * 8192 + k * 32, 16, 1024);
              const uint64_t bd = kBwd ? make_sdesc_sw128(b_addr + c * 8192 + k * 32, 16, 1024)
                                       : make_sdesc_sw128(b_addr + (c * 4 + k) * (UK * 128), BK * 128, 1024);
              mma_bf16_ss(d_tmem, ad, bd, idesc_base, (st | c | k) != 0);
            }
          }
          mma_commit(&empty_bar[s]);
        }
        __syncwarp();
        if (++s == S_STAGES) { s = 0; ph ^= 1; }
      }
      if (p.any_lora) {
        const int cc = p.tiles[mb].chunk_count;
        for (int ls = 0; ls * 4 < cc; ++ls) {
          const int nq = min(4, cc - ls * 4);
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(smem + s * S_STAGE);
            const uint32_t b_addr = a_addr + S_A_BYTES;
            for (int q = 0; q < nq; ++q) {
              const uint64_t ad = make_sdesc_sw128(a_addr + q * 32, 16, 1024);
              const uint64_t bd = make_sdesc_sw128(b_addr + q * LORA_CHUNK_BYTES, BK * 128, 1024);
              mma_bf16_ss(d_tmem, ad, bd, idesc_lora, 1u);
            }
            mma_commit(&empty_bar[s]);
          }
          __syncwarp();
          if (++s == S_STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (lane == 0) mma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  } else if (warp >= 4) {
    const uint32_t ew = warp - 4;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      const TileDesc td = p.tiles[mb];
      epilogue_tile<TBN>(p, tmem_base + acc * TBN, ew, lane, td, 0, nb * TBN, &tfull_bar[acc], acc_ph,
                         epi_stage, tempty0 + acc * 8);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
    if (ew == 0 && lane == 0) bulk_wait_all();
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * TBN);
  }
}

// ============================================================================ K1/K2/K5, 2-CTA
// CTA pair (cluster of 2 on one TPC), tcgen05 cta_group::2: UMMA 256 x 256 x 16 per K step and
// 256-column group. Each CTA stages its own 128 rows of A and half of the pair's B columns, so
// per SM the MMA reads 4 KB of A + 4 KB of B per 128-cycle UMMA (the 1-CTA kernel is
// smem-bandwidth bound, profiles/r01_ncu_gemm_full.md). The leader CTA (rank 0) issues the
// MMAs; both CTAs run TMA producers (bytes counted on the leader's full barrier) and epilogues
// (each drains its own 128 TMEM lanes).
//   PN = 256: pair tile 256 x 256, double-buffered TMEM accumulator (epilogue overlaps MMA).
//   PN = 512: pair tile 256 x 512 (two UMMAs per K step into TMEM columns 0-255 / 256-511),
//             one 512-column accumulator; 25 % fewer operand bytes per FLOP from L2.
// B columns are interleaved between the CTAs in 128-column groups (group g of CTA c covers
// pair columns g*256 + c*128 .. +128), so each UMMA's N=256 output maps linearly onto TMEM.
constexpr int BM2 = 256;                        // rows per pair tile

// PN = 512 runs 12 warps: the single 512-column accumulator cannot be double-buffered, so its
// drain is the bubble between tiles; two groups of 4 epilogue warps (each its own TMEM-lane
// quarter mapping, chunk half, staging buffers and named barrier) halve it. setmaxnreg moves
// registers from the producer / MMA warp group to the epilogue groups.
template <int PN>
struct PairCfg {
  static constexpr int G = PN / 256;            // 256-column UMMA groups per K step
  static constexpr int NACC = PN == 256 ? 2 : 1;
  static constexpr int EPI_GROUPS = PN == 256 ? 1 : 2;
  static constexpr int THREADS = 128 + 128 * EPI_GROUPS;
  static constexpr int B_BYTES = (PN / 2) * BK * 2;   // this CTA's B slice per stage
  static constexpr int STAGE = A_STAGE_BYTES + B_BYTES;
#ifndef SS_PAIR512_STAGES
#define SS_PAIR512_STAGES 3
#endif
  static constexpr int STAGES_ = PN == 256 ? 6 : SS_PAIR512_STAGES;
  // 512: 3 stages + 2 x 16 KB staging per epilogue group, or 4 stages + one 16 KB buffer each
  static constexpr int EPI_BUFS = (PN == 512 && STAGES_ > 3) ? 1 : 2;
  static constexpr int EPI_GROUP_BYTES = EPI_BUFS * EPI_STAGE_BYTES;
  static constexpr int SMEM = STAGES_ * STAGE + EPI_GROUPS * EPI_GROUP_BYTES + 1024 + 256;
};
constexpr int GEMM2_SMEM = PairCfg<256>::SMEM;
constexpr int GEMM2W_SMEM = PairCfg<512>::SMEM;

template <bool kBwd, int PN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<PN>::THREADS, 1)
    seg_gemm2_kernel(const __grid_constant__ CUtensorMap tmB,   // W: fwd box {64,64}; bwd {64,128}
                     const __grid_constant__ CUtensorMap tmAL,  // A_lora [M, R_w], box {64,128}
                     const __grid_constant__ CUtensorMap tmBP,  // pack [R, N], box {64,16}
                     const GemmParams p) {
  using Cfg = PairCfg<PN>;
  constexpr int STAGES2 = Cfg::STAGES_;
  constexpr int G = Cfg::G;
  constexpr int NACC = Cfg::NACC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES2 * A_STAGE_BYTES;
  uint8_t* epi_stage = smem + STAGES2 * Cfg::STAGE;  // per epilogue group: 2 x 16 KB staging
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi_stage + Cfg::EPI_GROUPS * Cfg::EPI_GROUP_BYTES);
  uint64_t* empty_bar = full_bar + STAGES2;
  uint64_t* tfull_bar = empty_bar + STAGES2;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    if (p.any_lora) {
      tma_prefetch_desc(&tmAL);
      tma_prefetch_desc(&tmBP);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full_bar[s], 1);    // leader: one arrive.expect_tx per stage (+ both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);   // one multicast commit per stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 8 * Cfg::EPI_GROUPS);  // leader: epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!p.wait_at_end) pdl_wait();
  pdl_trigger();

  const int num_tiles = p.tiles_total > 0 ? p.tiles_total : p.num_m_tiles * p.num_n_tiles;
  const int nkb = (p.K + BK - 1) / BK;
  const int cluster_id = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;

  // 384 threads (PN = 512): warp group 0 (producer, MMA issuer, TMEM owner) hands registers
  // to the two epilogue groups
  if constexpr (Cfg::EPI_GROUPS == 2) {
    if (warp < 4) reg_dealloc<56>();   // 128 x 56 + 256 x 224 = 168 x 384
  }
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      const uint64_t pol_a = l2_policy(p.hint_a), pol_b = l2_policy(p.hint_b);
      int s = 0;
      uint32_t ph = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        int mb, nb;
        tile_coords(t, p, mb, nb);
        const TileDesc td = p.tiles[mb];
        const CUtensorMap* tmA = p.tmaps + td.amap;
        const CUtensorMap* tmA_lo = p.tmaps + (td.amap_lo >= 0 ? td.amap_lo : td.amap);
        const int arow = td.arow + crank * BM;
        tensormap_acquire(tmA);
        if (td.amap_lo >= 0) tensormap_acquire(tmA_lo);
        const int m0 = mb * BM2 + crank * BM;       // row of this CTA's half in A_lora
        const int nh = nb * PN + crank * 128;      // first column of this CTA's group 0
        const int nkb_t = td.amap_lo >= 0 ? 2 * nkb : nkb;
        for (int kb2 = 0; kb2 < nkb_t; ++kb2) {
          const int kb = kb2 < nkb ? kb2 : kb2 - nkb;
          mbar_wait(&empty_bar[s], ph ^ 1);
          const uint32_t fb = full0 + s * 8;
          if (leader) mbar_expect_tx(&full_bar[s], 2 * Cfg::STAGE);
          load_a_or_b_2sm(smA + s * A_STAGE_BYTES, kb2 < nkb ? tmA : tmA_lo, fb, kb * BK, arow, p.hint_a, pol_a);
          uint8_t* b = smB + s * Cfg::B_BYTES;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            if (kBwd) {
              load_a_or_b_2sm(b + g * 16384, &tmB, fb, kb * BK, nh + g * 256, p.hint_b, pol_b);
            } else {
#pragma unroll
              for (int j = 0; j < 2; ++j)
                load_a_or_b_2sm(b + g * 16384 + j * (BK * 128), &tmB, fb, nh + g * 256 + 64 * j, kb * BK,
                                p.hint_b, pol_b);
            }
          }
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
        if (p.any_lora) {
          const int cb = td.chunk_begin;
          const int cc = td.chunk_count;
          for (int ls = 0; ls * 4 < cc; ++ls) {
            const int nq = min(4, cc - ls * 4);
            mbar_wait(&empty_bar[s], ph ^ 1);
            const uint32_t fb = full0 + s * 8;
            if (leader)
              mbar_expect_tx(&full_bar[s], 2 * (A_STAGE_BYTES + nq * G * 2 * LORA_CHUNK_BYTES));
            tma_load_2d_2sm(smA + s * A_STAGE_BYTES, &tmAL, fb, ls * BK, m0);
            uint8_t* b = smB + s * Cfg::B_BYTES;
            for (int q = 0; q < nq; ++q) {
              const int prow = p.chunks[cb + ls * 4 + q];
#pragma unroll
              for (int g = 0; g < G; ++g)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                  tma_load_2d_2sm(b + g * 16384 + j * (BK * 128) + q * LORA_CHUNK_BYTES, &tmBP, fb,
                                  nh + g * 256 + 64 * j, prow);
            }
            if (++s == STAGES2) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      constexpr uint32_t idesc_base = make_idesc_bf16(BM2, 256, false, !kBwd);
      constexpr uint32_t idesc_lora = make_idesc_bf16(BM2, 256, false, true);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        int mb, nb;
        tile_coords(t, p, mb, nb);
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        const int nkb_t = p.tiles[mb].amap_lo >= 0 ? 2 * nkb : nkb;
        for (int kb = 0; kb < nkb_t; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(smA + s * A_STAGE_BYTES);
            const uint32_t b_addr = smem_u32(smB + s * Cfg::B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
              const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
#pragma unroll
              for (int g = 0; g < G; ++g) {
                const uint32_t bg = b_addr + g * 16384;
                const uint64_t bd = kBwd ? make_sdesc_sw128(bg + k * 32, 16, 1024)
                                         : make_sdesc_sw128(bg + k * (UK * 128), BK * 128, 1024);
                mma_bf16_ss_2sm(d_tmem + g * 256, ad, bd, idesc_base, (kb | k) != 0);
              }
            }
            mma_commit_2sm_mc(&empty_bar[s], 0x3);
          }
          __syncwarp();
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
        if (p.any_lora) {
          const int cc = p.tiles[mb].chunk_count;
          for (int ls = 0; ls * 4 < cc; ++ls) {
            const int nq = min(4, cc - ls * 4);
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t a_addr = smem_u32(smA + s * A_STAGE_BYTES);
              const uint32_t b_addr = smem_u32(smB + s * Cfg::B_BYTES);
              for (int q = 0; q < nq; ++q)
#pragma unroll
                for (int g = 0; g < G; ++g)
                  mma_bf16_ss_2sm(d_tmem + g * 256, make_sdesc_sw128(a_addr + q * 32, 16, 1024),
                                  make_sdesc_sw128(b_addr + g * 16384 + q * LORA_CHUNK_BYTES, BK * 128, 1024),
                                  idesc_lora, 1u);
              mma_commit_2sm_mc(&empty_bar[s], 0x3);
            }
            __syncwarp();
            if (++s == STAGES2) { s = 0; ph ^= 1; }
          }
        }
        if (lane == 0) mma_commit_2sm_mc(&tfull_bar[acc], 0x3);
        __syncwarp();
        if (++acc == NACC) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    if constexpr (Cfg::EPI_GROUPS == 2) reg_alloc<224>();
    const uint32_t ew = warp & 3;              // TMEM lane quarter (warp % 4)
    const int grp = (int)(warp - 4) >> 2;      // epilogue group: chunk half for PN = 512
    constexpr int CPG = PN / EPI_CHUNK / Cfg::EPI_GROUPS;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = cluster_id; t < num_tiles; t += num_clusters) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      const TileDesc td = p.tiles[mb];
      if constexpr (Cfg::EPI_GROUPS == 2)
        epilogue_tile_hold<CPG, Cfg::EPI_BUFS>(p, tmem_base + acc * 256, ew, lane, td, crank * BM, nb * PN,
                                               &tfull_bar[acc], acc_ph, epi_stage + grp * Cfg::EPI_GROUP_BYTES,
                                               tempty0 + acc * 8, grp * CPG, 1 + grp);
      else
        epilogue_tile<PN>(p, tmem_base + acc * 256, ew, lane, td, crank * BM, nb * PN, &tfull_bar[acc],
                          acc_ph, epi_stage, tempty0 + acc * 8);
      if (++acc == NACC) { acc = 0; acc_ph ^= 1; }
    }
    if (ew == 0 && lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
  if (p.wait_at_end) pdl_wait();   // complete only after the launch before this one
}

// ============================================================================ K1/K2/K5, 2 pairs
// Cluster of 4 = two CTA pairs on the same N tile and consecutive M tiles: each pair keeps
// 256 x 256 tiles with double-buffered accumulators (epilogue overlaps the MMAs), while the
// pair's B columns are fetched once for both pairs — CTA (pair q, rank c) loads the 64-column
// half q of rank c's 128 columns and multicasts it to ranks c and 2 + c. L2 -> SM bytes per
// FLOP fall by 25 % (as with 256 x 512 tiles) without the single-accumulator drain bubble.
// A stage is refilled only after BOTH pairs' MMAs released it (empty barriers count 2 commits).
// The pairs walk the same stage ring in lockstep: LoRA K-extension stages are padded to the
// larger chunk count of the two M tiles. A missing second M tile runs as a dummy (no stores).
constexpr int GEMM4_STAGES = 6;
constexpr int GEMM4_STAGE = A_STAGE_BYTES + 128 * BK * 2;
constexpr int GEMM4_SMEM = GEMM4_STAGES * GEMM4_STAGE + EPI_SMEM + 1024 + 256;

template <bool kBwd>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    seg_gemm4_kernel(const __grid_constant__ CUtensorMap tmB,   // W: fwd box {64,64}; bwd {64,64}
                     const __grid_constant__ CUtensorMap tmAL,  // A_lora [M, R_w], box {64,128}
                     const __grid_constant__ CUtensorMap tmBP,  // pack [R, N], box {64,16}
                     const GemmParams p) {
  constexpr int STAGES2 = GEMM4_STAGES;
  constexpr int B_BYTES = 128 * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES2 * A_STAGE_BYTES;
  uint8_t* epi_stage = smem + STAGES2 * GEMM4_STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi_stage + EPI_SMEM);
  uint64_t* empty_bar = full_bar + STAGES2;
  uint64_t* tfull_bar = empty_bar + STAGES2;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t crank = rank & 1;           // rank within the pair
  const uint32_t pq = rank >> 1;             // pair within the cluster
  const bool leader = crank == 0;
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pq));
  const uint16_t bmc_mask = (uint16_t)((1u << crank) | (1u << (2 + crank)));

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    if (p.any_lora) {
      tma_prefetch_desc(&tmAL);
      tma_prefetch_desc(&tmBP);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full_bar[s], 1);    // pair leader: one arrive.expect_tx per stage
      mbar_init(&empty_bar[s], 2);   // one commit from each pair's MMA issuer
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 8);  // pair leader: 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  const int num_m2 = (p.num_m_tiles + 1) >> 1;             // M-tile pairs
  const int num_tiles = num_m2 * p.num_n_tiles;
  const int nkb = (p.K + BK - 1) / BK;
  const int cluster_id = blockIdx.x >> 2;
  const int num_clusters = gridDim.x >> 2;
  GemmParams q2 = p;
  q2.num_m_tiles = num_m2;                                 // raster over M-tile pairs

  // this pair's tile of super-tile (mb2, nb); a missing second M tile is a dummy (rows = 0)
  auto pair_tile = [&](int mb2, TileDesc& td, int& mb, int& lora_stages) {
    mb = 2 * mb2 + (int)pq;
    const bool real = mb < p.num_m_tiles;
    td = p.tiles[real ? mb : 2 * mb2];
    if (!real) {
      td.rows = 0;
      td.chunk_count = 0;
      td.store_count = 0;
    }
    int cc = td.chunk_count;
    if (2 * mb2 + 1 - (int)pq < p.num_m_tiles) cc = max(cc, p.tiles[2 * mb2 + 1 - (int)pq].chunk_count);
    lora_stages = p.any_lora ? (cc + 3) / 4 : 0;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t fullL = mapa_shared(smem_u32(full_bar), 2 * pq);
      int s = 0;
      uint32_t ph = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        int mb2, nb, mb, nls;
        tile_coords(t, q2, mb2, nb);
        TileDesc td;
        pair_tile(mb2, td, mb, nls);
        const CUtensorMap* tmA = p.tmaps + td.amap;
        const int arow = td.arow + crank * BM;
        tensormap_acquire(tmA);
        const int m0 = mb * BM2 + crank * BM;
        const int nh = nb * 256 + crank * 128;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          const uint32_t fb = fullL + s * 8;
          if (leader) mbar_expect_tx(&full_bar[s], 2 * GEMM4_STAGE);
          tma_load_2d_2sm(smA + s * A_STAGE_BYTES, tmA, fb, kb * BK, arow);
          uint8_t* b = smB + s * B_BYTES;
          if (kBwd)
            tma_load_2d_2sm_mc(b + pq * (64 * 128), &tmB, &full_bar[s], bmc_mask, kb * BK, nh + 64 * pq);
          else
            tma_load_2d_2sm_mc(b + pq * (BK * 128), &tmB, &full_bar[s], bmc_mask, nh + 64 * pq, kb * BK);
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
        const int cb = td.chunk_begin;
        const int cc = td.chunk_count;
        for (int ls = 0; ls < nls; ++ls) {
          const int nq = max(0, min(4, cc - ls * 4));
          mbar_wait(&empty_bar[s], ph ^ 1);
          const uint32_t fb = fullL + s * 8;
          if (nq > 0) {
            if (leader) mbar_expect_tx(&full_bar[s], 2 * (A_STAGE_BYTES + nq * 2 * LORA_CHUNK_BYTES));
            tma_load_2d_2sm(smA + s * A_STAGE_BYTES, &tmAL, fb, ls * BK, m0);
            uint8_t* b = smB + s * B_BYTES;
            for (int qq = 0; qq < nq; ++qq) {
              const int prow = p.chunks[cb + ls * 4 + qq];
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tma_load_2d_2sm(b + j * (BK * 128) + qq * LORA_CHUNK_BYTES, &tmBP, fb, nh + 64 * j, prow);
            }
          } else if (leader) {
            mbar_expect_tx(&full_bar[s], 0);       // padding stage (the other pair has more chunks)
          }
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc_base = make_idesc_bf16(BM2, 256, false, !kBwd);
      constexpr uint32_t idesc_lora = make_idesc_bf16(BM2, 256, false, true);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        int mb2, nb, mb, nls;
        tile_coords(t, q2, mb2, nb);
        TileDesc td;
        pair_tile(mb2, td, mb, nls);
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(smA + s * A_STAGE_BYTES);
            const uint32_t b_addr = smem_u32(smB + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
              const uint64_t ad = make_sdesc_sw128(a_addr + k * 32, 16, 1024);
              const uint64_t bd = kBwd ? make_sdesc_sw128(b_addr + k * 32, 16, 1024)
                                       : make_sdesc_sw128(b_addr + k * (UK * 128), BK * 128, 1024);
              mma_bf16_ss_2sm(d_tmem, ad, bd, idesc_base, (kb | k) != 0);
            }
            mma_commit_2sm_mc(&empty_bar[s], 0xF);
          }
          __syncwarp();
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
        const int cc = td.chunk_count;
        for (int ls = 0; ls < nls; ++ls) {
          const int nq = max(0, min(4, cc - ls * 4));
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(smA + s * A_STAGE_BYTES);
            const uint32_t b_addr = smem_u32(smB + s * B_BYTES);
            for (int qq = 0; qq < nq; ++qq)
              mma_bf16_ss_2sm(d_tmem, make_sdesc_sw128(a_addr + qq * 32, 16, 1024),
                              make_sdesc_sw128(b_addr + qq * LORA_CHUNK_BYTES, BK * 128, 1024), idesc_lora, 1u);
            mma_commit_2sm_mc(&empty_bar[s], 0xF);
          }
          __syncwarp();
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
        if (lane == 0) mma_commit_2sm_mc(&tfull_bar[acc], pair_mask);
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const uint32_t ew = warp - 4;
    const uint32_t temptyL = mapa_shared(smem_u32(tempty_bar), 2 * pq);
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = cluster_id; t < num_tiles; t += num_clusters) {
      int mb2, nb, mb, nls;
      tile_coords(t, q2, mb2, nb);
      TileDesc td;
      pair_tile(mb2, td, mb, nls);
      epilogue_tile<256>(p, tmem_base + acc * 256, ew, lane, td, crank * BM, nb * 256, &tfull_bar[acc],
                         acc_ph, epi_stage, temptyL + acc * 8);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
    if (ew == 0 && lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
}

// ============================================================================ K3 shrink
// One CTA per item = (M-tile, LoRA segment piece of that tile, <= 128 rows):
//   T[rows, rank_pad] = A_src[rows, K] . P[rank rows, K]^T (tcgen05, M=128, N=rank_pad),
// scaled by alpha/r, rounded to bf16 and written into A_lora rows tile*TM + p0 .. at the piece's
// column block col0 (zeros elsewhere come from a memset) — the block-diagonal LoRA operand.
// The shrink is HBM-bound (it re-reads the LoRA segments' rows once, N = rank is tiny), so it
// runs 2 CTAs per SM (110 KB smem, 256 TMEM columns each) with as many pipeline stages as the
// item's rank leaves room for: stage = 16 KB of A + rank_pad x 128 B of the pack.
//
// K is split into fixed chunks of SHRINK_KB_CHUNK k-blocks (blockIdx.y = chunk): a slab of a
// few decode rows would otherwise be one CTA walking all of K serially, and a prefill dispatch
// would be one unbalanced wave. Each chunk's fp32 partial goes to a workspace; the LAST chunk
// CTA of the slab to finish (atomic ticket) adds the partials in chunk order 0..S-1, scales,
// rounds to bf16 and writes A_lora. The chunking depends only on K, and the order of every sum
// is fixed, so a row's result never depends on the dispatch it rides in (batching invisible).
constexpr int SHRINK_KB_CHUNK = 20;   // default k-blocks per chunk (1280 of K); ss_set_option("shrink_kb_chunk")
constexpr int SHRINK_MAXN = 256;
constexpr int SHRINK_MAX_STAGES = 12;
constexpr int SHRINK_SMEM = 110 * 1024;

struct ShrinkItem {
  int32_t seg;
  int32_t amap;   // A source tensor map (0 = X, 1 + i = direct source i)
  int32_t arow;   // row coordinate of the item's first row in that map
  int32_t rows;   // <= 128
  int32_t orow;   // first output row in A_lora (tile * TM + row offset within tile)
  int32_t col0;   // column of this segment's rank block in its tile
  int32_t pack;   // 0: pack map tmP, contraction K = p.K; 1: tmP2, K = p.K2 (gradient shrinks)
  int32_t a_rows; // rows one A box delivers (128, or 16 for short pieces: MMA rows past the box
                  // are stale smem whose outputs are never written); 0 = 128
  // block-diagonal zeros: the first slab of a piece writes zeros into its column block for the
  // tile's rows OUTSIDE the piece [piece_lo, piece_hi) (tile-relative; tile rows tile_row0 ..
  // + tm), so rows of other clients in the tile get no contribution from this adapter
  int32_t zero_fill;
  int32_t tile_row0, tm, piece_lo, piece_hi;
  // 1: the segment's column block is 2 x rank_pad wide: hi = bf16(v) in the first half and
  // lo = bf16(v - hi) in the second, the GEMM's K-extension reading the same B rows for both
  // (v = s*x.A kept to ~2^-17 instead of bf16's 2^-9: the fp32-output tier)
  int32_t hilo;
  // > 0: tensor map of the lo halves (X_lo, same box) of an SEGF_IA3_LO backward segment: every
  // K chunk runs a second pass over them into the same accumulator (g = hi + lo, fp32 tier)
  int32_t amap_lo;
  int32_t pad_;
};

struct ShrinkParams {
  int K, K2;
  int lora_ld;  // A_lora row stride (elements)
  const DevSeg* segs;
  const ShrinkItem* items;
  const CUtensorMap* tmaps;
  __nv_bfloat16* a_lora;
  float* part;            // [items, max chunks, 128, part_ld] fp32 chunk partials
  int part_ld;            // >= every item's rank_pad
  int max_chunks;         // gridDim.y
  int* ticket;            // [items] arrival counters (zero between launches)
  int kb_chunk;           // k-blocks per chunk (a per-context constant: the chunking must not vary)
  int* done_ctr = nullptr;  // overlap mode: every CTA adds 1 after its writes (the GEMM waits on it)
};

__host__ __device__ inline int shrink_chunks(int K, int kb_chunk) {
  return ((K + BK - 1) / BK + kb_chunk - 1) / kb_chunk;
}

// One shrink item (bx) and K chunk (by of gy; gy == 1: every chunk, whole mode) per CTA; the
// kernel below, and the fused adapter-gradient kernel (grads.cuh), which picks items itself.
__device__ __forceinline__ void lora_shrink_body(const CUtensorMap& tmP,   // pack [R, K] (K-major rows)
                                                 const CUtensorMap& tmP2,  // second pack (items with pack = 1)
                                                 const ShrinkParams& p, const int bx, const int by,
                                                 const int gy) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const ShrinkItem it = p.items[bx];
  const DevSeg sg = p.segs[it.seg];
  const int npad = sg.rank_pad;  // multiple of 16, <= 256
  const CUtensorMap* tmA = p.tmaps + it.amap;
  const CUtensorMap* tmPk = it.pack ? &tmP2 : &tmP;
  const int Kc = it.pack ? p.K2 : p.K;
  const int nkb_all = (Kc + BK - 1) / BK;
  const int nchk = shrink_chunks(Kc, p.kb_chunk);
  // whole mode (gridDim.y == 1): this CTA runs every chunk of the slab, double-buffering the
  // chunk accumulators in TMEM and summing them in registers (npad <= 64); split mode: one
  // chunk per CTA, partials through the workspace, the slab's last CTA sums them. Both add the
  // chunk partials in the same order, so the two modes give bitwise-identical rows.
  const bool whole = gy == 1;
  const int c0 = whole ? 0 : by;
  const int c1 = whole ? nchk : c0 + 1;
  if (c0 >= nchk) {         // (gradient launches mix two K's; uniform exit before any barrier)
    if (p.done_ctr && threadIdx.x == 0) atomicAdd(p.done_ctr, 1);
    return;
  }
  const int b_bytes = npad * BK * 2;
  const int stage_bytes = A_STAGE_BYTES + b_bytes;
  const int SHRINK_STAGES = min(SHRINK_MAX_STAGES, (SHRINK_SMEM - 2048) / stage_bytes);
  // barriers in the first KB, then stages (each A | B, 1 KB aligned)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty_bar = full_bar + SHRINK_MAX_STAGES;
  uint64_t* tfull = empty_bar + SHRINK_MAX_STAGES;     // [2]
  uint64_t* tempty = tfull + 2;                        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* stage0 = smem + 1024;
#define SHRINK_A(s) (stage0 + (s) * stage_bytes)
#define SHRINK_B(s) (stage0 + (s) * stage_bytes + A_STAGE_BYTES)

  const CUtensorMap* tmAlo = p.tmaps + (it.amap_lo > 0 ? it.amap_lo : it.amap);
  const int npass = it.amap_lo > 0 ? 2 : 1;
  if (warp == 0 && lane == 0) {
    tensormap_acquire(tmA);
    tma_prefetch_desc(tmA);
    tma_prefetch_desc(tmPk);
    if (npass == 2) tensormap_acquire(tmAlo);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < SHRINK_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();
  const int nchunk = npad / LORA_CHUNK;
  __shared__ int last_flag;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int c = c0; c < c1; ++c)
        for (int pass = 0; pass < npass; ++pass)
          for (int kb = c * p.kb_chunk; kb < min(nkb_all, (c + 1) * p.kb_chunk); ++kb) {
            mbar_wait(&empty_bar[s], ph ^ 1);
            mbar_expect_tx(&full_bar[s], (it.a_rows ? it.a_rows * 128 : A_STAGE_BYTES) + nchunk * LORA_CHUNK_BYTES);
            tma_load_2d(SHRINK_A(s), pass ? tmAlo : tmA, &full_bar[s], kb * BK, it.arow);
            for (int q = 0; q < nchunk; ++q)
              tma_load_2d(SHRINK_B(s) + q * LORA_CHUNK_BYTES, tmPk, &full_bar[s], kb * BK,
                          sg.pack_row + q * LORA_CHUNK);
            if (++s == SHRINK_STAGES) { s = 0; ph ^= 1; }
          }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(BM, (uint32_t)npad, false, false);
    int s = 0;
    uint32_t ph = 0;
    for (int c = c0; c < c1; ++c) {
      const int buf = (c - c0) & 1;
      const uint32_t tph = (((c - c0) >> 1) & 1) ^ 1;
      mbar_wait(&tempty[buf], tph);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * 128;
      const int kb0 = c * p.kb_chunk, kb1 = min(nkb_all, kb0 + p.kb_chunk);
      for (int pass = 0; pass < npass; ++pass)
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(SHRINK_A(s));
            const uint32_t b_addr = smem_u32(SHRINK_B(s));
#pragma unroll
            for (int k = 0; k < BK / UK; ++k)
              mma_bf16_ss(d_tmem, make_sdesc_sw128(a_addr + k * 32, 16, 1024),
                          make_sdesc_sw128(b_addr + k * 32, 16, 1024), idesc, (pass | (kb - kb0) | k) != 0);
            mma_commit(&empty_bar[s]);
          }
          __syncwarp();
          if (++s == SHRINK_STAGES) { s = 0; ph ^= 1; }
        }
      if (lane == 0) mma_commit(&tfull[buf]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const uint32_t ew = warp - 4;
    const int lr = ew * 32 + lane;  // row within the item
    const bool ok = lr < it.rows;
    __nv_bfloat16* out = p.a_lora + (int64_t)(it.orow + lr) * p.lora_ld + it.col0;
    auto store_bf16 = [&](int c, const float* v) {
      uint4* o = reinterpret_cast<uint4*>(out + c * 16);
      o[0] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                        pack_bf16x2(v[6], v[7]));
      o[1] = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                        pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
      if (it.hilo) {
        float lo[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) lo[j] = v[j] - __bfloat162float(__float2bfloat16_rn(v[j]));
        uint4* q = reinterpret_cast<uint4*>(out + npad + c * 16);
        q[0] = make_uint4(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]), pack_bf16x2(lo[4], lo[5]),
                          pack_bf16x2(lo[6], lo[7]));
        q[1] = make_uint4(pack_bf16x2(lo[8], lo[9]), pack_bf16x2(lo[10], lo[11]),
                          pack_bf16x2(lo[12], lo[13]), pack_bf16x2(lo[14], lo[15]));
      }
    };
    if (whole && nchk > 1) {
      // running fp32 sums of the chunk partials, in chunk order (npad <= 64: host-guaranteed)
      float acc[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = 0.f;
      for (int c = c0; c < c1; ++c) {
        const int buf = (c - c0) & 1;
        mbar_wait(&tfull[buf], ((c - c0) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (g < nchunk) {
            uint32_t r[16];
            tmem_ld_32x32b_x16(tmem_base + buf * 128 + g * 16 + ((ew * 32u) << 16), r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[g * 16 + j] += __uint_as_float(r[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
      if (ok) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (g < nchunk) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = acc[g * 16 + j] * sg.lora_scale;
            store_bf16(g, v);
          }
        }
      }
    } else if (nchk == 1) {
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      for (int c = 0; c < nchunk; ++c) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem_base + c * 16 + ((ew * 32u) << 16), r);
        tmem_wait_ld();
        if (ok) {
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) * sg.lora_scale;
          store_bf16(c, v);
        }
      }
      tc_fence_before();
    } else {
      // split mode: this chunk's fp32 partial -> workspace, the slab's last chunk sums in order
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      float* mine = p.part + (((int64_t)bx * p.max_chunks + c0) * BM + lr) * p.part_ld;
      for (int c = 0; c < nchunk; ++c) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem_base + c * 16 + ((ew * 32u) << 16), r);
        tmem_wait_ld();
        if (ok) {
          float4* o = reinterpret_cast<float4*>(mine + c * 16);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcg(o + j, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                      __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
      }
      tc_fence_before();
      __threadfence();
      named_bar_sync(1, 128);
      if (ew == 0 && lane == 0) last_flag = atomicAdd(p.ticket + bx, 1) == nchk - 1;
      named_bar_sync(1, 128);
      if (last_flag) {
        __threadfence();
        if (ok) {
          const float* base = p.part + ((int64_t)bx * p.max_chunks * BM + lr) * p.part_ld;
          for (int c = 0; c < nchunk; ++c) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
            for (int q = 0; q < nchk; ++q) {
              const float4* src = reinterpret_cast<const float4*>(base + (int64_t)q * BM * p.part_ld + c * 16);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 f = __ldcg(src + j);
                v[4 * j] += f.x; v[4 * j + 1] += f.y; v[4 * j + 2] += f.z; v[4 * j + 3] += f.w;
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] *= sg.lora_scale;
            store_bf16(c, v);
          }
        }
        if (ew == 0 && lane == 0) p.ticket[bx] = 0;   // ready for the next launch
      }
    }
    if (it.zero_fill && c0 == 0) {
      // zeros of the block-diagonal operand (replaces a memset of the whole operand)
      const int vec_per_row = (it.hilo ? 2 : 1) * npad / 8;  // 16-byte vectors of bf16
      const int nrow = it.tm - (it.piece_hi - it.piece_lo);
      for (int v = (int)(ew * 32 + lane); v < nrow * vec_per_row; v += 128) {
        const int k = v / vec_per_row;
        const int row = k < it.piece_lo ? k : k + (it.piece_hi - it.piece_lo);
        reinterpret_cast<uint4*>(p.a_lora + (int64_t)(it.tile_row0 + row) * p.lora_ld + it.col0)[v % vec_per_row] =
            make_uint4(0, 0, 0, 0);
      }
    }
  }
  __syncthreads();
  if (p.done_ctr && threadIdx.x == 0) {
    __threadfence();                 // this CTA's A_lora writes before the arrival (cumulative)
    atomicAdd(p.done_ctr, 1);
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 256);
  }
}

__global__ void __launch_bounds__(GEMM_THREADS, 2)
    lora_shrink_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmP2,
                       const ShrinkParams p) {
  lora_shrink_body(tmP, tmP2, p, (int)blockIdx.x, (int)blockIdx.y, (int)gridDim.y);
}
#undef SHRINK_A
#undef SHRINK_B

// ============================================================================ K4 gather
// Packs the rows that cannot be TMA-loaded in place (tails of segments shorter than a tile,
// f32 sources, IA3 backward rows that need g = dy * l) into X, in segment order
// (concat_rows order restricted to packed pieces), and records each X row's segment.
struct GatherParams {
  int MX, K;              // packed rows, width
  int ldx;
  int n_piece;
  int nsplit;             // column chunks per row (several warps per row for small dispatches)
  int ia3_in_prologue;    // backward: g = dy * l
  const DevSeg* segs;
  const int32_t* piece_seg;  // segment of each packed piece, in X order
  __nv_bfloat16* X;
  int32_t* row_seg;
  // != nullptr when some segment is SEGF_IA3_LO: its rows get lo = bf16(g - bf16(g)) here (the
  // second K pass of their tiles), every other packed row zeros
  __nv_bfloat16* X_lo = nullptr;
};


__device__ __forceinline__ int find_piece(const GatherParams& p, int xrow) {
  int lo = 0, hi = p.n_piece - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.segs[p.piece_seg[mid]].xrow0 <= xrow) lo = mid; else hi = mid - 1;
  }
  return p.piece_seg[lo];
}

// One warp per (row, column chunk), grid-stride.
// Block `bx` of `nb` (the kernel below; or a share of a combined launch, decode.cuh).
__device__ __forceinline__ void gather_rows_body(const GatherParams& p, const int bx, const int nb) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  // work item = (row, column chunk): a decode-size dispatch (tens of rows) still spreads over
  // the whole GPU instead of one latency-bound warp per row
  const int nchunk8 = (p.K / 8 + p.nsplit - 1) / p.nsplit;     // 8-element units per chunk
  for (int w = bx * wpb + (threadIdx.x >> 5); w < p.MX * p.nsplit; w += nb * wpb) {
    const int row = w / p.nsplit, part = w - row * p.nsplit;
    const int u0 = part * nchunk8, u1 = min(p.K / 8, u0 + nchunk8);   // vector units [u0, u1)
    const int e0 = part == 0 ? 0 : u0 * 8, e1 = part == p.nsplit - 1 ? p.K : u1 * 8;  // scalar range
    const int si = find_piece(p, row);
    const DevSeg& sg = p.segs[si];
    if (lane == 0 && part == 0) p.row_seg[row] = si;
    const int64_t lr = row - sg.xrow0 + sg.xlocal0;
    __nv_bfloat16* xr = p.X + (int64_t)row * p.ldx;
    const bool scale = p.ia3_in_prologue && (sg.flags & SEGF_IA3);
    const float* l = sg.ia3;
    const bool vec = (sg.flags & SEGF_SRC_VEC) && ((p.K & 7) == 0);
    if (p.X_lo) {
      __nv_bfloat16* xl = p.X_lo + (int64_t)row * p.ldx;
      if (!(scale && (sg.flags & SEGF_IA3_LO))) {
        for (int i = e0 + lane; i < e1; i += 32) xl[i] = __float2bfloat16_rn(0.f);
      } else {
        // IA3 backward with the lo pass: g = dy * l as hi (X) + lo (X_lo), scalar per element
        // (these dispatches are fine-tune backward slabs of f32-output clients; not the hot path)
        for (int i = e0 + lane; i < e1; i += 32) {
          const float v = ((sg.flags & SEGF_SRC_BF16)
                               ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(sg.src)[lr * sg.src_ld + i])
                               : reinterpret_cast<const float*>(sg.src)[lr * sg.src_ld + i]) * __ldg(l + i);
          const __nv_bfloat16 h = __float2bfloat16_rn(v);
          xr[i] = h;
          xl[i] = __float2bfloat16_rn(v - __bfloat162float(h));
        }
        continue;
      }
    }
    if (sg.flags & SEGF_SRC_BF16) {
      const __nv_bfloat16* sr = reinterpret_cast<const __nv_bfloat16*>(sg.src) + lr * sg.src_ld;
      if (vec && !scale) {
        const uint4* s4 = reinterpret_cast<const uint4*>(sr);
        uint4* d4 = reinterpret_cast<uint4*>(xr);
#pragma unroll 4
        for (int i = u0 + lane; i < u1; i += 32) d4[i] = __ldg(s4 + i);
      } else if (vec) {
        // IA3 backward prologue, 8 bf16 per lane per step: g = dy * l (client.py:291-294)
        const uint4* s4 = reinterpret_cast<const uint4*>(sr);
        uint4* d4 = reinterpret_cast<uint4*>(xr);
        for (int i = u0 + lane; i < u1; i += 32) {
          const uint4 raw = __ldg(s4 + i);
          const float4 la = __ldg(reinterpret_cast<const float4*>(l) + 2 * i);
          const float4 lb = __ldg(reinterpret_cast<const float4*>(l) + 2 * i + 1);
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
          const float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
          const float2 f2 = __bfloat1622float2(h[2]), f3 = __bfloat1622float2(h[3]);
          d4[i] = make_uint4(pack_bf16x2(f0.x * la.x, f0.y * la.y), pack_bf16x2(f1.x * la.z, f1.y * la.w),
                             pack_bf16x2(f2.x * lb.x, f2.y * lb.y), pack_bf16x2(f3.x * lb.z, f3.y * lb.w));
        }
      } else {
        for (int i = e0 + lane; i < e1; i += 32) {
          float v = __bfloat162float(sr[i]);
          if (scale) v *= __ldg(l + i);
          xr[i] = __float2bfloat16_rn(v);
        }
      }
    } else {
      const float* sr = reinterpret_cast<const float*>(sg.src) + lr * sg.src_ld;
      if (vec) {
        const float4* s4 = reinterpret_cast<const float4*>(sr);
        uint4* d4 = reinterpret_cast<uint4*>(xr);
        for (int i = u0 + lane; i < u1; i += 32) {
          float4 a = __ldg(s4 + 2 * i), b = __ldg(s4 + 2 * i + 1);
          if (scale) {
            const float4 la = __ldg(reinterpret_cast<const float4*>(l) + 2 * i);
            const float4 lb = __ldg(reinterpret_cast<const float4*>(l) + 2 * i + 1);
            a.x *= la.x; a.y *= la.y; a.z *= la.z; a.w *= la.w;
            b.x *= lb.x; b.y *= lb.y; b.z *= lb.z; b.w *= lb.w;
          }
          d4[i] = make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                             pack_bf16x2(b.z, b.w));
        }
      } else {
        for (int i = e0 + lane; i < e1; i += 32) {
          float v = sr[i];
          if (scale) v *= __ldg(l + i);
          xr[i] = __float2bfloat16_rn(v);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) gather_rows_kernel(const GatherParams p) {
  pdl_wait();
  pdl_trigger();
  gather_rows_body(p, (int)blockIdx.x, (int)gridDim.x);
}

// f32 -> bf16 conversion for weight / pack uploads.
__global__ void f32_to_bf16_2d_kernel(const float* __restrict__ src, int64_t src_ld,
                                      __nv_bfloat16* __restrict__ dst, int64_t dst_ld, int rows,
                                      int cols) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    dst[r * dst_ld + c] = __float2bfloat16_rn(src[r * src_ld + c]);
  }
}

// Transposing copy: dst[c, r] = src[r, c]  (A [d_in, r] -> A^T pack rows), f32 or bf16 source.
__global__ void transpose_to_bf16_kernel(const void* __restrict__ src, int src_bf16, int64_t src_ld,
                                         __nv_bfloat16* __restrict__ dst, int64_t dst_ld, int rows,
                                         int cols) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const float v = src_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[r * src_ld + c])
                             : reinterpret_cast<const float*>(src)[r * src_ld + c];
    dst[c * dst_ld + r] = __float2bfloat16_rn(v);
  }
}

__global__ void copy_to_bf16_kernel(const void* __restrict__ src, int src_bf16, int64_t src_ld,
                                    __nv_bfloat16* __restrict__ dst, int64_t dst_ld, int rows,
                                    int cols) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const float v = src_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[r * src_ld + c])
                             : reinterpret_cast<const float*>(src)[r * src_ld + c];
    dst[r * dst_ld + c] = __float2bfloat16_rn(v);
  }
}

__global__ void copy_to_f32_kernel(const void* __restrict__ src, int src_bf16,
                                   float* __restrict__ dst, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[i])
                      : reinterpret_cast<const float*>(src)[i];
}

// Row copies device staging -> (pinned host) destination rows, one warp per row, 16-byte
// vectors: the reply leg of a zero-copy host dispatch (coalesced PCIe writes, one launch
// instead of one D2H memcpy per segment).
struct RowCopy {
  const char* src;     // first row (device)
  char* dst;           // first row (host, UVA)
  int64_t src_ld, dst_ld;  // bytes
  int32_t rows, row_bytes; // row_bytes % 16 == 0 when vec
};

__global__ void __launch_bounds__(256) copy_rows_kernel(const RowCopy* __restrict__ ops, int n_ops,
                                                        int total_rows) {
  const int lane = threadIdx.x & 31;
  for (int w = blockIdx.x * 8 + (threadIdx.x >> 5); w < total_rows; w += gridDim.x * 8) {
    int o = 0, r = w;
    while (o < n_ops - 1 && r >= ops[o].rows) { r -= ops[o].rows; ++o; }
    const RowCopy& op = ops[o];
    const char* s = op.src + r * op.src_ld;
    char* d = op.dst + r * op.dst_ld;
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | op.row_bytes) & 15) == 0;
    if (vec) {
      for (int i = lane; i < op.row_bytes / 16; i += 32)
        reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
    } else {
      for (int i = lane; i < op.row_bytes; i += 32) d[i] = s[i];
    }
  }
}

}  // namespace ss
