// K1d: split-K persistent GEMM for decode-class segments (SURVEY §8a affine_forward /
// affine_backward_input / noise matmul + the fused adapter epilogue, for requests of a few rows).
//
// Why a separate kernel and a separate summation order. A decode dispatch streams W (HBM-bound in
// principle), but every output column of the single-chain kernels is K/16 dependent UMMAs
// accumulating into one TMEM accumulator, and at decode sizes that chain, not HBM, sets the time
// (DESIGN.md "Decode"). Only a shorter chain helps, and a shorter chain is a different fp32
// summation order. Rows of a decode-class segment (its own row count <= decode_rows, a property
// of the request alone) therefore use their own fixed order, independent of the dispatch:
//
//   K is cut into C = min(decode_chunks, ceil(K / 128)) contiguous chunks of whole 128-deep
//   stages (a function of K only); chunk c is one UMMA chain in K order; the LoRA expand of the
//   tile (its rank chunks, block-diagonal over the tile's segments as in the other kernels) is a
//   chain of its own. y = ((p_0 + p_1) + ... + p_{C-1}) + p_lora, then bias / y_base / IA3.
//
// A row's bits depend only on its segment's class, K and its own values (foreign rows of the
// block-diagonal LoRA operand contribute exact zeros): batched == solo holds for decode-class rows
// exactly as for the single-chain kernels (tests/test_gpu_decode.py).
//
// Work item = (64-row decode tile m, 128-column tile n, chunk c in 0..C, c == C the LoRA chain),
// chunk fastest. A persistent grid walks the items: the producer streams stage after stage
// across items, the MMA warp alternates two TMEM accumulators, and the epilogue warps write each
// item's fp32 partial to an L2-resident workspace ([row][col], 512 B per row). No CTA waits on
// another: the fixed-order sum, bias / y_base / IA3 and the stores run in dec_fixup_kernel,
// launched behind the GEMM with programmatic dependent launch.
// The UMMA is M = 128: A boxes deliver 64 rows, MMA rows 64-127 read the stage bytes that follow
// and their outputs are never read. Stage = 128 of K: A {64 k, 64 rows, 2 k-chunks} (16 KB), W
// two {64 n, 128 k} boxes (forward, MN-major) or {64 k, 128 n, 2 k-chunks} (backward) (32 KB).
#pragma once
#include "kernels.cuh"

namespace ss {

constexpr int DEC_ROWS = 64;                            // packed rows per tile
constexpr int DEC_TN = 128;                             // output columns per tile
constexpr int DEC_KB = 2;                               // 64-deep k-blocks per stage
constexpr int DEC_SK = DEC_KB * BK;                     // 128 of K per stage
constexpr int DEC_A_BYTES = DEC_KB * DEC_ROWS * 128;    // 16 KB
constexpr int DEC_WBOX = DEC_SK * 128;                  // one {64 n, 128 k} box: 16 KB
constexpr int DEC_B_BYTES = DEC_TN * DEC_SK * 2;        // 32 KB
constexpr int DEC_STAGE = DEC_A_BYTES + DEC_B_BYTES;    // 48 KB
#ifndef SS_DEC_STAGES
#define SS_DEC_STAGES 4
#endif
constexpr int DEC_STAGES = SS_DEC_STAGES;
constexpr int DEC_MAX_C = 16;
constexpr int DEC_PART = DEC_TN * DEC_ROWS;             // fp32 values per item partial (32 KB)
constexpr int DEC_SMEM = DEC_STAGES * DEC_STAGE + 1024 + 256;

struct DecTile {
  int32_t arow;          // first packed (X) row
  int32_t rows;          // valid rows (<= DEC_ROWS), whole segments
  int32_t al_row;        // first row of the tile's block-diagonal LoRA operand
  int32_t lo;            // 1: some row is SEGF_IA3_LO -> every chunk runs a second pass over X_lo
  int32_t chunk_begin;   // LoRA rank chunks (pack rows) of the tile in `chunks`
  int32_t chunk_count;   // 0: no LoRA item for this tile
};

struct DecParams {
  int N, K;
  int C;                 // K chunks
  int nst;               // 128-deep stages over K
  int n_m, n_n;          // decode tiles, 128-column tiles
  int items_per_n;       // sum over decode tiles of C + (chunk_count > 0)
  int has_bias, ia3_in_epilogue;
  const float* bias;
  const DevSeg* segs;
  const int32_t* row_seg;
  const DecTile* tiles;
  const int32_t* chunks;
  const CUtensorMap* tmaps;
  int amap, alo_map;     // X / X_lo as {64 k, 64 rows, 2 k-chunks} boxes
  float* part;           // [n_n * n_m * (C + 1)][DEC_ROWS][DEC_TN] fp32 partials (item c of tile
                         // nt * n_m + mt at (tile * (C + 1) + c))
};

__host__ __device__ inline int dec_stages(int K) { return (K / BK + DEC_KB - 1) / DEC_KB; }

// item w -> (n tile, decode tile m, chunk c); c == C is the tile's LoRA item
__device__ __forceinline__ void dec_item(const DecParams& p, int w, int& n, int& m, int& c) {
  n = w / p.items_per_n;
  int r = w - n * p.items_per_n;
  m = 0;
  for (;;) {
    const int k = p.C + (p.tiles[m].chunk_count > 0 ? 1 : 0);
    if (r < k) break;
    r -= k;
    ++m;
  }
  c = r;
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

template <bool kBwd>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    seg_gemm_dec_kernel(const __grid_constant__ CUtensorMap tmB,   // W (see above)
                        const __grid_constant__ CUtensorMap tmAL,  // A_lora, box {64, 64 rows}
                        const __grid_constant__ CUtensorMap tmBP,  // pack [R, N] (MN-major B), box {64, 16}
                        const DecParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + DEC_STAGES * DEC_STAGE);
  uint64_t* empty_bar = full_bar + DEC_STAGES;
  uint64_t* tfull_bar = empty_bar + DEC_STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const int n_items = p.n_n * p.items_per_n;
  const int nkb = p.K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmAL);
    tma_prefetch_desc(&tmBP);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2);   // warps 4 and 5 (TMEM lanes 0-63) read the accumulator
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * DEC_TN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const CUtensorMap* tmA = p.tmaps + p.amap;
      const CUtensorMap* tmAlo = p.tmaps + p.alo_map;
      tensormap_acquire(tmA);
      if (p.alo_map != p.amap) tensormap_acquire(tmAlo);
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        int nt, mt, c;
        dec_item(p, w, nt, mt, c);
        const DecTile td = p.tiles[mt];
        const int n0 = nt * DEC_TN;
        if (c < p.C) {
          const int st0 = c * p.nst / p.C, st1 = (c + 1) * p.nst / p.C;
          for (int pass = 0; pass < (td.lo ? 2 : 1); ++pass) {
            for (int st = st0; st < st1; ++st) {
              mbar_wait(&empty_bar[s], ph ^ 1);
              mbar_expect_tx(&full_bar[s], DEC_STAGE);
              uint8_t* a = smem + s * DEC_STAGE;
              uint8_t* b = a + DEC_A_BYTES;
              tma_load_3d(a, pass ? tmAlo : tmA, &full_bar[s], 0, td.arow, st * DEC_KB);
              if (kBwd) {
                tma_load_3d(b, &tmB, &full_bar[s], 0, n0, st * DEC_KB);
              } else {
                tma_load_2d(b, &tmB, &full_bar[s], n0, st * DEC_SK);
                tma_load_2d(b + DEC_WBOX, &tmB, &full_bar[s], n0 + 64, st * DEC_SK);
              }
              if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
            }
          }
        } else {
          for (int ls = 0; ls * 4 < td.chunk_count; ++ls) {
            const int nq = min(4, td.chunk_count - ls * 4);
            mbar_wait(&empty_bar[s], ph ^ 1);
            mbar_expect_tx(&full_bar[s], DEC_ROWS * 128 + nq * 2 * LORA_CHUNK_BYTES);
            uint8_t* a = smem + s * DEC_STAGE;
            uint8_t* b = a + DEC_A_BYTES;
            tma_load_2d(a, &tmAL, &full_bar[s], ls * BK, td.al_row);
            for (int q = 0; q < nq; ++q) {
              const int prow = p.chunks[td.chunk_begin + ls * 4 + q];
              tma_load_2d(b + q * LORA_CHUNK_BYTES, &tmBP, &full_bar[s], n0, prow);
              tma_load_2d(b + BK * 128 + q * LORA_CHUNK_BYTES, &tmBP, &full_bar[s], n0 + 64, prow);
            }
            if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_base = make_idesc_bf16(BM, DEC_TN, false, !kBwd);
    constexpr uint32_t idesc_lora = make_idesc_bf16(BM, DEC_TN, false, true);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      int nt, mt, c;
      dec_item(p, w, nt, mt, c);
      const DecTile td = p.tiles[mt];
      mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * DEC_TN;
      uint32_t accum = 0;
      if (c < p.C) {
        const int st0 = c * p.nst / p.C, st1 = (c + 1) * p.nst / p.C;
        for (int pass = 0; pass < (td.lo ? 2 : 1); ++pass) {
          for (int st = st0; st < st1; ++st) {
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t a_addr = smem_u32(smem + s * DEC_STAGE);
              const uint32_t b_addr = a_addr + DEC_A_BYTES;
              const int kbs = min(DEC_KB, nkb - st * DEC_KB);
              for (int cc = 0; cc < kbs; ++cc) {
#pragma unroll
                for (int k = 0; k < BK / UK; ++k) {
                  const uint64_t ad = make_sdesc_sw128(a_addr + cc * (DEC_ROWS * 128) + k * 32, 16, 1024);
                  const uint64_t bd = kBwd ? make_sdesc_sw128(b_addr + cc * (DEC_TN * 128) + k * 32, 16, 1024)
                                           : make_sdesc_sw128(b_addr + (cc * 4 + k) * (UK * 128), DEC_WBOX, 1024);
                  mma_bf16_ss(d_tmem, ad, bd, idesc_base, accum);
                  accum = 1;
                }
              }
              mma_commit(&empty_bar[s]);
            }
            __syncwarp();
            if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
          }
        }
      } else {
        for (int ls = 0; ls * 4 < td.chunk_count; ++ls) {
          const int nq = min(4, td.chunk_count - ls * 4);
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(smem + s * DEC_STAGE);
            const uint32_t b_addr = a_addr + DEC_A_BYTES;
            for (int q = 0; q < nq; ++q) {
              const uint64_t ad = make_sdesc_sw128(a_addr + q * 32, 16, 1024);
              const uint64_t bd = make_sdesc_sw128(b_addr + q * LORA_CHUNK_BYTES, BK * 128, 1024);
              mma_bf16_ss(d_tmem, ad, bd, idesc_lora, accum);
              accum = 1;
            }
            mma_commit(&empty_bar[s]);
          }
          __syncwarp();
          if (++s == DEC_STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (lane == 0) mma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  } else if (warp == 4 || warp == 5) {
    // ------------------------------------------------------------ item partial -> workspace
    // TMEM lane = tile row (warps 4 and 5 own lanes 0-63); layout [row][col], 512 B per row
    const int row = (int)((warp - 4) * 32 + lane);
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      int nt, mt, c;
      dec_item(p, w, nt, mt, c);
      const bool ok = row < p.tiles[mt].rows;
      float4* dst = reinterpret_cast<float4*>(
          p.part + ((int64_t)(nt * p.n_m + mt) * (p.C + 1) + c) * DEC_PART + (int64_t)row * DEC_TN);
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < DEC_TN / 32; ++h) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + acc * DEC_TN + h * 32 + (((warp - 4) * 32u) << 16), r);
        tmem_wait_ld();
        if (ok) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(dst + h * 8 + j, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                                __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * DEC_TN);
  }
}

// K1d fixup: y = ((p_0 + p_1) + ... + p_{C-1}) + p_lora, then bias / y_base / IA3 / dst, for
// every valid row of every decode tile. Launched behind the GEMM (PDL: the grid is resident
// early and waits on griddepcontrol.wait, which covers the GEMM's partial stores). One CTA per
// 16 rows x 128 columns of a tile; a thread owns one row x 8 columns and issues the loads of all
// C (+1) partials before the first add (the sum order is fixed, the loads are not serialised).
constexpr int DEC_FIX_ROWS = 16;
constexpr int DEC_FIX_THREADS = DEC_FIX_ROWS * (DEC_TN / 8);   // 256

__global__ void __launch_bounds__(DEC_FIX_THREADS)
    dec_fixup_kernel(const DecParams p) {
  const int q = blockIdx.x % (DEC_ROWS / DEC_FIX_ROWS);
  const int tile = blockIdx.x / (DEC_ROWS / DEC_FIX_ROWS);
  const int nt = tile / p.n_m, mt = tile - nt * p.n_m;
  const int row = q * DEC_FIX_ROWS + (int)(threadIdx.x / (DEC_TN / 8));
  const int col = (int)(threadIdx.x % (DEC_TN / 8)) * 8;
  const DecTile td = p.tiles[mt];
  pdl_wait();
  pdl_trigger();
  const int n = nt * DEC_TN + col;
  if (row >= td.rows || n >= p.N) return;
  const float4* src = reinterpret_cast<const float4*>(p.part + (int64_t)tile * (p.C + 1) * DEC_PART +
                                                      (int64_t)row * DEC_TN + col);
  constexpr int P4 = DEC_PART / 4;
  float4 buf[DEC_MAX_C + 1][2];
#pragma unroll
  for (int c = 0; c <= DEC_MAX_C; ++c) {
    if (c < p.C || (c == p.C && td.chunk_count > 0)) {
      buf[c][0] = __ldcg(src + c * P4);
      buf[c][1] = __ldcg(src + c * P4 + 1);
    }
  }
  float v[8] = {buf[0][0].x, buf[0][0].y, buf[0][0].z, buf[0][0].w,
                buf[0][1].x, buf[0][1].y, buf[0][1].z, buf[0][1].w};
#pragma unroll
  for (int c = 1; c <= DEC_MAX_C; ++c) {
    if (c < p.C || (c == p.C && td.chunk_count > 0)) {
      v[0] += buf[c][0].x; v[1] += buf[c][0].y; v[2] += buf[c][0].z; v[3] += buf[c][0].w;
      v[4] += buf[c][1].x; v[5] += buf[c][1].y; v[6] += buf[c][1].z; v[7] += buf[c][1].w;
    }
  }
  const int ncols = min(8, p.N - n);
  const int xrow = td.arow + row;
  const DevSeg sg = p.segs[p.row_seg[xrow]];
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

}  // namespace ss
