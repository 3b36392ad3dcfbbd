// Probe: how fast can a persistent grid stream a decode-shaped weight matrix W [K, N] (bf16,
// row-major, the forward decode GEMM's B operand) through TMA, with no MMA behind it?
// Units are (k chunk of `kbc` 64-row k-blocks) x (group of `g` adjacent 64-column tiles), one
// {64 n, 64 k} 128B-swizzled box per tile per stage, exactly the K1d producer's access pattern
// (csrc/decode.cuh); units are claimed through an atomic ticket. Mode 1 streams the same bytes
// as contiguous 1-D bulk copies (the access-pattern upper bound).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2507_03220_b200/csrc
//        tools/probes/tma_stream.cu -o runs/tma_stream -lcuda
// Run:   runs/tma_stream K N g kbc stages mode [copies]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ss;

__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

struct P {
  int K, N, g, kbc, stages, mode, n_groups, n_chunks;
  const char* base;   // mode 1
  int* claim;
};

__global__ void __launch_bounds__(128, 1) stream_k(const __grid_constant__ CUtensorMap tm, P p) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = p.g * 8192;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  __shared__ int q_id[64];
  __shared__ int q_n;
  __shared__ int q_issued;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    q_n = 0; q_issued = 0;
    for (int s = 0; s < p.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int nkb = p.K / 64;
  const int total = p.n_groups * p.n_chunks;
  if (warp == 0 && lane == 0) {
    const uint64_t pol = policy_evict_first();
    int s = 0; uint32_t ph = 0;
    for (;;) {
      const int id = atomicAdd(p.claim, 1);
      if (id >= total) break;
      const int c = id / p.n_groups, gi = id % p.n_groups;
      const int kb0 = c * p.kbc, kb1 = min(nkb, kb0 + p.kbc);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], stage_bytes);
        uint8_t* b = smem + s * stage_bytes;
        if (p.mode == 0) {
          for (int j = 0; j < p.g; ++j)
            tma_load_2d_hint(b + j * 8192, &tm, &full[s], (gi * p.g + j) * 64, kb * 64, pol);
        } else {
          // same bytes, contiguous: unit = the k-block's rows of the group as one flat piece
          const size_t off = ((size_t)kb * p.n_groups + gi) * (size_t)stage_bytes;
          bulk_load_1d(b, p.base + off, stage_bytes, &full[s], pol);
        }
        *(volatile int*)&q_issued += 1;
        if (++s == p.stages) { s = 0; ph ^= 1; }
      }
    }
    // poison: tell the consumer how many stages were issued
    __threadfence_block();
    *(volatile int*)&q_n = -1;
  } else if (warp == 1 && lane == 0) {
    // consumer: releases each stage as soon as it lands, until the producer is done
    int s = 0, consumed = 0; uint32_t ph = 0;
    for (;;) {
      if (consumed < *(volatile int*)&q_issued) {
        mbar_wait(&full[s], ph);
        mbar_arrive(&empty[s]);
        ++consumed;
        if (++s == p.stages) { s = 0; ph ^= 1; }
      } else if (*(volatile int*)&q_n == -1 && consumed == *(volatile int*)&q_issued) {
        break;
      }
    }
  }
  (void)q_id;
}

typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int K = atoi(argv[1]), N = atoi(argv[2]), g = atoi(argv[3]), kbc = atoi(argv[4]), stages = atoi(argv[5]),
      mode = atoi(argv[6]);
  int copies = argc > 7 ? atoi(argv[7]) : 0;
  const size_t wbytes = (size_t)K * N * 2;
  if (!copies) copies = (int)((600ull << 20) / wbytes) + 2;
  std::vector<char*> W(copies);
  for (auto& w : W) { cudaMalloc(&w, wbytes); cudaMemset(w, 1, wbytes); }
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc_t enc = (enc_t)fn;
  std::vector<CUtensorMap> tm(copies);
  for (int i = 0; i < copies; ++i) {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
    cuuint64_t str[1] = {(cuuint64_t)N * 2};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    if (enc(&tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W[i], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
      printf("encode failed\n"); return 1;
    }
  }
  const int iters = 60;
  int* claims; cudaMalloc(&claims, (iters + 8) * sizeof(int));
  const size_t smem = (size_t)stages * g * 8192 + 1024 + 256;
  cudaFuncSetAttribute(stream_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  P p{K, N, g, kbc, stages, mode, N / 64 / g, (K / 64 + kbc - 1) / kbc, nullptr, nullptr};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaMemset(claims, 0, (iters + 8) * sizeof(int));
  for (int i = 0; i < 3; ++i) { p.base = W[i % copies]; p.claim = claims + iters + i; stream_k<<<sms, 128, smem>>>(tm[i % copies], p); }
  cudaDeviceSynchronize();
  // single launches (cold in L2: a fresh copy each time), each timed alone
  float single = 0;
  for (int i = 0; i < 5; ++i) {
    int c = (3 + i) % copies;
    cudaMemset(claims, 0, sizeof(int));
    p.base = W[c]; p.claim = claims;
    cudaEventRecord(e0);
    stream_k<<<sms, 128, smem>>>(tm[c], p);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); single += ms / 5;
  }
  cudaMemset(claims, 0, (iters + 8) * sizeof(int));
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) {
    p.base = W[i % copies]; p.claim = claims + i;
    stream_k<<<sms, 128, smem>>>(tm[i % copies], p);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  printf("K=%5d N=%5d g=%2d kbc=%2d stages=%d mode=%d units=%4d: back-to-back %7.2f us (%5.0f GB/s), single %7.2f us (%5.0f GB/s) %s\n",
         K, N, g, kbc, stages, mode, p.n_groups * p.n_chunks, ms / iters * 1e3, wbytes / (ms / iters * 1e-3) / 1e9,
         single * 1e3, wbytes / (single * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  return 0;
}
