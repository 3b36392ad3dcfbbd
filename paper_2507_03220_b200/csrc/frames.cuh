// GPU-direct LSV1 framing (reference protocol.py:6-25, 96-153).
//
// A run of request frames is copied to the device as raw bytes; payloads sit behind 30-byte
// headers, so their f32 values are not 4-byte aligned in general. K8 decodes every valid frame's
// little-endian f32 payload into a bf16 operand block (the GEMM's operand precision), reading
// aligned 32-bit words and funnel-shifting the misaligned ones; K9 encodes the reply stream on
// the device — each frame's 30-byte header (or a PASS_ERROR header + UTF-8 message) followed by
// its f32 payload written with 16-bit stores at the unaligned offset — so one D2H copy returns
// the whole stream (byte stores where an odd-length error message shifted the alignment).
// Both are HBM-bound copies (4 B read + 2 B written per decoded value; 4 B
// read + 4 B written per encoded value).
#pragma once
#include "ptx.cuh"

namespace ss {

struct FrameDesc {
  int64_t in_off;     // byte offset of the request payload in the device copy of the stream
  int64_t out_off;    // byte offset of the reply frame in the device reply stream
  int64_t x_off;      // element offset of the decoded bf16 rows [t, w]
  int64_t o_off;      // element offset of the f32 reply rows [t, out_w] from the GEMM
  int32_t t, w, out_w;
  int32_t msg_off, msg_len;  // PASS_ERROR frames: message bytes in the message blob
  int32_t is_err;
  uint8_t hdr[32];    // the reply header (30 bytes used)
};

// f32 at any byte offset: the two aligned words around it, funnel-shifted (the device copy of
// the stream is padded so the word after the last value is readable).
__device__ __forceinline__ float load_f32_unaligned(const uint8_t* base, int64_t o) {
  const int64_t a = o & ~int64_t(3);
  const uint32_t lo = __ldg(reinterpret_cast<const uint32_t*>(base + a));
  if ((o & 3) == 0) return __uint_as_float(lo);
  const uint32_t hi = __ldg(reinterpret_cast<const uint32_t*>(base + a + 4));
  return __uint_as_float(__funnelshift_r(lo, hi, 8 * (uint32_t)(o & 3)));
}

// blockIdx.y = frame; grid-stride over the frame's t*w values, 2 values per thread step.
__global__ void __launch_bounds__(256) frame_decode_kernel(const uint8_t* __restrict__ in,
                                                           const FrameDesc* __restrict__ fd,
                                                           __nv_bfloat16* __restrict__ fx) {
  const FrameDesc& f = fd[blockIdx.y];
  if (f.is_err) return;
  const int64_t n = (int64_t)f.t * f.w;
  __nv_bfloat16* dst = fx + f.x_off;
  for (int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i < n;
       i += 2 * (int64_t)gridDim.x * blockDim.x) {
    const float a = load_f32_unaligned(in, f.in_off + 4 * i);
    if (i + 1 < n) {
      const float b = load_f32_unaligned(in, f.in_off + 4 * i + 4);
      if ((f.x_off + i) % 2 == 0) {
        *reinterpret_cast<uint32_t*>(dst + i) = pack_bf16x2(a, b);
      } else {
        dst[i] = __float2bfloat16_rn(a);
        dst[i + 1] = __float2bfloat16_rn(b);
      }
    } else {
      dst[i] = __float2bfloat16_rn(a);
    }
  }
}

// blockIdx.y = frame; header / message bytes by block 0, payload values grid-stride.
__global__ void __launch_bounds__(256) frame_encode_kernel(uint8_t* __restrict__ out,
                                                           const FrameDesc* __restrict__ fd,
                                                           const float* __restrict__ fo,
                                                           const uint8_t* __restrict__ msgs) {
  const FrameDesc& f = fd[blockIdx.y];
  uint8_t* o = out + f.out_off;
  if (blockIdx.x == 0) {
    if (threadIdx.x < 30) o[threadIdx.x] = f.hdr[threadIdx.x];
    if (f.is_err)
      for (int i = threadIdx.x; i < f.msg_len; i += blockDim.x) o[30 + i] = msgs[f.msg_off + i];
  }
  if (f.is_err) return;
  const int64_t n = (int64_t)f.t * f.out_w;
  const float* src = fo + f.o_off;
  uint8_t* pay = o + 30;
  const bool even = ((f.out_off + 30) & 1) == 0;  // odd only after an odd-length error message
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = __float_as_uint(src[i]);
    if (even) {
      uint16_t* p = reinterpret_cast<uint16_t*>(pay + 4 * i);
      p[0] = (uint16_t)(v & 0xffffu);
      p[1] = (uint16_t)(v >> 16);
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) pay[4 * i + b] = (uint8_t)(v >> (8 * b));
    }
  }
}

}  // namespace ss
