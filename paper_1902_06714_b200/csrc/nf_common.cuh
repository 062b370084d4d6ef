// nf_common.cuh -- device helpers shared by the CUDA kernels of the hot path.
// Activation pairs (sigma, sigma') of P:108-109 / S:40, evaluated from
// z in numerically stable fp32 forms (reading R6 in DESIGN.md): sigma' is
// computed from z inside the forward epilogue and stashed, so no cancellation
// of the a(1-a) / 1-a^2 kind ever happens.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nf {

enum Act : int { ACT_SIGMOID = 0, ACT_TANH = 1, ACT_RELU = 2, ACT_GAUSSIAN = 3, ACT_STEP = 4 };

// a = sigma(z), s = sigma'(z).  Accurate libdevice expf/tanhf (no fast-math).
__device__ __forceinline__ void act_fwd(int kind, float z, float &a, float &s) {
  switch (kind) {
    case ACT_SIGMOID: {            // t = e^{-|z|}:  sigma = 1/(1+t) or t/(1+t);  sigma' = t/(1+t)^2
      const float t = expf(-fabsf(z));
      const float r = __frcp_rn(1.0f + t);  // == 1.0f / (1.0f + t), correctly rounded
      a = z >= 0.0f ? r : t * r;
      s = t * r * r;
      break;
    }
    case ACT_TANH: {               // t = e^{-2|z|}, e = expm1(-2|z|) = t - 1 (both accurate):
      const float t = expf(-2.0f * fabsf(z));    // tanh|z| = (1 - t)/(1 + t) = -e / (2 + e),
      const float e = expm1f(-2.0f * fabsf(z));  // sigma' = sech^2 z = 4t/(1+t)^2; 1 + t and
      const float r = __frcp_rn(1.0f + t);       // 2 + e carry no cancellation, and t keeps its
      a = copysignf(-e * __frcp_rn(2.0f + e), z);  // own precision when sigma' is tiny (reading
      s = 4.0f * t * r * r;                      // R6; a compact replacement of tanhf)
      break;
    }
    case ACT_RELU:                 // relu'(0) = 0 (reading R8)
      a = z > 0.0f ? z : 0.0f;
      s = z > 0.0f ? 1.0f : 0.0f;
      break;
    case ACT_GAUSSIAN: {           // e^{-z^2}, -2z e^{-z^2}
      const float e = expf(-z * z);
      a = e;
      s = -2.0f * z * e;
      break;
    }
    default:                       // step: [z>0], derivative 0
      a = z > 0.0f ? 1.0f : 0.0f;
      s = 0.0f;
      break;
  }
}

// Compile-time-activation forms (same arithmetic) for unrolled epilogue strips.
template <int K>
__device__ __forceinline__ void act_fwd_t(float z, float &a, float &s) { act_fwd(K, z, a, s); }
template <int K>
__device__ __forceinline__ float act_only_t(float z) {
  float a, s;
  act_fwd(K, z, a, s);
  return a;
}

__device__ __forceinline__ float act_only(int kind, float z) {
  switch (kind) {
    case ACT_SIGMOID: {
      const float t = expf(-fabsf(z));
      const float r = __frcp_rn(1.0f + t);  // == 1.0f / (1.0f + t), correctly rounded
      return z >= 0.0f ? r : t * r;
    }
    case ACT_TANH: {
      const float e = expm1f(-2.0f * fabsf(z));
      return copysignf(-e * __frcp_rn(2.0f + e), z);
    }
    case ACT_RELU: return z > 0.0f ? z : 0.0f;
    case ACT_GAUSSIAN: return expf(-z * z);
    default: return z > 0.0f ? 1.0f : 0.0f;
  }
}

// Blackwell packed fp32 FMA (FFMA2): d.{x,y} = a * b.{x,y} + d.{x,y}, a broadcast.  Two
// correctly rounded fp32 FMAs per instruction (same arithmetic as two fmaf calls).
__device__ __forceinline__ void ffma2(float2 &d, float a, float2 b) {
  unsigned long long dd, bb, aa;
  asm("mov.b64 %0, {%1, %2};" : "=l"(dd) : "f"(d.x), "f"(d.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(dd));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace nf
