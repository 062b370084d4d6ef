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

// e^x for x <= 0 through the SFU: ex2.approx(x log2 e).  Relative error <= 2^-21 + |x| 2^-24
// (the rounding of x log2 e), i.e. < 1e-6 for |x| < 16 -- far inside the 1e-4 parity bar, and
// ~20 dependent instructions shorter than libdevice expf (the epilogues are latency-bound).
__device__ __forceinline__ float exp_neg(float x) { return __expf(x); }

// 1/d for d in [1, 2] (d = 1 + t, t in [0, 1]): SFU rcp.approx + one Newton step, <= 1 ulp.
// Branch-free: __frcp_rn / '/' carry a special-case test and a slow-path CALL per use, whose
// reconvergence regions stop the compiler from interleaving the independent activation chains
// of an epilogue strip (measured: the tanh epilogue of a 4096x1024 tile GEMM 17 us -> see R6).
__device__ __forceinline__ float rcp_1p(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return fmaf(r, fmaf(-d, r, 1.0f), r);
}

// tanh |z| for |z| < 0.5: odd Taylor series to z^15 (truncation < 5e-8 relative).
__device__ __forceinline__ float tanh_small(float z) {
  const float q = z * z;
  float p = 929569.0f / 638512875.0f;
  p = fmaf(p, q, -21844.0f / 6081075.0f);
  p = fmaf(p, q, 1382.0f / 155925.0f);
  p = fmaf(p, q, -62.0f / 2835.0f);
  p = fmaf(p, q, 17.0f / 315.0f);
  p = fmaf(p, q, -2.0f / 15.0f);
  p = fmaf(p, q, 1.0f / 3.0f);
  return fmaf(-z * q, p, z);  // z - z^3 (1/3 - 2 z^2/15 + ...)
}

// a = sigma(z), s = sigma'(z), branch-free stable forms (no fast-math elsewhere).
__device__ __forceinline__ void act_fwd(int kind, float z, float &a, float &s) {
  switch (kind) {
    case ACT_SIGMOID: {            // t = e^{-|z|}:  sigma = 1/(1+t) or t/(1+t);  sigma' = t/(1+t)^2
      const float t = exp_neg(-fabsf(z));
      const float r = rcp_1p(1.0f + t);     // 1 / (1 + t) within 1 ulp
      a = z >= 0.0f ? r : t * r;
      s = t * r * r;
      break;
    }
    case ACT_TANH: {               // t = e^{-2|z|}: tanh|z| = (1 - t)/(1 + t) for |z| >= 1/2 (no
      const float t = exp_neg(-2.0f * fabsf(z));  // cancellation there), series below;
      const float r = rcp_1p(1.0f + t);           // sigma' = sech^2 z = 4t/(1+t)^2 from t itself
      a = fabsf(z) < 0.5f ? tanh_small(z) : copysignf((1.0f - t) * r, z);  // (exact when tiny)
      s = 4.0f * t * r * r;
      break;
    }
    case ACT_RELU:                 // relu'(0) = 0 (reading R8)
      a = z > 0.0f ? z : 0.0f;
      s = z > 0.0f ? 1.0f : 0.0f;
      break;
    case ACT_GAUSSIAN: {           // e^{-z^2}, -2z e^{-z^2}
      const float e = exp_neg(-z * z);
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
  float a, s;
  act_fwd(kind, z, a, s);
  return a;
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

// d += a * b elementwise on float pairs (one packed fp32x2 FMA)
__device__ __forceinline__ void ffma2v(float2 &d, float2 a, float2 b) {
  unsigned long long dd, aa, bb;
  asm("mov.b64 %0, {%1, %2};" : "=l"(dd) : "f"(d.x), "f"(d.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(dd));
}

// x rounded to the nearest TF32 value (10-bit mantissa, ties away: cvt.rna), an fp32 bit
// pattern whose low 13 mantissa bits are zero.  In NF_MATH_TF32 every tensor-core operand this
// library produces (hidden activations, deltas, the weight shadow) is stored this way, so the
// tensor core -- which reads fp32 bit patterns and truncates them to TF32 -- multiplies
// round-to-nearest operands (reading R13).
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Transposed copy of a 32 x 32 epilogue block (rows m0.., columns nc..; buf[r * 33 + c] holds the
// value stored at (m0 + r, nc + c)): thread `lane` writes row m0 + lane of T^T, i.e. one
// coalesced 128-B run T[nc + c][m0 .. m0 + 31] per column c.
__device__ __forceinline__ void store_t(float *T, int ldT, int m0, int mlim, int nc, int nlim, const float *buf,
                                        int lane) {
  if (m0 + lane >= mlim) return;
  const int cols = min(32, nlim - nc);
#pragma unroll 8
  for (int c = 0; c < cols; ++c) T[(int64_t)(nc + c) * ldT + m0 + lane] = buf[lane * 33 + c];
}

// Pre-split 3xTF32 (reading R13): every tensor-core operand x reaches the MMA as hi + lo.
//  * RN split (activations, weights): hi = tf32_rn(x) is stored as its own array, lo = tf32_rn(x - hi)
//    (x - hi exact in fp32, |lo| <= 2^-11 |x|): the dropped lo*lo is <= 2^-22 relative and of either
//    sign.
//  * truncation split (deltas): the tensor core reads x itself as hi, i.e. its truncated TF32 bits,
//    and lo = tf32_rn(x - trunc(x)) (|lo| < 2^-10 |x|, the sign of x).  Its lo*lo term alone would
//    be biased (same sign as the product), so every contraction pairs a truncation-split operand
//    with an RN-split one: the dropped lo_a*lo_b then has zero mean.
__device__ __forceinline__ float tf32_lo(float x) {  // truncation split
  return tf32_rn(x - __uint_as_float(__float_as_uint(x) & 0xffffe000u));
}
__device__ __forceinline__ float tf32_lo_rn(float x) { return tf32_rn(x - tf32_rn(x)); }  // RN split

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace nf
