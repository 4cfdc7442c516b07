// wv_f32x2.cuh -- packed FP32x2 arithmetic (sm_100a FFMA2 / FADD2 / FMUL2).
//
// The all-pairs kernels are issue-bound: ~75% of their instructions are FP32
// ops on a pipe that stays ~67% busy.  Blackwell's packed f32x2 instructions
// do two lanes' worth of FP32 work per issue slot, and accept a scalar
// operand broadcast to both halves (SASS `Rn.F32`), so two QUERY POINTS are
// processed per instruction against the same (scalar) face data.  Measured
// on this pool: FFMA2 reaches the same 74 TFLOP/s FP32 ceiling as FFMA
// (tools/ffma2_probe.cu), while halving the issue slots spent on FP32.
#pragma once

#include <cstdint>

#include "wv_common.cuh"

namespace wv {

struct F2 {
  unsigned long long v;
};

__device__ __forceinline__ F2 f2(float lo, float hi) {
  F2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ F2 f2s(float s) { return f2(s, s); }  // folds to a .F32 broadcast
__device__ __forceinline__ void split(F2 a, float& lo, float& hi) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
}
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
  F2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
  F2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
  F2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
// (a.b) for packed 3-vectors
__device__ __forceinline__ F2 dot2(F2 ax, F2 ay, F2 az, F2 bx, F2 by, F2 bz) {
  return fma2(az, bz, fma2(ay, by, mul2(ax, bx)));
}
// scalar MUFU on each half
__device__ __forceinline__ F2 sqrt2(F2 a) {
  float l, h;
  split(a, l, h);
  return f2(sqrt_approx(l), sqrt_approx(h));
}
__device__ __forceinline__ F2 rsqrt2(F2 a) {
  float l, h;
  split(a, l, h);
  return f2(rsqrt_approx(l), rsqrt_approx(h));
}
__device__ __forceinline__ F2 rcp2(F2 a) {
  float l, h;
  split(a, l, h);
  return f2(rcp_approx(l), rcp_approx(h));
}

// 1/|x| per half: the exact backward's edge denominators are >= 0 in exact
// arithmetic but can round to small NEGATIVE values next to an edge; with the
// magnitude their ill-conditioning ratios stay >= 0, so a near-edge pair can
// never pass the ratio test with a negative (cancelled) ratio.  (The abs
// folds into MUFU.RCP's source operand.)
__device__ __forceinline__ F2 rcp2_abs(F2 a) {
  float l, h;
  split(a, l, h);
  return f2(rcp_approx(fabsf(l)), rcp_approx(fabsf(h)));
}

// NaN-propagating max (max.NaN.f32, ALU pipe): the exact backward screens a
// row run for ill-conditioned pairs with a running max of their reciprocal
// edge products; a NaN (a point ON a vertex) must poison the run, so the run
// is redone with per-lane masking
__device__ __forceinline__ float maxnan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
// NaN-propagating min (min.NaN.f32, ALU pipe): the trail backward's per-edge
// screen keeps the run's smallest edge denominator (a NaN poisons the run)
__device__ __forceinline__ float minnan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ F2 minnan2(F2 a, F2 b) {
  float al, ah, bl, bh;
  split(a, al, ah);
  split(b, bl, bh);
  return f2(minnan(al, bl), minnan(ah, bh));
}
__device__ __forceinline__ F2 maxnan2(F2 a, F2 b) {
  float al, ah, bl, bh;
  split(a, al, ah);
  split(b, bl, bh);
  return f2(maxnan(al, bl), maxnan(ah, bh));
}

}  // namespace wv
