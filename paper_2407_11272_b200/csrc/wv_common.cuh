// wv_common.cuh -- shared device helpers for the winding-number kernels
// (sm_100a only).  Record layouts, grid-node generation, mbarrier + TMA bulk
// copy wrappers (cp.async.bulk, SASS UBLKCP), approximate MUFU math.
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "windvox_b200 kernels target sm_100a only"
#endif

namespace wv {

constexpr double kPi = 3.14159265358979311599796346854;  // np.pi

// ---------------------------------------------------------------------------
// Packed face records (written once per mesh by wv_pack.cu, streamed into
// shared memory tile by tile by every forward CTA).
//
// ExactRecF32 (64 B): corners + the face normal N = (v1-v0)x(v2-v0) computed
//   in f64 without FMA contraction (so flipping a face negates N exactly),
//   and epsN = eps*|N|, the plane-distance threshold in alpha units
//   (alpha = N.(v0-q) = signed distance * |N|).  Degenerate faces (|N|==0 in
//   f64, dropped by the reference at winding.py:258-268) carry epsN = +inf.
struct __align__(16) ExactRecF32 {
  float4 v0e;  // v0.xyz, epsN
  float4 v1;   // v1.xyz, |v1-v0|^2/2
  float4 v2;   // v2.xyz, |v2-v1|^2/2
  float4 n;    // N.xyz,  |v0-v2|^2/2
};
static_assert(sizeof(ExactRecF32) == 64, "record size");

// SoftRecF32 (32 B): centroid c = v0 + (u+w)/3 and N = u x w, both computed
//   in f64 exactly as _kernels.py:139-155 does per pair (from the
//   f32-rounded corners), then rounded.  The centroid is kept as hi + lo:
//   d = c - q = (c_hi - q) + c_lo is then accurate to ~ulp(|d|) instead of
//   ulp(|c|), which matters at nodes next to a centroid (the dipole term
//   grows like 1/|d|^2).  The lo parts ride as bf16 (they are <= ulp(c)/2,
//   so 8 bits of them is ~1e-10 absolute) with K2 = (8e6 |N| |c_lo|)^2, the
//   "near" threshold on |d|^6: a pair with |d|^6 >= K2 changes by less than
//   2e-8 (in W) when c_lo is dropped, so far pairs skip the lo arithmetic.
struct __align__(16) SoftRecF32 {
  float4 c;   // c_hi.xyz, N.x
  float4 n;   // N.y, N.z, bits: bf16(c_lo.x) | bf16(c_lo.y) << 16,
              //           bits: bf16(c_lo.z) | bf16(K2) << 16
};
static_assert(sizeof(SoftRecF32) == 32, "record size");
__host__ __device__ __forceinline__ uint32_t bf16_bits(float x) {  // round to nearest even
  uint32_t b;
  memcpy(&b, &x, 4);
  b += 0x7fffu + ((b >> 16) & 1u);
  return b >> 16;
}
__device__ __forceinline__ float lo_x(const SoftRecF32& R) {
  return __uint_as_float(__float_as_uint(R.n.z) << 16);
}
__device__ __forceinline__ float lo_y(const SoftRecF32& R) {
  return __uint_as_float(__float_as_uint(R.n.z) & 0xffff0000u);
}
__device__ __forceinline__ float lo_z(const SoftRecF32& R) {
  return __uint_as_float(__float_as_uint(R.n.w) << 16);
}
__device__ __forceinline__ float near_k2(const SoftRecF32& R) {
  return __uint_as_float(__float_as_uint(R.n.w) & 0xffff0000u);
}

// SoftGradRecF32 (64 B): what the soft backward needs per face -- centroid
//   (hi + lo, as SoftRecF32), N = u x w, u = v1-v0, w = v2-v0 (all from the
//   f32-rounded corners in f64, then rounded).
struct __align__(16) SoftGradRecF32 {
  float4 c;  // c_hi.xyz, c_lo.x
  float4 n;  // N.xyz, c_lo.y
  float4 u;  // u.xyz, c_lo.z
  float4 w;  // w.xyz, K2 (SoftRecF32)
};
static_assert(sizeof(SoftGradRecF32) == 64, "record size");

// ExactGradRecF32 (48 B): one ACTIVE face of the exact backward -- corners
//   plus the net weights of its three directed edges (v0->v1, v1->v2,
//   v2->v0).  The exact d(Omega)/dv of a triangle is a sum of per-edge
//   Biot-Savart terms that cancel exactly between the two faces sharing an
//   interior edge, so only faces with a non-cancelling edge are packed.
struct __align__(16) ExactGradRecF32 {
  float4 a;  // v0.xyz, w01
  float4 b;  // v1.xyz, w12
  float4 c;  // v2.xyz, w20
  float4 u;  // squared edge lengths |v1-v0|^2, |v2-v1|^2, |v0-v2|^2 (from f64), 0
};
static_assert(sizeof(ExactGradRecF32) == 64, "record size");

// Edge-trail window (wv_trail.cu): K consecutive edges of a trail through
// the position-welded edge graph, positions p[0..K] (f32-rounded mesh),
// p[e].w = |p[e+1] - p[e]|^2 (from f64) for e < K, p[K].w = 0.
#ifndef WV_TRAIL_K
#define WV_TRAIL_K 4
#endif
constexpr int kTrailK = WV_TRAIL_K;
static_assert(kTrailK == 3 || kTrailK == 4, "trail windows of 3 or 4 edges");
struct __align__(16) TrailRecF32 {
  float4 p[kTrailK + 1];
};

// f64 twin of a trail window (the f64 mesh, no rounding)
struct __align__(16) TrailRecF64 {
  double p[kTrailK + 1][4];  // x, y, z, 0
};

struct __align__(16) ExactGradRecF64 {
  double v[9];
  double w[3];
  double pad[4];
};
static_assert(sizeof(ExactGradRecF64) == 128, "record size");

// SoftGradRecF64 (128 B): f64 twin for the parity backward.
struct __align__(16) SoftGradRecF64 {
  double c[3];
  double n[3];
  double u[3];
  double w[3];
  double pad[4];
};
static_assert(sizeof(SoftGradRecF64) == 128, "record size");

// ExactRecF64 (128 B): the reference's own per-face arrays (tri, nhat, pld,
//   winding.py:258-268) plus a dead flag for degenerate faces.
struct __align__(16) ExactRecF64 {
  double v[9];     // tri[f] row-major
  double nhat[3];
  double pld;
  double dead;     // 1.0 for |N| == 0 faces (skipped, never flagged)
  double pad[2];
};
static_assert(sizeof(ExactRecF64) == 128, "record size");

// SoftRecF64 (64 B): centroid and N in f64 (bit-identical to the reference's
//   per-pair expressions, which do not depend on q).
struct __align__(16) SoftRecF64 {
  double c[3];
  double n[3];
  double pad[2];
};
static_assert(sizeof(SoftRecF64) == 64, "record size");

// Header at the start of every packed buffer (64 B), so the kernels read eps
// from device memory and the device-resident path never syncs the host.
struct __align__(16) PackHeader {
  double eps;       // 1e-9 * bbox diagonal (winding.py:193-197)
  float eps_f32;    // float32(eps)  (winding.py:367)
  int32_t kind;     // 1 exact f32, 2 soft f32, 3 exact f64, 4 soft f64,
                    // 5 soft-grad f32, 6 soft-grad f64
  int64_t n_faces;
  int64_t n_live;   // non-degenerate faces (exact kinds)
  double pad[4];
};
static_assert(sizeof(PackHeader) == 64, "header size");

// Regular lattice (GridSpec): node (i,j,k) at lo + (hi-lo)*(i/(R-1)),
// midpoint for R == 1, flat index ((i*Ry)+j)*Rz+k (winding.py:118-140).
struct GridDesc {
  double lo[3];
  double hi[3];
  int64_t res[3];
};

__device__ __forceinline__ double axis_node(double lo, double hi, int64_t r,
                                            int64_t i) {
  // Same IEEE operations as numpy: lo + (hi - lo) * (i / (r - 1)).
  if (r == 1) return __dmul_rn(__dadd_rn(lo, hi), 0.5);
  const double frac = __ddiv_rn((double)i, (double)(r - 1));
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), frac));
}

__device__ __forceinline__ void grid_node(const GridDesc& g, int64_t n,
                                          double& x, double& y, double& z) {
  const int64_t ryz = g.res[1] * g.res[2];
  const int64_t i = n / ryz;
  const int64_t rem = n - i * ryz;
  const int64_t j = rem / g.res[2];
  const int64_t k = rem - j * g.res[2];
  x = axis_node(g.lo[0], g.hi[0], g.res[0], i);
  y = axis_node(g.lo[1], g.hi[1], g.res[1], j);
  z = axis_node(g.lo[2], g.hi[2], g.res[2], k);
}

// ---------------------------------------------------------------------------
// MUFU approximations (one SASS instruction each)
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// atan(t) for |t| <= 1: odd minimax polynomial t*P(t^2), 8 coefficients,
// fitted for RELATIVE error (max 1.0e-7 in exact arithmetic, 2.2e-7 when
// evaluated in fp32 Horner form), so the many tiny far-face terms carry no
// systematic bias.  Fit script: DESIGN.md section "atan polynomial".
__device__ __forceinline__ float atan_poly(float t, float s) {
  float p = -0.0046932753175497055f;
  p = fmaf(p, s, 0.024252397939562798f);
  p = fmaf(p, s, -0.05948638170957565f);
  p = fmaf(p, s, 0.09914291650056839f);
  p = fmaf(p, s, -0.14019480347633362f);
  p = fmaf(p, s, 0.19969724118709564f);
  p = fmaf(p, s, -0.33331990242004395f);
  p = fmaf(p, s, 0.9999998807907104f);
  return t * p;
}
__device__ __forceinline__ float atan_poly_coef(float s) {
  float p = -0.0046932753175497055f;
  p = fmaf(p, s, 0.024252397939562798f);
  p = fmaf(p, s, -0.05948638170957565f);
  p = fmaf(p, s, 0.09914291650056839f);
  p = fmaf(p, s, -0.14019480347633362f);
  p = fmaf(p, s, 0.19969724118709564f);
  p = fmaf(p, s, -0.33331990242004395f);
  p = fmaf(p, s, 0.9999998807907104f);
  return p;
}

// Full-range atan2(y, x) in units of radians, built on atan_poly; odd in y
// (so orientation flips negate exactly).  atan2(0, 0) = 0.
__device__ __forceinline__ float atan2_full(float y, float x) {
  const float ay = fabsf(y), ax = fabsf(x);
  if (ay == 0.0f && ax == 0.0f) return (x < 0.0f) ? copysignf((float)kPi, y) : y;
  const bool swap = ay > ax;
  const float num = swap ? x : y;
  const float den = swap ? y : x;
  const float t = __fdividef(num, den);
  const float phi = atan_poly(t, t * t);
  if (swap) return copysignf((float)(kPi / 2), y) - phi;
  if (x < 0.0f) return phi + copysignf((float)kPi, y);
  return phi;
}

// ---------------------------------------------------------------------------
// mbarrier + 1D TMA bulk copy (cp.async.bulk -> SASS UBLKCP)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar,
                                                      uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* smem_dst, const void* gmem_src,
                                             uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Face-tile ring without a producer warp.  TILE-record tiles of the packed
// face array stream into STAGES shared-memory slots by TMA bulk copy
// (cp.async.bulk, completion counted on the slot's mbarrier).  Every warp
// waits on full[s], computes, then bumps a CTA-scope counter; the LAST warp to
// finish a tile re-arms the slot and issues the copy of tile t+STAGES into it.
// Nobody ever waits for a slot to drain, so no warp spins: a dedicated
// producer warp polling an "empty" barrier measurably stole ~15% of the issue
// slots (profiles/README.md, round 1).
template <typename Rec, int TILE, int STAGES>
struct FaceRing {
  Rec tiles[STAGES][TILE];
  uint64_t full[STAGES];
  int done[STAGES];
};

template <typename Rec, int TILE, int STAGES>
__device__ __forceinline__ void ring_issue(FaceRing<Rec, TILE, STAGES>& r, int s,
                                           const Rec* __restrict__ recs, int64_t n_recs,
                                           int64_t t) {
  const int64_t first = t * TILE;
  const int64_t cnt = (n_recs - first) < TILE ? (n_recs - first) : TILE;
  const uint32_t bytes = (uint32_t)(cnt * (int64_t)sizeof(Rec));
  mbar_arrive_expect_tx(&r.full[s], bytes);
  tma_bulk_g2s(&r.tiles[s][0], recs + first, bytes, &r.full[s]);
}

// Initialise barriers and issue the first STAGES tiles of [t_begin, t_end).
template <typename Rec, int TILE, int STAGES>
__device__ __forceinline__ void ring_start(FaceRing<Rec, TILE, STAGES>& r,
                                           const Rec* __restrict__ recs, int64_t n_recs,
                                           int64_t t_begin, int64_t t_end) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&r.full[s], 1);
      r.done[s] = 0;
    }
    fence_barrier_init();
    for (int s = 0; s < STAGES && t_begin + s < t_end; ++s)
      ring_issue(r, s, recs, n_recs, t_begin + s);
  }
  __syncthreads();
}

// Called by lane 0 of every warp after it finished tile t (slot s).
template <typename Rec, int TILE, int STAGES>
__device__ __forceinline__ void ring_release(FaceRing<Rec, TILE, STAGES>& r, int s,
                                             int n_warps, const Rec* __restrict__ recs,
                                             int64_t n_recs, int64_t t, int64_t t_end) {
  __threadfence_block();  // this warp's reads of slot s precede the counter bump
  // monotonically increasing: round k of slot s takes the values
  // [k*n_warps, (k+1)*n_warps); round k+1 cannot start before round k's
  // last increment re-issued the slot, so rounds never interleave
  const int old = atomicAdd(&r.done[s], 1);
  if (old % n_warps == n_warps - 1) {  // last reader of this slot
    __threadfence_block();
    fence_proxy_async();  // generic-proxy reads before the async-proxy overwrite
    if (t + STAGES < t_end) ring_issue(r, s, recs, n_recs, t + STAGES);
  }
}

}  // namespace wv
