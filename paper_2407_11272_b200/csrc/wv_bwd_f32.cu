// wv_bwd_f32.cu -- FP32 backward kernels: per-face vertex gradients of the
// exact and soft winding numbers, reduced over query points.
//
// Mapping (the transpose of the forward): every thread OWNS one face; the CTA
// streams chunks of query points (coordinates + coefficient) through shared
// memory, so every warp reads the same point at the same time (broadcast
// LDS) and the per-point "coef == 0" skip of the reference
// (_kernels.py:182-184) is warp-uniform.  Generic sources keep fp32 partials
// per chunk; lattice sources (RowSrc) cut each chunk into k-row runs and keep
// a few running sums per run that are expanded into the face's corner sums
// once per run (flush_row) -- see ExactEdgeBwd / SoftBwd "Lattice-row form".
// The face's fp64 accumulators live in shared memory (5 CTAs per SM).
// No shuffles and no atomics: each (face block, point split) CTA writes its
// partials once, a fixed-order reduction sums the splits, and a CSR gather
// (wv_face_to_vertex) sums face corners into vertices -- bit-reproducible
// run to run, as the reference's chunk-ordered merge is (grad.py:113-127).
//
// Exact  (NEW, no reference kernel): d(Omega)/dv in its edge (Biot-Savart)
//   form, equal to the face-wise closed form of SURVEY.md A.4; only faces
//   with a non-cancelling edge are launched (see ExactEdgeBwd).
// Soft   (replaces _kernels.soft_grad_accum, _kernels.py:161-232):
//   dW/dv_k = [(G_k + N/3) / r^3 - S d / r^5] / (8 pi),  G_1 = w x d,
//   G_2 = d x u, G_0 = -G_1 - G_2; the N/3 and d terms are shared by the three
//   corners, so they are accumulated once per face.
// fp32 partials (per chunk or per run) are folded into fp64 accumulators.
#include <cmath>
#include <type_traits>

#include "wv_f32x2.cuh"
#include "wv_kernels.h"

namespace wv {

constexpr int kBwdThreads = 128;   // faces per CTA
#ifndef WV_BWD_CHUNK
#define WV_BWD_CHUNK 256
#endif
constexpr int kBwdChunk = WV_BWD_CHUNK;  // query points per shared-memory chunk
constexpr int kBwdMinBlocks = 5;  // CTAs per SM (launch bounds and split plan)
constexpr int kRowStep = 4;       // point pairs per basic block in the row loop
constexpr int kAxisMax = 1024;    // lattice axes up to this length use node tables

// Exact backward, edge form.  For a triangle seen from q, the variation of
// its solid angle is a boundary integral (the integrand (x-q)/|x-q|^3 is
// divergence-free), so d(Omega)/dv is a sum of per-edge Biot-Savart terms.
// For the directed edge P->Q with a = P-q, b = Q-q, m = a x b:
//   dW/dP = -m / (4 pi |a| (|a||b| + a.b)),  dW/dQ = -m / (4 pi |b| (|a||b| + a.b))
// (identical to the face-wise closed form of SURVEY.md A.4, oracle
// wvo_exact_grad_accum; stable: no differences of large terms).  Terms of an
// interior edge cancel exactly between its two faces, so each face carries
// the NET weight of its edges (0 for cancelled ones) and faces whose three
// weights vanish are not packed at all.  The sign and 1/(4 pi) are folded
// into coef_scale by the launcher.
// One ill-conditioned (face, point) pair of the exact backward in FP64,
// straight into the face's fp64 accumulators.  Used where the point lies
// close to an edge's segment ((|a|+|b|)^2 - |e|^2 < |e|^2 / 100): there the
// fp32 denominator cancels (relative error ~1e-7 |e|^2 / d).  Here
// |a||b| + a.b = |a x b|^2 / (|a||b| - a.b) has no cancellation, and the
// contributions bypass the fp32 run sums.  c already carries coef_scale and
// kCoefScale; corner k's three components are acc[3k .. 3k+2].
__device__ __noinline__ void exact_pair_f64(const ExactGradRecF32& R, double qx, double qy,
                                            double qz, double c, double (*acc)[kBwdThreads]) {
  if (c == 0.0) return;
  const double P[3][3] = {{(double)R.a.x - qx, (double)R.a.y - qy, (double)R.a.z - qz},
                          {(double)R.b.x - qx, (double)R.b.y - qy, (double)R.b.z - qz},
                          {(double)R.c.x - qx, (double)R.c.y - qy, (double)R.c.z - qz}};
  const double w[3] = {R.a.w, R.b.w, R.c.w};
  double len[3];
  for (int k = 0; k < 3; ++k) len[k] = sqrt(P[k][0] * P[k][0] + P[k][1] * P[k][1] + P[k][2] * P[k][2]);
  const int t = threadIdx.x;
  for (int e = 0; e < 3; ++e) {
    if (w[e] == 0.0) continue;
    const int i = e, j = (e + 1) % 3;
    const double* A = P[i];
    const double* B = P[j];
    const double m[3] = {A[1] * B[2] - A[2] * B[1], A[2] * B[0] - A[0] * B[2],
                         A[0] * B[1] - A[1] * B[0]};
    const double L = len[i] * len[j], ab = A[0] * B[0] + A[1] * B[1] + A[2] * B[2];
    const double mm = m[0] * m[0] + m[1] * m[1] + m[2] * m[2];
    const double den = (L - ab) > 0.0 ? mm / (L - ab) : L + ab;  // |a||b| + a.b
    if (!(den > 0.0) || !(len[i] > 0.0) || !(len[j] > 0.0)) continue;  // on the edge: flagged
    const double f = c * w[e] / (2.0 * den);  // c / d with d = 2 (|a||b| + a.b)
    for (int x = 0; x < 3; ++x) {
      acc[3 * i + x][t] += m[x] * (f / len[i]);
      acc[3 * j + x][t] += m[x] * (f / len[j]);
    }
  }
}

#ifndef WV_EDGE_PREFETCH
#define WV_EDGE_PREFETCH 0
#endif
struct ExactEdgeBwd {
  static constexpr bool kPrefetch = WV_EDGE_PREFETCH;  // next chunk's coefficients in registers
  using Rec = ExactGradRecF32;
  static constexpr int kFaces = 1;  // faces per thread (per record)
  static constexpr int kOut = 9;
  static constexpr bool kScaled = true;
  static constexpr bool kPairRuns = false;
  #ifndef WV_EDGE_STEP
#define WV_EDGE_STEP 4
#endif
#ifndef WV_EDGE_MINB
#define WV_EDGE_MINB 5
#endif
  static constexpr int kRowStep = WV_EDGE_STEP;
  __device__ __forceinline__ static void scale(Rec& R, float s) {
    R.a.x *= s; R.a.y *= s; R.a.z *= s;
    R.b.x *= s; R.b.y *= s; R.b.z *= s;
    R.c.x *= s; R.c.y *= s; R.c.z *= s;
    R.u.x *= s * s; R.u.y *= s * s; R.u.z *= s * s;
  }
  static constexpr int kMinBlocks = WV_EDGE_MINB;
  // -1/(4 pi) and the factor 2 of d = 2 (|a||b| + a.b) below
  static constexpr double kCoefScale = -2.0 / (4.0 * kPi);
  static constexpr int kAcc = 9;
  __device__ __forceinline__ static bool unit_weights(const Rec& R) {
    return R.a.w == 1.0f && R.b.w == 1.0f && R.c.w == 1.0f;
  }
  // Two query points per instruction (packed f32x2).  |a||b| + a.b =
  // ((|a|+|b|)^2 - |P-Q|^2) / 2  (a.b = (|a|^2+|b|^2-|a-b|^2)/2, a-b = P-Q):
  // no dot products, one FADD + one FFMA per edge, and the FFMA rounds
  // (|a|+|b|)^2 - U once.
  // a pair is ill-conditioned when some edge has d_e < |e|^2 / kIllRatio
  // (fp32 keeps ~1e-7 kIllRatio relative accuracy up to there: 1e-5)
  // (tested on the product of the three ratios |e|^2 / d_e; non-finite
  // counts as ill): its lanes take exact_pair_f64 instead
  static constexpr float kIllRatio = 100.0f;
  template <bool kUnit>
  __device__ __forceinline__ static uint32_t pair2(const Rec& R, F2 qx, F2 qy, F2 qz, F2 coef,
                                                   float, F2* g) {
    const F2 ax = sub2(f2s(R.a.x), qx), ay = sub2(f2s(R.a.y), qy), az = sub2(f2s(R.a.z), qz);
    const F2 bx = sub2(f2s(R.b.x), qx), by = sub2(f2s(R.b.y), qy), bz = sub2(f2s(R.b.z), qz);
    const F2 cx = sub2(f2s(R.c.x), qx), cy = sub2(f2s(R.c.y), qy), cz = sub2(f2s(R.c.z), qz);
    const F2 a2 = dot2(ax, ay, az, ax, ay, az);
    const F2 b2 = dot2(bx, by, bz, bx, by, bz);
    const F2 c2 = dot2(cx, cy, cz, cx, cy, cz);
    const F2 ia = rsqrt2(a2), ib = rsqrt2(b2), ic = rsqrt2(c2);
    const F2 lb = mul2(b2, ib), lc = mul2(c2, ic);
    const F2 s01 = fma2(a2, ia, lb), s12 = add2(lb, lc), s20 = fma2(a2, ia, lc);
    const F2 r01 = rcp2_abs(fma2(s01, s01, f2s(-R.u.x)));
    const F2 r12 = rcp2_abs(fma2(s12, s12, f2s(-R.u.y)));
    const F2 r20 = rcp2_abs(fma2(s20, s20, f2s(-R.u.z)));
    float q0, q1;
    split(mul2(mul2(r01, r12), mul2(r20, f2s(R.u.x * R.u.y * R.u.z))), q0, q1);
    const bool ill0 = !(q0 < kIllRatio), ill1 = !(q1 < kIllRatio);
    const F2 z2 = f2s(0.0f);
    const F2 t01 = (ill0 || ill1) ? z2 : mul2(kUnit ? coef : mul2(coef, f2s(R.a.w)), r01);
    const F2 t12 = (ill0 || ill1) ? z2 : mul2(kUnit ? coef : mul2(coef, f2s(R.b.w)), r12);
    const F2 t20 = (ill0 || ill1) ? z2 : mul2(kUnit ? coef : mul2(coef, f2s(R.c.w)), r20);
    // (a rare ill lane zeroes both lanes' fp32 terms; the caller redoes the
    // other lane in fp64 too, so no inf * 0 can reach the sums)
    // m01 = a x b, m12 = b x c, m20 = c x a
    const F2 m01x = sub2(mul2(ay, bz), mul2(az, by)), m01y = sub2(mul2(az, bx), mul2(ax, bz)),
             m01z = sub2(mul2(ax, by), mul2(ay, bx));
    const F2 m12x = sub2(mul2(by, cz), mul2(bz, cy)), m12y = sub2(mul2(bz, cx), mul2(bx, cz)),
             m12z = sub2(mul2(bx, cy), mul2(by, cx));
    const F2 m20x = sub2(mul2(cy, az), mul2(cz, ay)), m20y = sub2(mul2(cz, ax), mul2(cx, az)),
             m20z = sub2(mul2(cx, ay), mul2(cy, ax));
    const F2 s01a = mul2(t01, ia), s20a = mul2(t20, ia);  // v0 is P of 01, Q of 20
    const F2 s01b = mul2(t01, ib), s12b = mul2(t12, ib);  // v1 is Q of 01, P of 12
    const F2 s12c = mul2(t12, ic), s20c = mul2(t20, ic);  // v2 is Q of 12, P of 20
    g[0] = fma2(m20x, s20a, fma2(m01x, s01a, g[0]));
    g[1] = fma2(m20y, s20a, fma2(m01y, s01a, g[1]));
    g[2] = fma2(m20z, s20a, fma2(m01z, s01a, g[2]));
    g[3] = fma2(m12x, s12b, fma2(m01x, s01b, g[3]));
    g[4] = fma2(m12y, s12b, fma2(m01y, s01b, g[4]));
    g[5] = fma2(m12z, s12b, fma2(m01z, s01b, g[5]));
    g[6] = fma2(m20x, s20c, fma2(m12x, s12c, g[6]));
    g[7] = fma2(m20y, s20c, fma2(m12y, s12c, g[7]));
    g[8] = fma2(m20z, s20c, fma2(m12z, s12c, g[8]));
    return (ill0 || ill1) ? 3u : 0u;
  }
  // Lattice-row form (points of one k-row share x and y).
  //  * The edge moment is m = a x b = a x e with the edge vector e = Q - P
  //    (a x a = 0): with a's x/y fixed along the row, m's x/y components are
  //    affine in a_z and its z component is a row constant -- and a x e has
  //    no |a|/|e|-fold cancellation (a x b has, for far points).
  //  * So sum_q m(q) s(q) = K sum_q s(q) + E sum_q s(q) a_z(q) per (edge,
  //    corner): a pair only adds to 12 running sums (6 sums of s, 6 of
  //    s * corner z); the moments are formed once per row run (flush_row, in
  //    fp64, into the face's accumulators).
  //  * The three edge reciprocals share ONE MUFU.RCP: 1/d01 = R d12 d20 with
  //    R = 1/(d01 d12 d20) (products of O(|x|^2) terms: safe for coordinates
  //    within ~1e6 of the origin and points farther than ~1e-6 from an edge;
  //    R is clamped so the rest stays finite).
  // Per pair: ~36 FP32 lane-ops + 4 MUFU (was 53 + 6).
  static constexpr int kRowAcc = 12;
  struct Row {
    float a2, b2, c2;              // x/y parts of |corner - q|^2
    float k01x, k01y, m01z;        // m01 = a x e01: x = k01x - e01y a_z, y = k01y + e01x a_z
    float k12x, k12y, m12z;        // m12 = b x e12 (b_z)
    float k20x, k20y, m20z;        // m20 = c x e20 (c_z)
    float qx, qy;                  // the row (for exact_pair_f64)
  };
  __device__ __forceinline__ static Row row(const Rec& R, float qx, float qy) {
    const float ax = R.a.x - qx, ay = R.a.y - qy;
    const float bx = R.b.x - qx, by = R.b.y - qy;
    const float cx = R.c.x - qx, cy = R.c.y - qy;
    const float e01x = R.b.x - R.a.x, e01y = R.b.y - R.a.y, e01z = R.b.z - R.a.z;
    const float e12x = R.c.x - R.b.x, e12y = R.c.y - R.b.y, e12z = R.c.z - R.b.z;
    const float e20x = R.a.x - R.c.x, e20y = R.a.y - R.c.y, e20z = R.a.z - R.c.z;
    Row w;
    w.a2 = fmaf(ay, ay, ax * ax);
    w.b2 = fmaf(by, by, bx * bx);
    w.c2 = fmaf(cy, cy, cx * cx);
    w.k01x = ay * e01z;
    w.k01y = -(ax * e01z);
    w.m01z = fmaf(ax, e01y, -(ay * e01x));
    w.k12x = by * e12z;
    w.k12y = -(bx * e12z);
    w.m12z = fmaf(bx, e12y, -(by * e12x));
    w.k20x = cy * e20z;
    w.k20y = -(cx * e20z);
    w.m20z = fmaf(cx, e20y, -(cy * e20x));
    w.qx = qx;
    w.qy = qy;
    return w;
  }
  // kMask = false (hot path): no masking; the pair's reciprocal edge product
  //   rr = 1/(d01 d12 d20) goes to *mr, whose running max over the run (ALU
  //   pipe, NaN-propagating) times |e01|^2 |e12|^2 |e20|^2 is the run's worst
  //   ill-conditioning ratio product (ill_run); a run that reaches kIllRatio
  //   is discarded and redone with kMask = true.  (Each pair's fp32 terms
  //   carry a relative error ~1e-7 x its ratio, so the worst pair bounds the
  //   run sum's relative error.)
  // kMask = true: ill lanes contribute nothing here (bits returned; the
  //   caller adds them with exact_pair_f64).
  template <bool kUnit, bool kMask = true>
  __device__ __forceinline__ static uint32_t pair_row2(const Rec& R, const Row& w, F2 qz, F2 coef,
                                                       float, F2* z, F2* mr = nullptr) {
    const F2 az = sub2(f2s(R.a.z), qz), bz = sub2(f2s(R.b.z), qz), cz = sub2(f2s(R.c.z), qz);
    const F2 a2 = fma2(az, az, f2s(w.a2));
    const F2 b2 = fma2(bz, bz, f2s(w.b2));
    const F2 c2 = fma2(cz, cz, f2s(w.c2));
    const F2 ia = rsqrt2(a2), ib = rsqrt2(b2), ic = rsqrt2(c2);
    const F2 lb = mul2(b2, ib), lc = mul2(c2, ic);
    const F2 s01 = fma2(a2, ia, lb), s12 = add2(lb, lc), s20 = fma2(a2, ia, lc);
    const F2 d01 = fma2(s01, s01, f2s(-R.u.x));
    const F2 d12 = fma2(s12, s12, f2s(-R.u.y));
    const F2 d20 = fma2(s20, s20, f2s(-R.u.z));
    const F2 p12 = mul2(d12, d20);
    const F2 rr = rcp2_abs(mul2(d01, p12));
    // ill-conditioned lanes (some d_e < |e|^2 / kIllRatio, or a non-finite
    // reciprocal) leave the fp32 sums: cr = 0 here, exact_pair_f64 later
    bool ill0 = false, ill1 = false;
    F2 cr;  // coef / (d01 d12 d20)
    if constexpr (kMask) {
      const F2 ru = mul2(rr, f2s(R.u.x * R.u.y * R.u.z));
      float ru0, ru1;
      split(ru, ru0, ru1);
      ill0 = !(ru0 < kIllRatio);
      ill1 = !(ru1 < kIllRatio);
      float r0, r1;
      split(mul2(coef, rr), r0, r1);
      cr = f2(ill0 ? 0.0f : r0, ill1 ? 0.0f : r1);
    } else {
      *mr = rr;  // (>= 0: rcp2_abs; inf / NaN propagate through maxnan)
      cr = mul2(coef, rr);
    }
    const F2 q0 = mul2(cr, d01);
    const F2 t01 = mul2(kUnit ? cr : mul2(cr, f2s(R.a.w)), p12);
    const F2 t12 = mul2(kUnit ? q0 : mul2(q0, f2s(R.b.w)), d20);
    const F2 t20 = mul2(kUnit ? q0 : mul2(q0, f2s(R.c.w)), d12);
    // s_eP = t_e / |P - q|: each sum is one fma, t_e (or t_e * the edge's
    // corner z) times 1/|P - q|
    const F2 u01 = mul2(t01, az), u12 = mul2(t12, bz), u20 = mul2(t20, cz);
    z[0] = fma2(t01, ia, z[0]);
    z[1] = fma2(u01, ia, z[1]);
    z[2] = fma2(t20, ia, z[2]);
    z[3] = fma2(u20, ia, z[3]);
    z[4] = fma2(t01, ib, z[4]);
    z[5] = fma2(u01, ib, z[5]);
    z[6] = fma2(t12, ib, z[6]);
    z[7] = fma2(u12, ib, z[7]);
    z[8] = fma2(t12, ic, z[8]);
    z[9] = fma2(u12, ic, z[9]);
    z[10] = fma2(t20, ic, z[10]);
    z[11] = fma2(u20, ic, z[11]);
    return (ill0 ? 1u : 0u) | (ill1 ? 2u : 0u);
  }
  template <bool kUnit, int N>
  __device__ __forceinline__ static void step_row(const Rec& R, const Row& w, const float4* zc,
                                                  float eps2, F2* z, F2* mr) {
    F2 ru[N];
#pragma unroll
    for (int u = 0; u < N; ++u)
      pair_row2<kUnit, false>(R, w, f2(zc[u].x, zc[u].y), f2(zc[u].z, zc[u].w), eps2, z, &ru[u]);
    // pairwise max (short dependency chain), then one max into the run's
#pragma unroll
    for (int h = 1; h < N; h *= 2)
#pragma unroll
      for (int u = 0; u + h < N; u += 2 * h) ru[u] = maxnan2(ru[u], ru[u + h]);
    *mr = maxnan2(*mr, ru[0]);
  }
  // the run's worst ratio product reached kIllRatio (or is NaN)
  __device__ __forceinline__ static bool ill_run(const Rec& R, F2 mr) {
    float m0, m1;
    split(mr, m0, m1);
    return !(maxnan(m0, m1) * (R.u.x * R.u.y * R.u.z) < kIllRatio);
  }
  __device__ __forceinline__ static void rare_pair(const Rec& R, float qx, float qy, float qz,
                                                   float c, double (*acc)[kBwdThreads],
                                                   uint32_t = 3u) {
    exact_pair_f64(R, qx, qy, qz, c, acc);
  }
  // a run [j, e) holding an ill-conditioned pair, redone: fp32 sums without
  // the ill lanes, the ill lanes in fp64 (out of line: rare)
  template <bool kUnit>
  __device__ __noinline__ static void redo_run(const Rec& R, const Row& w, const float4* zcs,
                                               int j, int e, float eps2, F2* z,
                                               double (*acc)[kBwdThreads]) {
    for (int i = 0; i < kRowAcc; ++i) z[i] = f2(0.0f, 0.0f);
    for (; j < e; ++j) {
      const float4 zc = zcs[j];
      if (zc.z == 0.0f && zc.w == 0.0f) continue;
      const uint32_t ill = pair_row2<kUnit, true>(R, w, f2(zc.x, zc.y), f2(zc.z, zc.w), eps2, z);
      if (ill & 1u) exact_pair_f64(R, w.qx, w.qy, zc.x, zc.z, acc);
      if (ill & 2u) exact_pair_f64(R, w.qx, w.qy, zc.y, zc.w, acc);
    }
  }
  // sum_q m s for every (edge, corner) from the run's sums, into the face's
  // fp64 accumulators (acc[j][thread], j = corner * 3 + axis)
  // kW: the sums were taken without edge weights (strip pairs); weight them
  // here (sums 0,1,4,5: edge 01; 6-9: edge 12; 2,3,10,11: edge 20)
  template <bool kW = false>
  __device__ __forceinline__ static void flush_row(const Rec& R, const Row& w, const F2* z,
                                                   double (*acc)[kBwdThreads]) {
    double S[kRowAcc];
#pragma unroll
    for (int j = 0; j < kRowAcc; ++j) {
      float lo, hi;
      split(z[j], lo, hi);
      S[j] = (double)lo + (double)hi;
      if constexpr (kW) {
        const int e = (j == 0 || j == 1 || j == 4 || j == 5) ? 0 : (j >= 6 && j <= 9) ? 1 : 2;
        S[j] *= (double)(e == 0 ? R.a.w : e == 1 ? R.b.w : R.c.w);
      }
    }
    const double e01x = (double)(R.b.x - R.a.x), e01y = (double)(R.b.y - R.a.y);
    const double e12x = (double)(R.c.x - R.b.x), e12y = (double)(R.c.y - R.b.y);
    const double e20x = (double)(R.a.x - R.c.x), e20y = (double)(R.a.y - R.c.y);
    const int t = threadIdx.x;
    // corner a: edges 01 (a_z sums S0,S1) and 20 (c_z sums S2,S3)
    acc[0][t] += w.k01x * S[0] - e01y * S[1] + w.k20x * S[2] - e20y * S[3];
    acc[1][t] += w.k01y * S[0] + e01x * S[1] + w.k20y * S[2] + e20x * S[3];
    acc[2][t] += w.m01z * S[0] + w.m20z * S[2];
    // corner b: edges 01 (S4,S5) and 12 (b_z sums S6,S7)
    acc[3][t] += w.k01x * S[4] - e01y * S[5] + w.k12x * S[6] - e12y * S[7];
    acc[4][t] += w.k01y * S[4] + e01x * S[5] + w.k12y * S[6] + e12x * S[7];
    acc[5][t] += w.m01z * S[4] + w.m12z * S[6];
    // corner c: edges 12 (S8,S9) and 20 (S10,S11)
    acc[6][t] += w.k12x * S[8] - e12y * S[9] + w.k20x * S[10] - e20y * S[11];
    acc[7][t] += w.k12y * S[8] + e12x * S[9] + w.k20y * S[10] + e20x * S[11];
    acc[8][t] += w.m12z * S[8] + w.m20z * S[10];
  }
  __device__ __forceinline__ static void finish(const Rec&, const double* acc, double* out9) {
    for (int j = 0; j < 9; ++j) out9[j] = acc[j];
  }
};

struct SoftBwd {
  static constexpr bool kPrefetch = false;  // next chunk's coefficients in registers
  using Rec = SoftGradRecF32;
  static constexpr int kFaces = 1;
  static constexpr int kOut = 9;
  static constexpr bool kScaled = false;
  static constexpr bool kPairRuns = false;
  static constexpr int kRowStep = wv::kRowStep;
  __device__ __forceinline__ static void scale(Rec&, float) {}
  static constexpr int kMinBlocks = kBwdMinBlocks;
  static constexpr double kCoefScale = 1.0 / (8.0 * kPi);
  static constexpr int kAcc = 10;  // acc1(3) acc2(3) T(1) D(3)
  __device__ __forceinline__ static bool unit_weights(const Rec&) { return true; }
  template <bool kUnit>
  __device__ __forceinline__ static uint32_t pair2(const Rec& R, F2 qx, F2 qy, F2 qz, F2 coef,
                                                   float eps2, F2* g) {
    // d = (c_hi - q) + c_lo (SoftGradRecF32)
    const F2 dx = add2(sub2(f2s(R.c.x), qx), f2s(R.c.w));
    const F2 dy = add2(sub2(f2s(R.c.y), qy), f2s(R.n.w));
    const F2 dz = add2(sub2(f2s(R.c.z), qz), f2s(R.u.w));
    const F2 r2 = dot2(dx, dy, dz, dx, dy, dz);
    const F2 rs = rsqrt2(r2);
    const F2 S = fma2(f2s(R.n.z), dz, fma2(f2s(R.n.y), dy, mul2(f2s(R.n.x), dx)));
    const F2 rs2 = mul2(rs, rs);
    float r2l, r2h, cl, ch;
    split(r2, r2l, r2h);
    split(mul2(mul2(coef, rs2), rs), cl, ch);
    // r < eps: that face is skipped for that point (_kernels.py:203-204)
    const F2 c3 = f2(r2l < eps2 ? 0.0f : cl, r2h < eps2 ? 0.0f : ch);
    const F2 c5 = mul2(mul2(c3, S), rs2);
    // G1 = w x d, G2 = d x u
    const F2 g1x = sub2(mul2(f2s(R.w.y), dz), mul2(f2s(R.w.z), dy));
    const F2 g1y = sub2(mul2(f2s(R.w.z), dx), mul2(f2s(R.w.x), dz));
    const F2 g1z = sub2(mul2(f2s(R.w.x), dy), mul2(f2s(R.w.y), dx));
    const F2 g2x = sub2(mul2(dy, f2s(R.u.z)), mul2(dz, f2s(R.u.y)));
    const F2 g2y = sub2(mul2(dz, f2s(R.u.x)), mul2(dx, f2s(R.u.z)));
    const F2 g2z = sub2(mul2(dx, f2s(R.u.y)), mul2(dy, f2s(R.u.x)));
    g[0] = fma2(c3, g1x, g[0]);
    g[1] = fma2(c3, g1y, g[1]);
    g[2] = fma2(c3, g1z, g[2]);
    g[3] = fma2(c3, g2x, g[3]);
    g[4] = fma2(c3, g2y, g[4]);
    g[5] = fma2(c3, g2z, g[5]);
    g[6] = add2(g[6], c3);
    g[7] = fma2(c5, dx, g[7]);
    g[8] = fma2(c5, dy, g[8]);
    g[9] = fma2(c5, dz, g[9]);
    return 0u;
  }
  // Lattice-row form: d = c - q has row-constant x/y parts, so r^2 and S take
  // one op each per pair, and since G1 = w x d and G2 = d x u are affine in
  // d_z, sum_q c3 G = K sum c3 + E sum c3 d_z: a pair only adds to 4 running
  // sums (c3, c3 d_z, c5, c5 d_z); flush_row forms the 10 face sums per run.
  // Per pair: 12 FP32 lane-ops + 1 MUFU (was 22 + 1).
  static constexpr int kRowAcc = 4;
  // Row: d's x/y parts from c_hi + c_lo (dx, dy: the flush, and r2c, sc: the
  // near steps) and from c_hi alone (r2, s: the far steps, which drop c_lo in
  // the nonlinear factors c3, c5 -- < 2e-8 relative change beyond the
  // face's near threshold K2 on |d|^6, SoftRecF32).  The run sums of c*dz
  // always use dz from c_hi; flush_row adds c_lo.z * (sum c).
  struct Row {
    float dxh, dyh, r2, s;  // d's x/y from c_hi; r^2, S x/y parts from c_hi
    float dx, dy;           // d's x/y with c_lo (the flush's moments)
  };
  __device__ __forceinline__ static Row row(const Rec& R, float qx, float qy) {
    Row w;
    w.dxh = R.c.x - qx;
    w.dyh = R.c.y - qy;
    w.r2 = fmaf(w.dyh, w.dyh, w.dxh * w.dxh);
    w.s = fmaf(R.n.y, w.dyh, R.n.x * w.dxh);
    w.dx = w.dxh + R.c.w;
    w.dy = w.dyh + R.n.w;
    return w;
  }
  // one point pair with the corrected d (near steps)
  template <bool kUnit>
  __device__ __forceinline__ static void pair_row2(const Rec& R, const Row& w, F2 qz, F2 coef,
                                                   float eps2, F2* z) {
    const float dx = w.dx, dy = w.dy;  // + c_lo (c3, c5)
    const float r2c = fmaf(dy, dy, dx * dx), sc = fmaf(R.n.y, dy, R.n.x * dx);
    const F2 dz = sub2(f2s(R.c.z), qz);            // c_hi (run sums)
    const F2 dzc = add2(dz, f2s(R.u.w));
    const F2 r2 = fma2(dzc, dzc, f2s(r2c));
    const F2 rs = rsqrt2(r2);
    const F2 S = fma2(f2s(R.n.z), dzc, f2s(sc));
    float r2l, r2h, cl, ch;
    split(r2, r2l, r2h);
    const F2 rs2 = mul2(rs, rs);
    split(mul2(mul2(coef, rs2), rs), cl, ch);
    // r < eps: that face is skipped for that point (_kernels.py:203-204)
    const F2 c3 = f2(r2l < eps2 ? 0.0f : cl, r2h < eps2 ? 0.0f : ch);
    const F2 c5 = mul2(mul2(c3, S), rs2);
    z[0] = add2(z[0], c3);
    z[1] = fma2(c3, dz, z[1]);
    z[2] = add2(z[2], c5);
    z[3] = fma2(c5, dz, z[3]);
  }
  // N point pairs; the r < eps test is done once on the minimum r^2 of the
  // step (nearly always passes), so the common path has no per-lane selects
  __device__ __forceinline__ static void rare_pair(const Rec&, float, float, float, float,
                                                   double (*)[kBwdThreads], uint32_t = 0u) {}
  template <bool kUnit, class W>
  __device__ __forceinline__ static void redo_run(const Rec&, const W&, const float4*, int, int,
                                                  float, F2*, double (*)[kBwdThreads]) {}
  __device__ __forceinline__ static bool ill_run(const Rec&, F2) { return false; }
  template <bool kUnit, int N>
  __device__ __forceinline__ static void step_row(const Rec& R, const Row& w, const float4* zc,
                                                  float eps2, F2* z, F2*) {
    F2 dz[N], r2[N];
    float m = __int_as_float(0x7f800000);
#pragma unroll
    for (int u = 0; u < N; ++u) {
      dz[u] = sub2(f2s(R.c.z), f2(zc[u].x, zc[u].y));
      r2[u] = fma2(dz[u], dz[u], f2s(w.r2));
      float l, h;
      split(r2[u], l, h);
      m = fminf(m, fminf(l, h));
    }
    // some point of the step near this face's centroid (or on it)
    if (m < eps2 || m * m * m < R.w.w) {
#pragma unroll
      for (int u = 0; u < N; ++u)
        pair_row2<kUnit>(R, w, f2(zc[u].x, zc[u].y), f2(zc[u].z, zc[u].w), eps2, z);
      return;
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const F2 rs = rsqrt2(r2[u]);
      const F2 S = fma2(f2s(R.n.z), dz[u], f2s(w.s));
      const F2 rs2 = mul2(rs, rs);
      const F2 c3 = mul2(mul2(f2(zc[u].z, zc[u].w), rs2), rs);
      const F2 c5 = mul2(mul2(c3, S), rs2);
      z[0] = add2(z[0], c3);
      z[1] = fma2(c3, dz[u], z[1]);
      z[2] = add2(z[2], c5);
      z[3] = fma2(c5, dz[u], z[3]);
    }
  }
  __device__ __forceinline__ static void flush_row(const Rec& R, const Row& w, const F2* z,
                                                   double (*acc)[kBwdThreads]) {
    // the run sums of c * dz used dz from c_hi: add c_lo.z * sum c
    const F2 zz[kRowAcc] = {z[0], fma2(z[0], f2s(R.u.w), z[1]), z[2],
                            fma2(z[2], f2s(R.u.w), z[3])};
    double S[kRowAcc];
#pragma unroll
    for (int j = 0; j < kRowAcc; ++j) {
      float lo, hi;
      split(zz[j], lo, hi);
      S[j] = (double)lo + (double)hi;
    }
    const double C = S[0], A = S[1], D = S[2], E = S[3];
    const double dx = w.dx, dy = w.dy;
    const int t = threadIdx.x;
    // G1 = w x d, G2 = d x u with d = (dx, dy, dz): sum c3 G = row part * C + dz part * A
    acc[0][t] += (double)R.w.y * A - (double)R.w.z * dy * C;
    acc[1][t] += (double)R.w.z * dx * C - (double)R.w.x * A;
    acc[2][t] += ((double)R.w.x * dy - (double)R.w.y * dx) * C;
    acc[3][t] += dy * (double)R.u.z * C - (double)R.u.y * A;
    acc[4][t] += (double)R.u.x * A - dx * (double)R.u.z * C;
    acc[5][t] += (dx * (double)R.u.y - dy * (double)R.u.x) * C;
    acc[6][t] += C;
    acc[7][t] += dx * D;
    acc[8][t] += dy * D;
    acc[9][t] += E;
  }
  __device__ __forceinline__ static void finish(const Rec& R, const double* a, double* out9) {
    const double t = a[6] / 3.0;
    const double cx = t * R.n.x - a[7], cy = t * R.n.y - a[8], cz = t * R.n.z - a[9];
    out9[0] = -a[0] - a[3] + cx;
    out9[1] = -a[1] - a[4] + cy;
    out9[2] = -a[2] - a[5] + cz;
    out9[3] = a[0] + cx;
    out9[4] = a[1] + cy;
    out9[5] = a[2] + cz;
    out9[6] = a[3] + cx;
    out9[7] = a[4] + cy;
    out9[8] = a[5] + cz;
  }
};

// Soft backward with TWO faces per thread (the C4 meshes): the point loads,
// loop control and on-centroid test of a step are shared by both faces, and
// their two independent dependency chains interleave.  Faces 2r and 2r+1 form
// record r (so the face count must be even); their corner sums are the 18
// consecutive doubles of faces 2r, 2r+1 in the output.
struct SoftPairRec {
  SoftGradRecF32 f[2];
};
struct SoftBwdPair {
  static constexpr bool kPrefetch = false;  // next chunk's coefficients in registers
  using One = SoftBwd;
  using Rec = SoftPairRec;
  static constexpr int kFaces = 2;
  static constexpr int kOut = 18;
#ifndef WV_SOFT_PAIR_STEP
#define WV_SOFT_PAIR_STEP 4
#endif
#ifndef WV_SOFT_PAIR_MINB
#define WV_SOFT_PAIR_MINB 4  // two faces' state: up to 128 registers
#endif
  static constexpr int kRowStep = WV_SOFT_PAIR_STEP;
  static constexpr bool kScaled = false;
  static constexpr bool kPairRuns = false;
  __device__ __forceinline__ static void scale(Rec&, float) {}
  static constexpr int kMinBlocks = WV_SOFT_PAIR_MINB;
  static constexpr double kCoefScale = One::kCoefScale;
  static constexpr int kAcc = 2 * One::kAcc;
  static constexpr int kRowAcc = 2 * One::kRowAcc;
  __device__ __forceinline__ static bool unit_weights(const Rec&) { return true; }
  template <bool kUnit>
  __device__ __forceinline__ static uint32_t pair2(const Rec& R, F2 qx, F2 qy, F2 qz, F2 coef,
                                                   float eps2, F2* g) {
    One::pair2<kUnit>(R.f[0], qx, qy, qz, coef, eps2, g);
    One::pair2<kUnit>(R.f[1], qx, qy, qz, coef, eps2, g + One::kAcc);
    return 0u;
  }
  __device__ __forceinline__ static void rare_pair(const Rec&, float, float, float, float,
                                                   double (*)[kBwdThreads], uint32_t = 0u) {}
  template <bool kUnit, class W>
  __device__ __forceinline__ static void redo_run(const Rec&, const W&, const float4*, int, int,
                                                  float, F2*, double (*)[kBwdThreads]) {}
  __device__ __forceinline__ static bool ill_run(const Rec&, F2) { return false; }
  struct Row {
    One::Row r[2];
  };
  __device__ __forceinline__ static Row row(const Rec& R, float qx, float qy) {
    Row w;
    w.r[0] = One::row(R.f[0], qx, qy);
    w.r[1] = One::row(R.f[1], qx, qy);
    return w;
  }
  template <bool kUnit>
  __device__ __forceinline__ static void pair_row2(const Rec& R, const Row& w, F2 qz, F2 coef,
                                                   float eps2, F2* z) {
    One::pair_row2<kUnit>(R.f[0], w.r[0], qz, coef, eps2, z);
    One::pair_row2<kUnit>(R.f[1], w.r[1], qz, coef, eps2, z + One::kRowAcc);
  }
  // both faces' r^2 first, one on-centroid test for the whole step
  template <bool kUnit, int N>
  __device__ __forceinline__ static void step_row(const Rec& R, const Row& w, const float4* zc,
                                                  float eps2, F2* z, F2*) {
    F2 dz[2][N], r2[2][N];
    float m = __int_as_float(0x7f800000);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
#pragma unroll
      for (int u = 0; u < N; ++u) {
        dz[k][u] = sub2(f2s(R.f[k].c.z), f2(zc[u].x, zc[u].y));
        r2[k][u] = fma2(dz[k][u], dz[k][u], f2s(w.r[k].r2));
        float l, h;
        split(r2[k][u], l, h);
        m = fminf(m, fminf(l, h));
      }
    }
    if (m < eps2 || m * m * m < fmaxf(R.f[0].w.w, R.f[1].w.w)) {
#pragma unroll
      for (int u = 0; u < N; ++u)
        pair_row2<kUnit>(R, w, f2(zc[u].x, zc[u].y), f2(zc[u].z, zc[u].w), eps2, z);
      return;
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        F2* zk = z + k * One::kRowAcc;
        const F2 rs = rsqrt2(r2[k][u]);
        const F2 S = fma2(f2s(R.f[k].n.z), dz[k][u], f2s(w.r[k].s));
        const F2 rs2 = mul2(rs, rs);
        const F2 c3 = mul2(mul2(f2(zc[u].z, zc[u].w), rs2), rs);
        const F2 c5 = mul2(mul2(c3, S), rs2);
        zk[0] = add2(zk[0], c3);
        zk[1] = fma2(c3, dz[k][u], zk[1]);
        zk[2] = add2(zk[2], c5);
        zk[3] = fma2(c5, dz[k][u], zk[3]);
      }
    }
  }
  __device__ __forceinline__ static void flush_row(const Rec& R, const Row& w, const F2* z,
                                                   double (*acc)[kBwdThreads]) {
    One::flush_row(R.f[0], w.r[0], z, acc);
    One::flush_row(R.f[1], w.r[1], z + One::kRowAcc, acc + One::kAcc);
  }
  __device__ __forceinline__ static void finish(const Rec& R, const double* a, double* out) {
    One::finish(R.f[0], a, out);
    One::finish(R.f[1], a + One::kAcc, out + 9);
  }
};

// Exact backward over STRIP PAIRS: a record holds two faces F1 = (A, B, C)
// and F2 = (B', C', D) whose corners are in strip-window order (see
// wv_strip.cu), with B', C' at the positions of B, C (welded by position).
// Per point the pair needs 4 corner distances instead of 6, 5 edge
// denominators instead of 6, and the shared edge BC's four run sums serve
// both faces (the Biot-Savart term of an edge depends only on its end
// points): ~32 lane-ops and 3 MUFU per face and pair instead of ~38 and 4.
// The run sums are taken WITHOUT edge weights, which are applied once per run
// in the fp64 flush (F1's BC weight and F2's may differ).  A record whose
// positions do not match bitwise (welds broken by a morph step) evaluates
// its two faces one after the other with the single-face row code.
struct ExactPairRec {
  ExactGradRecF32 f[2];
};
struct ExactEdgeBwdPair {
  static constexpr bool kPrefetch = true;  // next chunk's coefficients in registers
  using One = ExactEdgeBwd;
  using Rec = ExactPairRec;
  static constexpr int kFaces = 2;
  static constexpr int kOut = 18;
  static constexpr bool kScaled = true;
  static constexpr bool kPairRuns = true;
#ifndef WV_PAIR_STEP
#define WV_PAIR_STEP 8  // c3s: 62.0 ms (8) vs 63.9 (6), 64.6 (4), 65.5 (16)
#endif
  static constexpr int kRowStep = WV_PAIR_STEP;
  __device__ __forceinline__ static void scale(Rec& R, float s) {
    One::scale(R.f[0], s);
    One::scale(R.f[1], s);
  }
#ifndef WV_PAIR_MINB
#define WV_PAIR_MINB 3  // 168 registers; 4 blocks spill
#endif
  static constexpr int kMinBlocks = WV_PAIR_MINB;
  static constexpr double kCoefScale = One::kCoefScale;
  static constexpr int kAcc = 18;
  static constexpr int kRowAcc = 20;
  __device__ __forceinline__ static bool unit_weights(const Rec&) { return true; }
  // generic point sources: the two faces independently (weighted)
  template <bool kUnit>
  __device__ __forceinline__ static uint32_t pair2(const Rec& R, F2 qx, F2 qy, F2 qz, F2 coef,
                                                   float eps2, F2* g) {
    const uint32_t i0 = One::pair2<false>(R.f[0], qx, qy, qz, coef, eps2, g);
    const uint32_t i1 = One::pair2<false>(R.f[1], qx, qy, qz, coef, eps2, g + One::kAcc);
    return (i0 ? 1u : 0u) | (i1 ? 2u : 0u);
  }
  __device__ __forceinline__ static void rare_pair(const Rec& R, float qx, float qy, float qz,
                                                   float c, double (*acc)[kBwdThreads],
                                                   uint32_t ill) {
    if (ill & 1u) exact_pair_f64(R.f[0], qx, qy, qz, c, acc);
    if (ill & 2u) exact_pair_f64(R.f[1], qx, qy, qz, c, acc + One::kAcc);
  }
  struct Row {
    float a2, b2, c2, d2;  // x/y parts of |corner - q|^2 (A, B, C, D)
    float qx, qy;
    bool paired;
  };
  __device__ __forceinline__ static Row row(const Rec& R, float qx, float qy) {
    const ExactGradRecF32& F = R.f[0];
    const ExactGradRecF32& G = R.f[1];
    Row w;
    const float ax = F.a.x - qx, ay = F.a.y - qy, bx = F.b.x - qx, by = F.b.y - qy;
    const float cx = F.c.x - qx, cy = F.c.y - qy, dx = G.c.x - qx, dy = G.c.y - qy;
    w.a2 = fmaf(ay, ay, ax * ax);
    w.b2 = fmaf(by, by, bx * bx);
    w.c2 = fmaf(cy, cy, cx * cx);
    w.d2 = fmaf(dy, dy, dx * dx);
    w.qx = qx;
    w.qy = qy;
    w.paired = G.a.x == F.b.x && G.a.y == F.b.y && G.a.z == F.b.z && G.b.x == F.c.x &&
               G.b.y == F.c.y && G.b.z == F.c.z;
    return w;
  }
  // sums 0-11: F1 in ExactEdgeBwd's layout; 12-19: F2's own sums 2,3,6-11
  // (its sums 0,1,4,5 are F1's 6,7,8,9: the shared edge)
  template <bool kUnit, int N>
  __device__ __forceinline__ static void step_row(const Rec& R, const Row& w, const float4* zc,
                                                  float, F2* z, F2* mr) {
    if (!w.paired) return;  // run_end evaluates the faces one by one
    const ExactGradRecF32& F = R.f[0];
    const ExactGradRecF32& G = R.f[1];
    F2 ru[N];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const F2 qz = f2(zc[u].x, zc[u].y), coef = f2(zc[u].z, zc[u].w);
      const F2 az = sub2(f2s(F.a.z), qz), bz = sub2(f2s(F.b.z), qz);
      const F2 cz = sub2(f2s(F.c.z), qz), dz = sub2(f2s(G.c.z), qz);
      const F2 a2 = fma2(az, az, f2s(w.a2)), b2 = fma2(bz, bz, f2s(w.b2));
      const F2 c2 = fma2(cz, cz, f2s(w.c2)), d2 = fma2(dz, dz, f2s(w.d2));
      const F2 ia = rsqrt2(a2), ib = rsqrt2(b2), ic = rsqrt2(c2), id = rsqrt2(d2);
      const F2 lb = mul2(b2, ib), lc = mul2(c2, ic);
      const F2 sab = fma2(a2, ia, lb), sbc = add2(lb, lc), sca = fma2(a2, ia, lc);
      const F2 scd = fma2(d2, id, lc), sdb = fma2(d2, id, lb);
      const F2 dab = fma2(sab, sab, f2s(-F.u.x)), dbc = fma2(sbc, sbc, f2s(-F.u.y));
      const F2 dca = fma2(sca, sca, f2s(-F.u.z));
      const F2 dcd = fma2(scd, scd, f2s(-G.u.y)), ddb = fma2(sdb, sdb, f2s(-G.u.z));
      const F2 p1 = mul2(dbc, dca), rr1 = rcp2_abs(mul2(dab, p1));
      const F2 rr2 = rcp2_abs(mul2(dcd, ddb));
      float r10, r11, r20, r21;  // lane max per face (ALU): F1's lo, F2's hi
      split(rr1, r10, r11);
      split(rr2, r20, r21);
      ru[u] = f2(maxnan(r10, r11), maxnan(r20, r21));
      const F2 cr1 = mul2(coef, rr1), q0 = mul2(cr1, dab);
      const F2 tab = mul2(cr1, p1), tbc = mul2(q0, dca), tca = mul2(q0, dbc);
      const F2 cr2 = mul2(coef, rr2);
      const F2 tcd = mul2(cr2, ddb), tdb = mul2(cr2, dcd);
      const F2 uab = mul2(tab, az), ubc = mul2(tbc, bz), uca = mul2(tca, cz);
      const F2 ucd = mul2(tcd, cz), udb = mul2(tdb, dz);
      z[0] = fma2(tab, ia, z[0]);
      z[1] = fma2(uab, ia, z[1]);
      z[2] = fma2(tca, ia, z[2]);
      z[3] = fma2(uca, ia, z[3]);
      z[4] = fma2(tab, ib, z[4]);
      z[5] = fma2(uab, ib, z[5]);
      z[6] = fma2(tbc, ib, z[6]);
      z[7] = fma2(ubc, ib, z[7]);
      z[8] = fma2(tbc, ic, z[8]);
      z[9] = fma2(ubc, ic, z[9]);
      z[10] = fma2(tca, ic, z[10]);
      z[11] = fma2(uca, ic, z[11]);
      z[12] = fma2(tdb, ib, z[12]);  // F2 edge D->B at its corner B'
      z[13] = fma2(udb, ib, z[13]);
      z[14] = fma2(tcd, ic, z[14]);  // F2 edge C->D at its corner C'
      z[15] = fma2(ucd, ic, z[15]);
      z[16] = fma2(tcd, id, z[16]);  // edge C->D at D
      z[17] = fma2(ucd, id, z[17]);
      z[18] = fma2(tdb, id, z[18]);  // edge D->B at D
      z[19] = fma2(udb, id, z[19]);
    }
#pragma unroll
    for (int h = 1; h < N; h *= 2)
#pragma unroll
      for (int u = 0; u + h < N; u += 2 * h) ru[u] = maxnan2(ru[u], ru[u + h]);
    *mr = maxnan2(*mr, ru[0]);
  }
  // one face over a run with the single-face row code (broken welds), flushed
  __device__ __noinline__ static void single_run(const ExactGradRecF32& Rk, float qx, float qy,
                                                 const float4* zcs, int j, int e, float eps2,
                                                 double (*acc)[kBwdThreads]) {
    const One::Row rk = One::row(Rk, qx, qy);
    F2 z[One::kRowAcc];
    for (int i = 0; i < One::kRowAcc; ++i) z[i] = f2(0.0f, 0.0f);
    F2 mr = f2(0.0f, 0.0f);
    const int j0 = j;
    for (; j < e; ++j) {
      const float4 zc = zcs[j];
      if (!(zc.z == 0.0f && zc.w == 0.0f)) One::step_row<true, 1>(Rk, rk, &zc, eps2, z, &mr);
    }
    if (One::ill_run(Rk, mr)) One::redo_run<true>(Rk, rk, zcs, j0, e, eps2, z, acc);
    One::flush_row<true>(Rk, rk, z, acc);
  }
  __device__ __noinline__ static void redo_pair(const Rec& R, float qx, float qy,
                                                const float4* zcs, int j0, int e, float eps2,
                                                double (*acc)[kBwdThreads]) {
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {
      const One::Row rk = One::row(R.f[k], qx, qy);
      F2 z[One::kRowAcc];
      One::redo_run<true>(R.f[k], rk, zcs, j0, e, eps2, z, acc + k * One::kAcc);
      One::flush_row<true>(R.f[k], rk, z, acc + k * One::kAcc);
    }
  }
  // end of a row run [j0, e): flush the sums (or redo / evaluate per face)
  template <bool kUnit>
  __device__ __forceinline__ static void run_end(const Rec& R, const Row& w, const float4* zcs,
                                                 int j0, int e, float eps2, const F2* z, F2 mr,
                                                 double (*acc)[kBwdThreads]) {
    if (!w.paired) {
      single_run(R.f[0], w.qx, w.qy, zcs, j0, e, eps2, acc);
      single_run(R.f[1], w.qx, w.qy, zcs, j0, e, eps2, acc + One::kAcc);
      return;
    }
    // mr = (max rr of F1, max rr of F2): ratio products with each face's
    // squared edge lengths (F2's shared edge BC is F1's)
    float m0, m1;
    split(mr, m0, m1);
    const float u1p = R.f[0].u.x * R.f[0].u.y * R.f[0].u.z, u2p = R.f[1].u.y * R.f[1].u.z;
    if (!(m0 * u1p < One::kIllRatio) || !(m1 * u2p < One::kIllRatio)) {  // rare: ill pair
      redo_pair(R, w.qx, w.qy, zcs, j0, e, eps2, acc);
      return;
    }
    One::flush_row<true>(R.f[0], One::row(R.f[0], w.qx, w.qy), z, acc);
    const F2 z2[One::kRowAcc] = {z[6], z[7], z[12], z[13], z[8], z[9],
                                 z[14], z[15], z[16], z[17], z[18], z[19]};
    One::flush_row<true>(R.f[1], One::row(R.f[1], w.qx, w.qy), z2, acc + One::kAcc);
  }
  __device__ __forceinline__ static void finish(const Rec& R, const double* a, double* out) {
    One::finish(R.f[0], a, out);
    One::finish(R.f[1], a + One::kAcc, out + 9);
  }
};

// ---------------------------------------------------------------------------
// Exact backward over edge TRAILS (wv_trail.cu): one thread owns a window of
// K = kTrailK (4) consecutive edges of a trail through the position-welded
// edge graph, p0 -> p1 -> ... -> pK.  Every distinct edge of the mesh is
// evaluated once (closed surface: 1.5 per face, strip pairs 2.5) and each
// position's distance serves both window edges at it: per point pair K+1
// MUFU.RSQ (distances and their reciprocals) + 1 MUFU.RCP (the K edge
// denominators share it) and ~13 FP32 lane-ops per edge, i.e. per face of a
// closed surface ~19.5 lane-ops + 2.25 MUFU (strip pairs: 28 + 3).  The
// terms are those of ExactEdgeBwd (edge form, row running sums, moments
// m = a_P x e formed once per row run in fp64); the kernel writes the 2 end
// vectors of each window edge (6K doubles per window) and the signed CSR
// gather (face_to_vertex_kernel) gives every vertex id its terms with the
// signs of its faces' edge directions.

// One ill-conditioned (window, point) pair in FP64 (ExactEdgeBwd's
// exact_pair_f64 for the window's edges): acc[6e + 3 end + axis].
__device__ __noinline__ void trail_pair_f64(const TrailRecF32& R, double qx, double qy,
                                            double qz, double c, double (*acc)[kBwdThreads]) {
  constexpr int K = kTrailK;
  if (c == 0.0) return;
  double P[K + 1][3], len[K + 1];
  for (int k = 0; k <= K; ++k) {
    P[k][0] = (double)R.p[k].x - qx;
    P[k][1] = (double)R.p[k].y - qy;
    P[k][2] = (double)R.p[k].z - qz;
    len[k] = sqrt(P[k][0] * P[k][0] + P[k][1] * P[k][1] + P[k][2] * P[k][2]);
  }
  const int t = threadIdx.x;
  for (int e = 0; e < K; ++e) {
    const double* A = P[e];
    const double* B = P[e + 1];
    const double m[3] = {A[1] * B[2] - A[2] * B[1], A[2] * B[0] - A[0] * B[2],
                         A[0] * B[1] - A[1] * B[0]};
    const double L = len[e] * len[e + 1], ab = A[0] * B[0] + A[1] * B[1] + A[2] * B[2];
    const double mm = m[0] * m[0] + m[1] * m[1] + m[2] * m[2];
    const double den = (L - ab) > 0.0 ? mm / (L - ab) : L + ab;  // |a||b| + a.b
    if (!(den > 0.0) || !(len[e] > 0.0) || !(len[e + 1] > 0.0)) continue;  // on the edge
    const double f = c / (2.0 * den);
    for (int x = 0; x < 3; ++x) {
      acc[6 * e + x][t] += m[x] * (f / len[e]);
      acc[6 * e + 3 + x][t] += m[x] * (f / len[e + 1]);
    }
  }
}

struct ExactEdgeBwdTrail {
  static constexpr int K = kTrailK;
  static constexpr bool kPrefetch = true;
  using Rec = TrailRecF32;
  static constexpr int kFaces = 1;
  static constexpr int kOut = 6 * K;  // (edge, end, axis)
  static constexpr bool kScaled = true;
  static constexpr bool kPairRuns = false;
#ifndef WV_TRAIL_STEP
#define WV_TRAIL_STEP 2  // C3: 1249 ms (2) vs 1275 (4), 1252 (6, 3 CTAs/SM), 1282 (K = 3, step 4)
#endif
#ifndef WV_TRAIL_MINB
#define WV_TRAIL_MINB 4
#endif
  static constexpr int kRowStep = WV_TRAIL_STEP;
  static constexpr int kMinBlocks = WV_TRAIL_MINB;
  static constexpr double kCoefScale = ExactEdgeBwd::kCoefScale;
  static constexpr int kAcc = 6 * K;
  static constexpr int kRowAcc = 4 * K;  // per edge: sum t/|P|, t a_z/|P|, t/|Q|, t a_z/|Q|
  static constexpr float kIllRatio = ExactEdgeBwd::kIllRatio;
  // The thread keeps only what every step reads in registers -- the
  // positions' z and the squared edge lengths, in the power-of-two scaled
  // frame (launch_bwd's grid_scale) -- and re-reads x / y from the record
  // (L1) once per row run: with all 20 floats live the compiler re-derived
  // the row parts of |p - q|^2 in every step to stay inside 128 registers.
  struct View {
    float z[K + 1];
    float u[K];
    const Rec* g;
    float gs;
  };
  __device__ __forceinline__ static View view(const Rec* g, float gs) {
    View v;
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      const float4 p = __ldg(&g->p[k]);
      v.z[k] = p.z * gs;
      if (k < K) v.u[k] = p.w * (gs * gs);
    }
    v.g = g;
    v.gs = gs;
    return v;
  }
  __device__ __forceinline__ static float2 xy(const View& V, int k) {
    const float4 p = __ldg(&V.g->p[k]);
    return make_float2(p.x * V.gs, p.y * V.gs);
  }
  // the full scaled record (rare fp64 path)
  __device__ __forceinline__ static Rec full(const View& V) {
    Rec R;
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      const float2 q = xy(V, k);
      R.p[k] = make_float4(q.x, q.y, V.z[k], k < K ? V.u[k] : 0.0f);
    }
    return R;
  }
  __device__ __forceinline__ static bool unit_weights(const View&) { return true; }
  struct Row {
    float a2[K + 1];  // x/y parts of |p_k - q|^2
    float qx, qy;
  };
  __device__ __forceinline__ static Row row(const View& V, float qx, float qy) {
    Row w;
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      const float2 p = xy(V, k);
      const float dx = p.x - qx, dy = p.y - qy;
      w.a2[k] = fmaf(dy, dy, dx * dx);
    }
    w.qx = qx;
    w.qy = qy;
    return w;
  }
  // Ill-conditioning screen, per EDGE: a pair is ill when some window edge
  // has d_e <= |e|^2 / kIllRatio (fp32 keeps ~1e-7 kIllRatio relative
  // accuracy above that), or d_e is NaN.  (ExactEdgeBwd screens the PRODUCT
  // of its face's three ratios, sound there because the other two edges of
  // a triangle bound their ratios from below for a point near one edge; a
  // window's far edges can be several edge lengths away, so the trail
  // screen keeps each edge's own minimum of d_e over the run -- NaN-
  // propagating mins on the ALU pipe.)
  struct Screen {
    F2 d[K];
  };
  __device__ __forceinline__ static Screen screen_init() {
    Screen s;
#pragma unroll
    for (int e = 0; e < K; ++e) s.d[e] = f2s(__int_as_float(0x7f800000));
    return s;
  }
  // one point pair (packed f32x2).  kMask = false: the hot path, the edge
  // denominators go to dd[K] for the run's screen; kMask = true: ill lanes
  // leave the fp32 sums (bits returned, trail_pair_f64 adds them)
  template <bool kMask>
  __device__ __forceinline__ static uint32_t pair_row2(const View& R, const Row& w, F2 qz, F2 coef,
                                                       F2* z, F2* dd = nullptr) {
    F2 az[K + 1], ip[K + 1], lp[K + 1];
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      az[k] = sub2(f2s(R.z[k]), qz);
      const F2 s2 = fma2(az[k], az[k], f2s(w.a2[k]));
      ip[k] = rsqrt2(s2);
      lp[k] = mul2(s2, ip[k]);
    }
    // 2 (|a||b| + a.b) = (|a| + |b|)^2 - |e|^2 per edge
    F2 d[K];
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const F2 se = add2(lp[e], lp[e + 1]);
      d[e] = fma2(se, se, f2s(-R.u[e]));
    }
    // one reciprocal for the K denominators
    F2 t[K];
    F2 rr, cr;
    F2 p01, p23;
    if constexpr (K == 3) {
      p23 = mul2(d[1], d[2]);
      rr = rcp2_abs(mul2(d[0], p23));
    } else {
      p01 = mul2(d[0], d[1]);
      p23 = mul2(d[2], d[3]);
      rr = rcp2_abs(mul2(p01, p23));
    }
    bool ill0 = false, ill1 = false;
    if constexpr (kMask) {
#pragma unroll
      for (int e = 0; e < K; ++e) {
        const float k = R.u[e] * (1.0f / kIllRatio);
        float lo, hi;
        split(d[e], lo, hi);
        ill0 |= !(lo > k);
        ill1 |= !(hi > k);
      }
      float r0, r1;
      split(mul2(coef, rr), r0, r1);
      cr = f2(ill0 ? 0.0f : r0, ill1 ? 0.0f : r1);
    } else {
#pragma unroll
      for (int e = 0; e < K; ++e) dd[e] = d[e];
      cr = mul2(coef, rr);
    }
    if constexpr (K == 3) {
      const F2 q0 = mul2(cr, d[0]);
      t[0] = mul2(cr, p23);
      t[1] = mul2(q0, d[2]);
      t[2] = mul2(q0, d[1]);
    } else {
      const F2 c01 = mul2(cr, p23), c23 = mul2(cr, p01);
      t[0] = mul2(c01, d[1]);
      t[1] = mul2(c01, d[0]);
      t[2] = mul2(c23, d[3]);
      t[3] = mul2(c23, d[2]);
    }
#pragma unroll
    for (int e = 0; e < K; ++e) {  // t_e = coef / d_e
      const F2 u = mul2(t[e], az[e]);
      z[4 * e + 0] = fma2(t[e], ip[e], z[4 * e + 0]);
      z[4 * e + 1] = fma2(u, ip[e], z[4 * e + 1]);
      z[4 * e + 2] = fma2(t[e], ip[e + 1], z[4 * e + 2]);
      z[4 * e + 3] = fma2(u, ip[e + 1], z[4 * e + 3]);
    }
    return (ill0 ? 1u : 0u) | (ill1 ? 2u : 0u);
  }
  template <bool kUnit, int N>
  __device__ __forceinline__ static void step_row(const View& R, const Row& w, const float4* zc,
                                                  float, F2* z, Screen* mr) {
    // the step's own minima first (short chains), then one min into the run's
    F2 m[K];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      F2 dd[K];
      pair_row2<false>(R, w, f2(zc[u].x, zc[u].y), f2(zc[u].z, zc[u].w), z, dd);
#pragma unroll
      for (int e = 0; e < K; ++e) m[e] = u == 0 ? dd[e] : minnan2(m[e], dd[e]);
    }
#pragma unroll
    for (int e = 0; e < K; ++e) mr->d[e] = minnan2(mr->d[e], m[e]);
  }
  __device__ __forceinline__ static bool ill_run(const View& R, const Screen& mr) {
    bool ill = false;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      float lo, hi;
      split(mr.d[e], lo, hi);
      ill |= !(minnan(lo, hi) > R.u[e] * (1.0f / kIllRatio));
    }
    return ill;
  }
  template <bool kUnit>
  __device__ __noinline__ static void redo_run(const View& R, const Row& w, const float4* zcs,
                                               int j, int e, float, F2* z,
                                               double (*acc)[kBwdThreads]) {
    const Rec Rf = full(R);
    for (int i = 0; i < kRowAcc; ++i) z[i] = f2(0.0f, 0.0f);
    for (; j < e; ++j) {
      const float4 zc = zcs[j];
      if (zc.z == 0.0f && zc.w == 0.0f) continue;
      const uint32_t ill = pair_row2<true>(R, w, f2(zc.x, zc.y), f2(zc.z, zc.w), z);
      if (ill & 1u) trail_pair_f64(Rf, w.qx, w.qy, zc.x, zc.z, acc);
      if (ill & 2u) trail_pair_f64(Rf, w.qx, w.qy, zc.y, zc.w, acc);
    }
  }
  // the run's sums -> sum_q m s per (edge, end) into the fp64 accumulators
  // (m = a_P x e: x/y affine in a_z of the edge's first position, z constant)
  __device__ __forceinline__ static void flush_row(const View& R, const Row& w, const F2* z,
                                                   double (*acc)[kBwdThreads]) {
    const int t = threadIdx.x;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      double s[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float lo, hi;
        split(z[4 * e + j], lo, hi);
        s[j] = (double)lo + (double)hi;
      }
      // (the moments in f64 from the f32 coordinates, exact differences)
      const float2 P = xy(R, e), Q = xy(R, e + 1);
      const double ax = (double)P.x - (double)w.qx, ay = (double)P.y - (double)w.qy;
      const double ex = (double)Q.x - (double)P.x, ey = (double)Q.y - (double)P.y;
      const double ez = (double)R.z[e + 1] - (double)R.z[e];
      const double kx = ay * ez, ky = -(ax * ez), mz = ax * ey - ay * ex;
      acc[6 * e + 0][t] += kx * s[0] - ey * s[1];
      acc[6 * e + 1][t] += ky * s[0] + ex * s[1];
      acc[6 * e + 2][t] += mz * s[0];
      acc[6 * e + 3][t] += kx * s[2] - ey * s[3];
      acc[6 * e + 4][t] += ky * s[2] + ex * s[3];
      acc[6 * e + 5][t] += mz * s[2];
    }
  }
  __device__ __forceinline__ static void finish(const View&, const double* acc, double* out) {
    for (int j = 0; j < kOut; ++j) out[j] = acc[j];
  }
};

// Query points of a chunk, stored as packed PAIRS: xy[j] = {x_2j, x_2j+1,
// y_2j, y_2j+1}, zc[j] = {z_2j, z_2j+1, coef_2j, coef_2j+1}; two LDS.128
// deliver one point pair already in f32x2 register pairs.
struct PointChunk {
  float4 xy[kBwdChunk / 2];
  float4 zc[kBwdChunk / 2];
};

template <class Pol, bool kUnit>
__device__ __forceinline__ void chunk_loop(const typename Pol::Rec& R, const PointChunk& ch,
                                           int n_pairs, float eps2, F2* g,
                                           double (*acc)[kBwdThreads]) {
#pragma unroll 2
  for (int j = 0; j < n_pairs; ++j) {
    const float4 zc = ch.zc[j];
    if (zc.z == 0.0f && zc.w == 0.0f) continue;  // warp-uniform (_kernels.py:182-184)
    const float4 xy = ch.xy[j];
    const uint32_t ill = Pol::template pair2<kUnit>(R, f2(xy.x, xy.y), f2(xy.z, xy.w),
                                                    f2(zc.x, zc.y), f2(zc.z, zc.w), eps2, g);
    if (ill != 0u) {  // both lanes redone in fp64 (see ExactEdgeBwd::pair2)
      Pol::rare_pair(R, xy.x, xy.z, zc.x, zc.z, acc, ill);
      Pol::rare_pair(R, xy.y, xy.w, zc.y, zc.w, acc, ill);
    }
  }
}

// Row mode: the chunk is cut at k-row boundaries (warp-uniform), each run of
// pairs shares the row's x/y, and the per-face row constants are computed
// once per run.  Needs rz and the range start even (pairs never straddle).
// Row mode: the chunk is cut at k-row boundaries (warp-uniform), each run of
// pairs shares the row's x/y, and the per-face row constants are computed
// once per run.  Needs rz and the range start even (pairs never straddle).
// the thread's register copy of its record: Pol::View when the policy
// defines one (a partial copy; the rest is re-read from global memory where
// needed), else the scaled record itself
template <class Pol, class = void>
struct RecOf {
  using T = typename Pol::Rec;
  __device__ __forceinline__ static T load(const typename Pol::Rec* recs, int64_t f, float gs) {
    T R = recs[f];
    if (gs != 1.0f) Pol::scale(R, gs);
    return R;
  }
};
template <class Pol>
struct RecOf<Pol, std::void_t<typename Pol::View>> {
  using T = typename Pol::View;
  __device__ __forceinline__ static T load(const typename Pol::Rec* recs, int64_t f, float gs) {
    return Pol::view(recs + f, gs);
  }
};

// the row loop's screen state: Pol::Screen when the policy defines one, else
// one F2 (a running max, 0 = clean)
template <class Pol, class = void>
struct ScreenOf {
  using T = F2;
  __device__ __forceinline__ static F2 init() { return f2(0.0f, 0.0f); }
};
template <class Pol>
struct ScreenOf<Pol, std::void_t<typename Pol::Screen>> {
  using T = typename Pol::Screen;
  __device__ __forceinline__ static T init() { return Pol::screen_init(); }
};

template <class Pol, bool kUnit>
__device__ __forceinline__ void chunk_rows(const typename RecOf<Pol>::T& R, const PointChunk& ch,
                                           int n_pairs, int64_t flat0, int64_t rz, float eps2,
                                           bool dense, double (*acc)[kBwdThreads]) {
  int j = 0;
  int k = (int)(flat0 % rz);  // k of the chunk's first node
  while (j < n_pairs) {
    int run = (int)((rz - k) >> 1);
    if (run > n_pairs - j) run = n_pairs - j;
    const float4 xy0 = ch.xy[j];
    const typename Pol::Row w = Pol::row(R, xy0.x, xy0.z);
    F2 z[Pol::kRowAcc];
#pragma unroll
    for (int i = 0; i < Pol::kRowAcc; ++i) z[i] = f2(0.0f, 0.0f);
    const int e = j + run, j0 = j;
    // running state of the ill-conditioning screen (exact only)
    typename ScreenOf<Pol>::T mr = ScreenOf<Pol>::init();
    // Pol::kRowStep point pairs per step under one (warp-uniform)
    // zero-coefficient test, so their dependency chains share a basic block
    // and interleave (a zero-coefficient pair next to a live one adds
    // 0 * finite: its point is parked far away)
#pragma unroll 1
    for (; j + Pol::kRowStep <= e; j += Pol::kRowStep) {
      float4 zc[Pol::kRowStep];
#pragma unroll
      for (int u = 0; u < Pol::kRowStep; ++u) zc[u] = ch.zc[j + u];
      if (!dense) {
        bool any = false;
#pragma unroll
        for (int u = 0; u < Pol::kRowStep; ++u) any |= zc[u].z != 0.0f || zc[u].w != 0.0f;
        if (!any) continue;
      }
      Pol::template step_row<kUnit, Pol::kRowStep>(R, w, zc, eps2, z, &mr);
    }
#pragma unroll 1
    for (; j < e; ++j) {
      const float4 zc = ch.zc[j];
      if (!(zc.z == 0.0f && zc.w == 0.0f))  // warp-uniform (_kernels.py:182-184)
        Pol::template step_row<kUnit, 1>(R, w, &zc, eps2, z, &mr);
    }
    if constexpr (Pol::kPairRuns) {
      Pol::template run_end<kUnit>(R, w, ch.zc, j0, e, eps2, z, mr, acc);
    } else {
      if (Pol::ill_run(R, mr))  // rare: an ill-conditioned pair in the run
        Pol::template redo_run<kUnit>(R, w, ch.zc, j0, e, eps2, z, acc);
      Pol::flush_row(R, w, z, acc);
    }
    k = 0;
  }
}

template <class Pol, class Src>
__global__ void __launch_bounds__(kBwdThreads, Pol::kMinBlocks)
bwd_f32_kernel(const PackHeader* __restrict__ hdr, const typename Pol::Rec* __restrict__ recs,
               size_t pack_stride, int64_t n_faces, Src src, const float* __restrict__ coefs,
               int64_t n_count, int64_t pts_per_split, float coef_scale,
               double* __restrict__ out, float gscale) {
  __shared__ PointChunk chunk;
  // batched launches: blockIdx.z selects the mesh (records pack_stride bytes
  // apart, coefficients n_count apart, partials (mesh, split)-major)
  hdr = reinterpret_cast<const PackHeader*>(reinterpret_cast<const char*>(hdr) +
                                            blockIdx.z * pack_stride);
  recs = reinterpret_cast<const typename Pol::Rec*>(hdr + 1);
  coefs += (int64_t)blockIdx.z * n_count;
  const int64_t f = (int64_t)blockIdx.x * kBwdThreads + threadIdx.x;
  const bool live = f < n_faces;
  const typename RecOf<Pol>::T R = RecOf<Pol>::load(recs, live ? f : 0, gscale);
  // power-of-two geometry scale (row mode of the exact backward, see
  // launch_bwd): exact in floating point, so the arithmetic is the unscaled
  // one; the corner sums are scaled back on the way out
  const float eps = hdr->eps_f32;
  const float eps2 = eps * eps;
  const int64_t p_begin = (int64_t)blockIdx.y * pts_per_split;
  int64_t p_end = p_begin + pts_per_split;
  if (p_end > n_count) p_end = n_count;

  // warp-uniform fast path when every face of the warp has unit edge
  // weights (soups, boundary strips): saves the per-edge weight multiply
  const bool unit = __all_sync(0xffffffffu, Pol::unit_weights(R));
  // fp64 accumulators in shared memory ([j][thread]), touched once per
  // 256-point chunk: keeps the pair arithmetic inside the register budget of
  // 5 CTAs per SM
  __shared__ double acc[Pol::kAcc][kBwdThreads];
#pragma unroll
  for (int j = 0; j < Pol::kAcc; ++j) acc[j][threadIdx.x] = 0.0;

  // Lattice sources: per-axis node tables in shared memory (the same IEEE
  // f64 node expression cast to f32 as GridSrc::point, evaluated once per
  // CTA instead of three f64 divisions per point per chunk) and 32-bit
  // index math -- the chunk fill otherwise costs ~1/3 of the soft pair work
  __shared__ float axt[3][kAxisMax];
  bool tab = false;
  if constexpr (Src::kGrid) {
    tab = src.g.res[0] <= kAxisMax && src.g.res[1] <= kAxisMax && src.g.res[2] <= kAxisMax &&
          src.n0 + n_count <= 0xffffffffll;
    if (tab) {
      for (int a = 0; a < 3; ++a)
        for (int t = threadIdx.x; t < src.g.res[a]; t += kBwdThreads)
          axt[a][t] = (float)axis_node(src.g.lo[a], src.g.hi[a], src.g.res[a], t) * gscale;
    }
  }

  // the coefficients of the NEXT chunk are loaded into registers while the
  // current chunk is evaluated (their global-load latency had stalled the
  // chunk fill; kPre per thread cover a chunk)
  constexpr int kPre = kBwdChunk / kBwdThreads;
  static_assert(kPre * kBwdThreads == kBwdChunk, "whole chunk per prefetch");
  // (the strip-pair kernel only: the others' register budgets spill with it)
  float cpre[kPre];
  if constexpr (Pol::kPrefetch) {
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int64_t gi = p_begin + threadIdx.x + k * kBwdThreads;
      cpre[k] = gi < p_end ? coefs[gi] : 0.0f;
    }
  }
  for (int64_t c0 = p_begin; c0 < p_end; c0 += kBwdChunk) {
    const int n = (int)((p_end - c0) < kBwdChunk ? (p_end - c0) : kBwdChunk);
    const int n_pairs = (n + 1) / 2;
    __syncthreads();
    int zero = 0;  // some coefficient of this chunk is zero (or padding)
    // one point of the chunk: coordinates (or parked), coefficient
    auto fill = [&](int i, float cv) {
      float x = 1.0e6f, y = 1.0e6f, z = 1.0e6f, c = 0.0f;
      if (i < n) {
        c = cv * coef_scale;
        // zero-coefficient points contribute nothing; park them far away so
        // the other half of their pair never sees an on-segment 0 * inf
        // (row mode keeps the row's x/y and parks z only)
        if (c != 0.0f || Src::kRows) {
          if constexpr (Src::kGrid) {
            if (tab) {
              const uint32_t gl = (uint32_t)(src.n0 + c0 + i);
              const uint32_t rz = (uint32_t)src.g.res[2], ry = (uint32_t)src.g.res[1];
              const uint32_t r = gl / rz, ii = r / ry;
              x = axt[0][ii];
              y = axt[1][r - ii * ry];
              z = axt[2][gl - r * rz];
            } else {
              src.point(c0 + i, x, y, z);
              x *= gscale;
              y *= gscale;
              z *= gscale;
            }
          } else {
            src.point(c0 + i, x, y, z);
          }
        }
        if (c == 0.0f) z = 1.0e6f;
      }
      float* xy = reinterpret_cast<float*>(&chunk.xy[i >> 1]);
      float* zc = reinterpret_cast<float*>(&chunk.zc[i >> 1]);
      xy[i & 1] = x;
      xy[2 + (i & 1)] = y;
      zc[i & 1] = z;
      zc[2 + (i & 1)] = c;
      zero |= c == 0.0f;
    };
    if constexpr (Pol::kPrefetch) {
#pragma unroll
      for (int k = 0; k < kPre; ++k) {
        const float cv = cpre[k];
        const int64_t gi = c0 + kBwdChunk + threadIdx.x + k * kBwdThreads;
        cpre[k] = gi < p_end ? coefs[gi] : 0.0f;
        const int i = threadIdx.x + k * kBwdThreads;
        if (i < 2 * n_pairs) fill(i, cv);
      }
    } else {
      for (int i = threadIdx.x; i < 2 * n_pairs; i += kBwdThreads)
        fill(i, i < n ? coefs[c0 + i] : 0.0f);
    }
    // a chunk without zero coefficients (the common case of a loss over a
    // grid) skips the per-step zero tests
    const bool dense = __syncthreads_or(zero) == 0;
    if constexpr (Src::kRows) {
      // row runs flush their sums straight into the fp64 accumulators
      const int64_t flat0 = src.n0 + c0;
      if (unit) {
        chunk_rows<Pol, true>(R, chunk, n_pairs, flat0, src.g.res[2], eps2, dense, acc);
      } else {
        chunk_rows<Pol, false>(R, chunk, n_pairs, flat0, src.g.res[2], eps2, dense, acc);
      }
    } else {
      F2 g[Pol::kAcc];
#pragma unroll
      for (int j = 0; j < Pol::kAcc; ++j) g[j] = f2(0.0f, 0.0f);
      if (unit) {
        chunk_loop<Pol, true>(R, chunk, n_pairs, eps2, g, acc);
      } else {
        chunk_loop<Pol, false>(R, chunk, n_pairs, eps2, g, acc);
      }
#pragma unroll
      for (int j = 0; j < Pol::kAcc; ++j) {
        float lo, hi;
        split(g[j], lo, hi);
        acc[j][threadIdx.x] += (double)lo + (double)hi;
      }
    }
  }
  if (live) {
    double o9[Pol::kOut];
    double a[Pol::kAcc];
#pragma unroll
    for (int j = 0; j < Pol::kAcc; ++j) a[j] = acc[j][threadIdx.x];
    Pol::finish(R, a, o9);
    double* dst = out + (((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * n_faces + f) * Pol::kOut;
#pragma unroll
    for (int j = 0; j < Pol::kOut; ++j) dst[j] = o9[j] * (double)gscale;  // dW/dv = s dW/d(s v)
  }
}
// out[f*9+j] = sum_s part[s][f*9+j], fixed split order
__global__ void reduce_splits_kernel(const double* __restrict__ part, int splits, int64_t n,
                                     int64_t batch, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * batch;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i / n, k = i - z * n;
    const double* p = part + z * splits * n + k;
    double a = 0.0;
    for (int s = 0; s < splits; ++s) a += p[(int64_t)s * n];
    out[i] = a;
  }
}

struct BwdPlan {
  int64_t blocks_x = 0;
  int splits = 1;
  int64_t pts_per_split = 0;
  static BwdPlan make(int64_t n_faces, int64_t n_count, int num_sms, int min_blocks,
                      int64_t batch = 1) {
    BwdPlan p;
    p.blocks_x = (n_faces + kBwdThreads - 1) / kBwdThreads;
    if (p.blocks_x < 1) p.blocks_x = 1;
    const int64_t slots = (int64_t)num_sms * min_blocks;
    const int64_t blocks = p.blocks_x * batch;
    int64_t lo = (4 * slots + blocks - 1) / blocks;  // >= ~4 waves
    int64_t hi = 4 * lo;  // then the split count with the fullest last wave
    int64_t max_s = (n_count + kBwdChunk - 1) / kBwdChunk;  // >= one chunk per split
    if (max_s > 4096) max_s = 4096;
    if (lo > max_s) lo = max_s;
    if (hi > max_s) hi = max_s;
    int64_t s = best_splits(blocks, lo, hi, slots);
    p.pts_per_split = (n_count + s - 1) / s;
    p.pts_per_split = ((p.pts_per_split + kBwdChunk - 1) / kBwdChunk) * kBwdChunk;
    p.splits = (int)((n_count + p.pts_per_split - 1) / p.pts_per_split);
    if (p.splits < 1) p.splits = 1;
    return p;
  }
  // n_rec records of k_out doubles each (9 per face)
  size_t workspace(int64_t n_rec, int64_t batch = 1, int k_out = 9) const {
    return splits > 1 ? (size_t)splits * (size_t)batch * (size_t)n_rec * k_out * sizeof(double)
                      : 0;
  }
};

// Power of two bringing the lattice's largest |coordinate| into [1, 2): the
// row backward's shared reciprocal forms d01 d12 d20 (~|x|^6), which must
// stay inside the f32 range for any input scale.
static float grid_scale(const GridDesc& g) {
  double m = 0.0;
  for (int a = 0; a < 3; ++a) m = fmax(m, fmax(fabs(g.lo[a]), fabs(g.hi[a])));
  if (!(m > 0.0) || !std::isfinite(m)) return 1.0f;
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  if (e > 120) e = 120;
  if (e < -120) e = -120;
  return (float)ldexp(1.0, 1 - e);
}

// two faces per thread for the soft backward whenever the face count is even
static bool soft_pairs(int64_t n_faces) { return n_faces >= 2 && n_faces % 2 == 0; }

template <class Pol>
static int launch_bwd(const void* packed, int64_t n_faces, const PointSource& ps,
                      int64_t n_count, const float* coefs, double coef_scale, double* face_grad,
                      void* workspace, size_t ws_bytes, int num_sms, cudaStream_t stream,
                      const Batch& bt) {
  if (n_faces <= 0 || bt.n <= 0) return kOk;
  if (bt.n > 65535 || (bt.n > 1 && ps.kind != PointSource::kGrid)) return kErrArg;
  if (n_count <= 0) {
    return cudaMemsetAsync(face_grad, 0, (size_t)bt.n * n_faces * 9 * sizeof(double), stream) ==
                   cudaSuccess ? kOk : kErrCuda;
  }
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const auto* recs = reinterpret_cast<const typename Pol::Rec*>(hdr + 1);
  const int64_t n_rec = n_faces / Pol::kFaces;  // callers pass a multiple of kFaces
  const BwdPlan pl = BwdPlan::make(n_rec, n_count, num_sms, Pol::kMinBlocks, bt.n);
  double* dst = face_grad;
  if (pl.splits > 1) {
    if (workspace == nullptr || ws_bytes < pl.workspace(n_rec, bt.n, Pol::kOut))
      return kErrWorkspace;
    dst = static_cast<double*>(workspace);
  }
  const float cs = (float)(coef_scale * Pol::kCoefScale);
  dim3 grid((unsigned)pl.blocks_x, (unsigned)pl.splits, (unsigned)bt.n);
  if (ps.kind == PointSource::kGrid && ps.grid.res[2] >= 16 &&
      row_aligned(ps.grid, ps.n0, 2 * ((n_count + 1) / 2), 2)) {
    RowSrc src{{ps.grid, ps.n0}};
    { bwd_f32_kernel<Pol, RowSrc><<<grid, kBwdThreads, 0, stream>>>(
        hdr, recs, bt.pack_stride, n_rec, src, coefs, n_count, pl.pts_per_split, cs, dst,
        Pol::kScaled ? grid_scale(ps.grid) : 1.0f); wv::note_launch(); }
  } else if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    { bwd_f32_kernel<Pol, GridSrc><<<grid, kBwdThreads, 0, stream>>>(
        hdr, recs, bt.pack_stride, n_rec, src, coefs, n_count, pl.pts_per_split, cs, dst, 1.0f); wv::note_launch(); }
  } else {
    ListSrc src{ps.points};
    { bwd_f32_kernel<Pol, ListSrc><<<grid, kBwdThreads, 0, stream>>>(
        hdr, recs, bt.pack_stride, n_rec, src, coefs, n_count, pl.pts_per_split, cs, dst, 1.0f); wv::note_launch(); }
  }
  if (pl.splits > 1) {
    const int64_t n = n_rec * Pol::kOut;
    int blocks = (int)((n * bt.n + 255) / 256);
    if (blocks > num_sms * 8) blocks = num_sms * 8;
    { reduce_splits_kernel<<<blocks, 256, 0, stream>>>(dst, pl.splits, n, bt.n, face_grad); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_exact_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, const float* coefs, double coef_scale,
                         double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                         cudaStream_t stream, const Batch& bt) {
  return launch_bwd<ExactEdgeBwd>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad, ws,
                                  ws_bytes, num_sms, stream, bt);
}
int launch_soft_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, const float* coefs, double coef_scale,
                        double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                        cudaStream_t stream, const Batch& bt) {
  if (soft_pairs(n_faces))
    return launch_bwd<SoftBwdPair>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad,
                                   ws, ws_bytes, num_sms, stream, bt);
  return launch_bwd<SoftBwd>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad, ws,
                             ws_bytes, num_sms, stream, bt);
}
size_t soft_bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch) {
  if (soft_pairs(n_faces))
    return BwdPlan::make(n_faces / 2, n_count, num_sms, SoftBwdPair::kMinBlocks, batch)
        .workspace(n_faces / 2, batch, SoftBwdPair::kOut);
  return BwdPlan::make(n_faces, n_count, num_sms, kBwdMinBlocks, batch).workspace(n_faces, batch);
}
// strip pairs (ExactEdgeBwdPair): n_faces = 2 x records, faces in pair order
int launch_exact_pair_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                              int64_t n_count, const float* coefs, double coef_scale,
                              double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                              cudaStream_t stream) {
  if (n_faces % 2 != 0) return kErrArg;
  return launch_bwd<ExactEdgeBwdPair>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad,
                                      ws, ws_bytes, num_sms, stream, Batch{});
}
size_t exact_pair_bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms) {
  return BwdPlan::make(n_faces / 2, n_count, num_sms, ExactEdgeBwdPair::kMinBlocks)
      .workspace(n_faces / 2, 1, ExactEdgeBwdPair::kOut);
}
// edge trails (ExactEdgeBwdTrail): lattice rows only (the trail records are
// chosen for row-aligned lattice ranges); out = (n_windows, 2K, 3) doubles
int launch_exact_trail_bwd_f32(const void* packed, int64_t n_windows, const PointSource& ps,
                               int64_t n_count, const float* coefs, double coef_scale,
                               double* out, void* workspace, size_t ws_bytes, int num_sms,
                               cudaStream_t stream) {
  using Pol = ExactEdgeBwdTrail;
  if (n_windows <= 0) return kOk;
  if (n_count <= 0)
    return cudaMemsetAsync(out, 0, (size_t)n_windows * Pol::kOut * sizeof(double), stream) ==
                   cudaSuccess ? kOk : kErrCuda;
  if (!(ps.kind == PointSource::kGrid && ps.grid.res[2] >= 16 &&
        row_aligned(ps.grid, ps.n0, 2 * ((n_count + 1) / 2), 2)))
    return kErrArg;
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const auto* recs = reinterpret_cast<const Pol::Rec*>(hdr + 1);
  const BwdPlan pl = BwdPlan::make(n_windows, n_count, num_sms, Pol::kMinBlocks);
  double* dst = out;
  if (pl.splits > 1) {
    if (workspace == nullptr || ws_bytes < pl.workspace(n_windows, 1, Pol::kOut))
      return kErrWorkspace;
    dst = static_cast<double*>(workspace);
  }
  const float cs = (float)(coef_scale * Pol::kCoefScale);
  dim3 grid((unsigned)pl.blocks_x, (unsigned)pl.splits, 1u);
  RowSrc src{{ps.grid, ps.n0}};
  bwd_f32_kernel<Pol, RowSrc><<<grid, kBwdThreads, 0, stream>>>(
      hdr, recs, 0, n_windows, src, coefs, n_count, pl.pts_per_split, cs, dst,
      grid_scale(ps.grid));
  wv::note_launch();
  if (pl.splits > 1) {
    const int64_t n = n_windows * Pol::kOut;
    int blocks = (int)((n + 255) / 256);
    if (blocks > num_sms * 8) blocks = num_sms * 8;
    reduce_splits_kernel<<<blocks, 256, 0, stream>>>(dst, pl.splits, n, 1, out);
    wv::note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}
size_t exact_trail_bwd_workspace_bytes(int64_t n_windows, int64_t n_count, int num_sms) {
  return BwdPlan::make(n_windows, n_count, num_sms, ExactEdgeBwdTrail::kMinBlocks)
      .workspace(n_windows, 1, ExactEdgeBwdTrail::kOut);
}
size_t bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch) {
  // the larger of the two single-face plans (exact and soft occupancies differ)
  const size_t a =
      BwdPlan::make(n_faces, n_count, num_sms, kBwdMinBlocks, batch).workspace(n_faces, batch);
  const size_t b = BwdPlan::make(n_faces, n_count, num_sms, ExactEdgeBwd::kMinBlocks, batch)
                       .workspace(n_faces, batch);
  return a > b ? a : b;
}

// ---------------------------------------------------------------------------
// face corners -> vertices, CSR order (deterministic); optional device scale
// (e.g. 1/sum(w) of the loss, read on the device so nothing syncs the host).
__global__ void face_to_vertex_kernel(const double* __restrict__ face_grad,
                                      const int64_t* __restrict__ off,
                                      const int64_t* __restrict__ slots, int64_t n_verts,
                                      const double* __restrict__ scale, int accumulate,
                                      double* __restrict__ out64, float* __restrict__ out32,
                                      int64_t fg_stride = 0, int64_t scale_stride = 0) {
  // batched launches: blockIdx.y = mesh (face_grad fg_stride doubles apart,
  // scale scale_stride apart, outputs n_verts x 3 apart)
  face_grad += blockIdx.y * fg_stride;
  if (scale) scale += blockIdx.y * scale_stride;
  if (out64) out64 += blockIdx.y * 3 * n_verts;
  if (out32) out32 += blockIdx.y * 3 * n_verts;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_verts;
       v += (int64_t)gridDim.x * blockDim.x) {
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      // slot = f*3 + corner (faces) or 6 w + 2 e + end (edge trails); a
      // negative entry -s-1 subtracts slot s (a trail edge walked against
      // the face's direction)
      const int64_t s = slots[e];
      const double* src = face_grad + (s >= 0 ? s : -s - 1) * 3;
      if (s >= 0) {
        gx += src[0];
        gy += src[1];
        gz += src[2];
      } else {
        gx -= src[0];
        gy -= src[1];
        gz -= src[2];
      }
    }
    if (scale) {
      const double s = *scale;
      gx *= s;
      gy *= s;
      gz *= s;
    }
    if (out64) {
      if (accumulate) {
        out64[3 * v] += gx;
        out64[3 * v + 1] += gy;
        out64[3 * v + 2] += gz;
      } else {
        out64[3 * v] = gx;
        out64[3 * v + 1] = gy;
        out64[3 * v + 2] = gz;
      }
    }
    if (out32) {
      if (accumulate) {
        out32[3 * v] += (float)gx;
        out32[3 * v + 1] += (float)gy;
        out32[3 * v + 2] += (float)gz;
      } else {
        out32[3 * v] = (float)gx;
        out32[3 * v + 1] = (float)gy;
        out32[3 * v + 2] = (float)gz;
      }
    }
  }
}

int launch_face_to_vertex(const double* face_grad, const int64_t* off, const int64_t* slots,
                          int64_t n_verts, const double* scale, int accumulate, double* out64,
                          float* out32, int num_sms, cudaStream_t stream) {
  if (n_verts <= 0) return kOk;
  int blocks = (int)((n_verts + 255) / 256);
  if (blocks > num_sms * 16) blocks = num_sms * 16;
  { face_to_vertex_kernel<<<blocks, 256, 0, stream>>>(face_grad, off, slots, n_verts, scale,
                                                    accumulate, out64, out32); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_face_to_vertex_batch(const double* face_grad, int64_t n_faces, const int64_t* off,
                                const int64_t* slots, int64_t n_verts, int64_t batch,
                                const double* scale, int64_t scale_stride, int accumulate,
                                double* out64, float* out32, int num_sms, cudaStream_t stream) {
  if (n_verts <= 0) return kOk;
  if (batch < 1 || batch > 65535) return kErrArg;
  int blocks = (int)((n_verts + 255) / 256);
  if (blocks > num_sms * 16) blocks = num_sms * 16;
  { face_to_vertex_kernel<<<dim3((unsigned)blocks, (unsigned)batch), 256, 0, stream>>>(
      face_grad, off, slots, n_verts, scale, accumulate, out64, out32, n_faces * 9, scale_stride); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
