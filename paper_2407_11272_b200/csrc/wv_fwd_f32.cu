// wv_fwd_f32.cu -- FP32 forward kernels (sm_100a): exact generalized winding
// number and the soft (dipole) winding number, both on the generic TMA-tiled
// all-pairs skeleton of wv_fwd.cuh.
//
// Exact (replaces _kernels.exact_batch_f32, _kernels.py:235-309, and the f64
// exact_batch hot loop, :34-116, under the 1e-5 tolerance of north_star):
//   theta = atan2(alpha, beta),  Omega = 2 theta,  W = sum(theta) / (2 pi)
//   alpha = N.(v0-q) (= det(a,b,c)), beta grouped as _kernels.py:98-103.
//   Common pairs (|alpha/beta| < 1/8, beta > |a||b||c|/2 and every corner
//   farther than eps: every far face) need one MUFU.RCP and a 3-term
//   polynomial; the rest (wide angles, ill-conditioned beta, vertex-hit and
//   other on-surface candidates, degenerate faces) go to exact_rare().
// Soft (replaces _kernels.soft_batch_f32, :312-349, and soft_batch, :119-158):
//   term = N.(c-q) / |c-q|^3 with one MUFU.RSQ,  W = sum(term) / (8 pi);
//   |c-q| < eps flags the point and skips the face.
#include "wv_fwd.cuh"

namespace wv {

// Rare exact pairs -- wide angles (|theta| >= atan(1/8), incl. beta <= 0),
// on-surface candidates and degenerate faces.  They are few (only faces
// within about a face size of the node), and they are where fp32 loses
// digits to cancellation in beta, so they are evaluated in FP64 on the same
// fp32-rounded inputs, in the reference kernel's operation order
// (_kernels.py:52-105): vertex test, plane + barycentric test (eps of the
// f64 header), triple product, beta grouping, atan2.  Returns theta =
// Omega/2 in f64, 0 for a degenerate face, NaN for an on-surface pair.
__device__ __noinline__ double exact_rare(float4 A, float4 B, float4 C, float qxf, float qyf,
                                          float qzf, double eps) {
  if (A.w == __int_as_float(0x7f800000)) return 0.0;  // degenerate (dropped) face
  const double qx = qxf, qy = qyf, qz = qzf;
  const double ax = (double)A.x - qx, ay = (double)A.y - qy, az = (double)A.z - qz;
  const double bx = (double)B.x - qx, by = (double)B.y - qy, bz = (double)B.z - qz;
  const double cx = (double)C.x - qx, cy = (double)C.y - qy, cz = (double)C.z - qz;
  const double na = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)), __dmul_rn(az, az)));
  const double nb = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(bx, bx), __dmul_rn(by, by)), __dmul_rn(bz, bz)));
  const double nc = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
  if (na < eps || nb < eps || nc < eps) return __longlong_as_double(0x7ff8000000000000ll);
  const double ux = (double)B.x - A.x, uy = (double)B.y - A.y, uz = (double)B.z - A.z;
  const double wx = (double)C.x - A.x, wy = (double)C.y - A.y, wz = (double)C.z - A.z;
  const double nx = uy * wz - uz * wy, ny = uz * wx - ux * wz, nz = ux * wy - uy * wx;
  const double nn = sqrt(nx * nx + ny * ny + nz * nz);
  const double pd = -(nx * ax + ny * ay + nz * az) / nn;  // nhat.(q - v0)
  if (-eps < pd && pd < eps) {
    const double d00 = ux * ux + uy * uy + uz * uz;
    const double d01 = ux * wx + uy * wy + uz * wz;
    const double d11 = wx * wx + wy * wy + wz * wz;
    const double denom = d00 * d11 - d01 * d01;
    const double ru = -(ax * ux + ay * uy + az * uz);
    const double rw = -(ax * wx + ay * wy + az * wz);
    const double b1 = (d11 * ru - d01 * rw) / denom;
    const double b2 = (d00 * rw - d01 * ru) / denom;
    if (b1 >= -1e-12 && b2 >= -1e-12 && b1 + b2 <= 1.0 + 1e-12)
      return __longlong_as_double(0x7ff8000000000000ll);
  }
  const double alpha = __dadd_rn(__dadd_rn(__dmul_rn(ax, __dsub_rn(__dmul_rn(by, cz), __dmul_rn(bz, cy))),
                                           __dmul_rn(ay, __dsub_rn(__dmul_rn(bz, cx), __dmul_rn(bx, cz)))),
                                 __dmul_rn(az, __dsub_rn(__dmul_rn(bx, cy), __dmul_rn(by, cx))));
  const double bc = __dadd_rn(__dadd_rn(__dmul_rn(bx, cx), __dmul_rn(by, cy)), __dmul_rn(bz, cz));
  const double ab = __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(ay, by)), __dmul_rn(az, bz));
  const double ca = __dadd_rn(__dadd_rn(__dmul_rn(cx, ax), __dmul_rn(cy, ay)), __dmul_rn(cz, az));
  const double beta = __dadd_rn(__dadd_rn(__dmul_rn(na, __dmul_rn(nb, nc)), __dmul_rn(bc, na)),
                                __dadd_rn(__dmul_rn(ab, nc), __dmul_rn(ca, nb)));
  return atan2(alpha, beta);
}

// Both policies evaluate TWO query points per instruction (packed f32x2, see
// wv_f32x2.cuh) against one face; common2 returns a 2-bit mask of the pairs
// that must go to the rare path (they contribute nothing here).
struct ExactPol {
  using Rec = ExactRecF32;
  static constexpr int kTile = 128;
  static constexpr int kStages = 4;
  static constexpr int kConsumerWarps = 4;
  static constexpr int kThreads = kConsumerWarps * 32;
#ifndef WV_EXACT_MINB
#define WV_EXACT_MINB 4
#endif
#ifndef WV_EXACT_MINB_ROW
#define WV_EXACT_MINB_ROW 4  // 5 (96 regs) spills and measured 2% slower (single faces)
#endif
  static constexpr int kMinBlocks = WV_EXACT_MINB;
  static constexpr int kMinBlocksRow = WV_EXACT_MINB_ROW;
  static constexpr int kP = 8;
  static constexpr double kScale = 1.0 / (2.0 * kPi);
  static constexpr bool kStrip = false;
  struct Slot {};
  // eps2: squared vertex-hit radius, eps (f32) inflated by 1% so that every
  // pair within the reference's f64 eps of a vertex (winding.py:65-67) leaves
  // the common path and is decided exactly by exact_rare
  struct Ctx {
    float eps2;
  };
  __device__ static Ctx make_ctx(float eps) {
    const float e = eps * 1.01f;
    return Ctx{e * e};
  }
  __device__ __forceinline__ static uint32_t common2(const Rec& R, F2 qx, F2 qy, F2 qz,
                                                     const Ctx& ctx, F2& tacc) {
    const F2 ax = sub2(f2s(R.v0e.x), qx), ay = sub2(f2s(R.v0e.y), qy), az = sub2(f2s(R.v0e.z), qz);
    const F2 bx = sub2(f2s(R.v1.x), qx), by = sub2(f2s(R.v1.y), qy), bz = sub2(f2s(R.v1.z), qz);
    const F2 cx = sub2(f2s(R.v2.x), qx), cy = sub2(f2s(R.v2.y), qy), cz = sub2(f2s(R.v2.z), qz);
    // alpha = N.(v0-q) = det(a,b,c)
    const F2 alpha = fma2(f2s(R.n.z), az, fma2(f2s(R.n.y), ay, mul2(f2s(R.n.x), ax)));
    const F2 la2 = dot2(ax, ay, az, ax, ay, az);
    const F2 lb2 = dot2(bx, by, bz, bx, by, bz);
    const F2 lc2 = dot2(cx, cy, cz, cx, cy, cz);
    return tail2(R, alpha, la2, lb2, lc2, ctx, tacc);
  }
  // Lattice-row form: the P points of a thread share x and y, so the x/y
  // parts of alpha and of the squared corner distances are per-face scalars
  // (same operation order as common2, hence bit-identical terms).
  struct Row {
    float a2, b2, c2, alpha;
  };
  __device__ __forceinline__ static Row row(const Rec& R, float qx, float qy) {
    const float ax = R.v0e.x - qx, ay = R.v0e.y - qy;
    const float bx = R.v1.x - qx, by = R.v1.y - qy;
    const float cx = R.v2.x - qx, cy = R.v2.y - qy;
    Row w;
    w.a2 = fmaf(ay, ay, ax * ax);
    w.b2 = fmaf(by, by, bx * bx);
    w.c2 = fmaf(cy, cy, cx * cx);
    w.alpha = fmaf(R.n.y, ay, R.n.x * ax);
    return w;
  }
  __device__ __forceinline__ static uint32_t common_row2(const Rec& R, const Row& w, F2 qz,
                                                         const Ctx& ctx, F2& tacc) {
    const F2 az = sub2(f2s(R.v0e.z), qz), bz = sub2(f2s(R.v1.z), qz), cz = sub2(f2s(R.v2.z), qz);
    const F2 alpha = fma2(f2s(R.n.z), az, f2s(w.alpha));
    const F2 la2 = fma2(az, az, f2s(w.a2));
    const F2 lb2 = fma2(bz, bz, f2s(w.b2));
    const F2 lc2 = fma2(cz, cz, f2s(w.c2));
    return tail2(R, alpha, la2, lb2, lc2, ctx, tacc);
  }
  __device__ __forceinline__ static uint32_t tail2(const Rec& R, F2 alpha, F2 la2, F2 lb2, F2 lc2,
                                                   const Ctx& ctx, F2& tacc) {
    const F2 la = sqrt2(la2), lb = sqrt2(lb2), lc = sqrt2(lc2);
    // a.b = (|a|^2 + |b|^2 - |v0-v1|^2)/2 etc. (half squared edge lengths are
    // packed): 2 ops instead of 3.  It can cancel only where beta itself is
    // ill-conditioned, and those pairs leave for the fp64 path below.
    const F2 half = f2s(0.5f);
    const F2 ab = fma2(add2(la2, lb2), half, f2s(-fabsf(R.v1.w)));
    const F2 bc = fma2(add2(lb2, lc2), half, f2s(-fabsf(R.v2.w)));
    const F2 ca = fma2(add2(lc2, la2), half, f2s(-R.n.w));
    // beta = |a||b||c| + (b.c)|a| + (a.b)|c| + (c.a)|b|  (_kernels.py:98-103)
    const F2 labc = mul2(la, mul2(lb, lc));
    const F2 beta = fma2(ca, lb, fma2(ab, lc, fma2(bc, la, labc)));
    // Common pairs: |theta| < atan(1/8) (|alpha/beta| < 1/8, beta > 0).  On
    // a face's closed triangle beta <= 0 (on a vertex alpha = beta = 0), so
    // every on-surface candidate fails this test and reaches exact_rare(), as
    // do degenerate faces (N = 0); far faces -- nearly all pairs of a fine
    // mesh -- stay here.  atan(t) = t (1 + s (c1 + c2 s)), s = t^2,
    // |t| <= 1/8: relative error 1.2e-7 in fp32 (fit: DESIGN.md 3.5).
    // Well-conditioned pairs only: beta = |a||b||c| (1 + sum cos) must not
    // have cancelled below |a||b||c|/2 (near-edge / grazing configurations,
    // where fp32 loses digits); those go to the fp64 rare path too.  The
    // angle test is |t| < 1/8 on the computed t = alpha / beta (t^2 < 1/64;
    // beta <= 0 already fails the conditioning test), the same operations
    // as the face-wide fast path of finish(), so both classify alike.
    float bl, bh, pl, ph;
    split(beta, bl, bh);
    split(labc, pl, ph);
    const float p2l = __int_as_float(__float_as_int(pl) - (1 << 23));  // |a||b||c| / 2
    const float p2h = __int_as_float(__float_as_int(ph) - (1 << 23));
    // vertex-hit candidates (some corner within eps: |a||b||c| can be 0 and
    // beta a rounding residue of either sign) are never common
    float a2l, a2h, b2l, b2h, c2l, c2h;
    split(la2, a2l, a2h);
    split(lb2, b2l, b2h);
    split(lc2, c2l, c2h);
    const bool vl = fminf(a2l, fminf(b2l, c2l)) >= ctx.eps2;
    const bool vh = fminf(a2h, fminf(b2h, c2h)) >= ctx.eps2;
    const F2 tt = mul2(alpha, rcp2(beta));
    const F2 s = mul2(tt, tt);
    // |t| < 1/8 on the computed t (the fast path's test, same operations)
    float sl, sh;
    split(add2(s, f2s(-1.0f / 64.0f)), sl, sh);
    const bool cl = sl < 0.0f && bl > p2l && vl, ch = sh < 0.0f && bh > p2h && vh;
    const F2 p = fma2(fma2(s, f2s(0.19669890403747559f), f2s(-0.33331409096717834f)), s,
                      f2s(1.0f));
    // select the updated sum per lane (a rare lane's t and p may be inf /
    // NaN -- beta cancelled to ~0 next to the surface -- so 0 * p is no
    // neutral term)
    float ul, uh, al, ah;
    split(fma2(tt, p, tacc), ul, uh);
    split(tacc, al, ah);
    tacc = f2(cl ? ul : al, ch ? uh : ah);
    return (cl ? 0u : 1u) | (ch ? 0u : 2u);
  }
  // All PP point pairs of a thread against one face.  The common-pair test
  // of tail2 (t^2 < 1/64 and beta > |a||b||c|/2) is evaluated for the whole
  // face as ONE predicate, max over lanes of (t^2 - 1/64, |a||b||c| - 2 beta)
  // < 0, from packed ops and a 3-input max tree: when
  // every point of the thread is a common pair (nearly always) the terms are
  // added without per-lane selects or rare-mask building, which had cost
  // ~1/3 of the issue slots.  Otherwise the per-lane path (tail2) runs.
  // near: some point of the group may be within eps of a vertex (then every
  // lane takes tail2, which routes the candidates to exact_rare)
  template <int PP>
  __device__ __forceinline__ static uint32_t finish(const Rec& R, const F2* alpha, const F2* la2,
                                                    const F2* lb2, const F2* lc2, const Ctx& ctx,
                                                    bool near, F2* tacc) {
    F2 la[PP], lb[PP], lc[PP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      la[pp] = sqrt2(la2[pp]);
      lb[pp] = sqrt2(lb2[pp]);
      lc[pp] = sqrt2(lc2[pp]);
    }
    return finish_len<PP>(R, alpha, la2, lb2, lc2, la, lb, lc, ctx, near, tacc);
  }
  // finish() with the corner distances given (the strip form carries them)
  template <int PP>
  __device__ __forceinline__ static uint32_t finish_len(const Rec& R, const F2* alpha,
                                                        const F2* la2, const F2* lb2,
                                                        const F2* lc2, const F2* la_,
                                                        const F2* lb_, const F2* lc_,
                                                        const Ctx& ctx, bool near, F2* tacc) {
    F2 tq[PP], tp[PP];
    float m = -1.0f;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 la = la_[pp], lb = lb_[pp], lc = lc_[pp];
      const F2 half = f2s(0.5f);
      const F2 ab = fma2(add2(la2[pp], lb2[pp]), half, f2s(-fabsf(R.v1.w)));
      const F2 bc = fma2(add2(lb2[pp], lc2[pp]), half, f2s(-fabsf(R.v2.w)));
      const F2 ca = fma2(add2(lc2[pp], la2[pp]), half, f2s(-R.n.w));
      const F2 labc = mul2(la, mul2(lb, lc));
      const F2 beta = fma2(ca, lb, fma2(ab, lc, fma2(bc, la, labc)));
      // |a||b||c| - 2 beta (exact scaling, one rounding: the sign is the
      // exact comparison's, as tail2's exponent-subtract test) and t^2 - 1/64
      // (tail2's operations); beta <= 0 makes ee >= 0, so a non-finite t
      // never passes
      const F2 ee = fma2(beta, f2s(-2.0f), labc);
      const F2 tt = mul2(alpha[pp], rcp2(beta));
      const F2 s = mul2(tt, tt);
      const F2 dd = add2(s, f2s(-1.0f / 64.0f));  // t^2 - 1/64
      float d0, d1, e0, e1;
      split(dd, d0, d1);
      split(ee, e0, e1);
      m = fmaxf(m, fmaxf(fmaxf(d0, d1), fmaxf(e0, e1)));
      tq[pp] = tt;
      tp[pp] = fma2(fma2(s, f2s(0.19669890403747559f), f2s(-0.33331409096717834f)), s,
                    f2s(1.0f));
    }
    if (m < 0.0f && !near) {  // tail2's operation for a common pair: tacc + t p, one rounding
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) tacc[pp] = fma2(tq[pp], tp[pp], tacc[pp]);
      return 0u;
    }
    uint32_t rare = 0;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp)
      rare |= tail2(R, alpha[pp], la2[pp], lb2[pp], lc2[pp], ctx, tacc[pp]) << (2 * pp);
    return rare;
  }
  // ---- two faces per angle (kPairFaces) --------------------------------
  // theta_a + theta_b = atan(T), T = tan(theta_a + theta_b)
  //   = (alpha_a beta_b + alpha_b beta_a) / (beta_a beta_b - alpha_a alpha_b),
  // so a PAIR of common faces needs one reciprocal and one polynomial instead
  // of two: 3.5 MUFU per pair instead of 4 (this kernel is bound by the MUFU
  // pipe).  Valid whenever |T| < 1/8 and both betas are well conditioned
  // (beta > |a||b||c|/2, as tail2): then |t_i| = |alpha_i|/beta_i < 2
  // (|alpha| <= |a||b||c|), so beta_a beta_b - alpha_a alpha_b <= 0 -- a sum
  // past pi/2 -- cannot come with |T| < 1/8, and num = den = 0 cannot
  // happen.  Accuracy: num and den are well conditioned when |T| < 1/8
  // (cancellation in num costs only ulp(t_i) absolute), so the pair's term
  // has the single-face error.  A pair that fails takes both faces through
  // the single-face path (nothing of the pair was added).
  static constexpr bool kPairFaces = true;
#ifndef WV_PAIR_GROUP
#define WV_PAIR_GROUP 2
#endif
  static constexpr int kPairGroup = WV_PAIR_GROUP;  // point pairs per pair decision
  __device__ __forceinline__ static void beta_ee(const Rec& R, F2 la2, F2 lb2, F2 lc2, F2& beta,
                                                 F2& ee) {
    const F2 la = sqrt2(la2), lb = sqrt2(lb2), lc = sqrt2(lc2);
    const F2 half = f2s(0.5f);
    const F2 ab = fma2(add2(la2, lb2), half, f2s(-fabsf(R.v1.w)));
    const F2 bc = fma2(add2(lb2, lc2), half, f2s(-fabsf(R.v2.w)));
    const F2 ca = fma2(add2(lc2, la2), half, f2s(-R.n.w));
    const F2 labc = mul2(la, mul2(lb, lc));
    beta = fma2(ca, lb, fma2(ab, lc, fma2(bc, la, labc)));
    ee = fma2(beta, f2s(-2.0f), labc);  // < 0: well conditioned (finish_len)
  }
  // geo(k, pp, alpha, la2, lb2, lc2): the pair quantities of face k (0: Ra,
  // 1: Rb) and point pair pp (row or generic form, same operations as
  // face_row / face)
  template <int PP, class Geo>
  __device__ __forceinline__ static bool pair_fast(const Rec& Ra, const Rec& Rb, Geo geo,
                                                   bool near, F2* tacc) {
    F2 tq[PP], tp[PP];
    float m = -1.0f;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      F2 aa, la2, lb2, lc2, ba, ea, ab_, bb, eb;
      geo(0, pp, aa, la2, lb2, lc2);
      beta_ee(Ra, la2, lb2, lc2, ba, ea);
      geo(1, pp, ab_, la2, lb2, lc2);
      beta_ee(Rb, la2, lb2, lc2, bb, eb);
      const F2 num = fma2(aa, bb, mul2(ab_, ba));
      const F2 den = fma2(mul2(aa, ab_), f2s(-1.0f), mul2(ba, bb));
      const F2 tt = mul2(num, rcp2(den));
      const F2 s2 = mul2(tt, tt);
      const F2 dd = add2(s2, f2s(-1.0f / 64.0f));
      float d0, d1, a0, a1, b0, b1;
      split(dd, d0, d1);
      split(ea, a0, a1);
      split(eb, b0, b1);
      m = fmaxf(m, fmaxf(fmaxf(d0, d1), fmaxf(fmaxf(a0, a1), fmaxf(b0, b1))));
      tq[pp] = tt;
      tp[pp] = fma2(fma2(s2, f2s(0.19669890403747559f), f2s(-0.33331409096717834f)), s2,
                    f2s(1.0f));
    }
    if (m < 0.0f && !near) {
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) tacc[pp] = fma2(tq[pp], tp[pp], tacc[pp]);
      return true;
    }
    return false;
  }
  template <int PP>
  __device__ __forceinline__ static bool face_row_pair(const Rec& Ra, const Row& wa,
                                                       const Rec& Rb, const Row& wb,
                                                       const F2* qz, const Ctx& ctx, F2* tacc) {
    const bool near = fminf(fminf(wa.a2, fminf(wa.b2, wa.c2)),
                            fminf(wb.a2, fminf(wb.b2, wb.c2))) < ctx.eps2;
    auto geo = [&](int k, int pp, F2& alpha, F2& la2, F2& lb2, F2& lc2) {
      const Rec& R = k ? Rb : Ra;
      const Row& w = k ? wb : wa;
      const F2 az = sub2(f2s(R.v0e.z), qz[pp]), bz = sub2(f2s(R.v1.z), qz[pp]);
      const F2 cz = sub2(f2s(R.v2.z), qz[pp]);
      alpha = fma2(f2s(R.n.z), az, f2s(w.alpha));
      la2 = fma2(az, az, f2s(w.a2));
      lb2 = fma2(bz, bz, f2s(w.b2));
      lc2 = fma2(cz, cz, f2s(w.c2));
    };
    return pair_fast<PP>(Ra, Rb, geo, near, tacc);
  }
  template <int PP>
  __device__ __forceinline__ static bool face_pair(const Rec& Ra, const Rec& Rb, const F2* qx,
                                                   const F2* qy, const F2* qz, const Ctx& ctx,
                                                   F2* tacc) {
    float mn = __int_as_float(0x7f800000);
    auto geo = [&](int k, int pp, F2& alpha, F2& la2, F2& lb2, F2& lc2) {
      const Rec& R = k ? Rb : Ra;
      const F2 ax = sub2(f2s(R.v0e.x), qx[pp]), ay = sub2(f2s(R.v0e.y), qy[pp]);
      const F2 az = sub2(f2s(R.v0e.z), qz[pp]);
      const F2 bx = sub2(f2s(R.v1.x), qx[pp]), by = sub2(f2s(R.v1.y), qy[pp]);
      const F2 bz = sub2(f2s(R.v1.z), qz[pp]);
      const F2 cx = sub2(f2s(R.v2.x), qx[pp]), cy = sub2(f2s(R.v2.y), qy[pp]);
      const F2 cz = sub2(f2s(R.v2.z), qz[pp]);
      alpha = fma2(f2s(R.n.z), az, fma2(f2s(R.n.y), ay, mul2(f2s(R.n.x), ax)));
      la2 = dot2(ax, ay, az, ax, ay, az);
      lb2 = dot2(bx, by, bz, bx, by, bz);
      lc2 = dot2(cx, cy, cz, cx, cy, cz);
      float a0, a1, b0, b1, c0, c1;
      split(la2, a0, a1);
      split(lb2, b0, b1);
      split(lc2, c0, c1);
      mn = fminf(mn, fminf(fminf(a0, a1), fminf(fminf(b0, b1), fminf(c0, c1))));
    };
    // the vertex-hit test needs every lane's distances: evaluate, then decide
    F2 tq[PP];
    for (int pp = 0; pp < PP; ++pp) tq[pp] = tacc[pp];
    const bool ok = pair_fast<PP>(Ra, Rb, geo, false, tq);
    if (!ok || mn < ctx.eps2) return false;
    for (int pp = 0; pp < PP; ++pp) tacc[pp] = tq[pp];
    return true;
  }
  template <int PP>
  __device__ __forceinline__ static uint32_t face_row(const Rec& R, const Row& w, const F2* qz,
                                                      const Ctx& ctx, F2* tacc) {
    F2 alpha[PP], la2[PP], lb2[PP], lc2[PP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 az = sub2(f2s(R.v0e.z), qz[pp]), bz = sub2(f2s(R.v1.z), qz[pp]);
      const F2 cz = sub2(f2s(R.v2.z), qz[pp]);
      alpha[pp] = fma2(f2s(R.n.z), az, f2s(w.alpha));
      la2[pp] = fma2(az, az, f2s(w.a2));
      lb2[pp] = fma2(bz, bz, f2s(w.b2));
      lc2[pp] = fma2(cz, cz, f2s(w.c2));
    }
    // the row's x/y part bounds every |corner - q|^2 of the row from below
    const bool near = fminf(w.a2, fminf(w.b2, w.c2)) < ctx.eps2;
    return finish<PP>(R, alpha, la2, lb2, lc2, ctx, near, tacc);
  }
  template <int PP>
  __device__ __forceinline__ static uint32_t face(const Rec& R, const F2* qx, const F2* qy,
                                                  const F2* qz, const Ctx& ctx, F2* tacc) {
    F2 alpha[PP], la2[PP], lb2[PP], lc2[PP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 ax = sub2(f2s(R.v0e.x), qx[pp]), ay = sub2(f2s(R.v0e.y), qy[pp]);
      const F2 az = sub2(f2s(R.v0e.z), qz[pp]);
      const F2 bx = sub2(f2s(R.v1.x), qx[pp]), by = sub2(f2s(R.v1.y), qy[pp]);
      const F2 bz = sub2(f2s(R.v1.z), qz[pp]);
      const F2 cx = sub2(f2s(R.v2.x), qx[pp]), cy = sub2(f2s(R.v2.y), qy[pp]);
      const F2 cz = sub2(f2s(R.v2.z), qz[pp]);
      alpha[pp] = fma2(f2s(R.n.z), az, fma2(f2s(R.n.y), ay, mul2(f2s(R.n.x), ax)));
      la2[pp] = dot2(ax, ay, az, ax, ay, az);
      lb2[pp] = dot2(bx, by, bz, bx, by, bz);
      lc2[pp] = dot2(cx, cy, cz, cx, cy, cz);
    }
    float mn = __int_as_float(0x7f800000);
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      float a0, a1, b0, b1, c0, c1;
      split(la2[pp], a0, a1);
      split(lb2[pp], b0, b1);
      split(lc2[pp], c0, c1);
      mn = fminf(mn, fminf(fminf(a0, a1), fminf(fminf(b0, b1), fminf(c0, c1))));
    }
    return finish<PP>(R, alpha, la2, lb2, lc2, ctx, mn < ctx.eps2, tacc);
  }
  __device__ __forceinline__ static double rare(const Rec& R, float qx, float qy, float qz,
                                                double eps) {
    return exact_rare(R.v0e, R.v1, R.v2, qx, qy, qz, eps);
  }
};

// Exact forward over STRIP-ordered records (wv_strip.cu): on lattice rows a
// thread carries |A - q|^2, |A - q| of the next face from the current
// face's B and C (bitwise the values a recomputation gives: the same
// operations on the same coordinates), so a face costs 1 square root + 1
// reciprocal per pair instead of 3 + 1 -- the MUFU pipe bounds this kernel.
// Records restart (recompute A and B) at strip starts and at every tile.
#ifndef WV_STRIP_P
#define WV_STRIP_P 8
#endif
#ifndef WV_STRIP_MINB
#define WV_STRIP_MINB 3  // 160 registers, no spills: 1% faster than 4 blocks with spills
#endif
struct ExactStripPol : ExactPol {
  static constexpr bool kStrip = true;
  static constexpr bool kPairFaces = false;  // strips pair their faces themselves
  static_assert(kTile == 128, "pack_strip_kernel restarts a strip every 128 records");
  static constexpr int kP = WV_STRIP_P;
  static constexpr int kMinBlocksRow = WV_STRIP_MINB;
#ifndef WV_STRIP_GROUP
#define WV_STRIP_GROUP 4
#endif
  static constexpr int kGroup = WV_STRIP_GROUP;  // point pairs per common-path decision
  // corner-distance slots per point pair: d = |v - q|, s = d + the next
  // slot's d.  Face k of a strip reads A, B from slots (k, k+1) mod 3 (and
  // s_A = |a| + |b| from the previous face) and writes C's distance to slot
  // (k+2) mod 3, so with the face loop unrolled by 3 nothing is moved.
#ifndef WV_STRIP_CARRY_S
#define WV_STRIP_CARRY_S 1
#endif
  struct Slot {
    F2 d;
#if WV_STRIP_CARRY_S
    F2 s;
#endif
  };
  // |a| + |b| of a face: carried from the previous face (s) or recomputed
  __device__ __forceinline__ static F2 sum_ab(const Slot& A, const Slot& B) {
#if WV_STRIP_CARRY_S
    return A.s;
#else
    return add2(A.d, B.d);
#endif
  }
  __device__ __forceinline__ static void set_s(Slot& S, F2 v) {
#if WV_STRIP_CARRY_S
    S.s = v;
#endif
  }
  // alpha = N.(C - q) (any corner of the face gives alpha; C's z part is
  // needed for |c - q| anyway, so alpha costs one FFMA2 per point pair)
  // Per face only C's row part is computed; A's and B's are carried from the
  // previous faces (row_ab at strip starts), bitwise what ExactPol::row gives
  __device__ __forceinline__ static Row row_c(const Rec& R, float qx, float qy) {
    const float cx = R.v2.x - qx, cy = R.v2.y - qy;
    Row w;
    w.c2 = fmaf(cy, cy, cx * cx);
    w.alpha = fmaf(R.n.y, cy, R.n.x * cx);
    return w;
  }
  __device__ __forceinline__ static void row_ab(const Rec& R, float qx, float qy, float& a2,
                                                float& b2) {
    const float ax = R.v0e.x - qx, ay = R.v0e.y - qy;
    const float bx = R.v1.x - qx, by = R.v1.y - qy;
    a2 = fmaf(ay, ay, ax * ax);
    b2 = fmaf(by, by, bx * bx);
  }
  // beta without the three dot products (no squared distances needed):
  //   a.b = (|a|^2 + |b|^2)/2 - h_ab  gives
  //   2 beta = (|a|+|b|)(|b|+|c|)(|c|+|a|) - 2 (|a| h_bc + |b| h_ca + |c| h_ab)
  //          = X - 2L                       (8 lane-ops with |a|+|b| carried)
  // Conditioning: 2 beta > X/8 (X >= 8 |a||b||c|, so this implies tail2's
  // beta > |a||b||c|/2), tested as L' > -X on the ALU with L' = 16/7 (-L);
  // angle: t^2 < 1/64 (max tree); no corner within eps (per-face scalar).
  // Lanes that fail take tail2 (recomputed from squared distances) or the
  // fp64 path.  The kernel decides two faces at a time (one branch per two
  // faces, so one face's tail overlaps the next face's square roots).
  // The common-path terms of one face for PP point pairs (tq, tp: the
  // accumulation is tacc = fma(tq, tp, tacc)); true when every pair is
  // common.  Always updates the distance slots.
  template <int PP>
  __device__ __forceinline__ static bool strip_fast(const Rec& R, const Row& w, const F2* qz,
                                                    const Ctx& ctx, bool restart, Slot* sA,
                                                    Slot* sB, Slot* sC, F2* tq, F2* tp) {
    if (restart) {
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) {
        const F2 az = sub2(f2s(R.v0e.z), qz[pp]), bz = sub2(f2s(R.v1.z), qz[pp]);
        sA[pp].d = sqrt2(fma2(az, az, f2s(w.a2)));
        sB[pp].d = sqrt2(fma2(bz, bz, f2s(w.b2)));
        set_s(sA[pp], add2(sA[pp].d, sB[pp].d));
      }
    }
    // the records carry (16/7) h (flags in the sign bits): -|.| folds into
    // the FFMA2 operands (SASS -|R|.F32), no per-face multiply
    const float kab = -fabsf(R.v1.w), kbc = -fabsf(R.v2.w), kca = -R.n.w;
    // t/2 = alpha / (2 beta) is what the division gives; the series is taken
    // in (t/2)^2 with its coefficients scaled by powers of 2, so
    // (t/2) (2 p(t^2)) rounds exactly as t p(t^2) does, without doubling alpha
    constexpr float kC2 = 32.0f * 0.19669890403747559f, kC1 = 8.0f * -0.33331409096717834f;
    float ms = 0.0f;
    bool cond = true;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 cz = sub2(f2s(R.v2.z), qz[pp]);
      const F2 alpha = fma2(f2s(R.n.z), cz, f2s(w.alpha));  // alpha from corner C (row_c())
      const F2 lc = sqrt2(fma2(cz, cz, f2s(w.c2)));
      const F2 la = sA[pp].d, lb = sB[pp].d;
      const F2 sbc = add2(lb, lc), sca = add2(lc, la);
      sC[pp].d = lc;
      const F2 sab = sum_ab(sA[pp], sB[pp]);  // |a| + |b|, the previous face's |b| + |c|
      set_s(sB[pp], sbc);
      const F2 x = mul2(mul2(sab, sbc), sca);
      const F2 lp = fma2(lc, f2s(kab), fma2(lb, f2s(kca), mul2(la, f2s(kbc))));  // 16/7 (-L)
      const F2 beta2 = fma2(lp, f2s(0.875f), x);  // X - 2L
      float x0, x1, l0, l1;
      split(x, x0, x1);
      split(lp, l0, l1);
      cond = cond && (l0 > -x0) && (l1 > -x1);
      const F2 th = mul2(alpha, rcp2(beta2));  // t/2
      const F2 s4 = mul2(th, th);               // t^2/4
      float s0, s1;
      split(s4, s0, s1);
      ms = fmaxf(ms, fmaxf(s0, s1));
      tq[pp] = th;
      tp[pp] = fma2(fma2(s4, f2s(kC2), f2s(kC1)), s4, f2s(2.0f));
    }
    const bool near = fminf(w.a2, fminf(w.b2, w.c2)) < ctx.eps2;
    return ms < 1.0f / 256.0f && cond && !near;  // t^2 < 1/64
  }
  // Two consecutive strip faces for ONE angle evaluation (tan addition, see
  // ExactPol::pair_fast): with B = 2 beta, the pair's t/2 is
  //   (alpha_a B_b + alpha_b B_a) / (B_a B_b - 4 alpha_a alpha_b),
  // one reciprocal and one polynomial for two faces (MUFU 2 -> 1.5 per pair).
  // Both faces' conditioning tests and vertex-hit screens must pass, and the
  // pair's angle test; the distance slots are updated exactly as two
  // strip_fast calls do (so a failed pair can redo the faces one by one).
#ifndef WV_STRIP_PAIR_ANGLE
#define WV_STRIP_PAIR_ANGLE 1
#endif
  static constexpr bool kPairAngle = WV_STRIP_PAIR_ANGLE;
  template <int PP>
  __device__ __forceinline__ static void restart_ab(const Rec& R, const Row& w, const F2* qz,
                                                    Slot* sA, Slot* sB) {
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 az = sub2(f2s(R.v0e.z), qz[pp]), bz = sub2(f2s(R.v1.z), qz[pp]);
      sA[pp].d = sqrt2(fma2(az, az, f2s(w.a2)));
      sB[pp].d = sqrt2(fma2(bz, bz, f2s(w.b2)));
      set_s(sA[pp], add2(sA[pp].d, sB[pp].d));
    }
  }
  // one face's alpha and 2 beta at point pair pp (strip_fast's operations)
  __device__ __forceinline__ static void ab_pp(const Rec& R, const Row& w, F2 qz, float kab,
                                               float kbc, float kca, Slot& sA, Slot& sB,
                                               Slot& sC, F2& alpha, F2& beta2, bool& cond) {
    const F2 cz = sub2(f2s(R.v2.z), qz);
    alpha = fma2(f2s(R.n.z), cz, f2s(w.alpha));
    const F2 lc = sqrt2(fma2(cz, cz, f2s(w.c2)));
    const F2 la = sA.d, lb = sB.d;
    const F2 sbc = add2(lb, lc), sca = add2(lc, la);
    const F2 x = mul2(mul2(sum_ab(sA, sB), sbc), sca);
    sC.d = lc;
    set_s(sB, sbc);
    const F2 lp = fma2(lc, f2s(kab), fma2(lb, f2s(kca), mul2(la, f2s(kbc))));
    beta2 = fma2(lp, f2s(0.875f), x);
    float x0, x1, l0, l1;
    split(x, x0, x1);
    split(lp, l0, l1);
    cond = cond && (l0 > -x0) && (l1 > -x1);
  }
  template <int PP>
  __device__ __forceinline__ static bool strip_pair_fast(const Rec& Ra, const Row& wa,
                                                         const Rec& Rb, const Row& wb,
                                                         const F2* qz, const Ctx& ctx,
                                                         Slot* s0, Slot* s1,
                                                         Slot* s2, Slot* s3, F2* tq, F2* tp) {
    // face a: slots (s0, s1) -> s2; face b: (s1, s2) -> s3 (= s0's storage).
    // Only for pairs that continue their strip (a restart takes strip_fast).
    const float kab_a = -fabsf(Ra.v1.w), kbc_a = -fabsf(Ra.v2.w), kca_a = -Ra.n.w;
    const float kab_b = -fabsf(Rb.v1.w), kbc_b = -fabsf(Rb.v2.w), kca_b = -Rb.n.w;
    constexpr float kC2 = 32.0f * 0.19669890403747559f, kC1 = 8.0f * -0.33331409096717834f;
    float ms = 0.0f;
    bool cond = true;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      F2 aa, ba, ab, bb;
      ab_pp(Ra, wa, qz[pp], kab_a, kbc_a, kca_a, s0[pp], s1[pp], s2[pp], aa, ba, cond);
      ab_pp(Rb, wb, qz[pp], kab_b, kbc_b, kca_b, s1[pp], s2[pp], s3[pp], ab, bb, cond);
      const F2 num = fma2(aa, bb, mul2(ab, ba));
      const F2 den = fma2(mul2(aa, ab), f2s(-4.0f), mul2(ba, bb));
      const F2 th = mul2(num, rcp2(den));  // T/2, T = tan(theta_a + theta_b)
      const F2 s4 = mul2(th, th);
      float u0, u1;
      split(s4, u0, u1);
      ms = fmaxf(ms, fmaxf(u0, u1));
      tq[pp] = th;
      tp[pp] = fma2(fma2(s4, f2s(kC2), f2s(kC1)), s4, f2s(2.0f));
    }
    const bool near = fminf(fminf(wa.a2, fminf(wa.b2, wa.c2)),
                            fminf(wb.a2, fminf(wb.b2, wb.c2))) < ctx.eps2;
    return ms < 1.0f / 256.0f && cond && !near;
  }
  // A face whose pairs are not all common: tail2 per lane, from squared
  // distances recomputed from the record (the row parts bitwise the carried
  // ones); returns the lanes for the fp64 path
  template <int PP>
  __device__ __forceinline__ static uint32_t strip_slow(const Rec& Rk, float qx, float qy,
                                                        const F2* qz, const Ctx& ctx, F2* tacc) {
    const Rec R = with_h(Rk);  // the face-ordered tail needs h itself
    Row w = row_c(R, qx, qy);
    row_ab(R, qx, qy, w.a2, w.b2);
    uint32_t rare = 0;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 az = sub2(f2s(R.v0e.z), qz[pp]), bz = sub2(f2s(R.v1.z), qz[pp]);
      const F2 cz = sub2(f2s(R.v2.z), qz[pp]);
      const F2 alpha = fma2(f2s(R.n.z), cz, f2s(w.alpha));
      rare |= tail2(R, alpha, fma2(az, az, f2s(w.a2)), fma2(bz, bz, f2s(w.b2)),
                    fma2(cz, cz, f2s(w.c2)), ctx, tacc[pp]) << (2 * pp);
    }
    return rare;
  }
  // strip records carry (16/7) h in the .w fields (flags in the sign bits);
  // the face-ordered paths (tail2, finish_len) take the record with h
  __device__ __forceinline__ static Rec with_h(const Rec& Rk) {
    Rec R = Rk;
    R.v1.w = fabsf(Rk.v1.w) * (7.0f / 16.0f);
    R.v2.w = fabsf(Rk.v2.w) * (7.0f / 16.0f);
    R.n.w = Rk.n.w * (7.0f / 16.0f);
    return R;
  }
  // point lists and unaligned ranges walk strip records face by face
  template <int PP>
  __device__ __forceinline__ static uint32_t face(const Rec& Rk, const F2* qx, const F2* qy,
                                                  const F2* qz, const Ctx& ctx, F2* tacc) {
    return ExactPol::face<PP>(with_h(Rk), qx, qy, qz, ctx, tacc);
  }
  // the fp64 path needs the face's own orientation (triple product): a
  // reflected window (v2.w < 0) swaps B and C back
  __device__ __forceinline__ static double rare(const Rec& R, float qx, float qy, float qz,
                                                double eps) {
    const bool refl = __float_as_int(R.v2.w) < 0;
    return exact_rare(R.v0e, refl ? R.v2 : R.v1, refl ? R.v1 : R.v2, qx, qy, qz, eps);
  }
};

struct SoftPol {
  using Rec = SoftRecF32;
  static constexpr int kTile = 256;
  static constexpr int kStages = 4;
  static constexpr int kConsumerWarps = 4;
  static constexpr int kThreads = kConsumerWarps * 32;
  static constexpr int kMinBlocks = 5;
  static constexpr int kMinBlocksRow = 5;
  static constexpr int kP = 8;
  static constexpr double kScale = 1.0 / (8.0 * kPi);
  static constexpr bool kStrip = false;
  static constexpr bool kPairFaces = false;
  struct Slot {};
  struct Ctx {
    float eps2;
  };
  __device__ static Ctx make_ctx(float eps) { return Ctx{eps * eps}; }
  __device__ __forceinline__ static uint32_t common2(const Rec& R, F2 qx, F2 qy, F2 qz,
                                                     const Ctx& ctx, F2& tacc) {
    // d = (c_hi - q) + c_lo (SoftRecF32)
    const F2 dx = add2(sub2(f2s(R.c.x), qx), f2s(lo_x(R)));
    const F2 dy = add2(sub2(f2s(R.c.y), qy), f2s(lo_y(R)));
    const F2 dz = add2(sub2(f2s(R.c.z), qz), f2s(lo_z(R)));
    const F2 r2 = dot2(dx, dy, dz, dx, dy, dz);
    const F2 s = fma2(f2s(R.n.y), dz, fma2(f2s(R.n.x), dy, mul2(f2s(R.c.w), dx)));
    return tail2(r2, s, ctx, tacc);
  }
  // Lattice rows: the x/y parts per face and row, from c_hi (r2, s) and from
  // c_hi + c_lo (r2c, sc).  A step whose points are all beyond the face's
  // near threshold (|d|^6 >= K2, SoftRecF32) takes the hi-only arithmetic
  // (the centroid's lo part changes such a term by < 2e-8); the rare steps
  // with a point nearer use the corrected d.
  struct Row {
    float dxh, dyh, r2, s, k2;
  };
  __device__ __forceinline__ static Row row(const Rec& R, float qx, float qy) {
    Row w;
    w.dxh = R.c.x - qx;
    w.dyh = R.c.y - qy;
    w.r2 = fmaf(w.dyh, w.dyh, w.dxh * w.dxh);
    w.s = fmaf(R.n.x, w.dyh, R.c.w * w.dxh);
    w.k2 = near_k2(R);
    return w;
  }
  // the corrected d (rare steps near a centroid)
  __device__ __forceinline__ static uint32_t common_row2(const Rec& R, const Row& w, F2 qz,
                                                         const Ctx& ctx, F2& tacc) {
    const float dx = w.dxh + lo_x(R), dy = w.dyh + lo_y(R);
    const float r2c = fmaf(dy, dy, dx * dx), sc = fmaf(R.n.x, dy, R.c.w * dx);
    const F2 dz = add2(sub2(f2s(R.c.z), qz), f2s(lo_z(R)));
    return tail2(fma2(dz, dz, f2s(r2c)), fma2(f2s(R.n.y), dz, f2s(sc)), ctx, tacc);
  }
  __device__ __forceinline__ static uint32_t tail2(F2 r2, F2 s, const Ctx& ctx, F2& tacc) {
    float r2l, r2h;
    split(r2, r2l, r2h);
    // |c - q| < eps: on a centroid, the face is skipped and the point flagged
    // (_kernels.py:150-152)
    const bool hl = r2l < ctx.eps2, hh = r2h < ctx.eps2;
    float rl, rh;
    split(rsqrt2(r2), rl, rh);
    const F2 rs = f2(hl ? 0.0f : rl, hh ? 0.0f : rh);
    tacc = fma2(s, mul2(rs, mul2(rs, rs)), tacc);
    return (hl ? 1u : 0u) | (hh ? 2u : 0u);
  }
  // All PP point pairs against one face.  The on-centroid test is done once
  // per face on the minimum r^2 of the thread's points (nearly every face is
  // far from every point): the common path has no per-lane selects, which
  // otherwise cost as many issue slots as the arithmetic (the soft term is
  // only ~7 FP32 ops + 1 MUFU per pair).
  template <int PP>
  __device__ __forceinline__ static uint32_t finish(const F2* r2, const F2* s, const Ctx& ctx,
                                                    F2* tacc) {
    float m = __int_as_float(0x7f800000);
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      float l, h;
      split(r2[pp], l, h);
      m = fminf(m, fminf(l, h));
    }
    if (m >= ctx.eps2) {
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) {
        const F2 rs = rsqrt2(r2[pp]);
        tacc[pp] = fma2(s[pp], mul2(rs, mul2(rs, rs)), tacc[pp]);
      }
      return 0u;
    }
    uint32_t rare = 0;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) rare |= tail2(r2[pp], s[pp], ctx, tacc[pp]) << (2 * pp);
    return rare;
  }
  template <int PP>
  __device__ __forceinline__ static uint32_t face_row(const Rec& R, const Row& w, const F2* qz,
                                                      const Ctx& ctx, F2* tacc) {
    F2 r2[PP], s[PP];
    float m = __int_as_float(0x7f800000);
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 dz = sub2(f2s(R.c.z), qz[pp]);
      r2[pp] = fma2(dz, dz, f2s(w.r2));
      s[pp] = fma2(f2s(R.n.y), dz, f2s(w.s));
      float l, h;
      split(r2[pp], l, h);
      m = fminf(m, fminf(l, h));
    }
    if (m * m * m >= w.k2 && m >= ctx.eps2) {  // every point far from the centroid
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) {
        const F2 rs = rsqrt2(r2[pp]);
        tacc[pp] = fma2(s[pp], mul2(rs, mul2(rs, rs)), tacc[pp]);
      }
      return 0u;
    }
    // rare: d with the centroid's lo part, per-lane on-centroid test
    uint32_t rare = 0;
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) rare |= common_row2(R, w, qz[pp], ctx, tacc[pp]) << (2 * pp);
    return rare;
  }
  template <int PP>
  __device__ __forceinline__ static uint32_t face(const Rec& R, const F2* qx, const F2* qy,
                                                  const F2* qz, const Ctx& ctx, F2* tacc) {
    F2 r2[PP], s[PP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      const F2 dx = add2(sub2(f2s(R.c.x), qx[pp]), f2s(lo_x(R)));
      const F2 dy = add2(sub2(f2s(R.c.y), qy[pp]), f2s(lo_y(R)));
      const F2 dz = add2(sub2(f2s(R.c.z), qz[pp]), f2s(lo_z(R)));
      r2[pp] = dot2(dx, dy, dz, dx, dy, dz);
      s[pp] = fma2(f2s(R.n.y), dz, fma2(f2s(R.n.x), dy, mul2(f2s(R.c.w), dx)));
    }
    return finish<PP>(r2, s, ctx, tacc);
  }
  __device__ __forceinline__ static double rare(const Rec&, float, float, float, double) {
    return __longlong_as_double(0x7ff8000000000000ll);  // always an on-surface (flagged) pair
  }
};
// Sum split partials in split order (deterministic), then W = sum * scale.
__global__ void finalize_theta_kernel(const double* __restrict__ part,
                                      const uint8_t* __restrict__ pflags, int splits,
                                      int64_t n_count, int policy, float* __restrict__ out_f32,
                                      uint8_t* __restrict__ flags, double scale) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n_count;
       l += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    uint8_t h = 0;
    for (int s = 0; s < splits; ++s) {
      acc += part[(int64_t)s * n_count + l];
      h |= pflags[(int64_t)s * n_count + l];
    }
    double w = acc * scale;
    if (h && policy == kPolicyHalf) w = 0.5;
    out_f32[l] = (float)w;
    if (flags) flags[l] = h;
  }
}

int launch_exact_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, int policy, float* out, uint8_t* flags,
                         void* workspace, size_t ws_bytes, int num_sms, cudaStream_t stream,
                         const Batch& bt) {
  return launch_fwd_f32<ExactPol>(packed, n_faces, ps, n_count, policy, out, flags, workspace,
                                  ws_bytes, num_sms, stream, bt);
}
int launch_exact_strip_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                               int64_t n_count, int policy, float* out, uint8_t* flags,
                               void* workspace, size_t ws_bytes, int num_sms,
                               cudaStream_t stream) {
  return launch_fwd_f32<ExactStripPol>(packed, n_faces, ps, n_count, policy, out, flags,
                                       workspace, ws_bytes, num_sms, stream, Batch{});
}
size_t exact_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch) {
  return FwdPlan<ExactPol>::workspace_bytes(n_faces, n_count, num_sms, batch);
}
int launch_soft_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, int policy, float* out, uint8_t* flags,
                        void* workspace, size_t ws_bytes, int num_sms, cudaStream_t stream,
                        const Batch& bt) {
  return launch_fwd_f32<SoftPol>(packed, n_faces, ps, n_count, policy, out, flags, workspace,
                                 ws_bytes, num_sms, stream, bt);
}
size_t exact_strip_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms) {
  return FwdPlan<ExactStripPol>::workspace_bytes(n_faces, n_count, num_sms, 1);
}
size_t soft_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch) {
  return FwdPlan<SoftPol>::workspace_bytes(n_faces, n_count, num_sms, batch);
}

}  // namespace wv
