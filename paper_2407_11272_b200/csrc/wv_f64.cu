// wv_f64.cu -- FP64 parity kernels (compiled with -fmad=false).
//
// These are the GPU twins of the reference's default-precision kernels,
// written in the reference's exact operation order so that the
// `precision="f64"` API path reproduces the reference to the last bit where
// the math library allows:
//   exact_fwd_f64  <- _kernels.exact_batch  (_kernels.py:34-116); identical
//                     except CUDA's atan2 vs libm's (<= 1-2 ulp per term)
//   soft_fwd_f64   <- _kernels.soft_batch   (_kernels.py:119-158); bit-exact
// Faces are streamed through the same TMA bulk-copy ring as the FP32 path and
// accumulated sequentially in face index order per point (no face splits), as
// the reference does.
#include "wv_kernels.h"

namespace wv {

constexpr int kF64Tile = 64;
constexpr int kF64Stages = 4;
constexpr int kF64ConsumerWarps = 4;
constexpr int kF64NC = kF64ConsumerWarps * 32;
constexpr int kF64Threads = kF64NC;
constexpr int kF64P = 1;
constexpr double kBaryTol = 1e-12;  // _kernels.py:31

// FP64 reciprocal / reciprocal square root without the IEEE slow-path
// branches of '/' and sqrt: the MUFU seed (rcp.approx.ftz.f64 /
// rsqrt.approx.ftz.f64, ~2^-22 relative) and two Newton steps (error ~2^-88
// before rounding: full f64 accuracy, within an ulp or two -- the parity
// tolerance is 1e-9).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // y <- y (3 - x y^2) / 2, twice
  double h = x * y;
  y = fma(y, fma(-h, y, 1.0) * 0.5, y);
  h = x * y;
  return fma(y, fma(-h, y, 1.0) * 0.5, y);
}

// |v| = v2 rsqrt(v2), 0 at the origin (the vertex-hit test needs the 0)
__device__ __forceinline__ double norm_nr(double v2) {
  return v2 > 0.0 ? v2 * rsqrt_nr(v2) : 0.0;
}

// One exact face term in the reference's operation order
// (_kernels.py:52-115).  The common pair -- a live face, no corner within
// eps, q off the face's plane band, |alpha| < beta/8 -- is decided by ONE
// predicate and evaluated branch-free (polynomial); everything else takes
// exact_f64_slow, the reference's tests in order.  Same results as the
// nested-branch form; far fewer divergent branches per pair.
__device__ __noinline__ void exact_f64_slow(const ExactRecF64& R, double ax, double ay,
                                            double az, double na, double nb, double nc,
                                            double pd, double alpha, double beta, double eps,
                                            int use_atan2, double& acc, bool& hit) {
  if (R.dead != 0.0) return;  // dropped by _prepare_exact
  if (na < eps || nb < eps || nc < eps) {
    hit = true;
    return;
  }
  const double* t = R.v;
  if (-eps < pd && pd < eps) {
    const double ux = t[3] - t[0], uy = t[4] - t[1], uz = t[5] - t[2];
    const double wx = t[6] - t[0], wy = t[7] - t[1], wz = t[8] - t[2];
    const double d00 = ux * ux + uy * uy + uz * uz;
    const double d01 = ux * wx + uy * wy + uz * wz;
    const double d11 = wx * wx + wy * wy + wz * wz;
    const double denom = d00 * d11 - d01 * d01;
    const double ru = -(ax * ux + ay * uy + az * uz);
    const double rw = -(ax * wx + ay * wy + az * wz);
    const double b1 = (d11 * ru - d01 * rw) / denom;
    const double b2 = (d00 * rw - d01 * ru) / denom;
    if (b1 >= -kBaryTol && b2 >= -kBaryTol && b1 + b2 <= 1.0 + kBaryTol) {
      hit = true;
      return;
    }
  }
  if (use_atan2) {
    acc += 2.0 * atan2(alpha, beta);
  } else {  // regression-demonstration branch, _kernels.py:106-114
    if (beta != 0.0)
      acc += 2.0 * atan(alpha / beta);
    else if (alpha > 0.0)
      acc += kPi;
    else if (alpha < 0.0)
      acc -= kPi;
  }
}

__device__ __forceinline__ void exact_f64_term(const ExactRecF64& R, double ax, double ay,
                                               double az, double bx, double by, double bz,
                                               double cx, double cy, double cz, double na,
                                               double nb, double nc, double qx, double qy,
                                               double qz, double eps, int use_atan2,
                                               double& acc, bool& hit) {
  const double pd = R.nhat[0] * qx + R.nhat[1] * qy + R.nhat[2] * qz - R.pld;
  const double alpha = (ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz)) +
                       az * (bx * cy - by * cx);
  const double beta = (na * (nb * nc) + (bx * cx + by * cy + bz * cz) * na) +
                      ((ax * bx + ay * by + az * bz) * nc + (cx * ax + cy * ay + cz * az) * nb);
  // atan2(alpha, beta) for |alpha| < beta/8 (nearly every pair of a fine
  // mesh): t = alpha/beta and the odd Taylor polynomial t (1 - s/3 + s^2/5
  // - ... + s^8/17), s = t^2 <= 1/64 (truncation < 2e-18 relative;
  // explicit fmas), a few ulp like libm's atan2 and exactly odd, so flipped
  // faces still negate exactly
  const bool common = use_atan2 && R.dead == 0.0 && na >= eps && nb >= eps && nc >= eps &&
                      !(-eps < pd && pd < eps) && fabs(alpha) * 8.0 < beta;
  if (common) {
    const double tt = alpha * rcp_nr(beta);  // (odd in alpha: flips negate exactly)
    const double ss = tt * tt;
    double p = 1.0 / 17.0;
    p = fma(p, ss, -1.0 / 15.0);
    p = fma(p, ss, 1.0 / 13.0);
    p = fma(p, ss, -1.0 / 11.0);
    p = fma(p, ss, 1.0 / 9.0);
    p = fma(p, ss, -1.0 / 7.0);
    p = fma(p, ss, 1.0 / 5.0);
    p = fma(p, ss, -1.0 / 3.0);
    p = fma(p * ss, tt, tt);  // t + t s P(s)
    acc += 2.0 * p;
  } else {
    exact_f64_slow(R, ax, ay, az, na, nb, nc, pd, alpha, beta, eps, use_atan2, acc, hit);
  }
}

struct ExactF64Pol {
  using Rec = ExactRecF64;
  static constexpr double kDiv = 4.0 * kPi;  // out = acc / _FOUR_PI
  __device__ __forceinline__ static void pair(const Rec& R, double qx, double qy, double qz,
                                              double eps, int use_atan2, double& acc,
                                              bool& hit) {
    const double* t = R.v;
    const double ax = t[0] - qx, ay = t[1] - qy, az = t[2] - qz;
    const double bx = t[3] - qx, by = t[4] - qy, bz = t[5] - qz;
    const double cx = t[6] - qx, cy = t[7] - qy, cz = t[8] - qz;
    const double na = norm_nr(ax * ax + ay * ay + az * az);
    const double nb = norm_nr(bx * bx + by * by + bz * bz);
    const double nc = norm_nr(cx * cx + cy * cy + cz * cz);
    exact_f64_term(R, ax, ay, az, bx, by, bz, cx, cy, cz, na, nb, nc, qx, qy, qz, eps,
                   use_atan2, acc, hit);
  }
};

struct SoftF64Pol {
  using Rec = SoftRecF64;
  static constexpr double kDiv = 8.0 * kPi;  // out = acc / _EIGHT_PI
  __device__ __forceinline__ static void pair(const Rec& R, double qx, double qy, double qz,
                                              double eps, int, double& acc, bool& hit) {
    const double dx = R.c[0] - qx, dy = R.c[1] - qy, dz = R.c[2] - qz;
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double r = sqrt(r2);
    if (r < eps) {
      hit = true;
      return;
    }
    acc += (R.n[0] * dx + R.n[1] * dy + R.n[2] * dz) / (r2 * r);
  }
};

template <class Pol, class Src>
__global__ void __launch_bounds__(kF64Threads, 6)
fwd_f64_kernel(const PackHeader* __restrict__ hdr, const typename Pol::Rec* __restrict__ recs,
               int64_t n_faces, Src src, int64_t n_count, int use_atan2, int policy,
               double* __restrict__ out, uint8_t* __restrict__ flags) {
  using Rec = typename Pol::Rec;
  __shared__ FaceRing<Rec, kF64Tile, kF64Stages> ring;
  const int64_t n_tiles = (n_faces + kF64Tile - 1) / kF64Tile;
  ring_start(ring, recs, n_faces, 0, n_tiles);
  const double eps = hdr->eps;
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * (kF64NC * kF64P);
  double qx[kF64P], qy[kF64P], qz[kF64P], acc[kF64P];
  bool hit[kF64P];
#pragma unroll
  for (int p = 0; p < kF64P; ++p) {
    int64_t l = base + p * kF64NC + tid;
    if (l >= n_count) l = n_count - 1;
    src.point(l, qx[p], qy[p], qz[p]);
    acc[p] = 0.0;
    hit[p] = false;
  }
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int s = (int)(t % kF64Stages);
    mbar_wait(&ring.full[s], (uint32_t)((t / kF64Stages) & 1));
    const int64_t first = t * kF64Tile;
    const int cnt = (int)((n_faces - first) < kF64Tile ? (n_faces - first) : kF64Tile);
    const Rec* tile = ring.tiles[s];
#pragma unroll 1
    for (int f = 0; f < cnt; ++f) {
      const Rec R = tile[f];
#pragma unroll
      for (int p = 0; p < kF64P; ++p) Pol::pair(R, qx[p], qy[p], qz[p], eps, use_atan2, acc[p], hit[p]);
    }
    __syncwarp();
    if ((tid & 31) == 0) ring_release(ring, s, kF64ConsumerWarps, recs, n_faces, t, n_tiles);
  }
#pragma unroll
  for (int p = 0; p < kF64P; ++p) {
    const int64_t l = base + p * kF64NC + tid;
    if (l < n_count) {
      double w = acc[p] / Pol::kDiv;
      if (hit[p] && policy == kPolicyHalf) w = 0.5;
      out[l] = w;
      if (flags) flags[l] = hit[p] ? 1 : 0;
    }
  }
}

template <class Pol>
static int launch_f64(const void* packed, int64_t n_faces, const PointSource& ps, int64_t n_count,
                      int use_atan2, int policy, double* out, uint8_t* flags,
                      cudaStream_t stream) {
  if (n_count <= 0) return kOk;
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const auto* recs = reinterpret_cast<const typename Pol::Rec*>(hdr + 1);
  const int64_t per_block = (int64_t)kF64NC * kF64P;
  const unsigned blocks = (unsigned)((n_count + per_block - 1) / per_block);
  if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    { fwd_f64_kernel<Pol, GridSrc><<<blocks, kF64Threads, 0, stream>>>(
        hdr, recs, n_faces, src, n_count, use_atan2, policy, out, flags); wv::note_launch(); }
  } else {
    ListSrc64 src{ps.points64};
    { fwd_f64_kernel<Pol, ListSrc64><<<blocks, kF64Threads, 0, stream>>>(
        hdr, recs, n_faces, src, n_count, use_atan2, policy, out, flags); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

// ---------------------------------------------------------------------------
// Strip-ordered f64 exact forward (records from pack_strip_f64_kernel): the
// reference's per-face term, bit for bit (true vertex order for alpha, beta
// and the on-surface tests), but the corner distances |v - q| of the strip's
// shared corners are carried between consecutive faces -- the same
// expression on the same coordinates, so the carried values are the ones the
// reference computes -- and a face costs one DP square root instead of
// three.  Only the order of the face sum differs from the index-order kernel
// (~1e-16 relative).
__device__ __forceinline__ double vdist(const double* v, double qx, double qy, double qz) {
  const double x = v[0] - qx, y = v[1] - qy, z = v[2] - qz;
  return norm_nr(x * x + y * y + z * z);
}
template <int kRot>
__device__ __forceinline__ void exact_f64_strip_face(const ExactRecF64& R, double qx, double qy,
                                                     double qz, double eps, int use_atan2,
                                                     double* d, double& acc, bool& hit) {
  const int code = (int)R.pad[1];
  const int iA = code % 3, iB = code / 3, iC = 3 - iA - iB;
  const double* t = R.v;
  if (R.pad[0] != 0.0) {
    d[kRot] = vdist(t + 3 * iA, qx, qy, qz);
    d[(kRot + 1) % 3] = vdist(t + 3 * iB, qx, qy, qz);
  }
  d[(kRot + 2) % 3] = vdist(t + 3 * iC, qx, qy, qz);
  // |v_k - q| in true corner order
  const double dA = d[kRot], dB = d[(kRot + 1) % 3], dC = d[(kRot + 2) % 3];
  const double na = iA == 0 ? dA : iB == 0 ? dB : dC;
  const double nb = iA == 1 ? dA : iB == 1 ? dB : dC;
  const double nc = iA == 2 ? dA : iB == 2 ? dB : dC;
  const double ax = t[0] - qx, ay = t[1] - qy, az = t[2] - qz;
  const double bx = t[3] - qx, by = t[4] - qy, bz = t[5] - qz;
  const double cx = t[6] - qx, cy = t[7] - qy, cz = t[8] - qz;
  // (a dead face is dropped by _prepare_exact; the carry still advanced)
  exact_f64_term(R, ax, ay, az, bx, by, bz, cx, cy, cz, na, nb, nc, qx, qy, qz, eps, use_atan2,
                 acc, hit);
}

template <class Src>
__global__ void __launch_bounds__(kF64Threads, 6)
fwd_f64_strip_kernel(const PackHeader* __restrict__ hdr, const ExactRecF64* __restrict__ recs,
                     int64_t n_faces, Src src, int64_t n_count, int use_atan2, int policy,
                     double* __restrict__ out, uint8_t* __restrict__ flags) {
  static_assert(kF64Tile == 64, "pack_strip_f64_kernel restarts a strip every 64 records");
  __shared__ FaceRing<ExactRecF64, kF64Tile, kF64Stages> ring;
  const int64_t n_tiles = (n_faces + kF64Tile - 1) / kF64Tile;
  ring_start(ring, recs, n_faces, 0, n_tiles);
  const double eps = hdr->eps;
  const int tid = threadIdx.x;
  int64_t l = (int64_t)blockIdx.x * kF64NC + tid;
  const int64_t lc = l < n_count ? l : n_count - 1;
  double qx, qy, qz;
  src.point(lc, qx, qy, qz);
  double acc = 0.0, d[3] = {0.0, 0.0, 0.0};
  bool hit = false;
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int s = (int)(t % kF64Stages);
    mbar_wait(&ring.full[s], (uint32_t)((t / kF64Stages) & 1));
    const int64_t first = t * kF64Tile;
    const int cnt = (int)((n_faces - first) < kF64Tile ? (n_faces - first) : kF64Tile);
    const ExactRecF64* tile = ring.tiles[s];
    int f = 0;
#pragma unroll 1
    for (; f + 3 <= cnt; f += 3) {
      exact_f64_strip_face<0>(tile[f], qx, qy, qz, eps, use_atan2, d, acc, hit);
      exact_f64_strip_face<1>(tile[f + 1], qx, qy, qz, eps, use_atan2, d, acc, hit);
      exact_f64_strip_face<2>(tile[f + 2], qx, qy, qz, eps, use_atan2, d, acc, hit);
    }
    if (f < cnt) exact_f64_strip_face<0>(tile[f], qx, qy, qz, eps, use_atan2, d, acc, hit);
    if (f + 1 < cnt)
      exact_f64_strip_face<1>(tile[f + 1], qx, qy, qz, eps, use_atan2, d, acc, hit);
    __syncwarp();
    if ((tid & 31) == 0) ring_release(ring, s, kF64ConsumerWarps, recs, n_faces, t, n_tiles);
  }
  if (l < n_count) {
    double w = acc / (4.0 * kPi);
    if (hit && policy == kPolicyHalf) w = 0.5;
    out[l] = w;
    if (flags) flags[l] = hit ? 1 : 0;
  }
}

int launch_exact_strip_fwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                               int64_t n_count, int use_atan2, int policy, double* out,
                               uint8_t* flags, cudaStream_t stream) {
  if (n_count <= 0) return kOk;
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const auto* recs = reinterpret_cast<const ExactRecF64*>(hdr + 1);
  const unsigned blocks = (unsigned)((n_count + kF64NC - 1) / kF64NC);
  if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    { fwd_f64_strip_kernel<GridSrc><<<blocks, kF64Threads, 0, stream>>>(
        hdr, recs, n_faces, src, n_count, use_atan2, policy, out, flags); wv::note_launch(); }
  } else {
    ListSrc64 src{ps.points64};
    { fwd_f64_strip_kernel<ListSrc64><<<blocks, kF64Threads, 0, stream>>>(
        hdr, recs, n_faces, src, n_count, use_atan2, policy, out, flags); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_exact_fwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, int use_atan2, int policy, double* out, uint8_t* flags,
                         cudaStream_t stream) {
  return launch_f64<ExactF64Pol>(packed, n_faces, ps, n_count, use_atan2, policy, out, flags,
                                 stream);
}

int launch_soft_fwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, int policy, double* out, uint8_t* flags,
                        cudaStream_t stream) {
  return launch_f64<SoftF64Pol>(packed, n_faces, ps, n_count, 1, policy, out, flags, stream);
}


// ---------------------------------------------------------------------------
// FP64 backward (parity path): same face-per-thread / point-broadcast mapping
// as wv_bwd_f32.cu, per-pair arithmetic in the reference's operation order.
constexpr int kBwd64Threads = 128;
constexpr int kBwd64Chunk = 256;
constexpr double kEightPi = 8.0 * kPi;

struct ExactBwd64 {
  using Rec = ExactGradRecF64;
  static constexpr int kOut = 9;
  static constexpr int kMinBlocks = 2;
  static constexpr int kUnroll = 1;
  // edge (Biot-Savart) form of d(Omega)/dv, see ExactEdgeBwd in wv_bwd_f32.cu;
  // coef carries the -1/(4 pi) factor.  Per pair: the three reciprocal corner
  // lengths once (Newton rsqrt), one Newton reciprocal per edge, no branches.
  // The reference has no exact gradient, so no operation order is pinned:
  // products and sums are fused explicitly (this file is built with
  // -fmad=false for the forwards' reference order).
  __device__ __forceinline__ static void edge(const double* a, const double* b, double la,
                                              double lb, double ia, double ib, double cw,
                                              double* gP, double* gQ) {
    const double m[3] = {fma(a[1], b[2], -a[2] * b[1]), fma(a[2], b[0], -a[0] * b[2]),
                         fma(a[0], b[1], -a[1] * b[0])};
    // |a||b| + a.b without cancellation next to the edge's segment (a.b < 0):
    // |a x b|^2 / (|a||b| - a.b), so cw / (|a||b| + a.b) = cw (|a||b| - a.b) / |a x b|^2
    const double L = la * lb, ab = fma(a[0], b[0], fma(a[1], b[1], a[2] * b[2]));
    const bool neg = ab < 0.0;
    const double num = neg ? cw * (L - ab) : cw;
    const double den = neg ? fma(m[0], m[0], fma(m[1], m[1], m[2] * m[2])) : L + ab;
    const double t = num * rcp_nr(den);
    if (cw == 0.0 || !(fabs(t) < INFINITY)) return;  // q on the segment: on-surface
    const double sp = t * ia, sq = t * ib;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      gP[d] = fma(m[d], sp, gP[d]);
      gQ[d] = fma(m[d], sq, gQ[d]);
    }
  }
  __device__ __forceinline__ static void pair(const Rec& R, double qx, double qy, double qz,
                                              double coef, double, double* g) {
    const double a[3] = {R.v[0] - qx, R.v[1] - qy, R.v[2] - qz};
    const double b[3] = {R.v[3] - qx, R.v[4] - qy, R.v[5] - qz};
    const double c[3] = {R.v[6] - qx, R.v[7] - qy, R.v[8] - qz};
    const double a2 = fma(a[0], a[0], fma(a[1], a[1], a[2] * a[2]));
    const double b2 = fma(b[0], b[0], fma(b[1], b[1], b[2] * b[2]));
    const double c2 = fma(c[0], c[0], fma(c[1], c[1], c[2] * c[2]));
    if (!(a2 > 0.0 && b2 > 0.0 && c2 > 0.0)) return;  // q on a vertex (flagged)
    const double ia = rsqrt_nr(a2), ib = rsqrt_nr(b2), ic = rsqrt_nr(c2);
    const double la = a2 * ia, lb = b2 * ib, lc = c2 * ic;
    edge(a, b, la, lb, ia, ib, coef * R.w[0], g + 0, g + 3);
    edge(b, c, lb, lc, ib, ic, coef * R.w[1], g + 3, g + 6);
    edge(c, a, lc, la, ic, ia, coef * R.w[2], g + 6, g + 0);
  }
};
// Edge trails (wv_trail.cu; the f32 kernel is ExactEdgeBwdTrail): one thread
// per window of K edges p0 -> .. -> pK of the f64 mesh; each position's
// reciprocal length serves both window edges at it, each distinct edge of
// the mesh is evaluated once (ExactBwd64::edge), and the signed CSR gather
// distributes the 2K end vectors to the vertex ids.  Per face of a closed
// surface: 1.5 edges and ~1.9 lengths instead of 3 and 3.
#ifndef WV_TRAIL64_MINB
#define WV_TRAIL64_MINB 3  // c3s f64 trail backward: 279 ms (3 CTAs/SM) vs 308 (2); unroll 2: 286-314
#endif
#ifndef WV_TRAIL64_UNROLL
#define WV_TRAIL64_UNROLL 1
#endif
struct ExactTrail64 {
  static constexpr int K = kTrailK;
  using Rec = TrailRecF64;
  static constexpr int kOut = 6 * K;
  static constexpr int kMinBlocks = WV_TRAIL64_MINB;
  static constexpr int kUnroll = WV_TRAIL64_UNROLL;  // points per loop body (ILP)
  __device__ __forceinline__ static void pair(const Rec& R, double qx, double qy, double qz,
                                              double coef, double, double* g) {
    double a[K + 1][3], l[K + 1], il[K + 1];
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      a[k][0] = R.p[k][0] - qx;
      a[k][1] = R.p[k][1] - qy;
      a[k][2] = R.p[k][2] - qz;
      const double a2 = fma(a[k][0], a[k][0], fma(a[k][1], a[k][1], a[k][2] * a[k][2]));
      if (!(a2 > 0.0)) return;  // q on a vertex (flagged; its coefficient is 0)
      il[k] = rsqrt_nr(a2);
      l[k] = a2 * il[k];
    }
#pragma unroll
    for (int e = 0; e < K; ++e)
      ExactBwd64::edge(a[e], a[e + 1], l[e], l[e + 1], il[e], il[e + 1], coef, g + 6 * e,
                       g + 6 * e + 3);
  }
};
struct SoftBwd64 {
  using Rec = SoftGradRecF64;
  static constexpr int kOut = 9;
  static constexpr int kMinBlocks = 2;
  static constexpr int kUnroll = 1;
  // _kernels.py:198-232, same expression order per pair
  __device__ __forceinline__ static void pair(const Rec& R, double qx, double qy, double qz,
                                              double coef, double eps, double* g) {
    const double dx = R.c[0] - qx, dy = R.c[1] - qy, dz = R.c[2] - qz;
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double r = sqrt(r2);
    if (r < eps) return;
    const double nx = R.n[0], ny = R.n[1], nz = R.n[2];
    const double s = nx * dx + ny * dy + nz * dz;
    const double inv3 = coef / (kEightPi * r2 * r);
    const double inv5 = coef * s / (kEightPi * r2 * r2 * r);
    const double ux = R.u[0], uy = R.u[1], uz = R.u[2];
    const double wx = R.w[0], wy = R.w[1], wz = R.w[2];
    const double g1x = wy * dz - wz * dy, g1y = wz * dx - wx * dz, g1z = wx * dy - wy * dx;
    const double g2x = dy * uz - dz * uy, g2y = dz * ux - dx * uz, g2z = dx * uy - dy * ux;
    const double n3x = nx / 3.0, n3y = ny / 3.0, n3z = nz / 3.0;
    g[0] += (-g1x - g2x + n3x) * inv3 - dx * inv5;
    g[1] += (-g1y - g2y + n3y) * inv3 - dy * inv5;
    g[2] += (-g1z - g2z + n3z) * inv3 - dz * inv5;
    g[3] += (g1x + n3x) * inv3 - dx * inv5;
    g[4] += (g1y + n3y) * inv3 - dy * inv5;
    g[5] += (g1z + n3z) * inv3 - dz * inv5;
    g[6] += (g2x + n3x) * inv3 - dx * inv5;
    g[7] += (g2y + n3y) * inv3 - dy * inv5;
    g[8] += (g2z + n3z) * inv3 - dz * inv5;
  }
};

template <class Pol, class Src>
__global__ void __launch_bounds__(kBwd64Threads, Pol::kMinBlocks)
bwd_f64_kernel(const PackHeader* __restrict__ hdr, const typename Pol::Rec* __restrict__ recs,
               int64_t n_faces, Src src, const double* __restrict__ coefs, int64_t n_count,
               int64_t pts_per_split, double coef_scale, double* __restrict__ out) {
  __shared__ double4 chunk[kBwd64Chunk];
  const int64_t f = (int64_t)blockIdx.x * kBwd64Threads + threadIdx.x;
  const bool live = f < n_faces;
  const typename Pol::Rec R = recs[live ? f : 0];
  const double eps = hdr->eps;
  const int64_t p_begin = (int64_t)blockIdx.y * pts_per_split;
  int64_t p_end = p_begin + pts_per_split;
  if (p_end > n_count) p_end = n_count;
  double g[Pol::kOut];
#pragma unroll
  for (int j = 0; j < Pol::kOut; ++j) g[j] = 0.0;
  for (int64_t c0 = p_begin; c0 < p_end; c0 += kBwd64Chunk) {
    const int n = (int)((p_end - c0) < kBwd64Chunk ? (p_end - c0) : kBwd64Chunk);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kBwd64Threads) {
      double x, y, z;
      src.point(c0 + i, x, y, z);
      chunk[i] = make_double4(x, y, z, coefs[c0 + i] * coef_scale);
    }
    __syncthreads();
    if constexpr (Pol::kUnroll > 1) {
      // chunk entries past n hold stale points: their coefficients are read
      // as 0 (the zero-coefficient skip of _kernels.py:182-184 is per point)
#pragma unroll 1
      for (int i = 0; i < n; i += Pol::kUnroll) {
#pragma unroll
        for (int u = 0; u < Pol::kUnroll; ++u) {
          const double4 q = chunk[i + u < n ? i + u : i];
          if (i + u < n && q.w != 0.0) Pol::pair(R, q.x, q.y, q.z, q.w, eps, g);
        }
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < n; ++i) {
        const double4 q = chunk[i];
        if (q.w == 0.0) continue;  // _kernels.py:182-184
        Pol::pair(R, q.x, q.y, q.z, q.w, eps, g);
      }
    }
  }
  if (live) {
    double* dst = out + ((int64_t)blockIdx.y * n_faces + f) * Pol::kOut;
    for (int j = 0; j < Pol::kOut; ++j) dst[j] = g[j];
  }
}

__global__ void reduce_splits64_kernel(const double* __restrict__ part, int splits, int64_t n,
                                       double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int s = 0; s < splits; ++s) a += part[(int64_t)s * n + i];
    out[i] = a;
  }
}

static void bwd64_plan(int64_t n_faces, int64_t n_count, int num_sms, int64_t* bx, int* splits,
                       int64_t* pps) {
  *bx = (n_faces + kBwd64Threads - 1) / kBwd64Threads;
  if (*bx < 1) *bx = 1;
  const int64_t want = (int64_t)num_sms * 8;
  int64_t s = (want + *bx - 1) / *bx;
  const int64_t max_s = (n_count + kBwd64Chunk - 1) / kBwd64Chunk;
  if (s > max_s) s = max_s;
  if (s > 4096) s = 4096;
  if (s < 1) s = 1;
  *pps = ((n_count + s - 1) / s + kBwd64Chunk - 1) / kBwd64Chunk * kBwd64Chunk;
  *splits = (int)((n_count + *pps - 1) / *pps);
  if (*splits < 1) *splits = 1;
}

static size_t bwd64_ws(int64_t n_faces, int64_t n_count, int num_sms, int k_out) {
  int64_t bx, pps;
  int s;
  bwd64_plan(n_faces, n_count, num_sms, &bx, &s, &pps);
  return s > 1 ? (size_t)s * n_faces * k_out * sizeof(double) : 0;
}
size_t bwd64_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms) {
  return bwd64_ws(n_faces, n_count, num_sms, 9);
}
size_t exact_trail_bwd64_workspace_bytes(int64_t n_windows, int64_t n_count, int num_sms) {
  return bwd64_ws(n_windows, n_count, num_sms, ExactTrail64::kOut);
}

template <class Pol>
static int launch_bwd64(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, const double* coefs, double coef_scale,
                        double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                        cudaStream_t stream) {
  constexpr int KO = Pol::kOut;
  if (n_faces <= 0) return kOk;
  if (n_count <= 0)
    return cudaMemsetAsync(face_grad, 0, (size_t)n_faces * KO * sizeof(double), stream) ==
                   cudaSuccess ? kOk : kErrCuda;
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const auto* recs = reinterpret_cast<const typename Pol::Rec*>(hdr + 1);
  int64_t bx, pps;
  int splits;
  bwd64_plan(n_faces, n_count, num_sms, &bx, &splits, &pps);
  double* dst = face_grad;
  if (splits > 1) {
    if (ws == nullptr || ws_bytes < (size_t)splits * n_faces * KO * sizeof(double))
      return kErrWorkspace;
    dst = static_cast<double*>(ws);
  }
  dim3 grid((unsigned)bx, (unsigned)splits);
  if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    { bwd_f64_kernel<Pol, GridSrc><<<grid, kBwd64Threads, 0, stream>>>(hdr, recs, n_faces, src,
                                                                     coefs, n_count, pps,
                                                                     coef_scale, dst); wv::note_launch(); }
  } else {
    ListSrc64 src{ps.points64};
    { bwd_f64_kernel<Pol, ListSrc64><<<grid, kBwd64Threads, 0, stream>>>(hdr, recs, n_faces, src,
                                                                       coefs, n_count, pps,
                                                                       coef_scale, dst); wv::note_launch(); }
  }
  if (splits > 1) {
    const int64_t n = n_faces * KO;
    int blocks = (int)((n + 255) / 256);
    if (blocks > num_sms * 8) blocks = num_sms * 8;
    { reduce_splits64_kernel<<<blocks, 256, 0, stream>>>(dst, splits, n, face_grad); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_exact_bwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, const double* coefs, double coef_scale,
                         double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                         cudaStream_t stream) {
  return launch_bwd64<ExactBwd64>(packed, n_faces, ps, n_count, coefs,
                                  coef_scale * (-1.0 / (4.0 * kPi)), face_grad,
                                  ws, ws_bytes, num_sms, stream);
}
int launch_exact_trail_bwd_f64(const void* packed, int64_t n_windows, const PointSource& ps,
                               int64_t n_count, const double* coefs, double coef_scale,
                               double* out, void* ws, size_t ws_bytes, int num_sms,
                               cudaStream_t stream) {
  return launch_bwd64<ExactTrail64>(packed, n_windows, ps, n_count, coefs,
                                    coef_scale * (-1.0 / (4.0 * kPi)), out, ws, ws_bytes,
                                    num_sms, stream);
}
int launch_soft_bwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, const double* coefs, double coef_scale,
                        double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                        cudaStream_t stream) {
  return launch_bwd64<SoftBwd64>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad,
                                 ws, ws_bytes, num_sms, stream);
}

}  // namespace wv
