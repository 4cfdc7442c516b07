// wv_bwd_f32.cu -- FP32 backward kernels: per-face vertex gradients of the
// exact and soft winding numbers, reduced over query points.
//
// Mapping (the transpose of the forward): every thread OWNS one face and keeps
// its 9 gradient partials in registers; the CTA streams chunks of query
// points (coordinates + coefficient) through shared memory, so every warp
// reads the same point at the same time (broadcast LDS) and the per-point
// "coef == 0" skip of the reference (_kernels.py:182-184) is warp-uniform.
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
// Per-chunk fp32 partials are folded into fp64 accumulators.
#include "wv_kernels.h"

namespace wv {

constexpr int kBwdThreads = 128;   // faces per CTA
constexpr int kBwdChunk = 256;     // query points per shared-memory chunk

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
struct ExactEdgeBwd {
  using Rec = ExactGradRecF32;
  static constexpr int kMinBlocks = 4;
  // -1/(4 pi) and the factor 2 of d = 2 (|a||b| + a.b) below
  static constexpr double kCoefScale = -2.0 / (4.0 * kPi);
  static constexpr int kAcc = 9;
  __device__ __forceinline__ static bool unit_weights(const Rec& R) {
    return R.a.w == 1.0f && R.b.w == 1.0f && R.c.w == 1.0f;
  }
  // |a||b| + a.b = ((|a|+|b|)^2 - |P-Q|^2) / 2 (a.b = (|a|^2+|b|^2-|a-b|^2)/2,
  // a-b = P-Q): no dot products, one FADD + one FFMA per edge, and the FFMA
  // rounds (|a|+|b|)^2 - U once.
  template <bool kUnit>
  __device__ __forceinline__ static void pair(const Rec& R, float qx, float qy, float qz,
                                              float coef, float, float, float* g) {
    const float ax = R.a.x - qx, ay = R.a.y - qy, az = R.a.z - qz;
    const float bx = R.b.x - qx, by = R.b.y - qy, bz = R.b.z - qz;
    const float cx = R.c.x - qx, cy = R.c.y - qy, cz = R.c.z - qz;
    const float a2 = fmaf(az, az, fmaf(ay, ay, ax * ax));
    const float b2 = fmaf(bz, bz, fmaf(by, by, bx * bx));
    const float c2 = fmaf(cz, cz, fmaf(cy, cy, cx * cx));
    const float ia = rsqrt_approx(a2), ib = rsqrt_approx(b2), ic = rsqrt_approx(c2);
    const float lb = b2 * ib, lc = c2 * ic;
    const float s01 = fmaf(a2, ia, lb), s12 = lb + lc, s20 = fmaf(a2, ia, lc);
    const float r01 = rcp_approx(fmaf(s01, s01, -R.u.x));
    const float r12 = rcp_approx(fmaf(s12, s12, -R.u.y));
    const float r20 = rcp_approx(fmaf(s20, s20, -R.u.z));
    const float t01 = (kUnit ? coef : coef * R.a.w) * r01;
    const float t12 = (kUnit ? coef : coef * R.b.w) * r12;
    const float t20 = (kUnit ? coef : coef * R.c.w) * r20;
    // m01 = a x b, m12 = b x c, m20 = c x a
    const float m01x = ay * bz - az * by, m01y = az * bx - ax * bz, m01z = ax * by - ay * bx;
    const float m12x = by * cz - bz * cy, m12y = bz * cx - bx * cz, m12z = bx * cy - by * cx;
    const float m20x = cy * az - cz * ay, m20y = cz * ax - cx * az, m20z = cx * ay - cy * ax;
    const float s01a = t01 * ia, s20a = t20 * ia;  // v0 is P of 01, Q of 20
    const float s01b = t01 * ib, s12b = t12 * ib;  // v1 is Q of 01, P of 12
    const float s12c = t12 * ic, s20c = t20 * ic;  // v2 is Q of 12, P of 20
    g[0] = fmaf(m20x, s20a, fmaf(m01x, s01a, g[0]));
    g[1] = fmaf(m20y, s20a, fmaf(m01y, s01a, g[1]));
    g[2] = fmaf(m20z, s20a, fmaf(m01z, s01a, g[2]));
    g[3] = fmaf(m12x, s12b, fmaf(m01x, s01b, g[3]));
    g[4] = fmaf(m12y, s12b, fmaf(m01y, s01b, g[4]));
    g[5] = fmaf(m12z, s12b, fmaf(m01z, s01b, g[5]));
    g[6] = fmaf(m20x, s20c, fmaf(m12x, s12c, g[6]));
    g[7] = fmaf(m20y, s20c, fmaf(m12y, s12c, g[7]));
    g[8] = fmaf(m20z, s20c, fmaf(m12z, s12c, g[8]));
  }
  __device__ __forceinline__ static void finish(const Rec&, const double* acc, double* out9) {
    for (int j = 0; j < 9; ++j) out9[j] = acc[j];
  }
};

struct SoftBwd {
  using Rec = SoftGradRecF32;
  static constexpr int kMinBlocks = 4;
  static constexpr double kCoefScale = 1.0 / (8.0 * kPi);
  static constexpr int kAcc = 10;  // acc1(3) acc2(3) T(1) D(3)
  __device__ __forceinline__ static bool unit_weights(const Rec&) { return true; }
  template <bool kUnit>
  __device__ __forceinline__ static void pair(const Rec& R, float qx, float qy, float qz,
                                              float coef, float, float eps2, float* g) {
    const float dx = R.c.x - qx, dy = R.c.y - qy, dz = R.c.z - qz;
    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    const float rs = rsqrt_approx(r2);
    const float S = fmaf(R.n.z, dz, fmaf(R.n.y, dy, R.n.x * dx));
    const float rs2 = rs * rs;
    const float c3 = (r2 < eps2) ? 0.0f : coef * rs2 * rs;  // r < eps: skipped (:203-204)
    const float c5 = c3 * S * rs2;
    // G1 = w x d, G2 = d x u
    const float g1x = R.w.y * dz - R.w.z * dy, g1y = R.w.z * dx - R.w.x * dz,
                g1z = R.w.x * dy - R.w.y * dx;
    const float g2x = dy * R.u.z - dz * R.u.y, g2y = dz * R.u.x - dx * R.u.z,
                g2z = dx * R.u.y - dy * R.u.x;
    g[0] = fmaf(c3, g1x, g[0]);
    g[1] = fmaf(c3, g1y, g[1]);
    g[2] = fmaf(c3, g1z, g[2]);
    g[3] = fmaf(c3, g2x, g[3]);
    g[4] = fmaf(c3, g2y, g[4]);
    g[5] = fmaf(c3, g2z, g[5]);
    g[6] += c3;
    g[7] = fmaf(c5, dx, g[7]);
    g[8] = fmaf(c5, dy, g[8]);
    g[9] = fmaf(c5, dz, g[9]);
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

template <class Pol, bool kUnit>
__device__ __forceinline__ void chunk_loop(const typename Pol::Rec& R, const float4* chunk, int n,
                                           float eps, float eps2, float* g) {
#pragma unroll 2
  for (int i = 0; i < n; ++i) {
    const float4 q = chunk[i];
    if (q.w == 0.0f) continue;  // warp-uniform: every lane reads the same point
    Pol::template pair<kUnit>(R, q.x, q.y, q.z, q.w, eps, eps2, g);
  }
}

template <class Pol, class Src>
__global__ void __launch_bounds__(kBwdThreads, Pol::kMinBlocks)
bwd_f32_kernel(const PackHeader* __restrict__ hdr, const typename Pol::Rec* __restrict__ recs,
               int64_t n_faces, Src src, const float* __restrict__ coefs, int64_t n_count,
               int64_t pts_per_split, float coef_scale, double* __restrict__ out) {
  __shared__ float4 chunk[kBwdChunk];
  const int64_t f = (int64_t)blockIdx.x * kBwdThreads + threadIdx.x;
  const bool live = f < n_faces;
  typename Pol::Rec R = recs[live ? f : 0];
  const float eps = hdr->eps_f32;
  const float eps2 = eps * eps;
  const int64_t p_begin = (int64_t)blockIdx.y * pts_per_split;
  int64_t p_end = p_begin + pts_per_split;
  if (p_end > n_count) p_end = n_count;

  // warp-uniform fast path when every face of the warp has unit edge
  // weights (soups, boundary strips): saves the per-edge weight multiply
  const bool unit = __all_sync(0xffffffffu, Pol::unit_weights(R));
  double acc[Pol::kAcc];
#pragma unroll
  for (int j = 0; j < Pol::kAcc; ++j) acc[j] = 0.0;

  for (int64_t c0 = p_begin; c0 < p_end; c0 += kBwdChunk) {
    const int n = (int)((p_end - c0) < kBwdChunk ? (p_end - c0) : kBwdChunk);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kBwdThreads) {
      float x, y, z;
      src.point(c0 + i, x, y, z);
      chunk[i] = make_float4(x, y, z, coefs[c0 + i] * coef_scale);
    }
    __syncthreads();
    float g[Pol::kAcc];
#pragma unroll
    for (int j = 0; j < Pol::kAcc; ++j) g[j] = 0.0f;
    if (unit) {
      chunk_loop<Pol, true>(R, chunk, n, eps, eps2, g);
    } else {
      chunk_loop<Pol, false>(R, chunk, n, eps, eps2, g);
    }
#pragma unroll
    for (int j = 0; j < Pol::kAcc; ++j) acc[j] += (double)g[j];
  }
  if (live) {
    double o9[9];
    Pol::finish(R, acc, o9);
    double* dst = out + ((int64_t)blockIdx.y * n_faces + f) * 9;
#pragma unroll
    for (int j = 0; j < 9; ++j) dst[j] = o9[j];
  }
}

// out[f*9+j] = sum_s part[s][f*9+j], fixed split order
__global__ void reduce_splits_kernel(const double* __restrict__ part, int splits, int64_t n,
                                     double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int s = 0; s < splits; ++s) a += part[(int64_t)s * n + i];
    out[i] = a;
  }
}

struct BwdPlan {
  int64_t blocks_x = 0;
  int splits = 1;
  int64_t pts_per_split = 0;
  static BwdPlan make(int64_t n_faces, int64_t n_count, int num_sms, int min_blocks) {
    BwdPlan p;
    p.blocks_x = (n_faces + kBwdThreads - 1) / kBwdThreads;
    if (p.blocks_x < 1) p.blocks_x = 1;
    const int64_t want = (int64_t)num_sms * min_blocks * 4;  // ~4 waves for balance
    int64_t s = (want + p.blocks_x - 1) / p.blocks_x;
    const int64_t max_s = (n_count + kBwdChunk - 1) / kBwdChunk;  // >= one chunk per split
    if (s > max_s) s = max_s;
    if (s > 4096) s = 4096;
    if (s < 1) s = 1;
    p.pts_per_split = (n_count + s - 1) / s;
    p.pts_per_split = ((p.pts_per_split + kBwdChunk - 1) / kBwdChunk) * kBwdChunk;
    p.splits = (int)((n_count + p.pts_per_split - 1) / p.pts_per_split);
    if (p.splits < 1) p.splits = 1;
    return p;
  }
  size_t workspace(int64_t n_faces) const {
    return splits > 1 ? (size_t)splits * (size_t)n_faces * 9 * sizeof(double) : 0;
  }
};

template <class Pol>
static int launch_bwd(const void* packed, int64_t n_faces, const PointSource& ps,
                      int64_t n_count, const float* coefs, double coef_scale, double* face_grad,
                      void* workspace, size_t ws_bytes, int num_sms, cudaStream_t stream) {
  if (n_faces <= 0) return kOk;
  if (n_count <= 0) {
    return cudaMemsetAsync(face_grad, 0, (size_t)n_faces * 9 * sizeof(double), stream) ==
                   cudaSuccess ? kOk : kErrCuda;
  }
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const auto* recs = reinterpret_cast<const typename Pol::Rec*>(hdr + 1);
  const BwdPlan pl = BwdPlan::make(n_faces, n_count, num_sms, Pol::kMinBlocks);
  double* dst = face_grad;
  if (pl.splits > 1) {
    if (workspace == nullptr || ws_bytes < pl.workspace(n_faces)) return kErrWorkspace;
    dst = static_cast<double*>(workspace);
  }
  const float cs = (float)(coef_scale * Pol::kCoefScale);
  dim3 grid((unsigned)pl.blocks_x, (unsigned)pl.splits);
  if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    bwd_f32_kernel<Pol, GridSrc><<<grid, kBwdThreads, 0, stream>>>(
        hdr, recs, n_faces, src, coefs, n_count, pl.pts_per_split, cs, dst);
  } else {
    ListSrc src{ps.points};
    bwd_f32_kernel<Pol, ListSrc><<<grid, kBwdThreads, 0, stream>>>(
        hdr, recs, n_faces, src, coefs, n_count, pl.pts_per_split, cs, dst);
  }
  if (pl.splits > 1) {
    const int64_t n = n_faces * 9;
    int blocks = (int)((n + 255) / 256);
    if (blocks > num_sms * 8) blocks = num_sms * 8;
    reduce_splits_kernel<<<blocks, 256, 0, stream>>>(dst, pl.splits, n, face_grad);
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_exact_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, const float* coefs, double coef_scale,
                         double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                         cudaStream_t stream) {
  return launch_bwd<ExactEdgeBwd>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad, ws,
                              ws_bytes, num_sms, stream);
}
int launch_soft_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, const float* coefs, double coef_scale,
                        double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                        cudaStream_t stream) {
  return launch_bwd<SoftBwd>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad, ws,
                             ws_bytes, num_sms, stream);
}
size_t bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms) {
  return BwdPlan::make(n_faces, n_count, num_sms, 4).workspace(n_faces);
}

// ---------------------------------------------------------------------------
// face corners -> vertices, CSR order (deterministic); optional device scale
// (e.g. 1/sum(w) of the loss, read on the device so nothing syncs the host).
__global__ void face_to_vertex_kernel(const double* __restrict__ face_grad,
                                      const int64_t* __restrict__ off,
                                      const int64_t* __restrict__ slots, int64_t n_verts,
                                      const double* __restrict__ scale, int accumulate,
                                      double* __restrict__ out64, float* __restrict__ out32) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_verts;
       v += (int64_t)gridDim.x * blockDim.x) {
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      const double* src = face_grad + slots[e] * 3;  // slot = f*3 + corner
      gx += src[0];
      gy += src[1];
      gz += src[2];
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
  face_to_vertex_kernel<<<blocks, 256, 0, stream>>>(face_grad, off, slots, n_verts, scale,
                                                    accumulate, out64, out32);
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
