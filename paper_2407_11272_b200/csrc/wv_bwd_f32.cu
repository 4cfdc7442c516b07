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
// Exact  (NEW, no reference kernel; closed form SURVEY.md A.4):
//   dW/dv_k = 1/(2 pi) (beta dalpha/dv_k - alpha dbeta/dv_k) / (alpha^2+beta^2)
// Soft   (replaces _kernels.soft_grad_accum, _kernels.py:161-232):
//   dW/dv_k = [(G_k + N/3) / r^3 - S d / r^5] / (8 pi),  G_1 = w x d,
//   G_2 = d x u, G_0 = -G_1 - G_2; the N/3 and d terms are shared by the three
//   corners, so they are accumulated once per face.
// Per-chunk fp32 partials are folded into fp64 accumulators.
#include "wv_kernels.h"

namespace wv {

constexpr int kBwdThreads = 128;   // faces per CTA
constexpr int kBwdChunk = 256;     // query points per shared-memory chunk

// Rare exact pair: plane distance below eps.  Returns 1 to keep the pair, 0
// when the forward skipped it (on-surface, _kernels.py:65-88, or a dead face).
__device__ __noinline__ float exact_keep(float4 A, float4 B, float4 C, float qx, float qy,
                                         float qz, float eps) {
  if (A.w == __int_as_float(0x7f800000)) return 0.0f;
  const float ax = A.x - qx, ay = A.y - qy, az = A.z - qz;
  const float bx = B.x - qx, by = B.y - qy, bz = B.z - qz;
  const float cx = C.x - qx, cy = C.y - qy, cz = C.z - qz;
  const float la = sqrt_approx(fmaf(az, az, fmaf(ay, ay, ax * ax)));
  const float lb = sqrt_approx(fmaf(bz, bz, fmaf(by, by, bx * bx)));
  const float lc = sqrt_approx(fmaf(cz, cz, fmaf(cy, cy, cx * cx)));
  if (la < eps || lb < eps || lc < eps) return 0.0f;
  const float ux = B.x - A.x, uy = B.y - A.y, uz = B.z - A.z;
  const float wx = C.x - A.x, wy = C.y - A.y, wz = C.z - A.z;
  const float d00 = fmaf(uz, uz, fmaf(uy, uy, ux * ux));
  const float d01 = fmaf(uz, wz, fmaf(uy, wy, ux * wx));
  const float d11 = fmaf(wz, wz, fmaf(wy, wy, wx * wx));
  const float denom = __fsub_rn(__fmul_rn(d00, d11), __fmul_rn(d01, d01));
  const float ru = -fmaf(az, uz, fmaf(ay, uy, ax * ux));
  const float rw = -fmaf(az, wz, fmaf(ay, wy, ax * wx));
  const float b1 = __fdiv_rn(__fsub_rn(__fmul_rn(d11, ru), __fmul_rn(d01, rw)), denom);
  const float b2 = __fdiv_rn(__fsub_rn(__fmul_rn(d00, rw), __fmul_rn(d01, ru)), denom);
  const float btol = 1e-12f;
  return (b1 >= -btol && b2 >= -btol && b1 + b2 <= 1.0f + btol) ? 0.0f : 1.0f;
}

struct ExactBwd {
  using Rec = ExactRecF32;
  static constexpr int kMinBlocks = 4;
  static constexpr double kCoefScale = 1.0 / (2.0 * kPi);
  static constexpr int kAcc = 9;
  __device__ __forceinline__ static void pair(const Rec& R, float qx, float qy, float qz,
                                              float coef, float eps, float eps2, float* g) {
    const float ax = R.v0e.x - qx, ay = R.v0e.y - qy, az = R.v0e.z - qz;
    const float bx = R.v1.x - qx, by = R.v1.y - qy, bz = R.v1.z - qz;
    const float cx = R.v2.x - qx, cy = R.v2.y - qy, cz = R.v2.z - qz;
    const float la2 = fmaf(az, az, fmaf(ay, ay, ax * ax));
    const float lb2 = fmaf(bz, bz, fmaf(by, by, bx * bx));
    const float lc2 = fmaf(cz, cz, fmaf(cy, cy, cx * cx));
    const float ia = rsqrt_approx(la2), ib = rsqrt_approx(lb2), ic = rsqrt_approx(lc2);
    const float la = la2 * ia, lb = lb2 * ib, lc = lc2 * ic;
    const float alpha = fmaf(R.n.z, az, fmaf(R.n.y, ay, R.n.x * ax));
    const float ab = fmaf(az, bz, fmaf(ay, by, ax * bx));
    const float bc = fmaf(bz, cz, fmaf(by, cy, bx * cx));
    const float ca = fmaf(az, cz, fmaf(ay, cy, ax * cx));
    const float lblc = lb * lc;
    const float beta = fmaf(ca, lb, fmaf(ab, lc, fmaf(bc, la, la * lblc)));
    float s = coef * rcp_approx(fmaf(alpha, alpha, beta * beta));
    if (fabsf(alpha) < R.v0e.w && exact_keep(R.v0e, R.v1, R.v2, qx, qy, qz, eps) == 0.0f)
      s = 0.0f;  // pair skipped by the forward's on-surface policy
    const float ga = s * beta;   // d theta / d alpha
    const float gb = -s * alpha; // d theta / d beta
    const float ka = (lblc + bc) * ia;
    const float kb = fmaf(la, lc, ca) * ib;
    const float kc = fmaf(la, lb, ab) * ic;
    // d alpha / d v0 = b x c, / d v1 = c x a, / d v2 = a x b
    const float x0 = by * cz - bz * cy, y0 = bz * cx - bx * cz, z0 = bx * cy - by * cx;
    const float x1 = cy * az - cz * ay, y1 = cz * ax - cx * az, z1 = cx * ay - cy * ax;
    const float x2 = ay * bz - az * by, y2 = az * bx - ax * bz, z2 = ax * by - ay * bx;
    // d beta / d a = ka a + lc b + lb c ; / d b = lc a + kb b + la c ;
    // d beta / d c = lb a + la b + kc c
    const float A0 = gb * ka, Bc = gb * lc, Cb = gb * lb, A1 = gb * kb, Da = gb * la,
                A2 = gb * kc;
    g[0] = fmaf(ga, x0, fmaf(Cb, cx, fmaf(Bc, bx, fmaf(A0, ax, g[0]))));
    g[1] = fmaf(ga, y0, fmaf(Cb, cy, fmaf(Bc, by, fmaf(A0, ay, g[1]))));
    g[2] = fmaf(ga, z0, fmaf(Cb, cz, fmaf(Bc, bz, fmaf(A0, az, g[2]))));
    g[3] = fmaf(ga, x1, fmaf(Da, cx, fmaf(A1, bx, fmaf(Bc, ax, g[3]))));
    g[4] = fmaf(ga, y1, fmaf(Da, cy, fmaf(A1, by, fmaf(Bc, ay, g[4]))));
    g[5] = fmaf(ga, z1, fmaf(Da, cz, fmaf(A1, bz, fmaf(Bc, az, g[5]))));
    g[6] = fmaf(ga, x2, fmaf(A2, cx, fmaf(Da, bx, fmaf(Cb, ax, g[6]))));
    g[7] = fmaf(ga, y2, fmaf(A2, cy, fmaf(Da, by, fmaf(Cb, ay, g[7]))));
    g[8] = fmaf(ga, z2, fmaf(A2, cz, fmaf(Da, bz, fmaf(Cb, az, g[8]))));
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
#pragma unroll 2
    for (int i = 0; i < n; ++i) {
      const float4 q = chunk[i];
      if (q.w == 0.0f) continue;  // warp-uniform: every lane reads the same point
      Pol::pair(R, q.x, q.y, q.z, q.w, eps, eps2, g);
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
  return launch_bwd<ExactBwd>(packed, n_faces, ps, n_count, coefs, coef_scale, face_grad, ws,
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
