// wv_exact_fwd.cu -- FP32 exact generalized-winding-number forward (sm_100a).
//
// Replaces the reference hot loop _kernels.py:34-116 (exact_batch) and its
// f32 twin _kernels.py:235-309.  N-body style all-pairs reduction:
//   * one producer warp per CTA streams 128-face tiles of the packed face
//     array (ExactRecF32, 64 B) into a 4-stage shared-memory ring with TMA
//     bulk copies (cp.async.bulk + mbarrier complete_tx);
//   * every consumer thread keeps P query points in registers and walks the
//     tiles in face order; per pair it evaluates the Van Oosterom-Strackee
//     half angle theta = atan2(alpha, beta) (Omega = 2 theta) with
//     alpha = N.(v0-q) and the reference's beta grouping;
//   * common pairs (beta > |alpha|, not near the face plane) take a branch-
//     free path: one MUFU.RCP + an 8-term minimax polynomial;  near-plane or
//     wide-angle pairs take the rare path (on-surface test of
//     _kernels.py:65-88, full-range atan2);
//   * each tile's terms are summed in fp32 and tile partials in fp64, which
//     keeps 100k-1M face sums inside the 1e-5 tolerance.
// W = sum(theta)/(2 pi).  Flagged (on-surface) pairs contribute nothing and
// flag the point, exactly as the reference.
#include "wv_common.cuh"
#include "wv_kernels.h"

namespace wv {

constexpr int kExactTile = 128;
constexpr int kExactStages = 4;
constexpr int kExactConsumerWarps = 4;
constexpr int kExactConsumers = kExactConsumerWarps * 32;
constexpr int kExactThreads = kExactConsumers + 32;
constexpr int kExactP = 8;  // query points per consumer thread

// Rare path, evaluated out of the hot loop for the few pairs whose plane
// distance is below eps (on-surface candidates, _kernels.py:65-88) or whose
// half angle exceeds pi/4 (|alpha| > beta, incl. beta < 0).  Recomputes the
// pair from scratch; returns theta, or NaN for an on-surface (flagged) pair.
__device__ __noinline__ float exact_rare(float4 A, float4 B, float4 C, float4 N, float qx,
                                         float qy, float qz, float eps) {
  const float ax = A.x - qx, ay = A.y - qy, az = A.z - qz;
  const float bx = B.x - qx, by = B.y - qy, bz = B.z - qz;
  const float cx = C.x - qx, cy = C.y - qy, cz = C.z - qz;
  const float alpha = fmaf(N.z, az, fmaf(N.y, ay, N.x * ax));
  const float la = sqrt_approx(fmaf(az, az, fmaf(ay, ay, ax * ax)));
  const float lb = sqrt_approx(fmaf(bz, bz, fmaf(by, by, bx * bx)));
  const float lc = sqrt_approx(fmaf(cz, cz, fmaf(cy, cy, cx * cx)));
  const float ab = fmaf(az, bz, fmaf(ay, by, ax * bx));
  const float bc = fmaf(bz, cz, fmaf(by, cy, bx * cx));
  const float ca = fmaf(az, cz, fmaf(ay, cy, ax * cx));
  const float g1 = fmaf(bc, la, la * (lb * lc));
  const float g2 = __fadd_rn(__fmul_rn(ab, lc), __fmul_rn(ca, lb));
  const float beta = g1 + g2;
  const float epsN = A.w;
  if (fabsf(alpha) < epsN) {
    if (epsN == __int_as_float(0x7f800000)) return 0.0f;  // degenerate face
    // _kernels.py:65-67 vertex test, then :70-88 plane + barycentric test
    if (la < eps || lb < eps || lc < eps) return __int_as_float(0x7fc00000);
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
    if (b1 >= -btol && b2 >= -btol && b1 + b2 <= 1.0f + btol)
      return __int_as_float(0x7fc00000);
  }
  return atan2_full(alpha, beta);
}

template <class Src>
__global__ void __launch_bounds__(kExactThreads, 3)
exact_fwd_f32_kernel(const PackHeader* __restrict__ hdr,
                     const ExactRecF32* __restrict__ recs, int64_t n_faces,
                     Src src, int64_t n_count, int64_t tiles_per_split,
                     OutF32 o) {
  __shared__ FaceRing<ExactRecF32, kExactTile, kExactStages> ring;
  ring_init(ring, kExactConsumerWarps);

  const int64_t n_tiles = (n_faces + kExactTile - 1) / kExactTile;
  const int64_t t_begin = (int64_t)blockIdx.y * tiles_per_split;
  int64_t t_end = t_begin + tiles_per_split;
  if (t_end > n_tiles) t_end = n_tiles;

  const int warp = threadIdx.x >> 5;
  if (warp == kExactConsumerWarps) {  // producer warp
    if ((threadIdx.x & 31) == 0 && t_begin < t_end)
      ring_produce(ring, recs, n_faces, t_begin, t_end);
    return;
  }

  const float eps = hdr->eps_f32;
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * (kExactConsumers * kExactP);
  float qx[kExactP], qy[kExactP], qz[kExactP];
  double accd[kExactP];
#pragma unroll
  for (int p = 0; p < kExactP; ++p) {
    int64_t l = base + p * kExactConsumers + tid;
    if (l >= n_count) l = n_count - 1;  // padded lanes recompute a valid node
    src.point(l, qx[p], qy[p], qz[p]);
    accd[p] = 0.0;
  }
  uint32_t hits = 0;

  for (int64_t t = t_begin; t < t_end; ++t) {
    const int64_t it = t - t_begin;
    const int s = (int)(it % kExactStages);
    mbar_wait(&ring.full[s], (uint32_t)((it / kExactStages) & 1));
    const int64_t first = t * kExactTile;
    const int cnt = (int)((n_faces - first) < kExactTile ? (n_faces - first) : kExactTile);
    const ExactRecF32* tile = ring.tiles[s];
    float tacc[kExactP];
#pragma unroll
    for (int p = 0; p < kExactP; ++p) tacc[p] = 0.0f;

#pragma unroll 1
    for (int f = 0; f < cnt; ++f) {
      const ExactRecF32 R = tile[f];
      uint32_t rare = 0;
#pragma unroll
      for (int p = 0; p < kExactP; ++p) {
        const float ax = R.v0e.x - qx[p], ay = R.v0e.y - qy[p], az = R.v0e.z - qz[p];
        const float bx = R.v1.x - qx[p], by = R.v1.y - qy[p], bz = R.v1.z - qz[p];
        const float cx = R.v2.x - qx[p], cy = R.v2.y - qy[p], cz = R.v2.z - qz[p];
        const float alpha = fmaf(R.n.z, az, fmaf(R.n.y, ay, R.n.x * ax));
        const float la = sqrt_approx(fmaf(az, az, fmaf(ay, ay, ax * ax)));
        const float lb = sqrt_approx(fmaf(bz, bz, fmaf(by, by, bx * bx)));
        const float lc = sqrt_approx(fmaf(cz, cz, fmaf(cy, cy, cx * cx)));
        const float ab = fmaf(az, bz, fmaf(ay, by, ax * bx));
        const float bc = fmaf(bz, cz, fmaf(by, cy, bx * cx));
        const float ca = fmaf(az, cz, fmaf(ay, cy, ax * cx));
        // beta grouped as _kernels.py:98-103 so that swapping v1<->v2 leaves
        // it bit-identical (orientation flips negate W exactly).
        const float g1 = fmaf(bc, la, la * (lb * lc));
        const float g2 = __fadd_rn(__fmul_rn(ab, lc), __fmul_rn(ca, lb));
        const float beta = g1 + g2;
        const float aa = fabsf(alpha);
        const bool r = (aa > beta) || (aa < R.v0e.w);
        const float tt = r ? 0.0f : alpha * rcp_approx(beta);
        tacc[p] = fmaf(tt, atan_poly_coef(tt * tt), tacc[p]);
        if (r) rare |= 1u << p;
      }
      if (rare != 0u) {
#pragma unroll
        for (int p = 0; p < kExactP; ++p) {
          if (rare & (1u << p)) {
            const float th = exact_rare(R.v0e, R.v1, R.v2, R.n, qx[p], qy[p], qz[p], eps);
            if (th != th) hits |= 1u << p;
            else tacc[p] += th;
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < kExactP; ++p) accd[p] += (double)tacc[p];
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&ring.empty[s]);
  }

#pragma unroll
  for (int p = 0; p < kExactP; ++p) {
    const int64_t l = base + p * kExactConsumers + tid;
    if (l < n_count) o.store(blockIdx.y, l, accd[p], (hits >> p) & 1u);
  }
}

// Sum split partials in split order (deterministic), then W = sum/(2 pi).
__global__ void finalize_theta_kernel(const double* __restrict__ part,
                                      const uint8_t* __restrict__ pflags,
                                      int splits, int64_t n_count, int policy,
                                      float* __restrict__ out_f32,
                                      double* __restrict__ out_f64,
                                      uint8_t* __restrict__ flags,
                                      double scale) {
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
    if (out_f32) out_f32[l] = (float)w;
    if (out_f64) out_f64[l] = w;
    if (flags) flags[l] = h;
  }
}

int launch_exact_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, int policy, float* out, uint8_t* flags,
                         void* workspace, size_t ws_bytes, int num_sms,
                         cudaStream_t stream) {
  if (n_count <= 0) return 0;
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const ExactRecF32* recs = reinterpret_cast<const ExactRecF32*>(hdr + 1);
  const int64_t per_block = (int64_t)kExactConsumers * kExactP;
  const int64_t bx = (n_count + per_block - 1) / per_block;
  const int64_t n_tiles = (n_faces + kExactTile - 1) / kExactTile;
  const int splits = choose_splits(bx, n_tiles, num_sms, 3);
  const int64_t tps = splits > 0 && n_tiles > 0 ? (n_tiles + splits - 1) / splits : 0;
  const int real_splits = tps > 0 ? (int)((n_tiles + tps - 1) / tps) : 1;
  OutF32 o;
  o.out = out;
  o.flags = flags;
  o.policy = policy;
  o.scale = 1.0 / (2.0 * kPi);
  if (real_splits > 1) {
    const size_t need = exact_fwd_workspace_bytes(n_faces, n_count, num_sms);
    if (workspace == nullptr || ws_bytes < need) return kErrWorkspace;
    o.part = static_cast<double*>(workspace);
    o.part_flags = reinterpret_cast<uint8_t*>(o.part + (size_t)real_splits * n_count);
    o.n_count = n_count;
  }
  dim3 grid((unsigned)bx, (unsigned)real_splits);
  if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    exact_fwd_f32_kernel<GridSrc><<<grid, kExactThreads, 0, stream>>>(
        hdr, recs, n_faces, src, n_count, tps, o);
  } else {
    ListSrc src{ps.points};
    exact_fwd_f32_kernel<ListSrc><<<grid, kExactThreads, 0, stream>>>(
        hdr, recs, n_faces, src, n_count, tps, o);
  }
  if (real_splits > 1) {
    const int threads = 256;
    int blocks = (int)((n_count + threads - 1) / threads);
    if (blocks > num_sms * 8) blocks = num_sms * 8;
    finalize_theta_kernel<<<blocks, threads, 0, stream>>>(
        o.part, o.part_flags, real_splits, n_count, policy, out, nullptr, flags,
        o.scale);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : kErrLaunch;
}

size_t exact_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms) {
  const int64_t per_block = (int64_t)kExactConsumers * kExactP;
  const int64_t bx = (n_count + per_block - 1) / per_block;
  const int64_t n_tiles = (n_faces + kExactTile - 1) / kExactTile;
  const int splits = choose_splits(bx, n_tiles, num_sms, 3);
  if (splits <= 1) return 0;
  return (size_t)splits * (size_t)n_count * (sizeof(double) + 1) + 256;
}

}  // namespace wv
