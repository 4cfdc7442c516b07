// wv_metrics.cu -- reconstruction quality on the device (
// reference metrics.py): counter-based SplitMix64 uniforms, area-weighted
// surface sampling, nearest-neighbour distances, and numpy's pairwise
// summation (for the Chamfer means and the total area).
//
// Compiled with -fmad=false: every expression below is the reference's numpy
// expression in the same IEEE operation order, so samples, distances and the
// Chamfer / Hausdorff values are BIT-IDENTICAL to the reference's
// (metrics.py:43-130; its k-d tree is documented and tested to equal a
// brute-force scan bit for bit, metrics.py:96-104, which is what we run).
//
//   splitmix64   u_i = (mix(seed + (i+1) * golden) >> 11) * 2^-53
//   areas        0.5 * sqrt((c0^2 + c1^2) + c2^2),  c = (v1-v0) x (v2-v0)
//   cdf          sequential prefix sum (np.cumsum), one thread
//   total        numpy pairwise sum of the areas (np.sum)
//   sample i     face = searchsorted(cdf, r[3i] * total, 'right'), folded
//                (u, v) = r[3i+1], r[3i+2]; p = (v0 + u e1) + v e2
//   nearest      min_j ((dx^2 + dy^2) + dz^2), then sqrt (monotone, so equal
//                to the min of the distances); targets staged through smem
//   pairwise     numpy's pairwise_sum: blocks of <= 128 summed with 8
//                accumulators, halves split at multiples of 8 -- leaves in
//                parallel, the (shape-only) tree combined by one thread
#include "wv_kernels.h"

namespace wv {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;

__device__ __forceinline__ double splitmix_u(uint64_t seed, int64_t i) {
  uint64_t z = seed + (uint64_t)(i + 1) * kGolden;  // wraps mod 2^64 (metrics.py:46)
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  z = z ^ (z >> 31);
  return (double)(z >> 11) * 0x1.0p-53;  // 53-bit integer: exact conversion
}

__global__ void splitmix_kernel(uint64_t seed, int64_t count, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = splitmix_u(seed, i);
}

__global__ void face_area_kernel(const double* __restrict__ v, const int64_t* __restrict__ f,
                                 int64_t n_faces, double* __restrict__ areas) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_faces;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double* p0 = v + 3 * f[3 * t];
    const double* p1 = v + 3 * f[3 * t + 1];
    const double* p2 = v + 3 * f[3 * t + 2];
    const double ax = p1[0] - p0[0], ay = p1[1] - p0[1], az = p1[2] - p0[2];
    const double bx = p2[0] - p0[0], by = p2[1] - p0[1], bz = p2[2] - p0[2];
    // np.cross: cp0 = a1 b2 - a2 b1, cp1 = a2 b0 - a0 b2, cp2 = a0 b1 - a1 b0
    const double c0 = ay * bz - az * by, c1 = az * bx - ax * bz, c2 = ax * by - ay * bx;
    areas[t] = 0.5 * sqrt((c0 * c0 + c1 * c1) + c2 * c2);
  }
}

__global__ void cumsum_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc = i == 0 ? x[0] : acc + x[i];
    out[i] = acc;
  }
}

__global__ void sample_kernel(const double* __restrict__ v, const int64_t* __restrict__ f,
                              int64_t n_faces, const double* __restrict__ cdf,
                              const double* __restrict__ total, uint64_t seed, int64_t n,
                              double* __restrict__ out) {
  const double tot = *total;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = splitmix_u(seed, 3 * i) * tot;
    // searchsorted(side="right"): first index with cdf > x
    int64_t lo = 0, hi = n_faces;
    while (lo < hi) {
      const int64_t mid = lo + ((hi - lo) >> 1);
      if (cdf[mid] <= x) lo = mid + 1;
      else hi = mid;
    }
    const int64_t t = lo < n_faces - 1 ? lo : n_faces - 1;
    double u = splitmix_u(seed, 3 * i + 1), w = splitmix_u(seed, 3 * i + 2);
    if (u + w > 1.0) {
      u = 1.0 - u;
      w = 1.0 - w;
    }
    const double* p0 = v + 3 * f[3 * t];
    const double* p1 = v + 3 * f[3 * t + 1];
    const double* p2 = v + 3 * f[3 * t + 2];
    for (int d = 0; d < 3; ++d) out[3 * i + d] = (p0[d] + u * (p1[d] - p0[d])) + w * (p2[d] - p0[d]);
  }
}

constexpr int kNnThreads = 256;
constexpr int kNnTile = 1024;

__global__ void __launch_bounds__(kNnThreads)
nearest_kernel(const double* __restrict__ q, int64_t nq, const double* __restrict__ t, int64_t nt,
               double* __restrict__ out) {
  __shared__ double tile[kNnTile * 3];
  const int64_t i = blockIdx.x * (int64_t)kNnThreads + threadIdx.x;
  const int64_t iq = i < nq ? i : nq - 1;
  const double qx = q[3 * iq], qy = q[3 * iq + 1], qz = q[3 * iq + 2];
  double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (int64_t t0 = 0; t0 < nt; t0 += kNnTile) {
    const int cnt = (int)((nt - t0) < kNnTile ? (nt - t0) : kNnTile);
    __syncthreads();
    for (int k = threadIdx.x; k < 3 * cnt; k += kNnThreads) tile[k] = t[3 * t0 + k];
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < cnt; ++k) {
      const double dx = qx - tile[3 * k], dy = qy - tile[3 * k + 1], dz = qz - tile[3 * k + 2];
      const double d2 = (dx * dx + dy * dy) + dz * dz;
      best = d2 < best ? d2 : best;
    }
  }
  if (i < nq) out[i] = sqrt(best);
}

// numpy pairwise_sum (loops_utils.h.src) on one range; n <= 128 here.
__device__ double pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

// Leaves of the pairwise tree in order (explicit stack; shape depends on n only).
__device__ int pairwise_leaves(int64_t n, int64_t* lo, int64_t* len, int max_leaves) {
  int64_t st_lo[64], st_n[64];
  int sp = 0, nl = 0;
  st_lo[sp] = 0;
  st_n[sp++] = n;
  while (sp > 0) {
    --sp;
    const int64_t l = st_lo[sp], m = st_n[sp];
    if (m <= 128) {
      if (nl >= max_leaves) return -1;
      lo[nl] = l;
      len[nl++] = m;
    } else {
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      st_lo[sp] = l + m2;  // right half pushed first: the left one is visited first
      st_n[sp++] = m - m2;
      st_lo[sp] = l;
      st_n[sp++] = m2;
    }
  }
  return nl;
}

// Combine leaf sums along the same tree: post-order with an explicit stack.
__device__ double pairwise_combine(int64_t n, const double* leaf, int* next) {
  // frame: (n, state, left value)
  int64_t st_n[64];
  int st_s[64];
  double st_v[64];
  int sp = 0;
  double ret = 0.0;
  st_n[sp] = n;
  st_s[sp++] = 0;
  while (sp > 0) {
    const int top = sp - 1;
    const int64_t m = st_n[top];
    if (m <= 128) {
      ret = leaf[(*next)++];
      --sp;
    } else {
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      if (st_s[top] == 0) {  // descend left
        st_s[top] = 1;
        st_n[sp] = m2;
        st_s[sp++] = 0;
        continue;
      }
      if (st_s[top] == 1) {  // left done: keep it, descend right
        st_v[top] = ret;
        st_s[top] = 2;
        st_n[sp] = m - m2;
        st_s[sp++] = 0;
        continue;
      }
      ret = st_v[top] + ret;  // left + right
      --sp;
    }
  }
  return ret;
}

__global__ void pairwise_sum_kernel(const double* __restrict__ x, int64_t n,
                                    double* __restrict__ out, int64_t* lo, int64_t* len,
                                    double* leaf, int max_leaves, int* status) {
  __shared__ int n_leaves;
  if (threadIdx.x == 0) n_leaves = pairwise_leaves(n, lo, len, max_leaves);
  __syncthreads();
  const int nl = n_leaves;
  if (nl < 0) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  for (int k = threadIdx.x; k < nl; k += blockDim.x) leaf[k] = pairwise_leaf(x + lo[k], len[k]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int next = 0;
    *out = pairwise_combine(n, leaf, &next);
    *status = 0;
  }
}

// ---------------------------------------------------------------------------
static int grid_for(int64_t n, int threads, int num_sms) {
  int64_t b = (n + threads - 1) / threads;
  if (b > (int64_t)num_sms * 16) b = (int64_t)num_sms * 16;
  return (int)(b < 1 ? 1 : b);
}

int launch_splitmix(uint64_t seed, int64_t count, double* out, int num_sms, cudaStream_t s) {
  if (count <= 0) return kOk;
  { splitmix_kernel<<<grid_for(count, 256, num_sms), 256, 0, s>>>(seed, count, out); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

size_t pairwise_workspace_bytes(int64_t n) {
  const int64_t leaves = n / 64 + 2;
  return (size_t)leaves * (2 * sizeof(int64_t) + sizeof(double)) + 16;
}

int launch_pairwise_sum(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes,
                        cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(out, 0, sizeof(double), s) == cudaSuccess ? kOk : kErrCuda;
  const size_t need = pairwise_workspace_bytes(n);
  if (ws == nullptr || ws_bytes < need) return kErrWorkspace;
  const int64_t leaves = n / 64 + 2;
  char* p = static_cast<char*>(ws);
  int64_t* lo = reinterpret_cast<int64_t*>(p);
  int64_t* len = lo + leaves;
  double* leaf = reinterpret_cast<double*>(len + leaves);
  int* status = reinterpret_cast<int*>(leaf + leaves);
  { pairwise_sum_kernel<<<1, 256, 0, s>>>(x, n, out, lo, len, leaf, (int)leaves, status); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_surface_cdf(const double* v, const int64_t* f, int64_t n_faces, double* areas,
                       double* cdf, double* total, void* ws, size_t ws_bytes, int num_sms,
                       cudaStream_t s) {
  if (n_faces <= 0) return kErrArg;
  { face_area_kernel<<<grid_for(n_faces, 256, num_sms), 256, 0, s>>>(v, f, n_faces, areas); wv::note_launch(); }
  { cumsum_kernel<<<1, 1, 0, s>>>(areas, n_faces, cdf); wv::note_launch(); }
  if (cudaGetLastError() != cudaSuccess) return kErrLaunch;
  return launch_pairwise_sum(areas, n_faces, total, ws, ws_bytes, s);
}

int launch_sample_surface(const double* v, const int64_t* f, int64_t n_faces, const double* cdf,
                          const double* total, uint64_t seed, int64_t n, double* out, int num_sms,
                          cudaStream_t s) {
  if (n <= 0) return kOk;
  { sample_kernel<<<grid_for(n, 256, num_sms), 256, 0, s>>>(v, f, n_faces, cdf, total, seed, n, out); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_nearest(const double* q, int64_t nq, const double* t, int64_t nt, double* out,
                   cudaStream_t s) {
  if (nq <= 0) return kOk;
  if (nt <= 0) return kErrArg;
  const int64_t blocks = (nq + kNnThreads - 1) / kNnThreads;
  { nearest_kernel<<<(unsigned)blocks, kNnThreads, 0, s>>>(q, nq, t, nt, out); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
