// wv_loss.cu -- occupancy-loss terms on the device (grad.py:101-110), fused so
// W never round-trips to the host:
//   loss   = sum_n w_n r_n^2 / sum_n w_n   over unflagged nodes, r = W - target
//   coef_n = 2 w_n r_n   (0 on flagged nodes; the 1/sum(w) factor is applied
//            after the face->vertex gather, reading sums[3] on the device, so
//            multi-GPU partial sums can be all-reduced first)
// sums[0..7] = {sum w r^2, sum w, n_flagged, 1/sum w, loss, 0, 0, 0}.
// Deterministic: fixed block count (a function of n only), per-block fp64
// partials, one final block sums them in a fixed order.
#include "wv_kernels.h"

namespace wv {

constexpr int kLossThreads = 256;

template <typename T>
__global__ void loss_terms_kernel(const T* __restrict__ values, const uint8_t* __restrict__ flags,
                                  const T* __restrict__ targets, const T* __restrict__ weights,
                                  int64_t n, T* __restrict__ coefs, double* __restrict__ part) {
  // batched launches: blockIdx.y = mesh (arrays n apart, partials per mesh)
  {
    const int64_t o = (int64_t)blockIdx.y * n;
    values += o;
    flags += o;
    targets += o;
    if (weights) weights += o;
    coefs += o;
    part += (int64_t)blockIdx.y * 3 * gridDim.x;
  }
  __shared__ double s0[kLossThreads], s1[kLossThreads], s2[kLossThreads];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kLossThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kLossThreads) {
    const bool flagged = flags[i] != 0;
    const double w = weights ? (double)weights[i] : 1.0;
    const double r = flagged ? 0.0 : (double)values[i] - (double)targets[i];
    if (flagged) a2 += 1.0;
    else a1 += w;
    a0 += w * r * r;
    coefs[i] = (T)(2.0 * w * r);
  }
  s0[threadIdx.x] = a0;
  s1[threadIdx.x] = a1;
  s2[threadIdx.x] = a2;
  __syncthreads();
  for (int s = kLossThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      s0[threadIdx.x] += s0[threadIdx.x + s];
      s1[threadIdx.x] += s1[threadIdx.x + s];
      s2[threadIdx.x] += s2[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = s0[0];
    part[3 * blockIdx.x + 1] = s1[0];
    part[3 * blockIdx.x + 2] = s2[0];
  }
}

__global__ void loss_final_kernel(const double* __restrict__ part, int nblocks,
                                  double* __restrict__ sums) {
  part += (int64_t)blockIdx.x * 3 * nblocks;  // batched: block b = mesh b
  sums += 8 * blockIdx.x;
  // fixed-order two-level sum (thread t takes partials t, t+256, ...; then a
  // shared-memory tree): deterministic, and ~30x faster than one thread
  __shared__ double s0[kLossThreads], s1[kLossThreads], s2[kLossThreads];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kLossThreads) {
    a0 += part[3 * b];
    a1 += part[3 * b + 1];
    a2 += part[3 * b + 2];
  }
  s0[threadIdx.x] = a0;
  s1[threadIdx.x] = a1;
  s2[threadIdx.x] = a2;
  __syncthreads();
  for (int s = kLossThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      s0[threadIdx.x] += s0[threadIdx.x + s];
      s1[threadIdx.x] += s1[threadIdx.x + s];
      s2[threadIdx.x] += s2[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sums[0] = s0[0];
    sums[1] = s1[0];
    sums[2] = s2[0];
    sums[3] = s1[0] != 0.0 ? 1.0 / s1[0] : 0.0;
    sums[4] = s1[0] != 0.0 ? s0[0] / s1[0] : 0.0;
  }
}

// recompute the derived entries after sums[0..2] were all-reduced
__global__ void loss_finalize_kernel(double* __restrict__ sums) {
  if (threadIdx.x != 0) return;
  sums[3] = sums[1] != 0.0 ? 1.0 / sums[1] : 0.0;
  sums[4] = sums[1] != 0.0 ? sums[0] / sums[1] : 0.0;
}

static int loss_blocks(int64_t n, int num_sms) {
  int64_t b = (n + kLossThreads - 1) / kLossThreads;
  const int64_t cap = 1024;
  (void)num_sms;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

size_t loss_workspace_bytes(int64_t n) { return (size_t)loss_blocks(n, 0) * 3 * sizeof(double); }

template <typename T>
static int launch_loss(const T* values, const uint8_t* flags, const T* targets, const T* weights,
                       int64_t n, T* coefs, double* sums, void* ws, size_t ws_bytes,
                       cudaStream_t stream) {
  const int nb = loss_blocks(n, 0);
  if (ws == nullptr || ws_bytes < loss_workspace_bytes(n)) return kErrWorkspace;
  double* part = static_cast<double*>(ws);
  if (n > 0)
    { loss_terms_kernel<T><<<nb, kLossThreads, 0, stream>>>(values, flags, targets, weights, n,
                                                          coefs, part); wv::note_launch(); }
  else
    cudaMemsetAsync(part, 0, 3 * sizeof(double), stream);
  { loss_final_kernel<<<1, kLossThreads, 0, stream>>>(part, n > 0 ? nb : 1, sums); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

// (batch, n) arrays, sums (batch, 8): one terms and one final launch for all
int launch_loss_f32_batch(const float* values, const uint8_t* flags, const float* targets,
                          const float* weights, int64_t n, int64_t batch, float* coefs,
                          double* sums, void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int nb = loss_blocks(n, 0);
  if (batch < 1 || batch > 65535 || n <= 0) return kErrArg;
  if (ws == nullptr || ws_bytes < (size_t)batch * loss_workspace_bytes(n)) return kErrWorkspace;
  double* part = static_cast<double*>(ws);
  { loss_terms_kernel<float><<<dim3((unsigned)nb, (unsigned)batch), kLossThreads, 0, stream>>>(
      values, flags, targets, weights, n, coefs, part); wv::note_launch(); }
  { loss_final_kernel<<<(unsigned)batch, kLossThreads, 0, stream>>>(part, nb, sums); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}
int launch_loss_f32(const float* values, const uint8_t* flags, const float* targets,
                    const float* weights, int64_t n, float* coefs, double* sums, void* ws,
                    size_t ws_bytes, cudaStream_t stream) {
  return launch_loss<float>(values, flags, targets, weights, n, coefs, sums, ws, ws_bytes,
                            stream);
}
int launch_loss_f64(const double* values, const uint8_t* flags, const double* targets,
                    const double* weights, int64_t n, double* coefs, double* sums, void* ws,
                    size_t ws_bytes, cudaStream_t stream) {
  return launch_loss<double>(values, flags, targets, weights, n, coefs, sums, ws, ws_bytes,
                             stream);
}
int launch_loss_finalize(double* sums, cudaStream_t stream) {
  { loss_finalize_kernel<<<1, 32, 0, stream>>>(sums); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
