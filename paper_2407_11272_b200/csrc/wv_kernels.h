// wv_kernels.h -- internal launch interface shared by the .cu files and the
// C-ABI layer (wv_capi.cu).  Not part of the public header.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "wv_common.cuh"

namespace wv {

// every kernel launch of the library bumps a process-wide counter
// (wv_launch_count): bench.py reports the launches of its timed region from
// it -- a count of OUR kernels that needs no profiler
void note_launch();
long long launch_count();

// status codes (mirrored in include/windvox_b200.h)
constexpr int kOk = 0;
constexpr int kErrArg = 1;
constexpr int kErrWorkspace = 2;
constexpr int kErrLaunch = 3;
constexpr int kErrCuda = 4;

// on-surface policy for stored values
constexpr int kPolicyRaw = 0;   // winding_number_batch: flagged keeps its partial sum
constexpr int kPolicyHalf = 1;  // voxelize: flagged -> exactly 0.5 (winding.py:358)

struct PointSource {
  enum Kind { kGrid = 0, kList = 1 };
  int kind;
  GridDesc grid;        // kGrid: nodes n0 .. n0+count-1 of the lattice
  int64_t n0;
  const float* points;  // kList f32 (count,3)
  const double* points64;  // kList f64 (count,3)
};

struct GridSrc {
  static constexpr bool kRows = false;
  static constexpr bool kGrid = true;
  GridDesc g;
  int64_t n0;
  __device__ __forceinline__ void point(int64_t l, float& x, float& y, float& z) const {
    double dx, dy, dz;
    grid_node(g, n0 + l, dx, dy, dz);
    x = (float)dx;  // winding.py:363: f64 node coordinates cast to f32
    y = (float)dy;
    z = (float)dz;
  }
  __device__ __forceinline__ void point(int64_t l, double& x, double& y, double& z) const {
    grid_node(g, n0 + l, x, y, z);
  }
};

// Lattice nodes taken in runs of consecutive k (the row-mode kernels):
// identical coordinates to GridSrc, different thread -> node mapping.
struct RowSrc : GridSrc {
  static constexpr bool kRows = true;
  static constexpr bool kWarpRow = false;
};
// Row mode where every warp's 32 P consecutive nodes lie in ONE k-row (the
// row length and the range start and count are multiples of them): the strip
// forward then computes each face's row terms once per warp (wv_fwd.cuh).
struct RowSrcW : RowSrc {
  static constexpr bool kWarpRow = true;
};
// Row mode needs every run of `run` nodes to stay inside one k-row.
inline bool row_aligned(const GridDesc& g, int64_t n0, int64_t count, int run) {
  return g.res[2] % run == 0 && n0 % run == 0 && count % run == 0 && count > 0;
}

struct ListSrc {
  static constexpr bool kRows = false;
  static constexpr bool kGrid = false;
  const float* pts;
  __device__ __forceinline__ void point(int64_t l, float& x, float& y, float& z) const {
    x = pts[3 * l + 0];
    y = pts[3 * l + 1];
    z = pts[3 * l + 2];
  }
};

struct ListSrc64 {
  static constexpr bool kRows = false;
  static constexpr bool kGrid = false;
  const double* pts;
  __device__ __forceinline__ void point(int64_t l, double& x, double& y, double& z) const {
    x = pts[3 * l + 0];
    y = pts[3 * l + 1];
    z = pts[3 * l + 2];
  }
};

// Forward output sink: final values (single split) or per-split partials.
// Batched launches over meshes with one connectivity and one query range:
// mesh z's packed records start z * pack_stride bytes after the first's
// (a multiple of 16 for the TMA copies), its outputs / coefficients lie
// z * count entries after the first's.
struct Batch {
  int64_t n = 1;
  size_t pack_stride = 0;
};

struct OutF32 {
  float* out = nullptr;
  uint8_t* flags = nullptr;
  double* part = nullptr;
  uint8_t* part_flags = nullptr;
  int64_t n_count = 0;
  int policy = kPolicyRaw;
  double scale = 1.0;
  __device__ __forceinline__ void store(int split, int64_t l, double acc, uint32_t hit) const {
    if (part != nullptr) {
      part[(int64_t)split * n_count + l] = acc;
      part_flags[(int64_t)split * n_count + l] = (uint8_t)hit;
      return;
    }
    double w = acc * scale;
    if (hit && policy == kPolicyHalf) w = 0.5;
    out[l] = (float)w;
    if (flags) flags[l] = (uint8_t)hit;
  }
};

// Face splits: when the node blocks alone cannot fill the chip, split the
// face range so that >= ~2 waves of CTAs exist; partials are summed in fixed
// split order by a finalize kernel (deterministic).  Depends only on the
// problem shape, never on timing.
// Work splits against wave quantization: every CTA of these kernels does the
// same work, so a grid of W waves (W = CTAs / resident slots) costs ceil(W)
// wave times.  Pick the split count in [s_lo, s_hi] whose last wave is
// fullest (a larger count must win by > 0.5% to be preferred).
inline int64_t best_splits(int64_t blocks, int64_t s_lo, int64_t s_hi, int64_t slots) {
  if (s_lo < 1) s_lo = 1;
  if (s_hi < s_lo) s_hi = s_lo;
  int64_t best = s_lo;
  double best_eff = -1.0;
  for (int64_t s = s_lo; s <= s_hi; ++s) {
    const int64_t ctas = blocks * s;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff > best_eff + 0.005) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

// Forward: split the face range over blockIdx.y when the node blocks alone
// give few waves (small grids, or one slab of a multi-GPU run).
inline int choose_splits(int64_t blocks_x, int64_t n_tiles, int num_sms, int ctas_per_sm) {
  if (n_tiles <= 1) return 1;
  const int64_t slots = (int64_t)num_sms * ctas_per_sm;
  if (blocks_x >= 16 * slots) return 1;  // >= 16 waves: the last one costs < 6%
  int64_t lo = (2 * slots + blocks_x - 1) / blocks_x;  // at least 2 waves
  int64_t hi = 4 * lo;
  const int64_t cap = n_tiles < 64 ? n_tiles : 64;
  if (lo > cap) lo = cap;
  if (hi > cap) hi = cap;
  return (int)best_splits(blocks_x, lo, hi, slots);
}

// packing (wv_pack.cu)
int launch_pack(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                const void* faces, int faces_i64, int64_t n_faces, const double* eps_dev,
                void* packed, cudaStream_t stream);
int launch_surface_eps(const void* vertices, int vert_f64, int64_t n_verts, double* eps_dev,
                       cudaStream_t stream);
size_t packed_bytes(int kind, int64_t n_faces);
int launch_vertex_normals(const double* verts, const int64_t* faces, int64_t n_faces,
                          const int64_t* off, const int64_t* slots, int64_t n_verts,
                          double* normals, uint8_t* zero, cudaStream_t stream);
int launch_pack_exact_grad(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                           const void* faces, int faces_i64, const int64_t* active,
                           const float* weights, int64_t n_active, void* packed,
                           cudaStream_t stream);

// forward (wv_exact_fwd.cu, wv_soft_fwd.cu, wv_f64.cu)
int launch_exact_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, int policy, float* out, uint8_t* flags,
                         void* workspace, size_t ws_bytes, int num_sms, cudaStream_t stream,
                         const Batch& bt = Batch());
size_t exact_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms,
                                 int64_t batch = 1);
// strip-pair exact backward (wv_bwd_f32.cu): records = ExactGradRecF32 pairs
int launch_exact_pair_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                              int64_t n_count, const float* coefs, double coef_scale,
                              double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                              cudaStream_t stream);
size_t exact_strip_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms);
size_t exact_pair_bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms);
// edge trails (wv_trail.cu builds and packs, wv_bwd_f32.cu runs)
int64_t weld_positions(const double* verts, int64_t n_verts, int64_t* canon);
int edge_trails(const double* verts, int64_t n_verts, const int64_t* faces, int64_t n_faces,
                const uint8_t* dead, int64_t* windows, int64_t* n_windows, int64_t* csr_off,
                int64_t* csr_slots, int64_t* n_slots, int64_t* vrep);
int launch_pack_trail(const void* verts, int vert_f64, int64_t n_verts, const int64_t* windows,
                      int64_t n_windows, void* packed, cudaStream_t stream);
int launch_exact_trail_bwd_f32(const void* packed, int64_t n_windows, const PointSource& ps,
                               int64_t n_count, const float* coefs, double coef_scale,
                               double* out, void* workspace, size_t ws_bytes, int num_sms,
                               cudaStream_t stream);
size_t exact_trail_bwd_workspace_bytes(int64_t n_windows, int64_t n_count, int num_sms);
int launch_pack_trail_f64(const void* verts, int vert_f64, int64_t n_verts,
                          const int64_t* windows, int64_t n_windows, void* packed,
                          cudaStream_t stream);
int launch_exact_trail_bwd_f64(const void* packed, int64_t n_windows, const PointSource& ps,
                               int64_t n_count, const double* coefs, double coef_scale,
                               double* out, void* ws, size_t ws_bytes, int num_sms,
                               cudaStream_t stream);
size_t exact_trail_bwd64_workspace_bytes(int64_t n_windows, int64_t n_count, int num_sms);
// strip-ordered exact forward (wv_strip.cu builds and packs, wv_fwd_f32.cu runs)
int strip_order(const double* verts, int64_t n_verts, const int64_t* faces, int64_t n_faces,
                int64_t* perm, int64_t* win, uint8_t* flags);
int launch_pack_strip(const void* verts, int vert_f64, int64_t n_verts, const void* faces,
                      int faces_i64, int64_t n_faces, const int64_t* perm, const int64_t* win,
                      const uint8_t* flags, void* packed, cudaStream_t stream);
int launch_pack_strip_f64(const void* verts, int vert_f64, int64_t n_verts, const void* faces,
                          int faces_i64, int64_t n_faces, const int64_t* perm,
                          const int64_t* win, const uint8_t* flags, void* packed,
                          cudaStream_t stream);
int launch_exact_strip_fwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                               int64_t n_count, int use_atan2, int policy, double* out,
                               uint8_t* flags, cudaStream_t stream);
int launch_exact_strip_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                               int64_t n_count, int policy, float* out, uint8_t* flags,
                               void* workspace, size_t ws_bytes, int num_sms,
                               cudaStream_t stream);
int launch_soft_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, int policy, float* out, uint8_t* flags,
                        void* workspace, size_t ws_bytes, int num_sms, cudaStream_t stream,
                         const Batch& bt = Batch());
size_t soft_fwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms,
                                int64_t batch = 1);
int launch_exact_fwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, int use_atan2, int policy, double* out, uint8_t* flags,
                         cudaStream_t stream);
int launch_soft_fwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, int policy, double* out, uint8_t* flags,
                        cudaStream_t stream);

// backward (wv_bwd_f32.cu, wv_f64.cu)
int launch_exact_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, const float* coefs, double coef_scale,
                         double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                         cudaStream_t stream,
                         const Batch& bt = Batch());
int launch_soft_bwd_f32(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, const float* coefs, double coef_scale,
                        double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                        cudaStream_t stream,
                         const Batch& bt = Batch());
size_t bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch = 1);
size_t soft_bwd_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms,
                                int64_t batch = 1);
int launch_exact_bwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                         int64_t n_count, const double* coefs, double coef_scale,
                         double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                         cudaStream_t stream);
int launch_soft_bwd_f64(const void* packed, int64_t n_faces, const PointSource& ps,
                        int64_t n_count, const double* coefs, double coef_scale,
                        double* face_grad, void* ws, size_t ws_bytes, int num_sms,
                        cudaStream_t stream);
size_t bwd64_workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms);
int launch_face_to_vertex_batch(const double* face_grad, int64_t n_faces, const int64_t* off,
                                const int64_t* slots, int64_t n_verts, int64_t batch,
                                const double* scale, int64_t scale_stride, int accumulate,
                                double* out64, float* out32, int num_sms, cudaStream_t stream);
int launch_pack_batch(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                      const void* faces, int faces_i64, int64_t n_faces, int64_t batch,
                      void* packed, size_t pack_stride, cudaStream_t stream);
int launch_loss_f32_batch(const float* values, const uint8_t* flags, const float* targets,
                          const float* weights, int64_t n, int64_t batch, float* coefs,
                          double* sums, void* ws, size_t ws_bytes, cudaStream_t stream);
int launch_face_to_vertex(const double* face_grad, const int64_t* off, const int64_t* slots,
                          int64_t n_verts, const double* scale, int accumulate, double* out64,
                          float* out32, int num_sms, cudaStream_t stream);

// marching cubes (wv_mc.cu)
int launch_mc_classify(const void* vals, int f64, int64_t rx, int64_t ry, int64_t rz, double iso,
                       const int8_t* count_tab, uint8_t* cases, int32_t* counts, int num_sms,
                       cudaStream_t stream);
int launch_mc_edges(const void* vals, int f64, int64_t rx, int64_t ry, int64_t rz, double iso,
                    int32_t* flags, int num_sms, cudaStream_t stream);
int launch_mc_vertices(const void* vals, int f64, const GridDesc& g, int64_t i0, int64_t rows,
                       double iso, const int32_t* flags, const int64_t* slot, double* verts,
                       int num_sms, cudaStream_t stream);
int launch_mc_emit(const uint8_t* cases, const int64_t* tri_off, const int8_t* tri_tab,
                   int max_tris, const int8_t* edge_axis, const int8_t* edge_base,
                   const int64_t* vidx, int64_t rx, int64_t ry, int64_t rz, int64_t* faces,
                   int num_sms, cudaStream_t stream);

// loss (wv_loss.cu)
size_t loss_workspace_bytes(int64_t n);
int launch_loss_f32(const float* values, const uint8_t* flags, const float* targets,
                    const float* weights, int64_t n, float* coefs, double* sums, void* ws,
                    size_t ws_bytes, cudaStream_t stream);
int launch_loss_f64(const double* values, const uint8_t* flags, const double* targets,
                    const double* weights, int64_t n, double* coefs, double* sums, void* ws,
                    size_t ws_bytes, cudaStream_t stream);
int launch_loss_finalize(double* sums, cudaStream_t stream);

// reconstruction metrics (wv_metrics.cu)
int launch_splitmix(uint64_t seed, int64_t count, double* out, int num_sms, cudaStream_t s);
size_t pairwise_workspace_bytes(int64_t n);
int launch_pairwise_sum(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes,
                        cudaStream_t s);
int launch_surface_cdf(const double* v, const int64_t* f, int64_t n_faces, double* areas,
                       double* cdf, double* total, void* ws, size_t ws_bytes, int num_sms,
                       cudaStream_t s);
int launch_sample_surface(const double* v, const int64_t* f, int64_t n_faces, const double* cdf,
                          const double* total, uint64_t seed, int64_t n, double* out, int num_sms,
                          cudaStream_t s);
int launch_nearest(const double* q, int64_t nq, const double* t, int64_t nt, double* out,
                   cudaStream_t s);

}  // namespace wv
