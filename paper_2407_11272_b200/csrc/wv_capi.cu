// wv_capi.cu -- extern "C" boundary (include/windvox_b200.h).  Argument
// validation, device-attribute caching, launch dispatch.  No exceptions cross
// the ABI; every entry point returns a status code.
#include <atomic>
#include "../../include/windvox_b200.h"
#include "wv_kernels.h"

namespace wv {
static std::atomic<long long> g_launch_count{0};
void note_launch() { g_launch_count.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launch_count.load(std::memory_order_relaxed); }
}  // namespace wv

namespace {

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static thread_local int cached_dev = -1;
  static thread_local int cached = 148;
  if (dev != cached_dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    cached_dev = dev;
  }
  return cached;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

bool grid_ok(const wv_grid_t& g, int64_t n0, int64_t count) {
  for (int i = 0; i < 3; ++i)
    if (g.res[i] < 1) return false;
  const int64_t n = g.res[0] * g.res[1] * g.res[2];
  return n0 >= 0 && count >= 0 && n0 + count <= n;
}

wv::PointSource grid_src(const wv_grid_t& g, int64_t n0) {
  wv::PointSource ps{};
  ps.kind = wv::PointSource::kGrid;
  for (int i = 0; i < 3; ++i) {
    ps.grid.lo[i] = g.lo[i];
    ps.grid.hi[i] = g.hi[i];
    ps.grid.res[i] = g.res[i];
  }
  ps.n0 = n0;
  return ps;
}

wv::PointSource list_src(const float* p32, const double* p64) {
  wv::PointSource ps{};
  ps.kind = wv::PointSource::kList;
  ps.points = p32;
  ps.points64 = p64;
  return ps;
}

bool fwd_args_ok(const void* packed, const void* out, int64_t n_faces, int64_t count) {
  return packed != nullptr && n_faces >= 0 && count >= 0 && (count == 0 || out != nullptr);
}

bool bwd_args_ok(const void* packed, const void* coefs, const double* face_grad,
                 int64_t n_faces, int64_t count) {
  return packed != nullptr && n_faces >= 0 && count >= 0 &&
         (n_faces == 0 || face_grad != nullptr) && (count == 0 || coefs != nullptr);
}

}  // namespace

extern "C" {

const char* wv_version(void) { return "windvox_b200 0.1.0 (sm_100a)"; }

const char* wv_status_string(int status) {
  switch (status) {
    case WV_OK: return "ok";
    case WV_ERR_ARG: return "invalid argument";
    case WV_ERR_WORKSPACE: return "workspace missing or too small";
    case WV_ERR_LAUNCH: return "kernel launch failed";
    case WV_ERR_CUDA: return "CUDA runtime error";
    default: return "unknown status";
  }
}

int wv_set_device(int device) {
  return cudaSetDevice(device) == cudaSuccess ? WV_OK : WV_ERR_CUDA;
}

long long wv_launch_count(void) { return wv::launch_count(); }

size_t wv_packed_bytes(int kind, int64_t n_faces) { return wv::packed_bytes(kind, n_faces); }

int wv_pack_faces(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                  const void* faces, int faces_i64, int64_t n_faces, void* packed,
                  void* stream) {
  if (packed == nullptr || n_verts < 0 || n_faces < 0) return WV_ERR_ARG;
  if ((n_verts > 0 && vertices == nullptr) || (n_faces > 0 && faces == nullptr))
    return WV_ERR_ARG;
  return wv::launch_pack(kind, vertices, vert_f64, n_verts, faces, faces_i64, n_faces, nullptr,
                         packed, as_stream(stream));
}

int wv_pack_exact_grad(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                       const void* faces, int faces_i64, const int64_t* active,
                       const float* weights, int64_t n_active, void* packed, void* stream) {
  if (packed == nullptr || n_verts < 0 || n_active < 0) return WV_ERR_ARG;
  if (n_active > 0 && (vertices == nullptr || faces == nullptr || active == nullptr ||
                       weights == nullptr))
    return WV_ERR_ARG;
  return wv::launch_pack_exact_grad(kind, vertices, vert_f64, n_verts, faces, faces_i64, active,
                                    weights, n_active, packed, as_stream(stream));
}

int wv_vertex_normals(const double* vertices, int64_t n_verts, const int64_t* faces,
                      int64_t n_faces, const int64_t* csr_offsets, const int64_t* csr_slots,
                      double* normals, uint8_t* zero, void* stream) {
  if (n_verts < 0 || n_faces < 0) return WV_ERR_ARG;
  if (n_verts > 0 && (vertices == nullptr || csr_offsets == nullptr || normals == nullptr))
    return WV_ERR_ARG;
  if (n_faces > 0 && (faces == nullptr || csr_slots == nullptr)) return WV_ERR_ARG;
  return wv::launch_vertex_normals(vertices, faces, n_faces, csr_offsets, csr_slots, n_verts,
                                   normals, zero, as_stream(stream));
}

// ---- forward ---------------------------------------------------------------
size_t wv_fwd_workspace_bytes(int kind, int64_t n_faces, int64_t count) {
  switch (kind) {
    case WV_PACK_EXACT_F32: return wv::exact_fwd_workspace_bytes(n_faces, count, sm_count());
    case WV_PACK_EXACTSTRIP_F32:
      return wv::exact_strip_fwd_workspace_bytes(n_faces, count, sm_count());
    case WV_PACK_SOFT_F32: return wv::soft_fwd_workspace_bytes(n_faces, count, sm_count());
    default: return 0;
  }
}

int wv_strip_order(const double* vertices, int64_t n_verts, const int64_t* faces,
                   int64_t n_faces, int64_t* perm, int64_t* window, uint8_t* flags) {
  if (n_verts < 0 || n_faces < 0 || n_faces >= ((int64_t)1 << 31)) return WV_ERR_ARG;
  if (n_faces == 0) return WV_OK;
  if (vertices == nullptr || faces == nullptr || perm == nullptr || window == nullptr ||
      flags == nullptr)
    return WV_ERR_ARG;
  for (int64_t i = 0; i < 3 * n_faces; ++i)
    if (faces[i] < 0 || faces[i] >= n_verts) return WV_ERR_ARG;
  return wv::strip_order(vertices, n_verts, faces, n_faces, perm, window, flags);
}

int wv_pack_exact_strip(const void* vertices, int vert_f64, int64_t n_verts, const void* faces,
                        int faces_i64, int64_t n_faces, const int64_t* perm,
                        const int64_t* window, const uint8_t* flags, void* packed,
                        void* stream) {
  if (packed == nullptr || n_verts < 0 || n_faces < 0) return WV_ERR_ARG;
  if (n_faces > 0 && (vertices == nullptr || faces == nullptr || perm == nullptr ||
                      window == nullptr || flags == nullptr))
    return WV_ERR_ARG;
  return wv::launch_pack_strip(vertices, vert_f64, n_verts, faces, faces_i64, n_faces, perm,
                               window, flags, packed, as_stream(stream));
}

int wv_exact_strip_fwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                                int64_t count, int policy, float* out, uint8_t* flags,
                                void* workspace, size_t workspace_bytes, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count)) return WV_ERR_ARG;
  return wv::launch_exact_strip_fwd_f32(packed, n_faces, grid_src(grid, n0), count, policy, out,
                                        flags, workspace, workspace_bytes, sm_count(),
                                        as_stream(stream));
}

int wv_exact_strip_fwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                                  int64_t count, int policy, float* out, uint8_t* flags,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_strip_fwd_f32(packed, n_faces, list_src(points, nullptr), count, policy,
                                        out, flags, workspace, workspace_bytes, sm_count(),
                                        as_stream(stream));
}

int wv_pack_exact_strip_f64(const void* vertices, int vert_f64, int64_t n_verts,
                            const void* faces, int faces_i64, int64_t n_faces,
                            const int64_t* perm, const int64_t* window, const uint8_t* flags,
                            void* packed, void* stream) {
  if (packed == nullptr || n_verts < 0 || n_faces < 0) return WV_ERR_ARG;
  if (n_faces > 0 && (vertices == nullptr || faces == nullptr || perm == nullptr ||
                      window == nullptr || flags == nullptr))
    return WV_ERR_ARG;
  return wv::launch_pack_strip_f64(vertices, vert_f64, n_verts, faces, faces_i64, n_faces, perm,
                                   window, flags, packed, as_stream(stream));
}
int wv_exact_strip_fwd_grid_f64(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                                int64_t count, int use_atan2, int policy, double* out,
                                uint8_t* flags, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count)) return WV_ERR_ARG;
  return wv::launch_exact_strip_fwd_f64(packed, n_faces, grid_src(grid, n0), count, use_atan2,
                                        policy, out, flags, as_stream(stream));
}
int wv_exact_strip_fwd_points_f64(const void* packed, int64_t n_faces, const double* points,
                                  int64_t count, int use_atan2, int policy, double* out,
                                  uint8_t* flags, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_strip_fwd_f64(packed, n_faces, list_src(nullptr, points), count,
                                        use_atan2, policy, out, flags, as_stream(stream));
}

int wv_exact_fwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, int policy, float* out, uint8_t* flags,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count)) return WV_ERR_ARG;
  return wv::launch_exact_fwd_f32(packed, n_faces, grid_src(grid, n0), count, policy, out, flags,
                                  workspace, workspace_bytes, sm_count(), as_stream(stream));
}

int wv_exact_fwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                            int64_t count, int policy, float* out, uint8_t* flags,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_fwd_f32(packed, n_faces, list_src(points, nullptr), count, policy, out,
                                  flags, workspace, workspace_bytes, sm_count(),
                                  as_stream(stream));
}

int wv_soft_fwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, int policy, float* out, uint8_t* flags, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count)) return WV_ERR_ARG;
  return wv::launch_soft_fwd_f32(packed, n_faces, grid_src(grid, n0), count, policy, out, flags,
                                 workspace, workspace_bytes, sm_count(), as_stream(stream));
}

int wv_soft_fwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                           int64_t count, int policy, float* out, uint8_t* flags,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_soft_fwd_f32(packed, n_faces, list_src(points, nullptr), count, policy, out,
                                 flags, workspace, workspace_bytes, sm_count(),
                                 as_stream(stream));
}

int wv_exact_fwd_grid_f64(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, int use_atan2, int policy, double* out, uint8_t* flags,
                          void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count)) return WV_ERR_ARG;
  return wv::launch_exact_fwd_f64(packed, n_faces, grid_src(grid, n0), count, use_atan2, policy,
                                  out, flags, as_stream(stream));
}

int wv_exact_fwd_points_f64(const void* packed, int64_t n_faces, const double* points,
                            int64_t count, int use_atan2, int policy, double* out,
                            uint8_t* flags, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_fwd_f64(packed, n_faces, list_src(nullptr, points), count, use_atan2,
                                  policy, out, flags, as_stream(stream));
}

int wv_soft_fwd_grid_f64(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, int policy, double* out, uint8_t* flags, void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count)) return WV_ERR_ARG;
  return wv::launch_soft_fwd_f64(packed, n_faces, grid_src(grid, n0), count, policy, out, flags,
                                 as_stream(stream));
}

int wv_soft_fwd_points_f64(const void* packed, int64_t n_faces, const double* points,
                           int64_t count, int policy, double* out, uint8_t* flags,
                           void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_soft_fwd_f64(packed, n_faces, list_src(nullptr, points), count, policy, out,
                                 flags, as_stream(stream));
}

// ---- backward --------------------------------------------------------------
size_t wv_bwd_workspace_bytes(int kind, int64_t n_faces, int64_t count) {
  switch (kind) {
    case WV_PACK_EXACTGRAD_F32: return wv::bwd_workspace_bytes(n_faces, count, sm_count());
    case WV_PACK_SOFTGRAD_F32: return wv::soft_bwd_workspace_bytes(n_faces, count, sm_count());
    case WV_PACK_EXACTGRAD_F64:
    case WV_PACK_SOFTGRAD_F64: return wv::bwd64_workspace_bytes(n_faces, count, sm_count());
    default: return 0;
  }
}

int wv_exact_bwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, const float* coefs, double coef_scale,
                          double* face_grad, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || !grid_ok(grid, n0, count))
    return WV_ERR_ARG;
  return wv::launch_exact_bwd_f32(packed, n_faces, grid_src(grid, n0), count, coefs, coef_scale,
                                  face_grad, workspace, workspace_bytes, sm_count(),
                                  as_stream(stream));
}

int wv_exact_bwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                            int64_t count, const float* coefs, double coef_scale,
                            double* face_grad, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_bwd_f32(packed, n_faces, list_src(points, nullptr), count, coefs,
                                  coef_scale, face_grad, workspace, workspace_bytes, sm_count(),
                                  as_stream(stream));
}

size_t wv_exact_pair_bwd_workspace_bytes(int64_t n_faces, int64_t count) {
  return n_faces > 0 && count > 0 ? wv::exact_pair_bwd_workspace_bytes(n_faces, count, sm_count())
                                  : 0;
}
int wv_exact_pair_bwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                               int64_t count, const float* coefs, double coef_scale,
                               double* face_grad, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || !grid_ok(grid, n0, count) ||
      n_faces % 2 != 0)
    return WV_ERR_ARG;
  return wv::launch_exact_pair_bwd_f32(packed, n_faces, grid_src(grid, n0), count, coefs,
                                       coef_scale, face_grad, workspace, workspace_bytes,
                                       sm_count(), as_stream(stream));
}
int wv_exact_pair_bwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                                 int64_t count, const float* coefs, double coef_scale,
                                 double* face_grad, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) ||
      (count > 0 && points == nullptr) || n_faces % 2 != 0)
    return WV_ERR_ARG;
  return wv::launch_exact_pair_bwd_f32(packed, n_faces, list_src(points, nullptr), count, coefs,
                                       coef_scale, face_grad, workspace, workspace_bytes,
                                       sm_count(), as_stream(stream));
}

int wv_trail_edges(void) { return wv::kTrailK; }
int wv_edge_trails(const double* vertices, int64_t n_verts, const int64_t* faces,
                   int64_t n_faces, const uint8_t* dead, int64_t* windows, int64_t* n_windows,
                   int64_t* csr_off, int64_t* csr_slots, int64_t* n_slots, int64_t* vrep) {
  if (n_verts < 0 || n_faces < 0 || n_windows == nullptr || n_slots == nullptr ||
      csr_off == nullptr || (n_verts > 0 && vertices == nullptr) ||
      (n_faces > 0 && (faces == nullptr || windows == nullptr || csr_slots == nullptr)))
    return WV_ERR_ARG;
  for (int64_t i = 0; i < 3 * n_faces; ++i)
    if (faces[i] < 0 || faces[i] >= n_verts) return WV_ERR_ARG;
  return wv::edge_trails(vertices, n_verts, faces, n_faces, dead, windows, n_windows, csr_off,
                         csr_slots, n_slots, vrep);
}
int wv_pack_exact_trail(const void* vertices, int vert_f64, int64_t n_verts,
                        const int64_t* windows, int64_t n_windows, void* packed, void* stream) {
  if (packed == nullptr || n_verts < 0 || n_windows < 0 ||
      (n_windows > 0 && (windows == nullptr || vertices == nullptr)))
    return WV_ERR_ARG;
  return wv::launch_pack_trail(vertices, vert_f64, n_verts, windows, n_windows, packed,
                               as_stream(stream));
}
size_t wv_exact_trail_bwd_workspace_bytes(int64_t n_windows, int64_t count) {
  return n_windows > 0 && count > 0
             ? wv::exact_trail_bwd_workspace_bytes(n_windows, count, sm_count())
             : 0;
}
int wv_exact_trail_bwd_grid_f32(const void* packed, int64_t n_windows, wv_grid_t grid,
                                int64_t n0, int64_t count, const float* coefs,
                                double coef_scale, double* out, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (!bwd_args_ok(packed, coefs, out, n_windows, count) || !grid_ok(grid, n0, count))
    return WV_ERR_ARG;
  return wv::launch_exact_trail_bwd_f32(packed, n_windows, grid_src(grid, n0), count, coefs,
                                        coef_scale, out, workspace, workspace_bytes, sm_count(),
                                        as_stream(stream));
}

int wv_pack_exact_trail_f64(const void* vertices, int vert_f64, int64_t n_verts,
                            const int64_t* windows, int64_t n_windows, void* packed,
                            void* stream) {
  if (packed == nullptr || n_verts < 0 || n_windows < 0 ||
      (n_windows > 0 && (windows == nullptr || vertices == nullptr)))
    return WV_ERR_ARG;
  return wv::launch_pack_trail_f64(vertices, vert_f64, n_verts, windows, n_windows, packed,
                                   as_stream(stream));
}
size_t wv_exact_trail_bwd_workspace_bytes_f64(int64_t n_windows, int64_t count) {
  return n_windows > 0 && count > 0
             ? wv::exact_trail_bwd64_workspace_bytes(n_windows, count, sm_count())
             : 0;
}
int wv_exact_trail_bwd_grid_f64(const void* packed, int64_t n_windows, wv_grid_t grid,
                                int64_t n0, int64_t count, const double* coefs,
                                double coef_scale, double* out, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (!bwd_args_ok(packed, coefs, out, n_windows, count) || !grid_ok(grid, n0, count))
    return WV_ERR_ARG;
  return wv::launch_exact_trail_bwd_f64(packed, n_windows, grid_src(grid, n0), count, coefs,
                                        coef_scale, out, workspace, workspace_bytes,
                                        sm_count(), as_stream(stream));
}
int wv_exact_trail_bwd_points_f64(const void* packed, int64_t n_windows, const double* points,
                                  int64_t count, const double* coefs, double coef_scale,
                                  double* out, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (!bwd_args_ok(packed, coefs, out, n_windows, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_trail_bwd_f64(packed, n_windows, list_src(nullptr, points), count,
                                        coefs, coef_scale, out, workspace, workspace_bytes,
                                        sm_count(), as_stream(stream));
}

int wv_soft_bwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, const float* coefs, double coef_scale,
                         double* face_grad, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || !grid_ok(grid, n0, count))
    return WV_ERR_ARG;
  return wv::launch_soft_bwd_f32(packed, n_faces, grid_src(grid, n0), count, coefs, coef_scale,
                                 face_grad, workspace, workspace_bytes, sm_count(),
                                 as_stream(stream));
}

int wv_soft_bwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                           int64_t count, const float* coefs, double coef_scale,
                           double* face_grad, void* workspace, size_t workspace_bytes,
                           void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_soft_bwd_f32(packed, n_faces, list_src(points, nullptr), count, coefs,
                                 coef_scale, face_grad, workspace, workspace_bytes, sm_count(),
                                 as_stream(stream));
}

int wv_exact_bwd_grid_f64(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, const double* coefs, double coef_scale,
                          double* face_grad, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || !grid_ok(grid, n0, count))
    return WV_ERR_ARG;
  return wv::launch_exact_bwd_f64(packed, n_faces, grid_src(grid, n0), count, coefs, coef_scale,
                                  face_grad, workspace, workspace_bytes, sm_count(),
                                  as_stream(stream));
}

int wv_exact_bwd_points_f64(const void* packed, int64_t n_faces, const double* points,
                            int64_t count, const double* coefs, double coef_scale,
                            double* face_grad, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_exact_bwd_f64(packed, n_faces, list_src(nullptr, points), count, coefs,
                                  coef_scale, face_grad, workspace, workspace_bytes, sm_count(),
                                  as_stream(stream));
}

int wv_soft_bwd_grid_f64(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, const double* coefs, double coef_scale,
                         double* face_grad, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || !grid_ok(grid, n0, count))
    return WV_ERR_ARG;
  return wv::launch_soft_bwd_f64(packed, n_faces, grid_src(grid, n0), count, coefs, coef_scale,
                                 face_grad, workspace, workspace_bytes, sm_count(),
                                 as_stream(stream));
}

int wv_soft_bwd_points_f64(const void* packed, int64_t n_faces, const double* points,
                           int64_t count, const double* coefs, double coef_scale,
                           double* face_grad, void* workspace, size_t workspace_bytes,
                           void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || (count > 0 && points == nullptr))
    return WV_ERR_ARG;
  return wv::launch_soft_bwd_f64(packed, n_faces, list_src(nullptr, points), count, coefs,
                                 coef_scale, face_grad, workspace, workspace_bytes, sm_count(),
                                 as_stream(stream));
}

int wv_face_to_vertex(const double* face_grad, const int64_t* csr_offsets,
                      const int64_t* csr_slots, int64_t n_verts, const double* scale,
                      int accumulate, double* out64, float* out32, void* stream) {
  if (n_verts < 0) return WV_ERR_ARG;
  if (n_verts > 0 && (csr_offsets == nullptr || (out64 == nullptr && out32 == nullptr)))
    return WV_ERR_ARG;
  return wv::launch_face_to_vertex(face_grad, csr_offsets, csr_slots, n_verts, scale, accumulate,
                                   out64, out32, sm_count(), as_stream(stream));
}

int wv_face_to_vertex_batch(const double* face_grad, int64_t n_faces, const int64_t* csr_offsets,
                            const int64_t* csr_slots, int64_t n_verts, int64_t batch,
                            const double* scale, int64_t scale_stride, int accumulate,
                            double* out64, float* out32, void* stream) {
  if (n_verts < 0 || n_faces < 0 || batch < 1) return WV_ERR_ARG;
  if (n_verts > 0 && (csr_offsets == nullptr || (out64 == nullptr && out32 == nullptr)))
    return WV_ERR_ARG;
  return wv::launch_face_to_vertex_batch(face_grad, n_faces, csr_offsets, csr_slots, n_verts,
                                         batch, scale, scale_stride, accumulate, out64, out32,
                                         sm_count(), as_stream(stream));
}
int wv_pack_faces_batch(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                        const void* faces, int faces_i64, int64_t n_faces, int64_t batch,
                        void* packed, size_t pack_stride, void* stream) {
  if (packed == nullptr || n_verts < 0 || n_faces < 0 || batch < 1) return WV_ERR_ARG;
  if ((n_verts > 0 && vertices == nullptr) || (n_faces > 0 && faces == nullptr))
    return WV_ERR_ARG;
  if (pack_stride < wv::packed_bytes(kind, n_faces)) return WV_ERR_ARG;
  return wv::launch_pack_batch(kind, vertices, vert_f64, n_verts, faces, faces_i64, n_faces,
                               batch, packed, pack_stride, as_stream(stream));
}
int wv_loss_terms_f32_batch(const float* values, const uint8_t* flags, const float* targets,
                            const float* weights, int64_t count, int64_t batch, float* coefs,
                            double* sums, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (count <= 0 || batch < 1 || values == nullptr || flags == nullptr || targets == nullptr ||
      coefs == nullptr || sums == nullptr)
    return WV_ERR_ARG;
  return wv::launch_loss_f32_batch(values, flags, targets, weights, count, batch, coefs, sums,
                                   workspace, workspace_bytes, as_stream(stream));
}

// ---- marching cubes ------------------------------------------------------------
int wv_mc_classify(const void* values, int values_f64, wv_grid_t grid, double iso,
                   const int8_t* tri_count, uint8_t* cases, int32_t* counts, void* stream) {
  if (values == nullptr || tri_count == nullptr || cases == nullptr || counts == nullptr)
    return WV_ERR_ARG;
  for (int i = 0; i < 3; ++i)
    if (grid.res[i] < 2) return WV_ERR_ARG;
  return wv::launch_mc_classify(values, values_f64, grid.res[0], grid.res[1], grid.res[2], iso,
                                tri_count, cases, counts, sm_count(), as_stream(stream));
}

int wv_mc_edges(const void* values, int values_f64, wv_grid_t grid, double iso, int32_t* flags,
                void* stream) {
  if (values == nullptr || flags == nullptr) return WV_ERR_ARG;
  for (int i = 0; i < 3; ++i)
    if (grid.res[i] < 2) return WV_ERR_ARG;
  return wv::launch_mc_edges(values, values_f64, grid.res[0], grid.res[1], grid.res[2], iso,
                             flags, sm_count(), as_stream(stream));
}

int wv_mc_vertices(const void* values, int values_f64, wv_grid_t grid, double iso,
                   const int32_t* flags, const int64_t* vertex_index, double* vertices,
                   void* stream) {
  if (values == nullptr || flags == nullptr || vertex_index == nullptr) return WV_ERR_ARG;
  return wv::launch_mc_vertices(values, values_f64, grid_src(grid, 0).grid, 0, grid.res[0], iso,
                                flags, vertex_index, vertices, sm_count(), as_stream(stream));
}

int wv_mc_vertices_slab(const void* values, int values_f64, wv_grid_t grid, int64_t i0,
                        int64_t rows, double iso, const int32_t* flags, const int64_t* slot,
                        double* vertices, void* stream) {
  if (values == nullptr || flags == nullptr || slot == nullptr || i0 < 0 || rows < 1 ||
      i0 + rows > grid.res[0])
    return WV_ERR_ARG;
  return wv::launch_mc_vertices(values, values_f64, grid_src(grid, 0).grid, i0, rows, iso, flags,
                                slot, vertices, sm_count(), as_stream(stream));
}

int wv_mc_emit(const uint8_t* cases, const int64_t* tri_offsets, const int8_t* tri_table,
               int max_tris, const int8_t* edge_axis, const int8_t* edge_base,
               const int64_t* vertex_index, wv_grid_t grid, int64_t* faces, void* stream) {
  if (cases == nullptr || tri_offsets == nullptr || tri_table == nullptr || max_tris < 1 ||
      edge_axis == nullptr || edge_base == nullptr || vertex_index == nullptr)
    return WV_ERR_ARG;
  return wv::launch_mc_emit(cases, tri_offsets, tri_table, max_tris, edge_axis, edge_base,
                            vertex_index, grid.res[0], grid.res[1], grid.res[2], faces,
                            sm_count(), as_stream(stream));
}

// ---- loss --------------------------------------------------------------------
size_t wv_loss_workspace_bytes(int64_t count) { return wv::loss_workspace_bytes(count); }

int wv_loss_terms_f32(const float* values, const uint8_t* flags, const float* targets,
                      const float* weights, int64_t count, float* coefs, double* sums,
                      void* workspace, size_t workspace_bytes, void* stream) {
  if (count < 0 || sums == nullptr) return WV_ERR_ARG;
  if (count > 0 && (values == nullptr || flags == nullptr || targets == nullptr || coefs == nullptr))
    return WV_ERR_ARG;
  return wv::launch_loss_f32(values, flags, targets, weights, count, coefs, sums, workspace,
                             workspace_bytes, as_stream(stream));
}

int wv_loss_terms_f64(const double* values, const uint8_t* flags, const double* targets,
                      const double* weights, int64_t count, double* coefs, double* sums,
                      void* workspace, size_t workspace_bytes, void* stream) {
  if (count < 0 || sums == nullptr) return WV_ERR_ARG;
  if (count > 0 && (values == nullptr || flags == nullptr || targets == nullptr || coefs == nullptr))
    return WV_ERR_ARG;
  return wv::launch_loss_f64(values, flags, targets, weights, count, coefs, sums, workspace,
                             workspace_bytes, as_stream(stream));
}

int wv_loss_finalize(double* sums, void* stream) {
  if (sums == nullptr) return WV_ERR_ARG;
  return wv::launch_loss_finalize(sums, as_stream(stream));
}

// ---- reconstruction metrics ---------------------------------------------------
int wv_splitmix64_uniform(uint64_t seed, int64_t count, double* out, void* stream) {
  if (count < 0 || (count > 0 && out == nullptr)) return WV_ERR_ARG;
  return wv::launch_splitmix(seed, count, out, sm_count(), as_stream(stream));
}

size_t wv_pairwise_sum_workspace_bytes(int64_t n) { return wv::pairwise_workspace_bytes(n); }

int wv_pairwise_sum(const double* x, int64_t n, double* out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (n < 0 || out == nullptr || (n > 0 && x == nullptr)) return WV_ERR_ARG;
  return wv::launch_pairwise_sum(x, n, out, workspace, workspace_bytes, as_stream(stream));
}

int wv_surface_cdf(const double* vertices, const int64_t* faces, int64_t n_faces, double* areas,
                   double* cdf, double* total, void* workspace, size_t workspace_bytes,
                   void* stream) {
  if (n_faces <= 0 || vertices == nullptr || faces == nullptr || areas == nullptr ||
      cdf == nullptr || total == nullptr)
    return WV_ERR_ARG;
  return wv::launch_surface_cdf(vertices, faces, n_faces, areas, cdf, total, workspace,
                                workspace_bytes, sm_count(), as_stream(stream));
}

int wv_sample_surface(const double* vertices, const int64_t* faces, int64_t n_faces,
                      const double* cdf, const double* total, uint64_t seed, int64_t n,
                      double* out, void* stream) {
  if (n < 0 || n_faces <= 0) return WV_ERR_ARG;
  if (n > 0 && (vertices == nullptr || faces == nullptr || cdf == nullptr || total == nullptr ||
                out == nullptr))
    return WV_ERR_ARG;
  return wv::launch_sample_surface(vertices, faces, n_faces, cdf, total, seed, n, out, sm_count(),
                                   as_stream(stream));
}

int wv_nearest_distances(const double* queries, int64_t n_queries, const double* targets,
                         int64_t n_targets, double* out, void* stream) {
  if (n_queries < 0 || n_targets < 1 || targets == nullptr) return WV_ERR_ARG;
  if (n_queries > 0 && (queries == nullptr || out == nullptr)) return WV_ERR_ARG;
  return wv::launch_nearest(queries, n_queries, targets, n_targets, out, as_stream(stream));
}

// ---- batched grid kernels ------------------------------------------------------
size_t wv_fwd_workspace_bytes_batch(int kind, int64_t n_faces, int64_t count, int64_t batch) {
  if (batch < 1) return 0;
  switch (kind) {
    case WV_PACK_EXACT_F32: return wv::exact_fwd_workspace_bytes(n_faces, count, sm_count(), batch);
    case WV_PACK_SOFT_F32: return wv::soft_fwd_workspace_bytes(n_faces, count, sm_count(), batch);
    default: return 0;
  }
}

static bool batch_ok(const void* packed, size_t stride, int64_t batch) {
  return packed != nullptr && batch >= 1 && batch <= 65535 && stride % 16 == 0 &&
         (batch == 1 || stride >= 64);
}

int wv_fwd_grid_f32_batch(int kind, const void* packed, size_t pack_stride, int64_t n_faces,
                          wv_grid_t grid, int64_t n0, int64_t count, int64_t batch, int policy,
                          float* out, uint8_t* flags, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (!fwd_args_ok(packed, out, n_faces, count) || !grid_ok(grid, n0, count) ||
      !batch_ok(packed, pack_stride, batch))
    return WV_ERR_ARG;
  wv::Batch bt;
  bt.n = batch;
  bt.pack_stride = pack_stride;
  if (kind == WV_PACK_EXACT_F32)
    return wv::launch_exact_fwd_f32(packed, n_faces, grid_src(grid, n0), count, policy, out,
                                    flags, workspace, workspace_bytes, sm_count(),
                                    as_stream(stream), bt);
  if (kind == WV_PACK_SOFT_F32)
    return wv::launch_soft_fwd_f32(packed, n_faces, grid_src(grid, n0), count, policy, out, flags,
                                   workspace, workspace_bytes, sm_count(), as_stream(stream), bt);
  return WV_ERR_ARG;
}

size_t wv_bwd_workspace_bytes_batch(int kind, int64_t n_faces, int64_t count, int64_t batch) {
  if (batch < 1) return 0;
  switch (kind) {
    case WV_PACK_EXACTGRAD_F32:
      return wv::bwd_workspace_bytes(n_faces, count, sm_count(), batch);
    case WV_PACK_SOFTGRAD_F32:
      return wv::soft_bwd_workspace_bytes(n_faces, count, sm_count(), batch);
    default: return 0;
  }
}

int wv_bwd_grid_f32_batch(int kind, const void* packed, size_t pack_stride, int64_t n_faces,
                          wv_grid_t grid, int64_t n0, int64_t count, int64_t batch,
                          const float* coefs, double coef_scale, double* face_grad,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (!bwd_args_ok(packed, coefs, face_grad, n_faces, count) || !grid_ok(grid, n0, count) ||
      !batch_ok(packed, pack_stride, batch))
    return WV_ERR_ARG;
  wv::Batch bt;
  bt.n = batch;
  bt.pack_stride = pack_stride;
  if (kind == WV_PACK_EXACTGRAD_F32)
    return wv::launch_exact_bwd_f32(packed, n_faces, grid_src(grid, n0), count, coefs, coef_scale,
                                    face_grad, workspace, workspace_bytes, sm_count(),
                                    as_stream(stream), bt);
  if (kind == WV_PACK_SOFTGRAD_F32)
    return wv::launch_soft_bwd_f32(packed, n_faces, grid_src(grid, n0), count, coefs, coef_scale,
                                   face_grad, workspace, workspace_bytes, sm_count(),
                                   as_stream(stream), bt);
  return WV_ERR_ARG;
}

}  // extern "C"
