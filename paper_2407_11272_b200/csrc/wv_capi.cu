// wv_capi.cu -- extern "C" boundary (include/windvox_b200.h).  Argument
// validation, device-attribute caching, launch dispatch.  No exceptions cross
// the ABI; every entry point returns a status code.
#include <cstdio>

#include "../../include/windvox_b200.h"
#include "wv_kernels.h"

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

wv::GridDesc to_desc(const wv_grid_t& g) {
  wv::GridDesc d;
  for (int i = 0; i < 3; ++i) {
    d.lo[i] = g.lo[i];
    d.hi[i] = g.hi[i];
    d.res[i] = g.res[i];
  }
  return d;
}

bool grid_ok(const wv_grid_t& g, int64_t n0, int64_t count) {
  for (int i = 0; i < 3; ++i)
    if (g.res[i] < 1) return false;
  const int64_t n = g.res[0] * g.res[1] * g.res[2];
  return n0 >= 0 && count >= 0 && n0 + count <= n;
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

size_t wv_packed_bytes(int kind, int64_t n_faces) { return wv::packed_bytes(kind, n_faces); }

int wv_pack_faces(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                  const void* faces, int faces_i64, int64_t n_faces, void* packed,
                  void* stream) {
  if (packed == nullptr || n_verts < 0 || n_faces < 0) return WV_ERR_ARG;
  if ((n_verts > 0 && vertices == nullptr) || (n_faces > 0 && faces == nullptr))
    return WV_ERR_ARG;
  return wv::launch_pack(kind, vertices, vert_f64, n_verts, faces, faces_i64, n_faces,
                         nullptr, packed, static_cast<cudaStream_t>(stream));
}

size_t wv_fwd_workspace_bytes(int kind, int64_t n_faces, int64_t count) {
  switch (kind) {
    case WV_PACK_EXACT_F32: return wv::exact_fwd_workspace_bytes(n_faces, count, sm_count());
    default: return 0;
  }
}

int wv_exact_fwd_grid_f32(const void* packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, int policy, float* out, uint8_t* flags,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (packed == nullptr || out == nullptr || n_faces < 0) return WV_ERR_ARG;
  if (!grid_ok(grid, n0, count)) return WV_ERR_ARG;
  wv::PointSource ps{};
  ps.kind = wv::PointSource::kGrid;
  ps.grid = to_desc(grid);
  ps.n0 = n0;
  return wv::launch_exact_fwd_f32(packed, n_faces, ps, count, policy, out, flags, workspace,
                                  workspace_bytes, sm_count(),
                                  static_cast<cudaStream_t>(stream));
}

int wv_exact_fwd_points_f32(const void* packed, int64_t n_faces, const float* points,
                            int64_t count, int policy, float* out, uint8_t* flags,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (packed == nullptr || out == nullptr || n_faces < 0 || count < 0) return WV_ERR_ARG;
  if (count > 0 && points == nullptr) return WV_ERR_ARG;
  wv::PointSource ps{};
  ps.kind = wv::PointSource::kList;
  ps.points = points;
  return wv::launch_exact_fwd_f32(packed, n_faces, ps, count, policy, out, flags, workspace,
                                  workspace_bytes, sm_count(),
                                  static_cast<cudaStream_t>(stream));
}

}  // extern "C"
