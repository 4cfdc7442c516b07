// wv_mc.cu -- marching cubes on the device-resident occupancy grid (SURVEY.md
// 8f, f2; reference recon.py:39-108).  Compiled with -fmad=false: crossing
// vertices use the reference's IEEE expression pa + t (pb - pa),
// t = (iso - va) / (vb - va), so the welded vertex array is bit-identical to
// the reference's (same crossing set, same global edge ids, same order).
//
// Pipeline (prefix sums between the passes are done by the caller):
//   classify : per cell, case index (bit c = corner c outside, value <= iso)
//              and its triangle count from the (classic) case table
//   edges    : per lattice edge (axis * N + base node), 1 if it crosses iso
//   vertices : per crossed edge, its interpolated position at its prefix slot
//   emit     : per cell, its triangles at its prefix offset, edge -> vertex id
#include "wv_kernels.h"

namespace wv {

__device__ __forceinline__ double mc_val(const void* v, int f64, int64_t i) {
  return f64 ? static_cast<const double*>(v)[i] : (double)static_cast<const float*>(v)[i];
}

__global__ void mc_classify_kernel(const void* __restrict__ vals, int f64, int64_t rx, int64_t ry,
                                   int64_t rz, double iso, const int8_t* __restrict__ count_tab,
                                   uint8_t* __restrict__ cases, int32_t* __restrict__ counts) {
  const int64_t cx = rx - 1, cy = ry - 1, cz = rz - 1;
  const int64_t n_cells = cx * cy * cz;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c / (cy * cz), rem = c - i * cy * cz, j = rem / cz, k = rem - j * cz;
    int cs = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int64_t n = ((i + (b & 1)) * ry + (j + ((b >> 1) & 1))) * rz + (k + ((b >> 2) & 1));
      if (mc_val(vals, f64, n) <= iso) cs |= 1 << b;
    }
    cases[c] = (uint8_t)cs;
    counts[c] = count_tab[cs];
  }
}

__global__ void mc_edge_kernel(const void* __restrict__ vals, int f64, int64_t rx, int64_t ry,
                               int64_t rz, double iso, int32_t* __restrict__ flags) {
  const int64_t n = rx * ry * rz;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < 3 * n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int axis = (int)(g / n);
    const int64_t node = g - axis * n;
    const int64_t i = node / (ry * rz), rem = node - i * ry * rz, j = rem / rz, k = rem - j * rz;
    const bool ok = axis == 0 ? i + 1 < rx : (axis == 1 ? j + 1 < ry : k + 1 < rz);
    int32_t f = 0;
    if (ok) {
      const int64_t stride = axis == 0 ? ry * rz : (axis == 1 ? rz : 1);
      f = (mc_val(vals, f64, node) <= iso) != (mc_val(vals, f64, node + stride) <= iso);
    }
    flags[g] = f;
  }
}

// rows i-rows of the grid starting at global row i0 (the whole grid: i0 = 0,
// rows = Rx); an edge with slot < 0 is not written (a slab's halo row)
__global__ void mc_vertex_kernel(const void* __restrict__ vals, int f64, GridDesc g, int64_t i0,
                                 int64_t rows, double iso, const int32_t* __restrict__ flags,
                                 const int64_t* __restrict__ slot, double* __restrict__ verts) {
  const int64_t ry = g.res[1], rz = g.res[2];
  const int64_t n = rows * ry * rz;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 3 * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[e] || slot[e] < 0) continue;
    const int axis = (int)(e / n);
    const int64_t node = e - axis * n;
    const int64_t i = node / (ry * rz), rem = node - i * ry * rz, j = rem / rz, k = rem - j * rz;
    const int64_t stride = axis == 0 ? ry * rz : (axis == 1 ? rz : 1);
    const double va = mc_val(vals, f64, node), vb = mc_val(vals, f64, node + stride);
    const double t = (iso - va) / (vb - va);
    const int64_t idx[3] = {i0 + i, j, k};
    double* out = verts + 3 * slot[e];
    for (int d = 0; d < 3; ++d) {
      const double pa = axis_node(g.lo[d], g.hi[d], g.res[d], idx[d]);
      const double pb = axis_node(g.lo[d], g.hi[d], g.res[d], idx[d] + (d == axis ? 1 : 0));
      out[d] = pa + t * (pb - pa);
    }
  }
}

__global__ void mc_emit_kernel(const uint8_t* __restrict__ cases,
                               const int64_t* __restrict__ tri_off,
                               const int8_t* __restrict__ tri_tab, int max_tris,
                               const int8_t* __restrict__ edge_axis,
                               const int8_t* __restrict__ edge_base, const int64_t* __restrict__ vidx,
                               int64_t rx, int64_t ry, int64_t rz, int64_t* __restrict__ faces) {
  const int64_t cx = rx - 1, cy = ry - 1, cz = rz - 1;
  const int64_t n_cells = cx * cy * cz;
  const int64_t n = rx * ry * rz;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int cs = cases[c];
    const int8_t* row = tri_tab + (int64_t)cs * 3 * max_tris;
    if (row[0] < 0) continue;
    const int64_t i = c / (cy * cz), rem = c - i * cy * cz, j = rem / cz, k = rem - j * cz;
    int64_t* out = faces + 3 * tri_off[c];
    for (int s = 0; s < 3 * max_tris && row[s] >= 0; ++s) {
      const int e = row[s];
      const int64_t node = ((i + edge_base[3 * e]) * ry + (j + edge_base[3 * e + 1])) * rz +
                           (k + edge_base[3 * e + 2]);
      out[s] = vidx[(int64_t)edge_axis[e] * n + node];
    }
  }
}

static int grid_blocks(int64_t n, int num_sms) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms * 32;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

int launch_mc_classify(const void* vals, int f64, int64_t rx, int64_t ry, int64_t rz, double iso,
                       const int8_t* count_tab, uint8_t* cases, int32_t* counts, int num_sms,
                       cudaStream_t stream) {
  const int64_t cells = (rx - 1) * (ry - 1) * (rz - 1);
  if (cells <= 0) return kOk;
  { mc_classify_kernel<<<grid_blocks(cells, num_sms), 256, 0, stream>>>(vals, f64, rx, ry, rz, iso,
                                                                      count_tab, cases, counts); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_mc_edges(const void* vals, int f64, int64_t rx, int64_t ry, int64_t rz, double iso,
                    int32_t* flags, int num_sms, cudaStream_t stream) {
  const int64_t n = 3 * rx * ry * rz;
  { mc_edge_kernel<<<grid_blocks(n, num_sms), 256, 0, stream>>>(vals, f64, rx, ry, rz, iso, flags); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_mc_vertices(const void* vals, int f64, const GridDesc& g, int64_t i0, int64_t rows,
                       double iso, const int32_t* flags, const int64_t* slot, double* verts,
                       int num_sms, cudaStream_t stream) {
  const int64_t n = 3 * rows * g.res[1] * g.res[2];
  if (n <= 0) return kOk;
  { mc_vertex_kernel<<<grid_blocks(n, num_sms), 256, 0, stream>>>(vals, f64, g, i0, rows, iso,
                                                                flags, slot, verts); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_mc_emit(const uint8_t* cases, const int64_t* tri_off, const int8_t* tri_tab,
                   int max_tris, const int8_t* edge_axis, const int8_t* edge_base,
                   const int64_t* vidx, int64_t rx, int64_t ry, int64_t rz, int64_t* faces,
                   int num_sms, cudaStream_t stream) {
  const int64_t cells = (rx - 1) * (ry - 1) * (rz - 1);
  if (cells <= 0) return kOk;
  { mc_emit_kernel<<<grid_blocks(cells, num_sms), 256, 0, stream>>>(
      cases, tri_off, tri_tab, max_tris, edge_axis, edge_base, vidx, rx, ry, rz, faces); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
