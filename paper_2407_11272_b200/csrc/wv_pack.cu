// wv_pack.cu -- per-mesh staging on the device (compiled with -fmad=false so
// every f64 expression is the same IEEE sequence as the numpy reference).
//
//  * surface_eps_kernel : eps = 1e-9 * |bbox max - bbox min|
//                         (winding.py:193-197, mesh_io.py:80-88)
//  * pack_kernel        : the reference's per-face staging
//                         (_prepare_exact, winding.py:258-268, and the soft
//                         path's triangle_corners, winding.py:301) folded into
//                         one record per face.  Exact-mode degenerate faces
//                         (|N| == 0) are kept in place but marked dead, so
//                         face order is preserved without a compaction pass.
#include "wv_kernels.h"

namespace wv {

template <typename V>
__device__ __forceinline__ void load_vertex(const V* v, int64_t i, double* out) {
  out[0] = (double)v[3 * i + 0];
  out[1] = (double)v[3 * i + 1];
  out[2] = (double)v[3 * i + 2];
}
// the FP32 records describe the f32-ROUNDED mesh (the inputs the kernels
// compute with, as the reference's f32 path rounds tri, winding.py:370-373):
// normals, edge lengths, centroids and the degenerate test are derived in f64
// from the rounded corners, so alpha = N.(v0 - q) etc. are consistent with
// the corners the kernels (and their fp64 rare paths) see
template <typename V>
__device__ __forceinline__ void load_vertex_f32(const V* v, int64_t i, double* out) {
  out[0] = (double)(float)v[3 * i + 0];
  out[1] = (double)(float)v[3 * i + 1];
  out[2] = (double)(float)v[3 * i + 2];
}

template <typename V>
__global__ void surface_eps_kernel(const V* __restrict__ verts, int64_t n_verts,
                                   PackHeader* __restrict__ hdr, int64_t vstride = 0,
                                   size_t hstride = 0) {
  // batched launches: block b handles mesh b (vertices vstride elements,
  // headers hstride bytes apart)
  verts += blockIdx.x * vstride;
  hdr = reinterpret_cast<PackHeader*>(reinterpret_cast<char*>(hdr) + blockIdx.x * hstride);
  __shared__ double smin[3][1024];
  __shared__ double smax[3][1024];
  double lo[3] = {INFINITY, INFINITY, INFINITY};
  double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = threadIdx.x; i < n_verts; i += blockDim.x) {
    double p[3];
    load_vertex(verts, i, p);
    for (int d = 0; d < 3; ++d) {
      lo[d] = fmin(lo[d], p[d]);
      hi[d] = fmax(hi[d], p[d]);
    }
  }
  for (int d = 0; d < 3; ++d) {
    smin[d][threadIdx.x] = lo[d];
    smax[d][threadIdx.x] = hi[d];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int d = 0; d < 3; ++d) {
        smin[d][threadIdx.x] = fmin(smin[d][threadIdx.x], smin[d][threadIdx.x + s]);
        smax[d][threadIdx.x] = fmax(smax[d][threadIdx.x], smax[d][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double eps = 0.0;
    if (n_verts > 0) {
      const double dx = smax[0][0] - smin[0][0];
      const double dy = smax[1][0] - smin[1][0];
      const double dz = smax[2][0] - smin[2][0];
      eps = 1e-9 * sqrt(dx * dx + dy * dy + dz * dz);
    }
    hdr->eps = eps;
    hdr->eps_f32 = (float)eps;
  }
}

template <typename V, typename I>
__global__ void pack_kernel(int kind, const V* __restrict__ verts,
                            const I* __restrict__ faces, int64_t n_faces,
                            PackHeader* __restrict__ hdr, void* __restrict__ recs,
                            int64_t vstride = 0, size_t pstride = 0) {
  // batched launches: blockIdx.y = mesh (vertices vstride elements, packed
  // buffers pstride bytes apart; one connectivity)
  verts += blockIdx.y * vstride;
  hdr = reinterpret_cast<PackHeader*>(reinterpret_cast<char*>(hdr) + blockIdx.y * pstride);
  recs = static_cast<void*>(reinterpret_cast<char*>(recs) + blockIdx.y * pstride);
  const double eps = hdr->eps;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_faces;
       f += (int64_t)gridDim.x * blockDim.x) {
    double v0[3], v1[3], v2[3];
    if (kind == 1 || kind == 2 || kind == 5) {  // FP32 records: the rounded mesh
      load_vertex_f32(verts, (int64_t)faces[3 * f + 0], v0);
      load_vertex_f32(verts, (int64_t)faces[3 * f + 1], v1);
      load_vertex_f32(verts, (int64_t)faces[3 * f + 2], v2);
    } else {
      load_vertex(verts, (int64_t)faces[3 * f + 0], v0);
      load_vertex(verts, (int64_t)faces[3 * f + 1], v1);
      load_vertex(verts, (int64_t)faces[3 * f + 2], v2);
    }
    const double ux = v1[0] - v0[0], uy = v1[1] - v0[1], uz = v1[2] - v0[2];
    const double wx = v2[0] - v0[0], wy = v2[1] - v0[1], wz = v2[2] - v0[2];
    // np.cross(u, w) component order (winding.py:262)
    const double nx = uy * wz - uz * wy;
    const double ny = uz * wx - ux * wz;
    const double nz = ux * wy - uy * wx;
    if (kind == 1 || kind == 3) {
      const double norm = sqrt(nx * nx + ny * ny + nz * nz);  // np.linalg.norm
      const bool dead = !(norm > 0.0);
      if (kind == 1) {
        ExactRecF32* r = static_cast<ExactRecF32*>(recs) + f;
        const float epsN = dead ? __int_as_float(0x7f800000) : (float)(eps * norm);
        r->v0e = make_float4((float)v0[0], (float)v0[1], (float)v0[2], epsN);
        // half squared edge lengths, for a.b = (|a|^2 + |b|^2 - |v0-v1|^2) / 2
        const double h01 = 0.5 * (ux * ux + uy * uy + uz * uz);
        const double h20 = 0.5 * (wx * wx + wy * wy + wz * wz);
        const double ex = v2[0] - v1[0], ey = v2[1] - v1[1], ez = v2[2] - v1[2];
        const double h12 = 0.5 * (ex * ex + ey * ey + ez * ez);
        r->v1 = make_float4((float)v1[0], (float)v1[1], (float)v1[2], (float)h01);
        r->v2 = make_float4((float)v2[0], (float)v2[1], (float)v2[2], (float)h12);
        r->n = make_float4((float)nx, (float)ny, (float)nz, (float)h20);
      } else {
        ExactRecF64* r = static_cast<ExactRecF64*>(recs) + f;
        for (int d = 0; d < 3; ++d) {
          r->v[d] = v0[d];
          r->v[3 + d] = v1[d];
          r->v[6 + d] = v2[d];
        }
        double hx = 0.0, hy = 0.0, hz = 0.0, pld = 0.0;
        if (!dead) {
          hx = nx / norm;
          hy = ny / norm;
          hz = nz / norm;
          pld = hx * v0[0] + hy * v0[1] + hz * v0[2];  // (nhat*tri[:,0]).sum(1)
        }
        r->nhat[0] = hx;
        r->nhat[1] = hy;
        r->nhat[2] = hz;
        r->pld = pld;
        r->dead = dead ? 1.0 : 0.0;
        r->pad[0] = r->pad[1] = 0.0;
      }
    } else {
      // centroid exactly as _kernels.py:145-147 minus the (-q) term
      const double cx = v0[0] + (ux + wx) / 3.0;
      const double cy = v0[1] + (uy + wy) / 3.0;
      const double cz = v0[2] + (uz + wz) / 3.0;
      // centroid hi + lo (SoftRecF32)
      const float hx = (float)cx, hy = (float)cy, hz = (float)cz;
      const double dlx = cx - (double)hx, dly = cy - (double)hy, dlz = cz - (double)hz;
      const float lx = (float)dlx, ly = (float)dly, lz = (float)dlz;
      // near threshold on |d|^6 (SoftRecF32): (8e6 |N| |c_lo|)^2, rounded up
      const double kk = 8e6 * sqrt(nx * nx + ny * ny + nz * nz) *
                        sqrt(dlx * dlx + dly * dly + dlz * dlz);
      const float k2 = (float)(kk * kk * 1.01);
      if (kind == 2) {
        SoftRecF32* r = static_cast<SoftRecF32*>(recs) + f;
        r->c = make_float4(hx, hy, hz, (float)nx);
        // bf16 of K2 rounded UP (a larger threshold is only more careful)
        const uint32_t kb = (__float_as_uint(k2) + 0xffffu) >> 16;
        r->n = make_float4((float)ny, (float)nz,
                           __uint_as_float(bf16_bits(lx) | (bf16_bits(ly) << 16)),
                           __uint_as_float(bf16_bits(lz) | (kb << 16)));
      } else if (kind == 5) {
        SoftGradRecF32* r = static_cast<SoftGradRecF32*>(recs) + f;
        r->c = make_float4(hx, hy, hz, lx);
        r->n = make_float4((float)nx, (float)ny, (float)nz, ly);
        r->u = make_float4((float)ux, (float)uy, (float)uz, lz);
        r->w = make_float4((float)wx, (float)wy, (float)wz, k2);
      } else if (kind == 6) {
        SoftGradRecF64* r = static_cast<SoftGradRecF64*>(recs) + f;
        r->c[0] = cx; r->c[1] = cy; r->c[2] = cz;
        r->n[0] = nx; r->n[1] = ny; r->n[2] = nz;
        r->u[0] = ux; r->u[1] = uy; r->u[2] = uz;
        r->w[0] = wx; r->w[1] = wy; r->w[2] = wz;
        r->pad[0] = r->pad[1] = r->pad[2] = r->pad[3] = 0.0;
      } else {
        SoftRecF64* r = static_cast<SoftRecF64*>(recs) + f;
        r->c[0] = cx;
        r->c[1] = cy;
        r->c[2] = cz;
        r->n[0] = nx;
        r->n[1] = ny;
        r->n[2] = nz;
        r->pad[0] = r->pad[1] = 0.0;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hdr->kind = kind;
    hdr->n_faces = n_faces;
    hdr->n_live = n_faces;
  }
}

// Active faces of the exact backward (kind 7 f32, 8 f64): corners + the net
// weights of the three directed edges, computed on the host from the
// connectivity (paper_2407_11272_b200/device.py:exact_edge_weights).
template <typename V, typename I>
__global__ void pack_exact_grad_kernel(int kind, const V* __restrict__ verts,
                                       const I* __restrict__ faces,
                                       const int64_t* __restrict__ active,
                                       const float* __restrict__ weights, int64_t n_active,
                                       void* __restrict__ recs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_active;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = active[i];
    double v0[3], v1[3], v2[3];
    if (kind == 7) {  // FP32 records: the rounded mesh (squared edge lengths too)
      load_vertex_f32(verts, (int64_t)faces[3 * f + 0], v0);
      load_vertex_f32(verts, (int64_t)faces[3 * f + 1], v1);
      load_vertex_f32(verts, (int64_t)faces[3 * f + 2], v2);
    } else {
      load_vertex(verts, (int64_t)faces[3 * f + 0], v0);
      load_vertex(verts, (int64_t)faces[3 * f + 1], v1);
      load_vertex(verts, (int64_t)faces[3 * f + 2], v2);
    }
    if (kind == 7) {
      ExactGradRecF32* r = static_cast<ExactGradRecF32*>(recs) + i;
      r->a = make_float4((float)v0[0], (float)v0[1], (float)v0[2], weights[3 * i + 0]);
      r->b = make_float4((float)v1[0], (float)v1[1], (float)v1[2], weights[3 * i + 1]);
      r->c = make_float4((float)v2[0], (float)v2[1], (float)v2[2], weights[3 * i + 2]);
      double U[3] = {0.0, 0.0, 0.0};
      for (int d = 0; d < 3; ++d) {
        U[0] += (v1[d] - v0[d]) * (v1[d] - v0[d]);
        U[1] += (v2[d] - v1[d]) * (v2[d] - v1[d]);
        U[2] += (v0[d] - v2[d]) * (v0[d] - v2[d]);
      }
      r->u = make_float4((float)U[0], (float)U[1], (float)U[2], 0.0f);
    } else {
      ExactGradRecF64* r = static_cast<ExactGradRecF64*>(recs) + i;
      for (int d = 0; d < 3; ++d) {
        r->v[d] = v0[d];
        r->v[3 + d] = v1[d];
        r->v[6 + d] = v2[d];
        r->w[d] = (double)weights[3 * i + d];
      }
      r->pad[0] = r->pad[1] = r->pad[2] = r->pad[3] = 0.0;
    }
  }
}

int launch_pack_exact_grad(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                           const void* faces, int faces_i64, const int64_t* active,
                           const float* weights, int64_t n_active, void* packed,
                           cudaStream_t stream) {
  if (kind != 7 && kind != 8) return kErrArg;
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  int rc = launch_surface_eps(vertices, vert_f64, n_verts, reinterpret_cast<double*>(hdr), stream);
  if (rc != kOk) return rc;
  if (n_active <= 0) return kOk;
  void* recs = hdr + 1;
  int64_t blocks = (n_active + 255) / 256;
  if (blocks > 4096) blocks = 4096;
#define WV_PACK_EG(VT, IT)                                                                    \
  pack_exact_grad_kernel<VT, IT><<<(unsigned)blocks, 256, 0, stream>>>(                       \
      kind, static_cast<const VT*>(vertices), static_cast<const IT*>(faces), active, weights, \
      n_active, recs)
  if (vert_f64) {
    if (faces_i64) WV_PACK_EG(double, int64_t);
    else WV_PACK_EG(double, int32_t);
  } else {
    if (faces_i64) WV_PACK_EG(float, int64_t);
    else WV_PACK_EG(float, int32_t);
  }
  wv::note_launch();
#undef WV_PACK_EG
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

// Area-weighted vertex normals (mesh_io.py:176-195): every face adds its
// unnormalised cross product to its three corners, then sums are normalised
// (zero sums flagged).  The gather walks a CSR whose slots are ordered
// corner-major (k*F + f), the exact order np.add.at(n, faces[:, k], fn),
// k = 0,1,2, accumulates in -- so results are bit-identical (-fmad=false).
__global__ void vertex_normals_kernel(const double* __restrict__ verts,
                                      const int64_t* __restrict__ faces, int64_t n_faces,
                                      const int64_t* __restrict__ off,
                                      const int64_t* __restrict__ slots, int64_t n_verts,
                                      double* __restrict__ normals, uint8_t* __restrict__ zero) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_verts;
       v += (int64_t)gridDim.x * blockDim.x) {
    double s[3] = {0.0, 0.0, 0.0};
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      const int64_t f = slots[e] % n_faces;
      double p0[3], p1[3], p2[3];
      load_vertex(verts, faces[3 * f + 0], p0);
      load_vertex(verts, faces[3 * f + 1], p1);
      load_vertex(verts, faces[3 * f + 2], p2);
      const double ux = p1[0] - p0[0], uy = p1[1] - p0[1], uz = p1[2] - p0[2];
      const double wx = p2[0] - p0[0], wy = p2[1] - p0[1], wz = p2[2] - p0[2];
      s[0] += uy * wz - uz * wy;
      s[1] += uz * wx - ux * wz;
      s[2] += ux * wy - uy * wx;
    }
    const double nrm = sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
    const bool z = nrm == 0.0;
    for (int d = 0; d < 3; ++d) normals[3 * v + d] = z ? s[d] : s[d] / nrm;
    if (zero) zero[v] = z ? 1 : 0;
  }
}

int launch_vertex_normals(const double* verts, const int64_t* faces, int64_t n_faces,
                          const int64_t* off, const int64_t* slots, int64_t n_verts,
                          double* normals, uint8_t* zero, cudaStream_t stream) {
  if (n_verts <= 0) return kOk;
  int64_t blocks = (n_verts + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  { vertex_normals_kernel<<<(unsigned)blocks, 256, 0, stream>>>(verts, faces, n_faces > 0 ? n_faces : 1,
                                                              off, slots, n_verts, normals, zero); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

size_t packed_bytes(int kind, int64_t n_faces) {
  size_t rec = 0;
  switch (kind) {
    case 1: rec = sizeof(ExactRecF32); break;
    case 2: rec = sizeof(SoftRecF32); break;
    case 3: rec = sizeof(ExactRecF64); break;
    case 4: rec = sizeof(SoftRecF64); break;
    case 5: rec = sizeof(SoftGradRecF32); break;
    case 6: rec = sizeof(SoftGradRecF64); break;
    case 7: rec = sizeof(ExactGradRecF32); break;
    case 8: rec = sizeof(ExactGradRecF64); break;
    case 9: rec = sizeof(ExactRecF32); break;  // strip-ordered exact records (wv_strip.cu)
    case 10: rec = sizeof(ExactRecF64); break;  // strip-ordered f64 parity records
    case 11: rec = sizeof(TrailRecF32); break;  // edge-trail windows (wv_trail.cu)
    case 12: rec = sizeof(TrailRecF64); break;  // f64 edge-trail windows
    default: return 0;
  }
  return sizeof(PackHeader) + rec * (size_t)(n_faces > 0 ? n_faces : 0);
}

int launch_surface_eps(const void* vertices, int vert_f64, int64_t n_verts, double* eps_dev,
                       cudaStream_t stream) {
  PackHeader* hdr = reinterpret_cast<PackHeader*>(eps_dev);
  if (vert_f64)
    { surface_eps_kernel<double><<<1, 1024, 0, stream>>>(static_cast<const double*>(vertices),
                                                       n_verts, hdr); wv::note_launch(); }
  else
    { surface_eps_kernel<float><<<1, 1024, 0, stream>>>(static_cast<const float*>(vertices),
                                                      n_verts, hdr); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_pack(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                const void* faces, int faces_i64, int64_t n_faces, const double* /*eps_dev*/,
                void* packed, cudaStream_t stream) {
  if (kind < 1 || kind > 6) return kErrArg;
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  int rc = launch_surface_eps(vertices, vert_f64, n_verts, reinterpret_cast<double*>(hdr),
                              stream);
  if (rc != kOk) return rc;
  void* recs = hdr + 1;
  const int threads = 256;
  int64_t blocks = (n_faces + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  if (vert_f64) {
    const double* v = static_cast<const double*>(vertices);
    if (faces_i64)
      { pack_kernel<double, int64_t><<<(unsigned)blocks, threads, 0, stream>>>(
          kind, v, static_cast<const int64_t*>(faces), n_faces, hdr, recs); wv::note_launch(); }
    else
      { pack_kernel<double, int32_t><<<(unsigned)blocks, threads, 0, stream>>>(
          kind, v, static_cast<const int32_t*>(faces), n_faces, hdr, recs); wv::note_launch(); }
  } else {
    const float* v = static_cast<const float*>(vertices);
    if (faces_i64)
      { pack_kernel<float, int64_t><<<(unsigned)blocks, threads, 0, stream>>>(
          kind, v, static_cast<const int64_t*>(faces), n_faces, hdr, recs); wv::note_launch(); }
    else
      { pack_kernel<float, int32_t><<<(unsigned)blocks, threads, 0, stream>>>(
          kind, v, static_cast<const int32_t*>(faces), n_faces, hdr, recs); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

// One connectivity, `batch` vertex sets ((batch, n_verts, 3) contiguous): the
// packed buffers lie pack_stride bytes apart (a multiple of 16).  Two
// launches for the whole batch; each mesh's buffer equals launch_pack's.
int launch_pack_batch(int kind, const void* vertices, int vert_f64, int64_t n_verts,
                      const void* faces, int faces_i64, int64_t n_faces, int64_t batch,
                      void* packed, size_t pack_stride, cudaStream_t stream) {
  if (kind < 1 || kind > 6 || batch < 1 || batch > 65535 || pack_stride % 16 != 0)
    return kErrArg;
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  const int64_t vs = 3 * n_verts;
  if (vert_f64)
    { surface_eps_kernel<double><<<(unsigned)batch, 1024, 0, stream>>>(
        static_cast<const double*>(vertices), n_verts, hdr, vs, pack_stride); wv::note_launch(); }
  else
    { surface_eps_kernel<float><<<(unsigned)batch, 1024, 0, stream>>>(
        static_cast<const float*>(vertices), n_verts, hdr, vs, pack_stride); wv::note_launch(); }
  void* recs = hdr + 1;
  const int threads = 256;
  int64_t blocks = (n_faces + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  const dim3 grid((unsigned)blocks, (unsigned)batch);
  if (vert_f64) {
    const double* v = static_cast<const double*>(vertices);
    if (faces_i64)
      { pack_kernel<double, int64_t><<<grid, threads, 0, stream>>>(
          kind, v, static_cast<const int64_t*>(faces), n_faces, hdr, recs, vs, pack_stride); wv::note_launch(); }
    else
      { pack_kernel<double, int32_t><<<grid, threads, 0, stream>>>(
          kind, v, static_cast<const int32_t*>(faces), n_faces, hdr, recs, vs, pack_stride); wv::note_launch(); }
  } else {
    const float* v = static_cast<const float*>(vertices);
    if (faces_i64)
      { pack_kernel<float, int64_t><<<grid, threads, 0, stream>>>(
          kind, v, static_cast<const int64_t*>(faces), n_faces, hdr, recs, vs, pack_stride); wv::note_launch(); }
    else
      { pack_kernel<float, int32_t><<<grid, threads, 0, stream>>>(
          kind, v, static_cast<const int32_t*>(faces), n_faces, hdr, recs, vs, pack_stride); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
