// wv_strip.cu -- face strips for the exact forward (host strip builder and
// the device packer of the strip-ordered records).
//
// The forward needs |v - q| for the three corners of every face; a vertex
// POSITION is shared by ~6 faces of a surface (triangle soups included: their
// copies of a position are bitwise equal).  Walking the faces as strips
// (face k+1 shares two corner positions with face k), a thread keeps the two
// shared distances in registers and evaluates ONE new square root per face
// instead of three.  Only the order of the faces and the roles of their
// corners change; W is a sum over faces, so the result is the same up to
// fp32 summation order.
//
// A strip record is an ExactRecF32 whose corners are in WINDOW order (A, B, C)
// with A, B at the positions of the previous record's B, C (unless the
// record restarts the strip); N is the face's own normal in its true
// orientation, so alpha = N.(A - q) keeps the true sign (any corner of the
// face gives the same alpha).  The .w fields carry (16/7) x the half squared
// edge lengths (>= 0; the strip kernel's beta constants, ExactStripPol), and
// flags live in their sign bits: v1.w < 0 marks a restart, v2.w < 0 a window that is a
// reflection of the face's vertex order (the fp64 rare path needs the true
// order for its triple product).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <parallel/algorithm>  // __gnu_parallel::sort (OpenMP: the host's cores)
#include <vector>

#include "wv_kernels.h"

namespace wv {

// Canonical position id per vertex (bitwise-equal f64 coordinates weld):
// ids are dense, in ascending order of the coordinate bit patterns; returns
// the number of distinct positions.  Total orders on both sides, so the
// parallel sort's result is independent of the thread count.
int64_t weld_positions(const double* verts, int64_t n_verts, int64_t* canon) {
  struct VK {
    uint64_t x, y, z;
    int64_t i;
  };
  std::vector<VK> ord((size_t)n_verts);
  for (int64_t i = 0; i < n_verts; ++i) {
    VK& o = ord[(size_t)i];
    std::memcpy(&o.x, verts + 3 * i, 8);
    std::memcpy(&o.y, verts + 3 * i + 1, 8);
    std::memcpy(&o.z, verts + 3 * i + 2, 8);
    o.i = i;
  }
  __gnu_parallel::sort(ord.begin(), ord.end(), [](const VK& a, const VK& b) {
    if (a.x != b.x) return a.x < b.x;
    if (a.y != b.y) return a.y < b.y;
    if (a.z != b.z) return a.z < b.z;
    return a.i < b.i;
  });
  int64_t id = -1;
  for (size_t r = 0; r < ord.size(); ++r) {
    if (r == 0 || ord[r].x != ord[r - 1].x || ord[r].y != ord[r - 1].y ||
        ord[r].z != ord[r - 1].z)
      ++id;
    canon[ord[r].i] = id;
  }
  return id + 1;
}

// perm[k]: face of strip position k; win[3k..3k+2]: its vertex indices in
// window order; flags[k]: bit0 restart, bit1 reflected window.
// Sort-based (no hash maps): ~20 ms per 100k faces on one core.
int strip_order(const double* verts, int64_t n_verts, const int64_t* faces, int64_t n_faces,
                int64_t* perm, int64_t* win, uint8_t* flags) {
  // canonical position id per vertex: sort by the coordinate bit patterns
  std::vector<int64_t> canon((size_t)n_verts);
  weld_positions(verts, n_verts, canon.data());
  auto cid = [&](int64_t f, int c) { return canon[(size_t)faces[3 * f + c]]; };
  // half-edges (canonical undirected key, face, local edge) sorted by key;
  // run[3f+e] = start of the run of face f's edge e (corners e, e+1)
  struct HE {
    uint64_t key;
    int64_t slot;  // 3 f + e
  };
  std::vector<HE> he;
  he.reserve((size_t)n_faces * 3);
  std::vector<uint8_t> dead((size_t)n_faces, 0);
  auto ekey = [](int64_t a, int64_t b) {
    const uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
    return (hi << 32) | lo;  // canonical ids < 2^32 (n_faces < 2^31)
  };
  for (int64_t f = 0; f < n_faces; ++f) {
    const int64_t a = cid(f, 0), b = cid(f, 1), c = cid(f, 2);
    if (a == b || b == c || c == a) {
      dead[(size_t)f] = 1;  // two coincident corners: zero area, never shares a window
      continue;
    }
    he.push_back({ekey(a, b), 3 * f});
    he.push_back({ekey(b, c), 3 * f + 1});
    he.push_back({ekey(c, a), 3 * f + 2});
  }
  __gnu_parallel::sort(he.begin(), he.end(), [](const HE& x, const HE& y) {
    return x.key < y.key || (x.key == y.key && x.slot < y.slot);
  });
  std::vector<int64_t> run((size_t)n_faces * 3, -1);
  for (size_t i = 0, r = 0; i < he.size(); ++i) {
    if (he[i].key != he[r].key) r = i;
    run[(size_t)he[i].slot] = (int64_t)r;
  }
  std::vector<uint8_t> used((size_t)n_faces, 0);
  // an unused face other than cur across the canonical edge (p, q) of cur
  auto next_face = [&](int64_t cur, int64_t p, int64_t q) -> int64_t {
    const uint64_t k = ekey(p, q);
    for (int e = 0; e < 3; ++e) {
      if (ekey(cid(cur, e), cid(cur, (e + 1) % 3)) != k) continue;
      const int64_t r0 = run[(size_t)(3 * cur + e)];
      if (r0 < 0) return -1;
      for (size_t i = (size_t)r0; i < he.size() && he[i].key == k; ++i) {
        const int64_t g = he[i].slot / 3;
        if (g != cur && !used[(size_t)g]) return g;
      }
      return -1;
    }
    return -1;
  };
  int64_t k = 0;
  auto emit = [&](int64_t f, int64_t A, int64_t B, int64_t C, bool restart) {
    perm[k] = f;
    win[3 * k] = A;
    win[3 * k + 1] = B;
    win[3 * k + 2] = C;
    // parity of the window against the face's own vertex order
    int pa = 0, pb = 0, pc = 0;
    for (int c = 0; c < 3; ++c) {
      if (faces[3 * f + c] == A) pa = c;
      if (faces[3 * f + c] == B) pb = c;
      if (faces[3 * f + c] == C) pc = c;
    }
    const bool even = (pb == (pa + 1) % 3) && (pc == (pb + 1) % 3);
    flags[k] = (uint8_t)((restart ? 1 : 0) | (even ? 0 : 2));
    used[(size_t)f] = 1;
    ++k;
  };
  // a face's indices at the positions p, q (the window's A, B) and its third
  auto orient = [&](int64_t g, int64_t p, int64_t q, int64_t& iA, int64_t& iB, int64_t& iC) {
    iA = iB = iC = -1;
    for (int c = 0; c < 3; ++c) {
      const int64_t v = faces[3 * g + c];
      if (canon[(size_t)v] == p && iA < 0) iA = v;
      else if (canon[(size_t)v] == q && iB < 0) iB = v;
      else iC = v;
    }
  };
  std::vector<int64_t> back;   // faces before the start face, nearest first
  std::vector<int64_t> bwin;
  for (int64_t f0 = 0; f0 < n_faces; ++f0) {
    if (used[(size_t)f0]) continue;
    const int64_t* t = faces + 3 * f0;
    if (dead[(size_t)f0]) {
      emit(f0, t[0], t[1], t[2], true);
      continue;
    }
    // rotation whose (B, C) edge continues the strip
    int rot = 0;
    for (int r = 0; r < 3; ++r)
      if (next_face(f0, canon[(size_t)t[(r + 1) % 3]], canon[(size_t)t[(r + 2) % 3]]) >= 0) {
        rot = r;
        break;
      }
    const int64_t A0 = t[rot], B0 = t[(rot + 1) % 3], C0 = t[(rot + 2) % 3];
    // grow backwards first: the face before a window (A, B, C) has the window
    // (X, A, B); it is emitted ahead of the start face
    used[(size_t)f0] = 1;
    back.clear();
    bwin.clear();
    {
      int64_t a = A0, b = B0, cur = f0;
      for (;;) {
        const int64_t g = next_face(cur, canon[(size_t)a], canon[(size_t)b]);
        if (g < 0) break;
        int64_t iA, iB, iC;  // g's corners at a, b and its third
        orient(g, canon[(size_t)a], canon[(size_t)b], iA, iB, iC);
        used[(size_t)g] = 1;
        back.push_back(g);
        bwin.push_back(iC);
        bwin.push_back(iA);
        bwin.push_back(iB);
        b = iA;
        a = iC;
        cur = g;
      }
    }
    for (size_t i = back.size(); i-- > 0;)
      emit(back[i], bwin[3 * i], bwin[3 * i + 1], bwin[3 * i + 2], i + 1 == back.size());
    emit(f0, A0, B0, C0, back.empty());
    int64_t B = B0, C = C0, cur = f0;
    for (;;) {
      const int64_t g = next_face(cur, canon[(size_t)B], canon[(size_t)C]);
      if (g < 0) break;
      int64_t nA, nB, nC;
      orient(g, canon[(size_t)B], canon[(size_t)C], nA, nB, nC);
      emit(g, nA, nB, nC, false);
      B = nB;
      C = nC;
      cur = g;
    }
  }
  return k == n_faces ? kOk : kErrArg;
}

template <typename V, typename I>
__global__ void pack_strip_kernel(const V* __restrict__ verts, const I* __restrict__ faces,
                                  const int64_t* __restrict__ perm,
                                  const int64_t* __restrict__ win,
                                  const uint8_t* __restrict__ flags, int64_t n_faces,
                                  PackHeader* __restrict__ hdr, ExactRecF32* __restrict__ recs) {
  const double eps = hdr->eps;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_faces;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = perm[k];
    double t[3][3], w[3][3];
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) {
        // the rounded mesh, as pack_kernel's FP32 kinds
        t[c][d] = (double)(float)verts[3 * (int64_t)faces[3 * f + c] + d];
        w[c][d] = (double)(float)verts[3 * win[3 * k + c] + d];
      }
    // true-orientation normal, as pack_kernel (winding.py:262)
    const double ux = t[1][0] - t[0][0], uy = t[1][1] - t[0][1], uz = t[1][2] - t[0][2];
    const double wx = t[2][0] - t[0][0], wy = t[2][1] - t[0][1], wz = t[2][2] - t[0][2];
    const double nx = uy * wz - uz * wy, ny = uz * wx - ux * wz, nz = ux * wy - uy * wx;
    const double norm = sqrt(nx * nx + ny * ny + nz * nz);
    const bool dead = !(norm > 0.0);
    const float epsN = dead ? __int_as_float(0x7f800000) : (float)(eps * norm);
    auto half2 = [&](int i, int j) {
      const double a = w[j][0] - w[i][0], b = w[j][1] - w[i][1], c = w[j][2] - w[i][2];
      return 0.5 * (a * a + b * b + c * c);
    };
    bool restart = (flags[k] & 1) != 0 || (k % 128) == 0;  // every tile (and split) restarts
    if (!restart) {
      // the carried distances are only valid for bitwise-equal f32 positions
      const int64_t* pw = win + 3 * (k - 1);
      for (int d = 0; d < 3; ++d) {
        restart |= (float)verts[3 * pw[1] + d] != (float)w[0][d];
        restart |= (float)verts[3 * pw[2] + d] != (float)w[1][d];
      }
    }
    // the strip kernel's beta uses (16/7) h (ExactStripPol::strip_fast), so
    // the records carry that, rounded once from f64 (its rare tail restores h)
    constexpr double kL = 16.0 / 7.0;
    const float hab = (float)(kL * half2(0, 1)), hbc = (float)(kL * half2(1, 2));
    const float hca = (float)(kL * half2(2, 0));
    ExactRecF32& r = recs[k];
    r.v0e = make_float4((float)w[0][0], (float)w[0][1], (float)w[0][2], epsN);
    // sign bits as flags (set on the bit pattern: a zero length gives -0.0)
    const float fab = restart ? __int_as_float(__float_as_int(hab) | 0x80000000) : hab;
    const float fbc = (flags[k] & 2) ? __int_as_float(__float_as_int(hbc) | 0x80000000) : hbc;
    r.v1 = make_float4((float)w[1][0], (float)w[1][1], (float)w[1][2], fab);
    r.v2 = make_float4((float)w[2][0], (float)w[2][1], (float)w[2][2], fbc);
    r.n = make_float4((float)nx, (float)ny, (float)nz, hca);
  }
}

// f64 parity records in strip order: the reference's own per-face arrays
// (true vertex order, nhat, pld, dead -- bit-identical to pack_kernel kind 3)
// plus pad[0] = strip restart (1.0 / 0.0) and pad[1] = the window as true
// corner indices, iA + 3 iB (iC = 3 - iA - iB).  Restarts every kF64Tile (64)
// records and wherever the window's A, B are not bitwise the previous B, C.
template <typename V, typename I>
__global__ void pack_strip_f64_kernel(const V* __restrict__ verts, const I* __restrict__ faces,
                                      const int64_t* __restrict__ perm,
                                      const int64_t* __restrict__ win,
                                      const uint8_t* __restrict__ flags, int64_t n_faces,
                                      ExactRecF64* __restrict__ recs) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_faces;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = perm[k];
    int64_t vi[3];
    double v[3][3];
    for (int c = 0; c < 3; ++c) {
      vi[c] = (int64_t)faces[3 * f + c];
      for (int d = 0; d < 3; ++d) v[c][d] = (double)verts[3 * vi[c] + d];
    }
    const double ux = v[1][0] - v[0][0], uy = v[1][1] - v[0][1], uz = v[1][2] - v[0][2];
    const double wx = v[2][0] - v[0][0], wy = v[2][1] - v[0][1], wz = v[2][2] - v[0][2];
    const double nx = uy * wz - uz * wy;
    const double ny = uz * wx - ux * wz;
    const double nz = ux * wy - uy * wx;
    const double norm = sqrt(nx * nx + ny * ny + nz * nz);
    const bool dead = !(norm > 0.0);
    ExactRecF64& r = recs[k];
    for (int d = 0; d < 3; ++d) {
      r.v[d] = v[0][d];
      r.v[3 + d] = v[1][d];
      r.v[6 + d] = v[2][d];
    }
    double hx = 0.0, hy = 0.0, hz = 0.0, pld = 0.0;
    if (!dead) {
      hx = nx / norm;
      hy = ny / norm;
      hz = nz / norm;
      pld = hx * v[0][0] + hy * v[0][1] + hz * v[0][2];
    }
    r.nhat[0] = hx;
    r.nhat[1] = hy;
    r.nhat[2] = hz;
    r.pld = pld;
    r.dead = dead ? 1.0 : 0.0;
    // window corners as true corner indices
    int ic[3] = {0, 1, 2};
    for (int c = 0; c < 3; ++c)
      for (int t = 0; t < 3; ++t)
        if (vi[t] == win[3 * k + c]) ic[c] = t;
    bool restart = (flags[k] & 1) != 0 || (k % 64) == 0;
    if (!restart) {
      const int64_t* pw = win + 3 * (k - 1);
      for (int d = 0; d < 3; ++d) {
        restart |= (double)verts[3 * pw[1] + d] != v[ic[0]][d];
        restart |= (double)verts[3 * pw[2] + d] != v[ic[1]][d];
      }
    }
    r.pad[0] = restart ? 1.0 : 0.0;
    r.pad[1] = (double)(ic[0] + 3 * ic[1]);
  }
}

int launch_pack_strip_f64(const void* verts, int vert_f64, int64_t n_verts, const void* faces,
                          int faces_i64, int64_t n_faces, const int64_t* perm,
                          const int64_t* win, const uint8_t* flags, void* packed,
                          cudaStream_t stream) {
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  const int rc = launch_surface_eps(verts, vert_f64, n_verts, reinterpret_cast<double*>(hdr),
                                    stream);
  if (rc != kOk) return rc;
  ExactRecF64* recs = reinterpret_cast<ExactRecF64*>(hdr + 1);
  const int blocks = (int)((n_faces + 255) / 256 > 0 ? (n_faces + 255) / 256 : 1);
#define WV_PSF(VT, IT)                                                                       \
  pack_strip_f64_kernel<VT, IT><<<blocks, 256, 0, stream>>>(                                  \
      static_cast<const VT*>(verts), static_cast<const IT*>(faces), perm, win, flags, n_faces, \
      recs)
  if (vert_f64) {
    if (faces_i64) WV_PSF(double, int64_t);
    else WV_PSF(double, int32_t);
  } else {
    if (faces_i64) WV_PSF(float, int64_t);
    else WV_PSF(float, int32_t);
  }
  wv::note_launch();
#undef WV_PSF
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_pack_strip(const void* verts, int vert_f64, int64_t n_verts, const void* faces,
                      int faces_i64, int64_t n_faces, const int64_t* perm, const int64_t* win,
                      const uint8_t* flags, void* packed, cudaStream_t stream) {
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  const int rc = launch_surface_eps(verts, vert_f64, n_verts, reinterpret_cast<double*>(hdr), stream);
  if (rc != kOk) return rc;
  ExactRecF32* recs = reinterpret_cast<ExactRecF32*>(hdr + 1);
  const int blocks = (int)((n_faces + 255) / 256 > 0 ? (n_faces + 255) / 256 : 1);
  if (vert_f64 && faces_i64)
    { pack_strip_kernel<double, int64_t><<<blocks, 256, 0, stream>>>(
        static_cast<const double*>(verts), static_cast<const int64_t*>(faces), perm, win, flags,
        n_faces, hdr, recs); wv::note_launch(); }
  else if (vert_f64)
    { pack_strip_kernel<double, int32_t><<<blocks, 256, 0, stream>>>(
        static_cast<const double*>(verts), static_cast<const int32_t*>(faces), perm, win, flags,
        n_faces, hdr, recs); wv::note_launch(); }
  else if (faces_i64)
    { pack_strip_kernel<float, int64_t><<<blocks, 256, 0, stream>>>(
        static_cast<const float*>(verts), static_cast<const int64_t*>(faces), perm, win, flags,
        n_faces, hdr, recs); wv::note_launch(); }
  else
    { pack_strip_kernel<float, int32_t><<<blocks, 256, 0, stream>>>(
        static_cast<const float*>(verts), static_cast<const int32_t*>(faces), perm, win, flags,
        n_faces, hdr, recs); wv::note_launch(); }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
