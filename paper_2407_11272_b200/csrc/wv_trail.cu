// wv_trail.cu -- edge trails for the exact backward (host builder and the
// device packer of the trail records).
//
// The exact gradient's edge (Biot-Savart) form makes every term a function of
// ONE edge's two end POSITIONS: for the directed edge P->Q seen from q,
// T_P = -m / (4 pi |a| (|a||b| + a.b)), T_Q likewise with |b| (wv_bwd_f32.cu,
// ExactEdgeBwd), and the reversed edge's terms are the negatives.  So over a
// mesh the work is one evaluation per distinct (position-welded) EDGE, not
// per face corner: a closed surface has 1.5 edges per face where the strip-
// pair kernel evaluates 2.5, and every vertex position is shared by ~6 edges.
//
// The builder welds vertices by bitwise-equal position (weld_positions),
// collects each live face's three directed edges, and nets, per (edge, end,
// vertex id), the signs of the terms that vertex receives (a vertex id that
// gets +T and -T -- an interior edge of an index-welded mesh -- gets nothing;
// edges whose every net weight vanishes are dropped, as exact_edge_weights
// drops cancelled face edges).  The remaining edges form a multigraph-free
// graph over positions; Hierholzer's algorithm covers it with trails
// (p0, p1, p2, ...), consecutive edges sharing a position.  A trail is cut
// into WINDOWS of K = kTrailK (4) consecutive edges (K+1 positions): one thread
// of the trail backward owns a window and evaluates K+1 corner distances, K
// edge denominators and ONE shared reciprocal per query point, i.e. 1.875
// distances and 1.5 denominators per face of a closed surface (strip pairs:
// 2 and 2.5).  A short last window repeats its own edges (never read).
//
// Outputs: windows (W x (K+1) vertex ids, one representative id per
// position), and a CSR from vertex id to SIGNED slots of the kernel's output
// (slot = 2K w + 2 e + end, end 0 = the window edge's first position; a
// negative entry -s-1 subtracts slot s), in a fixed order: the gather is
// deterministic.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <parallel/algorithm>
#include <vector>

#include "wv_kernels.h"

namespace wv {

int edge_trails(const double* verts, int64_t n_verts, const int64_t* faces, int64_t n_faces,
                const uint8_t* dead, int64_t* windows, int64_t* n_windows, int64_t* csr_off,
                int64_t* csr_slots, int64_t* n_slots, int64_t* vrep) {
  *n_windows = 0;
  *n_slots = 0;
  std::vector<int64_t> canon((size_t)n_verts);
  const int64_t n_pos = weld_positions(verts, n_verts, canon.data());
  if (n_pos >= ((int64_t)1 << 31)) return kErrArg;
  std::vector<int64_t> rep((size_t)n_pos, -1);  // representative vertex id per position
  for (int64_t v = n_verts - 1; v >= 0; --v) rep[(size_t)canon[(size_t)v]] = v;
  if (vrep != nullptr)
    for (int64_t v = 0; v < n_verts; ++v) vrep[v] = rep[(size_t)canon[(size_t)v]];
  // (edge key, end, vertex, sign) of every live face's directed edges: the
  // vertex receives sign * (the canonical lo->hi edge's term at that end)
  struct Ent {
    uint64_t key;
    int64_t vert;
    int32_t end;
    int32_t sign;
  };
  std::vector<Ent> ent;
  ent.reserve((size_t)n_faces * 6);
  for (int64_t f = 0; f < n_faces; ++f) {
    if (dead != nullptr && dead[f]) continue;  // dropped by the reference forward
    for (int k = 0; k < 3; ++k) {
      const int64_t u = faces[3 * f + k], w = faces[3 * f + (k + 1) % 3];
      const int64_t pu = canon[(size_t)u], pw = canon[(size_t)w];
      if (pu == pw) continue;  // zero-length edge: its moment vanishes
      const uint64_t lo = (uint64_t)(pu < pw ? pu : pw), hi = (uint64_t)(pu < pw ? pw : pu);
      const uint64_t key = (hi << 32) | lo;
      const int32_t dir = pu < pw ? 1 : -1;  // T(u->w) = dir * T(lo->hi)
      ent.push_back({key, u, pu == (int64_t)lo ? 0 : 1, dir});
      ent.push_back({key, w, pw == (int64_t)lo ? 0 : 1, dir});
    }
  }
  __gnu_parallel::sort(ent.begin(), ent.end(), [](const Ent& a, const Ent& b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.end != b.end) return a.end < b.end;
    return a.vert < b.vert;
  });
  // net weights per (key, end, vertex); live edges = keys with a nonzero one
  std::vector<Ent> net;
  net.reserve(ent.size());
  for (size_t i = 0; i < ent.size();) {
    size_t j = i;
    int32_t s = 0;
    while (j < ent.size() && ent[j].key == ent[i].key && ent[j].end == ent[i].end &&
           ent[j].vert == ent[i].vert)
      s += ent[j++].sign;
    if (s != 0) net.push_back({ent[i].key, ent[i].vert, ent[i].end, s});
    i = j;
  }
  std::vector<uint64_t> ekeys;  // live edges, ascending key
  for (const Ent& e : net)
    if (ekeys.empty() || ekeys.back() != e.key) ekeys.push_back(e.key);
  const int64_t n_e = (int64_t)ekeys.size();
  // edge end points: live edges first, then VIRTUAL edges pairing the
  // odd-degree positions (every degree even: the graph splits into closed
  // circuits; cutting them at the virtual edges leaves trails of real ones)
  std::vector<int64_t> elo((size_t)n_e), ehi((size_t)n_e);
  std::vector<int64_t> deg((size_t)n_pos, 0);
  for (int64_t e = 0; e < n_e; ++e) {
    elo[(size_t)e] = (int64_t)(ekeys[(size_t)e] & 0xffffffffull);
    ehi[(size_t)e] = (int64_t)(ekeys[(size_t)e] >> 32);
    ++deg[(size_t)elo[(size_t)e]];
    ++deg[(size_t)ehi[(size_t)e]];
  }
  {
    int64_t pending = -1;
    for (int64_t q = 0; q < n_pos; ++q) {
      if (deg[(size_t)q] % 2 == 0) continue;
      if (pending < 0) {
        pending = q;
      } else {
        elo.push_back(pending);
        ehi.push_back(q);
        pending = -1;
      }
    }
  }
  const int64_t n_all = (int64_t)elo.size();
  auto e_lo = [&](int64_t e) { return elo[(size_t)e]; };
  // position -> incident edges (CSR, ascending edge id)
  std::vector<int64_t> aoff((size_t)n_pos + 1, 0), adj((size_t)(2 * n_all));
  for (int64_t e = 0; e < n_all; ++e) {
    ++aoff[(size_t)elo[(size_t)e] + 1];
    ++aoff[(size_t)ehi[(size_t)e] + 1];
  }
  for (int64_t q = 0; q < n_pos; ++q) aoff[(size_t)q + 1] += aoff[(size_t)q];
  {
    std::vector<int64_t> fill(aoff.begin(), aoff.end() - 1);
    for (int64_t e = 0; e < n_all; ++e) {
      adj[(size_t)fill[(size_t)elo[(size_t)e]]++] = e;
      adj[(size_t)fill[(size_t)ehi[(size_t)e]]++] = e;
    }
  }
  // Hierholzer (iterative): the popped (vertex, arrival edge) sequence is an
  // Euler circuit of the component; edge k joins popped vertices k and k+1
  std::vector<uint8_t> used((size_t)n_all, 0);
  std::vector<int64_t> ptr(aoff.begin(), aoff.end() - 1);
  std::vector<int64_t> sv, se, cv, ce, seq;
  // edge slot of each live edge: window * 3 + e, and whether the window walks it lo -> hi
  std::vector<int64_t> eslot((size_t)n_e, -1);
  std::vector<uint8_t> efwd((size_t)n_e, 0);
  int64_t W = 0;
  auto find_edge = [&](int64_t p, int64_t q) -> int64_t {
    const uint64_t lo = (uint64_t)(p < q ? p : q), hi = (uint64_t)(p < q ? q : p);
    const uint64_t key = (hi << 32) | lo;
    const auto it = std::lower_bound(ekeys.begin(), ekeys.end(), key);
    return (it != ekeys.end() && *it == key) ? (int64_t)(it - ekeys.begin()) : -1;
  };
  // seq: the positions of one trail of real edges
  constexpr int K = kTrailK;
  auto emit_trail = [&]() {
    const int64_t L = (int64_t)seq.size() - 1;  // edges
    for (int64_t j = 0; j < L; j += K) {
      const int64_t r = L - j < K ? L - j : K;  // real edges of this window
      // pad a short window by walking its own edges back and forth:
      // (p0 p1 p0 p1 ..), (p0 p1 p2 p1 ..), (p0 p1 p2 p3 p2)
      int64_t p[K + 1];
      for (int i = 0; i <= K; ++i) {
        int k = i;
        if (k > r) {
          const int b = (int)(k - r) % (2 * (int)r);
          k = b <= r ? (int)r - b : b - (int)r;
        }
        p[i] = seq[(size_t)(j + k)];
      }
      for (int i = 0; i <= K; ++i) windows[(K + 1) * W + i] = rep[(size_t)p[i]];
      for (int i = 0; i < r; ++i) {
        const int64_t e = find_edge(p[i], p[i + 1]);
        if (e < 0 || eslot[(size_t)e] >= 0) return false;
        eslot[(size_t)e] = K * W + i;
        efwd[(size_t)e] = p[i] == e_lo(e) ? 1 : 0;
      }
      ++W;
    }
    return true;
  };
  for (int64_t s0 = 0; s0 < n_pos; ++s0) {
    for (;;) {
      int64_t& p0 = ptr[(size_t)s0];
      while (p0 < aoff[(size_t)s0 + 1] && used[(size_t)adj[(size_t)p0]]) ++p0;
      if (p0 == aoff[(size_t)s0 + 1]) break;
      sv.assign(1, s0);
      se.assign(1, -1);
      cv.clear();
      ce.clear();
      while (!sv.empty()) {
        const int64_t v = sv.back();
        int64_t& pv = ptr[(size_t)v];
        while (pv < aoff[(size_t)v + 1] && used[(size_t)adj[(size_t)pv]]) ++pv;
        if (pv < aoff[(size_t)v + 1]) {
          const int64_t e = adj[(size_t)pv++];
          used[(size_t)e] = 1;
          sv.push_back(elo[(size_t)e] == v ? ehi[(size_t)e] : elo[(size_t)e]);
          se.push_back(e);
        } else {
          cv.push_back(v);
          ce.push_back(se.back());
          sv.pop_back();
          se.pop_back();
        }
      }
      // circuit: positions cv[0..K], edges ce[0..K-1] (ce[K] = -1); cut at
      // the virtual edges (rotated to start after one, if any)
      const int64_t K = (int64_t)cv.size() - 1;
      int64_t start = 0;
      for (int64_t k = 0; k < K; ++k)
        if (ce[(size_t)k] >= n_e) {
          start = k + 1;
          break;
        }
      seq.assign(1, cv[(size_t)(start % K)]);
      for (int64_t i = 0; i < K; ++i) {
        const int64_t k = (start + i) % K;
        if (ce[(size_t)k] >= n_e) {
          if (seq.size() > 1 && !emit_trail()) return kErrArg;
          seq.assign(1, cv[(size_t)((k + 1) % K)]);
        } else {
          seq.push_back(cv[(size_t)((k + 1) % K)]);
        }
      }
      if (seq.size() > 1 && !emit_trail()) return kErrArg;
    }
  }
  for (int64_t e = 0; e < n_e; ++e)
    if (eslot[(size_t)e] < 0) return kErrArg;
  // vertex -> signed output slots (entries in (key, end, vertex) order)
  std::vector<int64_t> cnt((size_t)n_verts + 1, 0);
  for (const Ent& x : net) cnt[(size_t)x.vert + 1] += std::abs(x.sign);
  for (int64_t v = 0; v < n_verts; ++v) cnt[(size_t)v + 1] += cnt[(size_t)v];
  for (int64_t v = 0; v <= n_verts; ++v) csr_off[v] = cnt[(size_t)v];
  size_t ei = 0;
  for (const Ent& x : net) {
    while (ekeys[ei] != x.key) ++ei;
    const int64_t e = (int64_t)ei;
    const int64_t w = eslot[(size_t)e] / K, k = eslot[(size_t)e] % K;
    // the window evaluates its own direction p_k -> p_k+1 (ends 0, 1); the
    // canonical lo -> hi term is that, or minus the reversed ends
    const bool fwd = efwd[(size_t)e] != 0;
    const int64_t slot = 2 * K * w + 2 * k + (fwd ? x.end : 1 - x.end);
    const int32_t sgn = (x.sign > 0 ? 1 : -1) * (fwd ? 1 : -1);
    for (int r = 0; r < std::abs(x.sign); ++r)
      csr_slots[cnt[(size_t)x.vert]++] = sgn > 0 ? slot : -slot - 1;
  }
  *n_windows = W;
  *n_slots = csr_off[n_verts];
  return kOk;
}

// Trail records (TrailRecF32): the window's K+1 positions of the f32-rounded
// mesh, p[e].w = |p[e+1] - p[e]|^2 of the rounded positions (f64, rounded
// once), p[K].w = 0.
template <typename V>
__global__ void pack_trail_kernel(const V* __restrict__ verts, const int64_t* __restrict__ win,
                                  int64_t n_windows, TrailRecF32* __restrict__ recs) {
  constexpr int K = kTrailK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_windows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p[K + 1][3];
    for (int k = 0; k <= K; ++k)
      for (int d = 0; d < 3; ++d) p[k][d] = (double)(float)verts[3 * win[(K + 1) * i + k] + d];
    TrailRecF32& r = recs[i];
    for (int k = 0; k <= K; ++k) {
      double U = 0.0;
      if (k < K)
        for (int d = 0; d < 3; ++d) U += (p[k + 1][d] - p[k][d]) * (p[k + 1][d] - p[k][d]);
      r.p[k] = make_float4((float)p[k][0], (float)p[k][1], (float)p[k][2], (float)U);
    }
  }
}

template <typename V>
__global__ void pack_trail_f64_kernel(const V* __restrict__ verts,
                                      const int64_t* __restrict__ win, int64_t n_windows,
                                      TrailRecF64* __restrict__ recs) {
  constexpr int K = kTrailK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_windows;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k <= K; ++k) {
      const int64_t v = win[(K + 1) * i + k];
      for (int d = 0; d < 3; ++d) recs[i].p[k][d] = (double)verts[3 * v + d];
      recs[i].p[k][3] = 0.0;
    }
  }
}

int launch_pack_trail_f64(const void* verts, int vert_f64, int64_t n_verts,
                          const int64_t* windows, int64_t n_windows, void* packed,
                          cudaStream_t stream) {
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  const int rc = launch_surface_eps(verts, vert_f64, n_verts, reinterpret_cast<double*>(hdr),
                                    stream);
  if (rc != kOk) return rc;
  if (n_windows <= 0) return kOk;
  TrailRecF64* recs = reinterpret_cast<TrailRecF64*>(hdr + 1);
  int64_t blocks = (n_windows + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (vert_f64)
    pack_trail_f64_kernel<double><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const double*>(verts), windows, n_windows, recs);
  else
    pack_trail_f64_kernel<float><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const float*>(verts), windows, n_windows, recs);
  wv::note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

int launch_pack_trail(const void* verts, int vert_f64, int64_t n_verts, const int64_t* windows,
                      int64_t n_windows, void* packed, cudaStream_t stream) {
  PackHeader* hdr = static_cast<PackHeader*>(packed);
  const int rc = launch_surface_eps(verts, vert_f64, n_verts, reinterpret_cast<double*>(hdr),
                                    stream);
  if (rc != kOk) return rc;
  if (n_windows <= 0) return kOk;
  TrailRecF32* recs = reinterpret_cast<TrailRecF32*>(hdr + 1);
  int64_t blocks = (n_windows + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (vert_f64)
    pack_trail_kernel<double><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const double*>(verts), windows, n_windows, recs);
  else
    pack_trail_kernel<float><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const float*>(verts), windows, n_windows, recs);
  wv::note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
