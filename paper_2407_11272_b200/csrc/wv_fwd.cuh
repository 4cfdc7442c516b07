// wv_fwd.cuh -- generic FP32 all-pairs forward (point per thread, faces
// streamed through a TMA ring).  Instantiated by wv_fwd_f32.cu with the exact
// (Van Oosterom-Strackee) and soft (dipole) pair policies.
//
//  * TILE-record tiles of the packed face array stream into a STAGES-deep
//    shared-memory ring with cp.async.bulk (TMA, SASS UBLKCP); the last warp
//    to finish a tile issues the refill of its slot (no producer warp);
//  * each consumer thread holds P query points in registers and walks the
//    tiles in face order; per face it evaluates the common path for all P
//    points branch-free and defers the few "rare" pairs (near-plane /
//    wide-angle / on-surface candidates) to an out-of-line handler;
//  * per tile the terms are summed in fp32, tile partials in fp64;
//  * lattice rows (RowSrc): when the node range is row-aligned, a thread
//    takes P CONSECUTIVE nodes of one k-row, so x and y are common to its
//    points and the x/y parts of each pair term are per-face scalars
//    (Pol::row, once per face) -- the per-pair work drops by ~1/3.
#pragma once

#include <type_traits>

#include "wv_f32x2.cuh"
#include "wv_kernels.h"

namespace wv {

template <class Pol, class Src>
__global__ void __launch_bounds__(Pol::kThreads, Src::kRows ? Pol::kMinBlocksRow : Pol::kMinBlocks)
fwd_f32_kernel(const PackHeader* __restrict__ hdr, const typename Pol::Rec* __restrict__ recs,
               size_t pack_stride, int64_t n_faces, Src src, int64_t n_count,
               int64_t tiles_per_split, OutF32 o) {
  using Rec = typename Pol::Rec;
  constexpr int TILE = Pol::kTile;
  constexpr int STAGES = Pol::kStages;
  constexpr int CW = Pol::kConsumerWarps;
  constexpr int NC = CW * 32;
  constexpr int P = Pol::kP;
  __shared__ FaceRing<Rec, TILE, STAGES> ring;
  // fp64 per-point accumulators live in shared memory ([p][thread]): they are
  // touched once per tile (and by rare pairs), and keeping them out of the
  // register file leaves the 128-register budget to the pair arithmetic
  __shared__ double accs[P][NC];
  // warp rows (RowSrcW, strip policies): per tile, lane i computes the row
  // terms of faces i, i+32, ... for the warp's k-row; every lane reads them
  // back (a broadcast LDS.64 per face instead of 6 FP32 ops per face)
  // (face-ordered pairs: all four row terms of each face the same way)
  constexpr bool kTab = [] {
    if constexpr (Src::kRows) return Src::kWarpRow && Pol::kStrip;
    else return false;
  }();
  constexpr bool kTabF = [] {
    if constexpr (Src::kRows) return Src::kWarpRow && !Pol::kStrip && Pol::kPairFaces;
    else return false;
  }();
  __shared__ float2 rtab[kTab ? CW : 1][kTab ? TILE : 1];
  // (half a tile at a time: the whole-tile table would pass the 48 KB of
  // static shared memory next to the 4-stage ring)
  constexpr int kHalf = TILE / 2;
  __shared__ typename Pol::Row rtabf[kTabF ? CW : 1][kTabF ? kHalf : 1];
  // batched launches: blockIdx.z selects the mesh (its packed records lie
  // pack_stride bytes apart; its outputs n_count apart)
  hdr = reinterpret_cast<const PackHeader*>(reinterpret_cast<const char*>(hdr) +
                                            blockIdx.z * pack_stride);
  recs = reinterpret_cast<const Rec*>(hdr + 1);
  const int64_t zoff = (int64_t)blockIdx.z * n_count;
  const int64_t n_tiles = (n_faces + TILE - 1) / TILE;
  const int64_t t_begin = (int64_t)blockIdx.y * tiles_per_split;
  int64_t t_end = t_begin + tiles_per_split;
  if (t_end > n_tiles) t_end = n_tiles;
  ring_start(ring, recs, n_faces, t_begin, t_end);

  const float eps = hdr->eps_f32;
  const double eps64 = hdr->eps;
  const int tid = threadIdx.x;
  constexpr bool kRows = Src::kRows;
  const int64_t base = (int64_t)blockIdx.x * (NC * P);
  // row mode: thread group g owns nodes g*P .. g*P+P-1 (one k-row segment)
  const int64_t n_groups = n_count / P;
  const int64_t grp = (int64_t)blockIdx.x * NC + tid;
  const int64_t g0 = (grp < n_groups ? grp : n_groups - 1) * P;
  constexpr int PP = P / 2;  // point pairs (packed f32x2)
  F2 qx[PP], qy[PP], qz[PP];
  float rx = 0.0f, ry = 0.0f;
#pragma unroll
  for (int pp = 0; pp < PP; ++pp) {
    float x[2], y[2], z[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t l = kRows ? g0 + 2 * pp + h : base + (2 * pp + h) * NC + tid;
      if (l >= n_count) l = n_count - 1;  // padded lanes recompute a valid node
      src.point(l, x[h], y[h], z[h]);
      accs[2 * pp + h][tid] = 0.0;
    }
    qx[pp] = f2(x[0], x[1]);
    qy[pp] = f2(y[0], y[1]);
    qz[pp] = f2(z[0], z[1]);
    rx = x[0];
    ry = y[0];
  }
  typename Pol::Ctx ctx = Pol::make_ctx(eps);
  uint32_t hits = 0;
  typename Pol::Slot slot[3][PP];  // strip policies: corner distances (ring of 3 slots)
  [[maybe_unused]] float rrow[3] = {0.0f, 0.0f, 0.0f};  // strip policies: row parts of |v - q|^2

  for (int64_t t = t_begin; t < t_end; ++t) {
    const int64_t it = t - t_begin;
    const int s = (int)(it % STAGES);
    mbar_wait(&ring.full[s], (uint32_t)((it / STAGES) & 1));
    const int64_t first = t * TILE;
    const int cnt = (int)((n_faces - first) < TILE ? (n_faces - first) : TILE);
    const Rec* tile = ring.tiles[s];
    F2 tacc[PP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) tacc[pp] = f2(0.0f, 0.0f);

    [[maybe_unused]] const int wrpf = tid >> 5;
    [[maybe_unused]] int tab0 = 0;  // first face of the table's half tile
    [[maybe_unused]] auto fill_half = [&](int h0) {
      __syncwarp();  // the previous half's terms are consumed
#pragma unroll
      for (int k = 0; k < kHalf / 32; ++k) {
        const int fi = h0 + (tid & 31) + 32 * k;
        if (fi < cnt) rtabf[wrpf][fi - h0] = Pol::row(tile[fi], rx, ry);
      }
      tab0 = h0;
      __syncwarp();
    };
    // the row terms of a face: the warp's table (warp rows) or computed
    auto row_f = [&](const Rec& R) {
      if constexpr (kTabF) return rtabf[wrpf][(&R - tile) - tab0];
      else return Pol::row(R, rx, ry);
    };
    // lanes of one face that the fp32 paths left to the fp64 path
    auto do_rare = [&](const Rec& R, uint32_t rare) {
      if (rare != 0u) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (rare & (1u << p)) {
            float xl, xh, yl, yh, zl, zh;
            split(qx[p / 2], xl, xh);
            split(qy[p / 2], yl, yh);
            split(qz[p / 2], zl, zh);
            const bool hi = p & 1;
            const float px = kRows ? rx : (hi ? xh : xl), py = kRows ? ry : (hi ? yh : yl);
            const double th = Pol::rare(R, px, py, hi ? zh : zl, eps64);
            if (th != th) hits |= 1u << p;  // NaN marks an on-surface pair
            else accs[p][tid] += th;        // rare terms go straight to fp64
          }
        }
      }
    };
    // one face against the thread's P points
    auto do_face = [&](const Rec& R, auto) {
      uint32_t rare;
      if constexpr (kRows) {
        // groups of (at most) 4 point pairs: the per-face row constants are
        // shared by all of a thread's points, the temporaries by one group
        rare = 0;
        {
          const typename Pol::Row w = row_f(R);
#pragma unroll
          for (int g0 = 0; g0 < PP; g0 += 4)
            rare |= Pol::template face_row<(PP < 4 ? PP : 4)>(R, w, qz + g0, ctx, tacc + g0)
                    << (2 * g0);
        }
      } else {
        rare = 0;
#pragma unroll
        for (int g0 = 0; g0 < PP; g0 += 4)
          rare |= Pol::template face<(PP < 4 ? PP : 4)>(R, qx + g0, qy + g0, qz + g0, ctx,
                                                          tacc + g0) << (2 * g0);
      }
      do_rare(R, rare);
    };
    using R0 = std::integral_constant<int, 0>;
    using R1 = std::integral_constant<int, 1>;
    using R2 = std::integral_constant<int, 2>;
    if constexpr (Pol::kStrip && kRows) {
      static_assert(PP <= Pol::kGroup, "strip faces are decided for all point pairs at once");
      [[maybe_unused]] const int wrp = tid >> 5;
      if constexpr (kTab) {
        __syncwarp();  // the previous tile's terms are consumed
#pragma unroll
        for (int k = 0; k < TILE / 32; ++k) {
          const int fi = (tid & 31) + 32 * k;
          if (fi < cnt) {
            const typename Pol::Row w = Pol::row_c(tile[fi], rx, ry);
            rtab[wrp][fi] = make_float2(w.c2, w.alpha);
          }
        }
        __syncwarp();
      }
      // the row terms of face R (its C corner): the warp's table or computed
      auto row_c = [&](const Rec& R) {
        if constexpr (kTab) {
          const float2 v = rtab[wrp][&R - tile];
          typename Pol::Row w;
          w.c2 = v.x;
          w.alpha = v.y;
          return w;
        } else {
          return Pol::row_c(R, rx, ry);
        }
      };
      // one strip face's common-path terms; the slots rotate by kRot
      // may_restart: false when the caller has checked that R continues its
      // strip (then the block has no restart branch)
      auto fast = [&](const Rec& R, auto rot, F2* tq, F2* tp, auto may_restart) -> bool {
        constexpr int kRot = decltype(rot)::value;
        const bool restart =
            decltype(may_restart)::value && __float_as_int(R.v1.w) < 0;  // uniform per face
        // the row parts of |A - q|^2, |B - q|^2 are the previous faces'
        // |C - q|^2 row parts (ring of 3, like the distance slots)
        typename Pol::Row w = row_c(R);
        if (restart) Pol::row_ab(R, rx, ry, rrow[kRot], rrow[(kRot + 1) % 3]);
        w.a2 = rrow[kRot];
        w.b2 = rrow[(kRot + 1) % 3];
        rrow[(kRot + 2) % 3] = w.c2;
        return Pol::template strip_fast<PP>(R, w, qz, ctx, restart, slot[kRot],
                                            slot[(kRot + 1) % 3], slot[(kRot + 2) % 3], tq, tp);
      };
      auto commit = [&](const Rec& R, bool ok, const F2* tq, const F2* tp) {
        if (ok) {
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) tacc[pp] = fma2(tq[pp], tp[pp], tacc[pp]);
        } else {
          do_rare(R, Pol::template strip_slow<PP>(R, rx, ry, qz, ctx, tacc));
        }
      };
      // two faces per decision: face k's tail overlaps face k+1's square
      // roots (one branch per two faces); terms are added in face order
#ifndef WV_STRIP_PAIR_TERMS
#define WV_STRIP_PAIR_TERMS 1  // 1287.6 ms vs 1290.7 (speculative tacc) on C3
#endif
      using Yes = std::true_type;
      using No = std::false_type;
      // the row part of a face: C's computed, A's and B's carried (ring of 3)
      auto row_of = [&](const Rec& R, auto rot, auto may_restart, bool& restart) {
        constexpr int kRot = decltype(rot)::value;
        restart = decltype(may_restart)::value && __float_as_int(R.v1.w) < 0;
        typename Pol::Row w = row_c(R);
        if (restart) Pol::row_ab(R, rx, ry, rrow[kRot], rrow[(kRot + 1) % 3]);
        w.a2 = rrow[kRot];
        w.b2 = rrow[(kRot + 1) % 3];
        rrow[(kRot + 2) % 3] = w.c2;
        return w;
      };
      auto pair_body = [&](const Rec& Ra, const Rec& Rb, auto rota, auto rotb, auto mr) {
       if constexpr (Pol::kPairAngle && !decltype(mr)::value) {
        // both faces continue their strip: one angle evaluation for the pair
        constexpr int ka = decltype(rota)::value, kb = decltype(rotb)::value;
        bool ra, rb;
        const typename Pol::Row wa = row_of(Ra, rota, mr, ra);
        const typename Pol::Row wb = row_of(Rb, rotb, mr, rb);
        {
          F2 tq[PP], tp[PP];
          if (Pol::template strip_pair_fast<PP>(Ra, wa, Rb, wb, qz, ctx, slot[ka],
                                                slot[(ka + 1) % 3], slot[(ka + 2) % 3],
                                                slot[(kb + 2) % 3], tq, tp)) {
#pragma unroll
            for (int pp = 0; pp < PP; ++pp) tacc[pp] = fma2(tq[pp], tp[pp], tacc[pp]);
            return;
          }
        }
        // rare: face by face (face a restarts: its A slot now holds b's C)
        F2 tqa[PP], tpa[PP], tqb[PP], tpb[PP];
        const bool oka = Pol::template strip_fast<PP>(Ra, wa, qz, ctx, true, slot[ka],
                                                      slot[(ka + 1) % 3], slot[(ka + 2) % 3],
                                                      tqa, tpa);
        const bool okb = Pol::template strip_fast<PP>(Rb, wb, qz, ctx, false, slot[kb],
                                                      slot[(kb + 1) % 3], slot[(kb + 2) % 3],
                                                      tqb, tpb);
        commit(Ra, oka, tqa, tpa);
        commit(Rb, okb, tqb, tpb);
       } else {
#if WV_STRIP_PAIR_TERMS
        F2 tqa[PP], tpa[PP], tqb[PP], tpb[PP];  // both faces' terms
        const bool oka = fast(Ra, rota, tqa, tpa, mr);
        const bool okb = fast(Rb, rotb, tqb, tpb, mr);
        if (oka && okb) {
#pragma unroll
          for (int pp = 0; pp < PP; ++pp)
            tacc[pp] = fma2(tqb[pp], tpb[pp], fma2(tqa[pp], tpa[pp], tacc[pp]));
        } else {
          commit(Ra, oka, tqa, tpa);
          commit(Rb, okb, tqb, tpb);
        }
#else
        F2 ta[PP];  // tacc with face a's common terms (taken if face a is common)
        bool oka;
        {
          F2 tq[PP], tp[PP];
          oka = fast(Ra, rota, tq, tp, mr);
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) ta[pp] = fma2(tq[pp], tp[pp], tacc[pp]);
        }
        F2 tq[PP], tp[PP];
        const bool okb = fast(Rb, rotb, tq, tp, mr);
        if (oka && okb) {
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) tacc[pp] = fma2(tq[pp], tp[pp], ta[pp]);
        } else {
          if (oka) {
#pragma unroll
            for (int pp = 0; pp < PP; ++pp) tacc[pp] = ta[pp];
          } else {
            do_rare(Ra, Pol::template strip_slow<PP>(Ra, rx, ry, qz, ctx, tacc));
          }
          commit(Rb, okb, tq, tp);
        }
#endif
       }
      };
      // one restart test per pair: the common case (both faces continue a
      // strip) runs as one basic block up to the commit test
      auto pair = [&](const Rec& Ra, const Rec& Rb, auto rota, auto rotb) {
        if ((__float_as_int(Ra.v1.w) | __float_as_int(Rb.v1.w)) < 0)
          pair_body(Ra, Rb, rota, rotb, Yes{});
        else
          pair_body(Ra, Rb, rota, rotb, No{});
      };
      auto one = [&](const Rec& R, auto rot) {
        F2 tq[PP], tp[PP];
        const bool ok = fast(R, rot, tq, tp, Yes{});
        commit(R, ok, tq, tp);
      };
      // unrolled by 6 so the slot rotation is static
      int f = 0;
#pragma unroll 1
      for (; f + 6 <= cnt; f += 6) {
        pair(tile[f], tile[f + 1], R0{}, R1{});
        pair(tile[f + 2], tile[f + 3], R2{}, R0{});
        pair(tile[f + 4], tile[f + 5], R1{}, R2{});
      }
      const int r = cnt - f;  // 0..5 faces left, rotation 0
      if (r >= 2) pair(tile[f], tile[f + 1], R0{}, R1{});
      else if (r == 1) one(tile[f], R0{});
      if (r >= 4) pair(tile[f + 2], tile[f + 3], R2{}, R0{});
      else if (r == 3) one(tile[f + 2], R2{});
      if (r == 5) one(tile[f + 4], R1{});
    } else if constexpr (Pol::kPairFaces) {
      // two faces per angle evaluation (Pol::pair_fast); a pair that is not
      // common everywhere goes face by face
      // (groups of 2 point pairs: a group whose pair is not common
      // everywhere goes face by face, the others keep the pair's terms)
      constexpr int G = Pol::kPairGroup;
      static_assert(PP % G == 0, "point pairs split into whole decision groups");
      auto do_pair = [&](const Rec& Ra, const Rec& Rb) {
        uint32_t rare_a = 0, rare_b = 0;
        if constexpr (kRows) {
          const typename Pol::Row wa = row_f(Ra), wb = row_f(Rb);
#pragma unroll
          for (int g0 = 0; g0 < PP; g0 += G) {
            if (!Pol::template face_row_pair<G>(Ra, wa, Rb, wb, qz + g0, ctx, tacc + g0)) {
              rare_a |= Pol::template face_row<G>(Ra, wa, qz + g0, ctx, tacc + g0) << (2 * g0);
              rare_b |= Pol::template face_row<G>(Rb, wb, qz + g0, ctx, tacc + g0) << (2 * g0);
            }
          }
        } else {
#pragma unroll
          for (int g0 = 0; g0 < PP; g0 += G) {
            if (!Pol::template face_pair<G>(Ra, Rb, qx + g0, qy + g0, qz + g0, ctx, tacc + g0)) {
              rare_a |= Pol::template face<G>(Ra, qx + g0, qy + g0, qz + g0, ctx, tacc + g0)
                        << (2 * g0);
              rare_b |= Pol::template face<G>(Rb, qx + g0, qy + g0, qz + g0, ctx, tacc + g0)
                        << (2 * g0);
            }
          }
        }
        do_rare(Ra, rare_a);
        do_rare(Rb, rare_b);
      };
      if constexpr (kTabF) {
        static_assert(kHalf % 2 == 0, "pairs never straddle the halves");
#pragma unroll 1
        for (int h0 = 0; h0 < cnt; h0 += kHalf) {
          fill_half(h0);
          const int he = cnt < h0 + kHalf ? cnt : h0 + kHalf;
          int f = h0;
#pragma unroll 1
          for (; f + 2 <= he; f += 2) do_pair(tile[f], tile[f + 1]);
          if (f < he) do_face(tile[f], R0{});
        }
      } else {
        int f = 0;
#pragma unroll 1
        for (; f + 2 <= cnt; f += 2) do_pair(tile[f], tile[f + 1]);
        if (f < cnt) do_face(tile[f], R0{});
      }
    } else {
#pragma unroll 1
      for (int f = 0; f < cnt; ++f) do_face(tile[f], R0{});
    }
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      float lo, hi;
      split(tacc[pp], lo, hi);
      accs[2 * pp][tid] += (double)lo;
      accs[2 * pp + 1][tid] += (double)hi;
    }
    __syncwarp();
    if ((tid & 31) == 0) ring_release(ring, s, CW, recs, n_faces, t, t_end);
  }

#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t l = kRows ? grp * P + p : base + p * NC + tid;
    if (kRows ? grp < n_groups : l < n_count)
      o.store(blockIdx.y, zoff + l, accs[p][tid], (hits >> p) & 1u);
  }
}

template <class Pol>
struct FwdPlan {
  int64_t blocks_x = 0;
  int splits = 1;
  int64_t tiles_per_split = 0;
  // rows: the launch takes the lattice-row kernel, whose occupancy
  // (kMinBlocksRow CTAs per SM) sets the wave size the split count fills
  static FwdPlan make(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch = 1,
                      bool rows = false) {
    FwdPlan pl;
    const int64_t per_block = (int64_t)Pol::kConsumerWarps * 32 * Pol::kP;
    pl.blocks_x = (n_count + per_block - 1) / per_block;
    const int64_t n_tiles = (n_faces + Pol::kTile - 1) / Pol::kTile;
    const int s = choose_splits(pl.blocks_x * batch, n_tiles, num_sms,
                                rows ? Pol::kMinBlocksRow : Pol::kMinBlocks);
    pl.tiles_per_split = n_tiles > 0 ? (n_tiles + s - 1) / s : 0;
    pl.splits = pl.tiles_per_split > 0 ? (int)((n_tiles + pl.tiles_per_split - 1) / pl.tiles_per_split) : 1;
    return pl;
  }
  size_t workspace(int64_t n_count) const {
    return splits > 1 ? (size_t)splits * (size_t)n_count * (sizeof(double) + 1) + 256 : 0;
  }
  // what a launch needs whichever kernel (row or generic) it takes
  static size_t workspace_bytes(int64_t n_faces, int64_t n_count, int num_sms, int64_t batch) {
    const size_t a = make(n_faces, n_count, num_sms, batch, false).workspace(n_count * batch);
    const size_t b = make(n_faces, n_count, num_sms, batch, true).workspace(n_count * batch);
    return a > b ? a : b;
  }
};

__global__ void finalize_theta_kernel(const double* __restrict__ part,
                                      const uint8_t* __restrict__ pflags, int splits,
                                      int64_t n_count, int policy, float* __restrict__ out_f32,
                                      uint8_t* __restrict__ flags, double scale);

template <class Pol>
int launch_fwd_f32(const void* packed, int64_t n_faces, const PointSource& ps, int64_t n_count,
                   int policy, float* out, uint8_t* flags, void* workspace, size_t ws_bytes,
                   int num_sms, cudaStream_t stream, const Batch& bt) {
  if (n_count <= 0 || bt.n <= 0) return kOk;
  if (bt.n > 65535 || (bt.n > 1 && ps.kind != PointSource::kGrid)) return kErrArg;
  const PackHeader* hdr = static_cast<const PackHeader*>(packed);
  const typename Pol::Rec* recs = reinterpret_cast<const typename Pol::Rec*>(hdr + 1);
  const bool rows = ps.kind == PointSource::kGrid && row_aligned(ps.grid, ps.n0, n_count, Pol::kP);
  const FwdPlan<Pol> pl = FwdPlan<Pol>::make(n_faces, n_count, num_sms, bt.n, rows);
  OutF32 o;
  o.out = out;
  o.flags = flags;
  o.policy = policy;
  o.scale = Pol::kScale;
  const int64_t total = n_count * bt.n;  // outputs of all meshes, mesh-major
  if (pl.splits > 1) {
    if (workspace == nullptr || ws_bytes < pl.workspace(total)) return kErrWorkspace;
    o.part = static_cast<double*>(workspace);
    o.part_flags = reinterpret_cast<uint8_t*>(o.part + (size_t)pl.splits * total);
    o.n_count = total;
  }
  dim3 grid((unsigned)pl.blocks_x, (unsigned)pl.splits, (unsigned)bt.n);
  const unsigned threads = Pol::kThreads;
  // every warp's 32 P nodes in one k-row: row length, start and count are
  // multiples of them
  constexpr int64_t kWarpNodes = 32 * Pol::kP;
  const bool warp_rows = rows && ps.grid.res[2] % kWarpNodes == 0 &&
                         ps.n0 % kWarpNodes == 0 && n_count % kWarpNodes == 0;
  constexpr bool kWarpRowPol = Pol::kStrip || (Pol::kPairFaces && std::is_same_v<typename Pol::Rec, ExactRecF32>);
  if (rows && warp_rows && kWarpRowPol) {
    if constexpr (kWarpRowPol) {
      RowSrcW src{{{ps.grid, ps.n0}}};
      fwd_f32_kernel<Pol, RowSrcW><<<grid, threads, 0, stream>>>(
          hdr, recs, bt.pack_stride, n_faces, src, n_count, pl.tiles_per_split, o);
      wv::note_launch();
    }
  } else if (rows) {
    RowSrc src{{ps.grid, ps.n0}};
    { fwd_f32_kernel<Pol, RowSrc><<<grid, threads, 0, stream>>>(
        hdr, recs, bt.pack_stride, n_faces, src, n_count, pl.tiles_per_split, o); wv::note_launch(); }
  } else if (ps.kind == PointSource::kGrid) {
    GridSrc src{ps.grid, ps.n0};
    { fwd_f32_kernel<Pol, GridSrc><<<grid, threads, 0, stream>>>(
        hdr, recs, bt.pack_stride, n_faces, src, n_count, pl.tiles_per_split, o); wv::note_launch(); }
  } else {
    ListSrc src{ps.points};
    { fwd_f32_kernel<Pol, ListSrc><<<grid, threads, 0, stream>>>(
        hdr, recs, bt.pack_stride, n_faces, src, n_count, pl.tiles_per_split, o); wv::note_launch(); }
  }
  if (pl.splits > 1) {
    const int t = 256;
    int blocks = (int)((total + t - 1) / t);
    if (blocks > num_sms * 8) blocks = num_sms * 8;
    { finalize_theta_kernel<<<blocks, t, 0, stream>>>(o.part, o.part_flags, pl.splits, total,
                                                    policy, out, flags, o.scale); wv::note_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrLaunch;
}

}  // namespace wv
