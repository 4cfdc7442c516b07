/*
 * windvox_b200.h -- C ABI of the B200 winding-number hot path.
 *
 * One shared library (paper_2407_11272_b200/_lib/libwindvox_b200.so, built for
 * sm_100a) exports the functions below.  Conventions, mirroring the
 * reference kernel ABI (/root/reference/pkg/src/windvox/_kernels.py:1-19,
 * _parallel.py:1-10):
 *   * plain pointers and sizes only; every buffer is caller-owned DEVICE
 *     memory (the caller pre-allocates outputs, exactly as the reference
 *     callers pre-allocate `out`/`flags`/`grad`, winding.py:288-289,
 *     grad.py:64,115);
 *   * kernels never raise: they return a status code (WV_OK == 0) and report
 *     on-surface query points through `flags`, like the reference kernels;
 *   * stream-ordered: `stream` is a cudaStream_t (NULL = legacy default);
 *     nothing synchronizes the host;
 *   * stateless and re-entrant, so one process per GPU or one host thread
 *     per device both work (_parallel.py:39-53);
 *   * a node range [n0, n0+count) of a lattice, or an explicit point list,
 *     plays the role of the reference's per-chunk slice `points[s:e]`.
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef WINDVOX_B200_H
#define WINDVOX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define WV_OK 0
#define WV_ERR_ARG 1       /* invalid argument (null pointer, bad kind, ...) */
#define WV_ERR_WORKSPACE 2 /* workspace missing or smaller than required    */
#define WV_ERR_LAUNCH 3    /* kernel launch failed                           */
#define WV_ERR_CUDA 4      /* CUDA runtime error                             */

/* packed face-array kinds (wv_pack_faces) */
#define WV_PACK_EXACT_F32 1
#define WV_PACK_SOFT_F32 2
#define WV_PACK_EXACT_F64 3
#define WV_PACK_SOFT_F64 4
#define WV_PACK_SOFTGRAD_F32 5
#define WV_PACK_SOFTGRAD_F64 6
#define WV_PACK_EXACTGRAD_F32 7 /* wv_pack_exact_grad: active faces of the exact backward */
#define WV_PACK_EXACTGRAD_F64 8
#define WV_PACK_EXACTSTRIP_F32 9 /* wv_pack_exact_strip: exact f32 records in strip order */
#define WV_PACK_EXACTSTRIP_F64 10 /* wv_pack_exact_strip_f64: f64 parity records in strip order */
#define WV_PACK_EXACTTRAIL_F32 11 /* wv_pack_exact_trail: edge-trail windows of the exact backward */
#define WV_PACK_EXACTTRAIL_F64 12 /* wv_pack_exact_trail_f64: their f64 twin */

/* stored value for on-surface (flagged) nodes */
#define WV_POLICY_RAW 0  /* keep the partial sum: winding_number_batch, winding.py:271-309 */
#define WV_POLICY_HALF 1 /* exactly 0.5: voxelize, winding.py:358                          */

/* GridSpec (winding.py:69-140): node (i,j,k) at lo + (hi-lo)*(i/(R-1)),
 * midpoint when R == 1; flat index ((i*Ry)+j)*Rz+k (k fastest). */
typedef struct wv_grid {
  double lo[3];
  double hi[3];
  int64_t res[3];
} wv_grid_t;

const char *wv_version(void);
const char *wv_status_string(int status);
/* CUDA device ordinal the calls on this thread use (cudaSetDevice). */
int wv_set_device(int device);

/* ---- per-mesh staging -------------------------------------------------
 * Replaces surface_epsilon (winding.py:193-197), _prepare_exact
 * (winding.py:258-268) and TriangleMesh.triangle_corners (mesh_io.py:90-92).
 * vertices: (V,3) f32 (vert_f64=0) or f64 (vert_f64=1); faces: (F,3) int32
 * (faces_i64=0) or int64.  `packed` must hold wv_packed_bytes(kind, F).
 * Exact kinds keep degenerate faces in place, marked dead (the reference
 * drops them; results are identical). */
/* Kernels launched by this library since load (all entry points, all
 * threads): bench.py's count of its own launches in a timed region. */
long long wv_launch_count(void);

size_t wv_packed_bytes(int kind, int64_t n_faces);
int wv_pack_faces(int kind, const void *vertices, int vert_f64, int64_t n_verts,
                  const void *faces, int faces_i64, int64_t n_faces, void *packed,
                  void *stream);
/* Staging for the exact backward (kinds 7/8): only the `active` faces
 * (A,) int64 -- those with a non-cancelling directed edge -- with the net
 * weights (A,3) f32 of their edges v0->v1, v1->v2, v2->v0.  Interior edges of
 * a consistently oriented mesh cancel exactly in d(Omega)/dv, so a closed
 * manifold packs no face (its exact gradient vanishes, test_grad.py:231-246).
 * Degenerate faces (dropped by the reference forward) must be excluded from
 * the edge count by the caller.  `packed` holds wv_packed_bytes(kind, A). */
int wv_pack_exact_grad(int kind, const void *vertices, int vert_f64, int64_t n_verts,
                       const void *faces, int faces_i64, const int64_t *active,
                       const float *weights, int64_t n_active, void *packed, void *stream);

/* Area-weighted vertex normals (mesh_io.vertex_normals, mesh_io.py:176-195),
 * the staging of flipped duplication for open meshes (openmesh.py:21-48).
 * vertices (V,3) f64, faces (F,3) int64; the CSR lists, per vertex, the slots
 * k*F + f of its face corners in ascending order (np.add.at's order, so the
 * result is bit-identical).  normals (V,3) f64; zero (V,) u8 may be NULL. */
int wv_vertex_normals(const double *vertices, int64_t n_verts, const int64_t *faces,
                      int64_t n_faces, const int64_t *csr_offsets, const int64_t *csr_slots,
                      double *normals, uint8_t *zero, void *stream);

/* ---- forward: winding numbers at lattice nodes or explicit points -------
 * exact f32: replaces _kernels.exact_batch_f32 (_kernels.py:235-309); FP32
 *   compute with fp64 tile-partial accumulation, within 1e-5 of the f64
 *   reference.  packed kind WV_PACK_EXACT_F32.
 * soft f32: replaces _kernels.soft_batch_f32 (_kernels.py:312-349).
 *   packed kind WV_PACK_SOFT_F32.
 * exact f64 / soft f64: replace _kernels.exact_batch / soft_batch
 *   (_kernels.py:34-116, 119-158) in the reference's operation order; kinds
 *   WV_PACK_EXACT_F64 / WV_PACK_SOFT_F64.  use_atan2=0 selects the
 *   single-argument arctan regression branch (_kernels.py:106-114).
 * Writes out[0..count) and flags[0..count) (1 = on-surface, may be NULL).
 * `workspace` may be NULL when wv_fwd_workspace_bytes(...) returns 0. */
size_t wv_fwd_workspace_bytes(int kind, int64_t n_faces, int64_t count);
int wv_exact_fwd_grid_f32(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, int policy, float *out, uint8_t *flags,
                          void *workspace, size_t workspace_bytes, void *stream);
int wv_exact_fwd_points_f32(const void *packed, int64_t n_faces, const float *points,
                            int64_t count, int policy, float *out, uint8_t *flags,
                            void *workspace, size_t workspace_bytes, void *stream);
int wv_soft_fwd_grid_f32(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, int policy, float *out, uint8_t *flags, void *workspace,
                         size_t workspace_bytes, void *stream);
int wv_soft_fwd_points_f32(const void *packed, int64_t n_faces, const float *points,
                           int64_t count, int policy, float *out, uint8_t *flags,
                           void *workspace, size_t workspace_bytes, void *stream);
int wv_exact_fwd_grid_f64(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, int use_atan2, int policy, double *out, uint8_t *flags,
                          void *stream);
int wv_exact_fwd_points_f64(const void *packed, int64_t n_faces, const double *points,
                            int64_t count, int use_atan2, int policy, double *out,
                            uint8_t *flags, void *stream);
int wv_soft_fwd_grid_f64(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, int policy, double *out, uint8_t *flags, void *stream);
int wv_soft_fwd_points_f64(const void *packed, int64_t n_faces, const double *points,
                           int64_t count, int policy, double *out, uint8_t *flags,
                           void *stream);

/* ---- strip-ordered exact f32 forward (same values as wv_exact_fwd_*_f32
 * up to fp32 summation order; fewer square roots on lattice rows) --------
 * wv_strip_order (HOST memory, CPU): welds vertices by bitwise-equal
 *   position and walks the faces as strips: perm[k] = face at strip position
 *   k, window[3k..3k+2] = its vertex indices in window order, flags[k] bit0
 *   = strip start, bit1 = window reflects the face's orientation.
 * wv_pack_exact_strip (device arrays): packs those records (kind
 *   WV_PACK_EXACTSTRIP_F32, wv_packed_bytes sizes it); n_faces < 2^31.
 * Outputs are per query point (face order does not matter to W). */
int wv_strip_order(const double *vertices, int64_t n_verts, const int64_t *faces,
                   int64_t n_faces, int64_t *perm, int64_t *window, uint8_t *flags);
int wv_pack_exact_strip(const void *vertices, int vert_f64, int64_t n_verts, const void *faces,
                        int faces_i64, int64_t n_faces, const int64_t *perm,
                        const int64_t *window, const uint8_t *flags, void *packed,
                        void *stream);
int wv_exact_strip_fwd_grid_f32(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                                int64_t count, int policy, float *out, uint8_t *flags,
                                void *workspace, size_t workspace_bytes, void *stream);
int wv_exact_strip_fwd_points_f32(const void *packed, int64_t n_faces, const float *points,
                                  int64_t count, int policy, float *out, uint8_t *flags,
                                  void *workspace, size_t workspace_bytes, void *stream);
/* f64 parity twin (replaces _kernels.exact_batch on large lattices): each
 * face term is the reference's bit for bit, the shared corners' |v - q| are
 * carried along the strip (one DP square root per pair instead of three),
 * and only the order of the face sum differs from wv_exact_fwd_*_f64. */
int wv_pack_exact_strip_f64(const void *vertices, int vert_f64, int64_t n_verts,
                            const void *faces, int faces_i64, int64_t n_faces,
                            const int64_t *perm, const int64_t *window, const uint8_t *flags,
                            void *packed, void *stream);
int wv_exact_strip_fwd_grid_f64(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                                int64_t count, int use_atan2, int policy, double *out,
                                uint8_t *flags, void *stream);
int wv_exact_strip_fwd_points_f64(const void *packed, int64_t n_faces, const double *points,
                                  int64_t count, int use_atan2, int policy, double *out,
                                  uint8_t *flags, void *stream);

/* ---- backward: per-face corner gradients reduced over query points ------
 * face_grad (F,3,3) f64 is OVERWRITTEN with
 *   sum_p coef_scale * coefs[p] * dW(q_p)/dv_{f,k}
 * over the node range / point list; points with coefs[p] == 0 are skipped
 * and pairs the forward skipped (on-surface) contribute nothing.
 * soft: replaces _kernels.soft_grad_accum (_kernels.py:161-232); packed kind
 *   WV_PACK_SOFTGRAD_F32 / _F64.
 * exact: NEW (no reference kernel, grad.py:9-12): d(Omega)/dv of the VOS
 *   solid angle in its per-edge (Biot-Savart) form; packed kind
 *   WV_PACK_EXACTGRAD_F32 / _F64 and n_faces = number of ACTIVE faces.
 *   Callers pass coefs == 0 at on-surface (flagged) points, where W is
 *   discontinuous and has no derivative.
 * Corner sums become vertex gradients with wv_face_to_vertex. */
size_t wv_bwd_workspace_bytes(int kind, int64_t n_faces, int64_t count);
int wv_exact_bwd_grid_f32(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, const float *coefs, double coef_scale,
                          double *face_grad, void *workspace, size_t workspace_bytes,
                          void *stream);
int wv_exact_bwd_points_f32(const void *packed, int64_t n_faces, const float *points,
                            int64_t count, const float *coefs, double coef_scale,
                            double *face_grad, void *workspace, size_t workspace_bytes,
                            void *stream);
/* exact f32 over STRIP PAIRS (same gradients, fewer operations on lattice
 * rows): the packed array is wv_pack_exact_grad's (kind
 * WV_PACK_EXACTGRAD_F32) over 2P faces given in pair order -- faces 2i and
 * 2i+1 with corners in strip-window order (A, B, C), (B', C', D), B' and C'
 * at B's and C's positions (a pair whose positions differ is evaluated as two
 * separate faces), edge weights in window order (negated for a window that
 * reflects the face).  face_grad rows follow that order.  n_faces even. */
size_t wv_exact_pair_bwd_workspace_bytes(int64_t n_faces, int64_t count);
int wv_exact_pair_bwd_grid_f32(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                               int64_t count, const float *coefs, double coef_scale,
                               double *face_grad, void *workspace, size_t workspace_bytes,
                               void *stream);
int wv_exact_pair_bwd_points_f32(const void *packed, int64_t n_faces, const float *points,
                                 int64_t count, const float *coefs, double coef_scale,
                                 double *face_grad, void *workspace, size_t workspace_bytes,
                                 void *stream);
/* exact f32 over EDGE TRAILS (same gradients, one evaluation per distinct
 * edge; lattice rows only):
 * wv_edge_trails (HOST memory, CPU): welds vertices by bitwise-equal
 *   position, nets each vertex id's signed edge terms over its live faces
 *   (dead: NULL or n_faces flags of faces the reference drops, winding.py:
 *   262-264), drops edges whose net weights all vanish, and covers the rest
 *   with trails (Hierholzer) cut into windows of K = wv_trail_edges()
 *   consecutive edges: windows (capacity 3 n_faces (K+1) int64) = K+1 vertex
 *   ids per window (one per position p0..pK), csr_off (n_verts + 1),
 *   csr_slots (capacity 6 n_faces) = signed output slots per vertex id
 *   (2K w + 2 e + end, or -slot-1 to subtract).  Sizes written to *n_windows, *n_slots.  vrep (NULL or
 *   n_verts): the representative vertex id of each vertex's position.
 * wv_pack_exact_trail: the window records (wv_packed_bytes(
 *   WV_PACK_EXACTTRAIL_F32, n_windows) bytes).
 * wv_exact_trail_bwd_grid_f32: out (n_windows, 2K, 3) doubles = the two end
 *   vectors of each window edge; row-aligned lattice ranges only (res_z >= 16
 *   and even, n0 even), else WV_ERR_ARG.  wv_face_to_vertex with the trail
 *   CSR turns them into vertex gradients (replaces the reference's FD-only
 *   exact gradient, grad.py:9-12; equal to wv_exact_bwd_* + gather). */
int wv_trail_edges(void); /* K, the edges per trail window of this build */
int wv_edge_trails(const double *vertices, int64_t n_verts, const int64_t *faces,
                   int64_t n_faces, const uint8_t *dead, int64_t *windows, int64_t *n_windows,
                   int64_t *csr_off, int64_t *csr_slots, int64_t *n_slots, int64_t *vrep);
int wv_pack_exact_trail(const void *vertices, int vert_f64, int64_t n_verts,
                        const int64_t *windows, int64_t n_windows, void *packed, void *stream);
size_t wv_exact_trail_bwd_workspace_bytes(int64_t n_windows, int64_t count);
int wv_exact_trail_bwd_grid_f32(const void *packed, int64_t n_windows, wv_grid_t grid,
                                int64_t n0, int64_t count, const float *coefs,
                                double coef_scale, double *out, void *workspace,
                                size_t workspace_bytes, void *stream);
/* f64 twin (the parity path's exact backward over the same trails, any
 * lattice range or point list): records of kind WV_PACK_EXACTTRAIL_F64 (the
 * f64 mesh), same output layout and CSR. */
int wv_pack_exact_trail_f64(const void *vertices, int vert_f64, int64_t n_verts,
                            const int64_t *windows, int64_t n_windows, void *packed,
                            void *stream);
size_t wv_exact_trail_bwd_workspace_bytes_f64(int64_t n_windows, int64_t count);
int wv_exact_trail_bwd_grid_f64(const void *packed, int64_t n_windows, wv_grid_t grid,
                                int64_t n0, int64_t count, const double *coefs,
                                double coef_scale, double *out, void *workspace,
                                size_t workspace_bytes, void *stream);
int wv_exact_trail_bwd_points_f64(const void *packed, int64_t n_windows, const double *points,
                                  int64_t count, const double *coefs, double coef_scale,
                                  double *out, void *workspace, size_t workspace_bytes,
                                  void *stream);
int wv_soft_bwd_grid_f32(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, const float *coefs, double coef_scale,
                         double *face_grad, void *workspace, size_t workspace_bytes,
                         void *stream);
int wv_soft_bwd_points_f32(const void *packed, int64_t n_faces, const float *points,
                           int64_t count, const float *coefs, double coef_scale,
                           double *face_grad, void *workspace, size_t workspace_bytes,
                           void *stream);
int wv_exact_bwd_grid_f64(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                          int64_t count, const double *coefs, double coef_scale,
                          double *face_grad, void *workspace, size_t workspace_bytes,
                          void *stream);
int wv_exact_bwd_points_f64(const void *packed, int64_t n_faces, const double *points,
                            int64_t count, const double *coefs, double coef_scale,
                            double *face_grad, void *workspace, size_t workspace_bytes,
                            void *stream);
int wv_soft_bwd_grid_f64(const void *packed, int64_t n_faces, wv_grid_t grid, int64_t n0,
                         int64_t count, const double *coefs, double coef_scale,
                         double *face_grad, void *workspace, size_t workspace_bytes,
                         void *stream);
int wv_soft_bwd_points_f64(const void *packed, int64_t n_faces, const double *points,
                           int64_t count, const double *coefs, double coef_scale,
                           double *face_grad, void *workspace, size_t workspace_bytes,
                           void *stream);

/* Vertex gradients from face-corner sums, in CSR order (deterministic):
 *   out[v] (+)= scale * sum_{e in [off[v], off[v+1])} face_grad[slots[e]]
 * slots[e] = 3*f + k for every corner k of face f incident to v, sorted by v
 * (stable); a negative entry -s-1 SUBTRACTS slot s (edge-trail CSRs).  `scale` is a DEVICE pointer (NULL = 1).  out64 / out32 may each
 * be NULL.  Replaces the chunk-ordered buffer merge of grad.py:113-127. */
int wv_face_to_vertex(const double *face_grad, const int64_t *csr_offsets,
                      const int64_t *csr_slots, int64_t n_verts, const double *scale,
                      int accumulate, double *out64, float *out32, void *stream);

/* ---- batched grid kernels (many meshes, one connectivity, one grid) ------
 * The C4 training batch / batched morph trials: `batch` meshes sharing the
 * face count and query range, evaluated by ONE launch per stage (blockIdx.z
 * = mesh).  Mesh z's packed buffer (wv_pack_faces / wv_pack_exact_grad)
 * starts at packed + z * pack_stride bytes (pack_stride a multiple of 16, at
 * least the packed size); its values / flags / coefficients sit at
 * z * count, its corner sums at z * n_faces * 9.  kind: WV_PACK_EXACT_F32 or
 * WV_PACK_SOFT_F32 (forward), WV_PACK_EXACTGRAD_F32 or WV_PACK_SOFTGRAD_F32
 * (backward).  Results equal `batch` single-mesh calls. */
size_t wv_fwd_workspace_bytes_batch(int kind, int64_t n_faces, int64_t count, int64_t batch);
int wv_fwd_grid_f32_batch(int kind, const void *packed, size_t pack_stride, int64_t n_faces,
                          wv_grid_t grid, int64_t n0, int64_t count, int64_t batch, int policy,
                          float *out, uint8_t *flags, void *workspace, size_t workspace_bytes,
                          void *stream);
size_t wv_bwd_workspace_bytes_batch(int kind, int64_t n_faces, int64_t count, int64_t batch);
int wv_bwd_grid_f32_batch(int kind, const void *packed, size_t pack_stride, int64_t n_faces,
                          wv_grid_t grid, int64_t n0, int64_t count, int64_t batch,
                          const float *coefs, double coef_scale, double *face_grad,
                          void *workspace, size_t workspace_bytes, void *stream);
/* The per-mesh stages around them, batched the same way (two, two and one
 * launches for the whole batch instead of per mesh):
 *   wv_pack_faces_batch: vertices (batch, n_verts, 3) contiguous, one face
 *     array; kinds 1-6; buffers pack_stride bytes apart (multiple of 16).
 *   wv_loss_terms_f32_batch: values / flags / targets / coefs (batch, count),
 *     weights NULL or (batch, count), sums (batch, 8); workspace
 *     batch * wv_loss_workspace_bytes(count).
 *   wv_face_to_vertex_batch: face_grad (batch, n_faces, 3, 3), one CSR,
 *     scale NULL or scale[b * scale_stride], outputs (batch, n_verts, 3).
 * Each mesh's results equal the single-mesh calls. */
int wv_pack_faces_batch(int kind, const void *vertices, int vert_f64, int64_t n_verts,
                        const void *faces, int faces_i64, int64_t n_faces, int64_t batch,
                        void *packed, size_t pack_stride, void *stream);
int wv_loss_terms_f32_batch(const float *values, const uint8_t *flags, const float *targets,
                            const float *weights, int64_t count, int64_t batch, float *coefs,
                            double *sums, void *workspace, size_t workspace_bytes,
                            void *stream);
int wv_face_to_vertex_batch(const double *face_grad, int64_t n_faces,
                            const int64_t *csr_offsets, const int64_t *csr_slots,
                            int64_t n_verts, int64_t batch, const double *scale,
                            int64_t scale_stride, int accumulate, double *out64, float *out32,
                            void *stream);

/* ---- marching cubes on the device-resident grid (recon.py:39-108) --------
 * Four stream-ordered passes; the caller computes exclusive prefix sums
 * between them (counts -> tri_offsets, flags -> vertex_index).
 *   wv_mc_classify: per cell (Rx-1)(Ry-1)(Rz-1): case (bit c = corner c
 *     outside, value <= iso; corner c at (c&1, c>>1&1, c>>2&1)) and its
 *     triangle count tri_count[case];
 *   wv_mc_edges: per lattice edge g = axis*N + node (N = Rx*Ry*Rz), 1 if it
 *     crosses iso (the reference's global edge id, recon.py:90-93);
 *   wv_mc_vertices: vertex vertex_index[g] = pa + t (pb - pa),
 *     t = (iso - va)/(vb - va), f64 -- bit-identical to the reference;
 *   wv_mc_emit: triangles of each cell at tri_offsets[cell] from the case
 *     table (max_tris triples per case, -1 terminated) and the per-edge
 *     axis / base-corner tables of the table's edge numbering.
 * values: the field, f32 (values_f64=0) or f64. */
int wv_mc_classify(const void *values, int values_f64, wv_grid_t grid, double iso,
                   const int8_t *tri_count, uint8_t *cases, int32_t *counts, void *stream);
int wv_mc_edges(const void *values, int values_f64, wv_grid_t grid, double iso, int32_t *flags,
                void *stream);
int wv_mc_vertices(const void *values, int values_f64, wv_grid_t grid, double iso,
                   const int32_t *flags, const int64_t *vertex_index, double *vertices,
                   void *stream);
int wv_mc_emit(const uint8_t *cases, const int64_t *tri_offsets, const int8_t *tri_table,
               int max_tris, const int8_t *edge_axis, const int8_t *edge_base,
               const int64_t *vertex_index, wv_grid_t grid, int64_t *faces, void *stream);
/* Slab-sharded marching cubes (one i-slab per GPU): a rank
 * runs wv_mc_classify / wv_mc_edges / wv_mc_emit on its block of `rows`
 * i-rows (its slab plus a 1-row halo from the next rank; `grid` with
 * res[0] = rows), vertex_index holding GLOBAL vertex ids, and
 * wv_mc_vertices_slab places the vertices of the block's crossed edges at
 * slot[g] (local output rows; slot < 0: skipped, e.g. the halo row's edges,
 * which the next rank owns), computing positions with the GLOBAL grid
 * `grid` (i = i0 + local row).  distributed.slab_marching_cubes does the
 * halo exchange and the id offsets; the result equals the one-GPU mesh. */
int wv_mc_vertices_slab(const void *values, int values_f64, wv_grid_t grid, int64_t i0,
                        int64_t rows, double iso, const int32_t *flags, const int64_t *slot,
                        double *vertices, void *stream);

/* ---- occupancy loss terms (grad.py:101-110), fused on the device ---------
 * coefs[n] = 2 w r (0 on flagged nodes); sums (8 doubles, device) =
 * {sum w r^2, sum w, n_flagged, 1/sum w, loss, 0, 0, 0}.  weights may be NULL
 * (all ones).  wv_loss_finalize recomputes sums[3..4] after sums[0..2] were
 * all-reduced across ranks. */
size_t wv_loss_workspace_bytes(int64_t count);
int wv_loss_terms_f32(const float *values, const uint8_t *flags, const float *targets,
                      const float *weights, int64_t count, float *coefs, double *sums,
                      void *workspace, size_t workspace_bytes, void *stream);
int wv_loss_terms_f64(const double *values, const uint8_t *flags, const double *targets,
                      const double *weights, int64_t count, double *coefs, double *sums,
                      void *workspace, size_t workspace_bytes, void *stream);
int wv_loss_finalize(double *sums, void *stream);

/* ---- reconstruction metrics (metrics.py:43-150), bit-identical ------------
 * wv_splitmix64_uniform: out[i] = (SplitMix64(seed + (i+1)*golden) >> 11)
 *   * 2^-53, i < count (replaces splitmix64_uniform, metrics.py:43-51).
 * wv_surface_cdf: per face area 0.5*|(v1-v0)x(v2-v0)| (numpy's expression
 *   order), cdf = np.cumsum(areas), *total = np.sum(areas) (numpy pairwise
 *   order); total stays on the device.  faces int64 (F,3), vertices f64.
 * wv_sample_surface: n points by area (metrics.py:58-93): face =
 *   searchsorted(cdf, r[3i]*total, 'right') clamped, folded barycentrics
 *   r[3i+1], r[3i+2]; out (n,3) f64.
 * wv_nearest_distances: out[i] = min_j |q_i - t_j| (brute force, equal bit
 *   for bit to the reference's k-d tree, metrics.py:96-104).  nt >= 1.
 * wv_pairwise_sum: *out = np.sum(x) (numpy pairwise summation order). */
int wv_splitmix64_uniform(uint64_t seed, int64_t count, double *out, void *stream);
size_t wv_pairwise_sum_workspace_bytes(int64_t n);
int wv_pairwise_sum(const double *x, int64_t n, double *out, void *workspace,
                    size_t workspace_bytes, void *stream);
int wv_surface_cdf(const double *vertices, const int64_t *faces, int64_t n_faces, double *areas,
                   double *cdf, double *total, void *workspace, size_t workspace_bytes,
                   void *stream);
int wv_sample_surface(const double *vertices, const int64_t *faces, int64_t n_faces,
                      const double *cdf, const double *total, uint64_t seed, int64_t n,
                      double *out, void *stream);
int wv_nearest_distances(const double *queries, int64_t n_queries, const double *targets,
                         int64_t n_targets, double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* WINDVOX_B200_H */
