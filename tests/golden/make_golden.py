"""Generate the golden fixtures that pin the oracle to the reference.

Run in the build container (needs the read-only reference checkout):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports the reference package ``windvox`` itself and records, for a set of
small seeded cases modelled on the reference's own tests
(pkg/tests/test_winding.py, test_grad.py, test_openmesh.py,
test_acceptance.py), the inputs (mesh arrays, points / grid) and the
reference outputs.  The fixtures are committed; nothing on the GPU box reads
/root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

import windvox as wv
from windvox import _kernels, shapes
from windvox.winding import _prepare_exact, surface_epsilon

OUT = Path(__file__).resolve().parent


def unit_grid(res, lo=-1.0, hi=1.0):
    return wv.GridSpec((lo,) * 3, (hi,) * 3, res)


def grid_dict(prefix, spec):
    return {f"{prefix}_lo": spec.bounds_min, f"{prefix}_hi": spec.bounds_max,
            f"{prefix}_res": np.array(spec.resolution)}


def random_generic_mesh(rng, max_vertices=50):
    # test_grad.py:16-27
    nv = int(rng.integers(6, max_vertices + 1))
    verts = rng.normal(size=(nv, 3))
    nf = int(rng.integers(4, 12))
    seen, faces = set(), []
    while len(faces) < nf:
        f = rng.choice(nv, size=3, replace=False)
        key = frozenset(f.tolist())
        if key not in seen:
            seen.add(key)
            faces.append(f.tolist())
    return wv.TriangleMesh(verts, faces)


def off_centroid_point(mesh, rng, min_dist=0.5):
    centroids = mesh.vertices[mesh.faces].mean(axis=1)
    while True:
        q = rng.normal(size=3) * 2
        if np.linalg.norm(centroids - q, axis=1).min() >= min_dist:
            return q


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({sum(a.nbytes for a in map(np.asarray, arrays.values()))} B raw)")


def main():
    # 1. census: cube(0.5) on [-1,1]^3 at R=9 (test_winding.py:276-288)
    mesh = shapes.cube(0.5)
    spec = unit_grid(9)
    field = wv.voxelize(mesh, spec)
    vals, flags = wv.winding_number_batch(mesh, spec.node_coordinates())
    save("census_cube_r9", vertices=mesh.vertices, faces=mesh.faces,
         values=field.values, raw=vals, flags=flags, **grid_dict("grid", spec))

    # 2. point batches, exact + soft + flipped (test_winding.py:114-140)
    rng = np.random.default_rng(101)
    cases = {}
    ico = shapes.icosahedron()
    pts = rng.normal(size=(64, 3)) * 1.5
    tor = shapes.torus(0.7, 0.3, 48, 24)
    tpts = np.concatenate([rng.uniform(-1.2, 1.2, size=(200, 3)),
                           rng.normal(size=(56, 3)) * 0.3 + [0.7, 0.0, 0.0]])
    for tag, m, p in (("ico", ico, pts), ("torus", tor, tpts)):
        ex, fe = wv.winding_number_batch(m, p, mode="exact")
        so, fs = wv.winding_number_batch(m, p, mode="soft")
        ar, fa = wv.winding_number_batch(m, p, mode="exact", use_atan2=False)
        cases.update({f"{tag}_vertices": m.vertices, f"{tag}_faces": m.faces,
                      f"{tag}_points": p, f"{tag}_exact": ex, f"{tag}_exact_flags": fe,
                      f"{tag}_soft": so, f"{tag}_soft_flags": fs,
                      f"{tag}_arctan": ar, f"{tag}_arctan_flags": fa})
    save("point_batches", **cases)

    # 3. voxelize icosphere(2) @13 on [-1.5,1.5] exact+soft, f64 and f32
    #    (test_winding.py:299-322)
    m = shapes.icosphere(2)
    spec = unit_grid(13, -1.5, 1.5)
    d = {"vertices": m.vertices, "faces": m.faces, **grid_dict("grid", spec)}
    for mode in ("exact", "soft"):
        d[f"{mode}_f64"] = wv.voxelize(m, spec, mode=mode).values
        d[f"{mode}_f32"] = wv.voxelize(m, spec, mode=mode, precision="f32").values
    save("voxelize_icosphere2_r13", **d)

    # 4. C1: icosphere(3) normalized, [-1,1]^3 at 32^3, exact f64 + f32 + soft
    m, _ = wv.normalize_to_unit_cube(shapes.icosphere(3, 1.0))
    spec = unit_grid(32)
    vals, flags = wv.winding_number_batch(m, spec.node_coordinates(), mode="exact")
    save("c1_icosphere3_r32", vertices=m.vertices, faces=m.faces, raw=vals, flags=flags,
         exact_f64=wv.voxelize(m, spec).values,
         exact_f32=wv.voxelize(m, spec, precision="f32").values,
         soft_f64=wv.voxelize(m, spec, mode="soft").values, **grid_dict("grid", spec))

    # 5. open hemisphere closed by flipped duplication (test_openmesh.py:44-55)
    hemi = shapes.hemisphere(3)
    shell = wv.flipped_duplication(hemi, epsilon=0.01)
    cen = hemi.vertices[hemi.faces].mean(axis=1)
    high = cen[cen[:, 2] > 0.5]
    probes = np.concatenate([high * (1.0 - 0.005 / np.linalg.norm(high, axis=1)[:, None]),
                             [[0.0, 0.0, 0.0], [60.0, 30.0, 40.0]]])
    w, f = wv.winding_number_batch(shell, probes)
    save("open_hemisphere_shell", hemi_vertices=hemi.vertices, hemi_faces=hemi.faces,
         vertices=shell.vertices, faces=shell.faces, points=probes, values=w, flags=f)

    # 6. soft Jacobians on random generic meshes (test_grad.py:64-72)
    rng = np.random.default_rng(17)
    jac = {}
    for i in range(12):
        m = random_generic_mesh(rng)
        q = off_centroid_point(m, rng)
        jac[f"m{i}_vertices"] = m.vertices
        jac[f"m{i}_faces"] = m.faces
        jac[f"m{i}_q"] = q
        jac[f"m{i}_jac"] = wv.soft_winding_vertex_jacobian(m, q).vectors
    save("soft_jacobians", n=np.array(12), **jac)

    # 7. occupancy loss + gradient (test_grad.py:135-164) and the
    #    excluded-node case (test_grad.py:183-202)
    rng = np.random.default_rng(43)
    verts = rng.normal(size=(20, 3)) * 0.4
    faces, seen = [], set()
    while len(faces) < 12:
        f = rng.choice(20, size=3, replace=False)
        key = frozenset(f.tolist())
        if key not in seen:
            seen.add(key)
            faces.append(f.tolist())
    m = wv.TriangleMesh(verts, faces)
    spec = unit_grid(8)
    target = rng.uniform(0, 1, size=spec.num_nodes)
    weights = rng.uniform(0.5, 2.0, size=spec.num_nodes)
    r = wv.occupancy_loss_grad(m, wv.ScalarField(spec, target))
    rw = wv.occupancy_loss_grad(m, wv.ScalarField(spec, target), weights=weights)
    ev = np.array([[0.0, -0.3, -0.3], [0.0, 0.6, -0.3], [0.0, -0.3, 0.6],
                   [2.0, 0.0, 0.0], [2.0, 1.0, 0.0], [2.0, 0.0, 1.0]])
    ef = np.array([[0, 1, 2], [3, 4, 5]])
    espec = unit_grid(3)
    etarget = np.random.default_rng(47).uniform(0, 1, size=espec.num_nodes)
    er = wv.occupancy_loss_grad(wv.TriangleMesh(ev, ef), wv.ScalarField(espec, etarget))
    save("loss_grad", vertices=verts, faces=np.array(faces), target=target, weights=weights,
         loss=np.array(r.loss), grads=r.grads.vectors, excluded=np.array(r.excluded_nodes),
         wloss=np.array(rw.loss), wgrads=rw.grads.vectors,
         ex_vertices=ev, ex_faces=ef, ex_target=etarget, ex_loss=np.array(er.loss),
         ex_grads=er.grads.vectors, ex_excluded=np.array(er.excluded_nodes),
         **grid_dict("grid", spec), **grid_dict("ex_grid", espec))

    # 8. exact d(W)/dv by central finite differences of the reference
    #    exact_batch itself (the package's FD authority, test_grad.py:3-6)
    rng = np.random.default_rng(5)
    fdd = {}
    for i in range(4):
        m = random_generic_mesh(rng, max_vertices=14)
        pts = rng.normal(size=(9, 3)) * 1.5
        coefs = rng.normal(size=len(pts))
        fd = np.zeros_like(m.vertices)
        h = 1e-6
        for vi in range(m.num_vertices):
            for c in range(3):
                vp = m.vertices.copy()
                vp[vi, c] += h
                vm = m.vertices.copy()
                vm[vi, c] -= h
                wp, _ = wv.winding_number_batch(wv.TriangleMesh(vp, m.faces), pts)
                wm, _ = wv.winding_number_batch(wv.TriangleMesh(vm, m.faces), pts)
                fd[vi, c] = float(((wp - wm) * coefs).sum()) / (2 * h)
        fdd.update({f"m{i}_vertices": m.vertices, f"m{i}_faces": m.faces,
                    f"m{i}_points": pts, f"m{i}_coefs": coefs, f"m{i}_fd": fd})
    save("exact_grad_fd", n=np.array(4), **fdd)

    # 9. raw reference kernel ABI on a random soup (f64 + f32 twins), plus
    #    the soft gradient accumulation kernel
    rng = np.random.default_rng(9)
    tri_v = rng.normal(size=(60, 3))
    tri_f = rng.integers(0, 60, size=(80, 3))
    tri_f[5] = [3, 3, 4]  # one degenerate face (dropped by _prepare_exact)
    m = wv.TriangleMesh(tri_v, tri_f)
    pts = rng.normal(size=(300, 3)) * 1.2
    pts[0] = tri_v[7]  # exactly on a vertex
    tri, nhat, pld = _prepare_exact(m)
    eps = surface_epsilon(m)
    out = np.zeros(len(pts))
    fl = np.zeros(len(pts), dtype=bool)
    _kernels.exact_batch(pts, tri, nhat, pld, eps, True, out, fl)
    out32 = np.zeros(len(pts), dtype=np.float32)
    fl32 = np.zeros(len(pts), dtype=bool)
    _kernels.exact_batch_f32(pts.astype(np.float32), tri.astype(np.float32),
                             nhat.astype(np.float32), pld.astype(np.float32),
                             np.float32(eps), out32, fl32)
    tri_all = np.ascontiguousarray(m.triangle_corners())
    sout = np.zeros(len(pts))
    sfl = np.zeros(len(pts), dtype=bool)
    _kernels.soft_batch(pts, tri_all, eps, sout, sfl)
    sout32 = np.zeros(len(pts), dtype=np.float32)
    sfl32 = np.zeros(len(pts), dtype=bool)
    _kernels.soft_batch_f32(pts.astype(np.float32), tri_all.astype(np.float32),
                            np.float32(eps), sout32, sfl32)
    coefs = rng.normal(size=len(pts))
    coefs[::7] = 0.0
    grad = np.zeros((m.num_vertices, 3))
    _kernels.soft_grad_accum(pts, coefs, tri_all, m.faces, eps, grad)
    save("kernel_abi_soup", vertices=tri_v, faces=tri_f, points=pts, exact=out, exact_flags=fl,
         exact32=out32, exact32_flags=fl32, soft=sout, soft_flags=sfl, soft32=sout32,
         soft32_flags=sfl32, coefs=coefs, soft_grad=grad)

    # 11. morph traces (test_acceptance.py:268-278 and test_morph.py setups)
    from windvox.morph import MorphConfig, morph
    tgt_spec = wv.GridSpec([-0.8] * 3, [0.8] * 3, 12)
    target = wv.voxelize(shapes.cube(0.5), tgt_spec)
    tmpl = shapes.icosphere(1, 0.4)
    res_mesh, rep = morph(tmpl, target, MorphConfig(iterations=10))
    res2, rep2 = morph(tmpl, target, MorphConfig(iterations=6, momentum=0.0, smooth_weight=0.0,
                                                 step_size=0.2))
    save("morph_traces", tmpl_vertices=tmpl.vertices, tmpl_faces=tmpl.faces,
         target=target.values, **grid_dict("grid", tgt_spec),
         final=res_mesh.vertices, losses=np.array([e["loss"] for e in rep.entries]),
         gnorms=np.array([e["grad_inf_norm"] for e in rep.entries]),
         final2=res2.vertices, losses2=np.array([e["loss"] for e in rep2.entries]))

    # 12. flipped duplication and WVOX1 bytes (openmesh.py:21-48, winding.py:403-443)
    import tempfile
    hemi = shapes.hemisphere(2)
    dup = wv.flipped_duplication(hemi, epsilon=0.02)
    fld = wv.ScalarField(wv.GridSpec((-1.0, 0.0, 0.5), (1.0, 2.0, 0.75), (4, 3, 5)),
                         np.random.default_rng(53).normal(size=60))
    with tempfile.TemporaryDirectory() as d:
        wv.save_field(fld, f"{d}/f.wvox")
        raw64 = np.frombuffer(open(f"{d}/f.wvox", "rb").read(), dtype=np.uint8)
        f32 = wv.ScalarField(fld.spec, fld.values.astype(np.float32))
        wv.save_field(f32, f"{d}/g.wvox")
        raw32 = np.frombuffer(open(f"{d}/g.wvox", "rb").read(), dtype=np.uint8)
    save("openmesh_and_io", hemi_vertices=hemi.vertices, hemi_faces=hemi.faces,
         dup_vertices=dup.vertices, dup_faces=dup.faces, field_values=fld.values,
         wvox_f64=raw64, wvox_f32=raw32)

    # 13. marching cubes + smoothing (recon.py:39-140) on a voxelized mesh and
    #     on a smooth random field
    mc = {}
    spec16 = wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 16)
    occ = wv.voxelize(shapes.icosphere(2, 0.7), spec16)
    m1 = wv.marching_cubes(occ, iso=0.5)
    s1 = wv.laplacian_smooth(m1, lam=0.15, iterations=10)
    rng = np.random.default_rng(21)
    spec14 = wv.GridSpec((-1.0, -0.5, 0.0), (1.0, 1.5, 2.0), (14, 12, 13))
    nodes = spec14.node_coordinates()
    cen = rng.uniform([-0.6, 0.0, 0.5], [0.6, 1.0, 1.5], size=(5, 3))
    smooth = sum(np.exp(-np.sum((nodes - c) ** 2, axis=1) / 0.08) for c in cen)
    m2 = wv.marching_cubes(wv.ScalarField(spec14, smooth), iso=0.3)
    mc.update(occ=occ.values, m1_vertices=m1.vertices, m1_faces=m1.faces,
              s1_vertices=s1.vertices, smooth=smooth, m2_vertices=m2.vertices,
              m2_faces=m2.faces, **grid_dict("g16", spec16), **grid_dict("g14", spec14))
    save("marching_cubes", **mc)

    # 10. solid-angle known answers (test_winding.py:45-83)
    save("solid_angle_known",
         octant=np.array(wv.solid_angle_triangle([1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, 0])),
         cube_face_center=np.array(wv.winding_number_exact(shapes.cube(0.5), [0.5, 0.0, 0.0])),
         nested=np.array(wv.winding_number_exact(
             shapes.concatenate(shapes.cube(0.5), shapes.cube(0.25)), [0, 0, 0])))
    return 0


if __name__ == "__main__":
    sys.exit(main())
