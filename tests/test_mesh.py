"""Map export to a mesh: extract_mesh / IncrementalMesher
(proj/src/mesh.cpp:105-287).

CPU: the marching-cubes tables against the reference header, and the oracle's C
restatement of extract_mesh against the reference's own mesh.cpp (oracle/_ref) on
hand-built SDF maps and on integrated scan sequences, bit for bit.
GPU: the device mesher (svx_mesh.cu through the C-ABI) against the oracle on the
same maps, and the IncrementalMesher against the reference's."""
import os
import re

import numpy as np
import pytest

import paper_2412_00291_b200 as svx
from oracle import bindings as ob

REF_MC = "/root/reference/proj/include/semvox/mc_tables.hpp"
MC_H = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2412_00291_b200", "csrc", "svx_mc_tables.h")

needs_oracle = pytest.mark.skipif(not ob.oracle_available(), reason="oracle not built")
needs_ref = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built here")


def _product_tables():
    src = open(MC_H).read()
    tris = re.findall(r'"([0-9a-f]*)"', src[src.index("kMcTris"):])
    assert len(tris) == 256
    return [[int(ch, 16) for ch in t] for t in tris]


@pytest.mark.skipif(not os.path.exists(REF_MC), reason="reference tree not mounted")
def test_mc_tables_match_reference():
    """Same triangulation, corner and edge numbering as the reference's tables."""
    src = open(REF_MC).read()
    tri = src[src.index("kTriTable"):]
    ref = [[int(x) for x in r.split(",") if x.strip()] for r in re.findall(r"\{([-0-9, ]+)\}", tri)]
    ref = [[x for x in r if x >= 0] for r in ref[:256]]
    assert _product_tables() == ref
    edges = re.findall(r"0x([0-9a-f]+)", src[src.index("kEdgeTable"):src.index("kTriTable")])
    EC = [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4), (0, 4), (1, 5), (2, 6), (3, 7)]
    for c in range(256):  # the edge mask the product derives equals the tabulated one
        m = sum(1 << e for e, (a, b) in enumerate(EC) if ((c >> a) & 1) != ((c >> b) & 1))
        assert m == int(edges[c], 16)


# ----------------------------------------------------------------- test maps

def sphere_map(cfg, radius, extent, center=(0.0, 0.0, 0.0), seed=0, sem_frac=0.0, holes=0.0):
    """Blocks {key: (tsdf[512], sem[512,K] | None)} holding the exact SDF of a sphere
    (fill_sphere, proj/tests/test_mesh.cpp:26-38), optionally with random semantic
    layers (some voxels left at the exact uniform prior) and unobserved holes."""
    rng = np.random.default_rng(seed)
    vs, tau, K = cfg.voxel_size, cfg.truncation, cfg.num_labels
    blocks = {}
    r = np.arange(-extent, extent + 1)
    z, y, x = np.meshgrid(r, r, r, indexing="ij")
    v = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.int32)
    c = v.astype(np.float64) * np.float64(np.float32(vs)) - np.asarray(center)
    nrm = np.sqrt((c[:, 0] * c[:, 0] + c[:, 1] * c[:, 1]) + c[:, 2] * c[:, 2])
    d = nrm - radius
    keep = np.abs(d) <= tau
    if holes:
        keep &= rng.uniform(size=len(keep)) >= holes
    v, c, nrm, d = v[keep], c[keep], nrm[keep], d[keep]
    g = np.where(nrm[:, None] > 1e-9, c / np.maximum(nrm, 1e-300)[:, None], [0, 0, 1]).astype(np.float32)
    dt = np.clip(d, -tau, tau).astype(np.float32)
    w = rng.choice(np.array([1.0, 0.5, 5e-5], np.float32), size=len(v), p=[0.8, 0.15, 0.05])
    bk = np.floor_divide(v, 8)
    lin = (v[:, 0] & 7) + 8 * (v[:, 1] & 7) + 64 * (v[:, 2] & 7)
    for key in np.unique(bk, axis=0):
        sel = np.all(bk == key, axis=1)
        t = np.zeros(512, svx.TSDF_DTYPE)
        t["distance"][lin[sel]] = dt[sel]
        t["weight"][lin[sel]] = w[sel]
        t["gradient"][lin[sel]] = g[sel]
        sem = None
        if rng.uniform() < sem_frac:
            sem = np.full((512, K), np.float32(1.0) / np.float32(K), np.float32)
            upd = rng.uniform(size=512) < 0.7
            p = rng.dirichlet(np.ones(K), size=int(upd.sum())).astype(np.float32)
            sem[upd] = p
            if rng.uniform() < 0.3:  # exact ties between classes
                sem[upd, 1] = sem[upd, 0]
        blocks[tuple(int(a) for a in key)] = (t, sem)
    return blocks


def load_into(m, blocks):
    for k, (t, s) in blocks.items():
        m.get_or_allocate_block(k)
        m.write_block(k, t, s, has_sem=s is not None) if isinstance(m, (ob.OracleMap, ob.RefMap)) \
            else m.write_block(k, t, s)


def assert_mesh_equal(a, b):
    for x, y, name in zip(a, b, ("vertices", "normals", "labels", "faces")):
        assert x.shape == y.shape, (name, x.shape, y.shape)
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), name  # bitwise


SPHERES = [
    dict(vs=0.05, tau=0.25, K=4, radius=0.5, extent=16),
    dict(vs=0.1, tau=0.5, K=20, radius=1.3, extent=20, center=(0.03, -0.41, 0.2), sem_frac=0.8,
         holes=0.02),
    dict(vs=0.2, tau=1.0, K=3, radius=2.9, extent=24, center=(-1.7, 0.9, -3.3), sem_frac=1.0),
]


@needs_ref
@pytest.mark.parametrize("case", range(len(SPHERES)))
@pytest.mark.parametrize("reserved", [False, True])
def test_oracle_mesh_equals_reference_spheres(case, reserved):
    sp = SPHERES[case]
    cfg = svx.MapConfig(sp["vs"], sp["tau"], sp["K"], 1 << 16)
    blocks = sphere_map(cfg, sp["radius"], sp["extent"], sp.get("center", (0, 0, 0)), seed=case,
                        sem_frac=sp.get("sem_frac", 0.0), holes=sp.get("holes", 0.0))
    o, r = ob.OracleMap(cfg), ob.RefMap(cfg)
    load_into(o, blocks)
    load_into(r, blocks)
    res = cfg.num_labels - 1 if reserved else -1
    mo = o.extract_mesh(1e-4, res)
    assert mo[3].shape[0] > 100
    assert_mesh_equal(mo, r.extract_mesh(1e-4, res))


@needs_ref
def test_oracle_mesh_equals_reference_integrated():
    """A labelled scan sequence integrated by the reference: its mesh, restated."""
    from tests.helpers import Golden
    g = Golden()
    o, r = ob.OracleMap(g.cfg), ob.RefMap(g.cfg)
    for i in range(g.n):
        d, h, n, v, _ = ob.OracleMap.project(g.model, g.points(i), g.pose(i))
        for m in (o, r):
            m.integrate(g.model, d, n, v, g.pose(i), svx.IntegratorConfig())
            m.integrate_labels(g.label_image(i), svx.SemanticConfig())
    assert o.save_bytes() == r.save_bytes()
    for res in (-1, g.cfg.num_labels - 1):
        mo = o.extract_mesh(1e-4, res)
        assert mo[3].shape[0] > 1000
        assert_mesh_equal(mo, r.extract_mesh(1e-4, res))


@needs_ref
def test_oracle_block_subset_equals_reference_incremental():
    """IncrementalMesher semantics: the stitched mesh after update(dirty) is the
    mesh of the cached block set (mesh.cpp:231-287), which the oracle's block-subset
    extraction restates; the cached-set bookkeeping is the product's Python mirror."""
    cfg = svx.MapConfig(0.05, 0.25, 4, 1 << 16)
    blocks = sphere_map(cfg, 0.5, 16, seed=3, sem_frac=0.5)
    o, r = ob.OracleMap(cfg), ob.RefMap(cfg)
    load_into(o, blocks)
    load_into(r, blocks)
    keys = np.array(sorted(blocks), np.int32)
    cache = set()
    rng = np.random.default_rng(5)
    for step in range(4):
        dirty = keys[rng.uniform(size=len(keys)) < 0.3] if step else keys[:5]
        if step == 3:
            dirty = np.concatenate([dirty, [[40, 40, 40]]]).astype(np.int32)  # absent block
        mr, rem = r.mesh_incremental(dirty)
        off = np.array([(x, y, z) for z in (-1, 0) for y in (-1, 0) for x in (-1, 0)], np.int32)
        aff = np.unique((dirty[:, None, :] + off[None]).reshape(-1, 3), axis=0)
        present = np.array([tuple(a) in blocks for a in aff.tolist()])
        assert np.array_equal(rem, aff[present])
        for a, p in zip(map(tuple, aff.tolist()), present):
            (cache.add if p else cache.discard)(a)
        mo = o.extract_mesh(1e-4, -1, np.array(sorted(cache), np.int32))
        assert_mesh_equal(mo, mr)


# ------------------------------------------------------------------------ GPU

@pytest.mark.gpu
@needs_oracle
@pytest.mark.parametrize("case", range(len(SPHERES)))
def test_gpu_mesh_equals_oracle_spheres(case):
    sp = SPHERES[case]
    cfg = svx.MapConfig(sp["vs"], sp["tau"], sp["K"], 1 << 16)
    blocks = sphere_map(cfg, sp["radius"], sp["extent"], sp.get("center", (0, 0, 0)), seed=case,
                        sem_frac=sp.get("sem_frac", 0.0), holes=sp.get("holes", 0.0))
    o = ob.OracleMap(cfg)
    load_into(o, blocks)
    gpu = svx.VoxelStore(cfg)
    load_into(gpu, blocks)
    for res in (-1, cfg.num_labels - 1):
        mg = svx.extract_mesh(gpu, 1e-4, ["c"] * (cfg.num_labels - 1) + ["unlabeled"]
                              if res >= 0 else None)
        got = (mg.vertices, mg.vertex_normals, mg.vertex_labels, mg.faces)
        assert_mesh_equal(got, o.extract_mesh(1e-4, res))
    for mw in (0.0, 0.6):  # the weight threshold decides cell usability
        mg = svx.extract_mesh(gpu, mw)
        assert_mesh_equal((mg.vertices, mg.vertex_normals, mg.vertex_labels, mg.faces),
                          o.extract_mesh(mw, -1))
    gpu.close()


@pytest.mark.gpu
@needs_oracle
def test_gpu_mesh_of_integrated_sequence():
    """Mesh of a map integrated on the GPU = oracle mesh of the oracle's map (the two
    maps are byte-identical, tests/test_gpu_parity.py)."""
    from paper_2412_00291_b200 import workload as W
    wl = W.make("cfg1", 4)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 18)
    gpu = svx.VoxelStore(cfg)
    o = ob.OracleMap(cfg)
    tsdf = svx.TsdfIntegrator(gpu, svx.IntegratorConfig())
    sem = svx.SemanticIntegrator(gpu, svx.SemanticConfig())
    for p, i in wl.scans():
        p = p.numpy()
        pose = wl.pose(i)
        tsdf.integrate_cloud(p, pose, wl.model)
        d, h, n, v, _ = ob.OracleMap.project(wl.model, p, pose)
        o.integrate(wl.model, d, n, v, pose, svx.IntegratorConfig())
        for li in wl.label_images(i):
            sem.integrate_labels(li)
            o.integrate_labels(li, svx.SemanticConfig())
    assert gpu.save_bytes() == o.save_bytes()
    names = ["c"] * (cfg.num_labels - 1) + ["unlabeled"]
    mg = svx.extract_mesh(gpu, label_names=names)
    assert mg.faces.shape[0] > 10000
    assert_mesh_equal((mg.vertices, mg.vertex_normals, mg.vertex_labels, mg.faces),
                      o.extract_mesh(1e-4, cfg.num_labels - 1))
    # watertight where closed: every face index in range, no degenerate faces
    f = mg.faces.astype(np.int64)
    assert f.max() < mg.vertex_count()
    assert np.all((f[:, 0] != f[:, 1]) & (f[:, 1] != f[:, 2]) & (f[:, 0] != f[:, 2]))
    gpu.close()


@pytest.mark.gpu
@needs_ref
def test_gpu_incremental_mesher_equals_reference():
    cfg = svx.MapConfig(0.05, 0.25, 4, 1 << 16)
    blocks = sphere_map(cfg, 0.5, 16, seed=3, sem_frac=0.5)
    r = ob.RefMap(cfg)
    load_into(r, blocks)
    gpu = svx.VoxelStore(cfg)
    load_into(gpu, blocks)
    mesher = svx.IncrementalMesher()
    keys = np.array(sorted(blocks), np.int32)
    rng = np.random.default_rng(5)
    m0 = mesher.update(gpu, np.zeros((0, 3), np.int32))
    assert m0.vertex_count() == 0 and len(mesher.last_remeshed) == 0
    for step in range(4):
        dirty = keys[rng.uniform(size=len(keys)) < 0.3] if step else keys[:5]
        if step == 3:
            dirty = np.concatenate([dirty, [[40, 40, 40]]]).astype(np.int32)
        mr, rem = r.mesh_incremental(dirty)
        mg = mesher.update(gpu, dirty)
        assert np.array_equal(mesher.last_remeshed, rem)
        assert_mesh_equal((mg.vertices, mg.vertex_normals, mg.vertex_labels, mg.faces), mr)
    gpu.close()
