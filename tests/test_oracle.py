"""CPU: the oracle (C restatement) pinned against the reference's golden vectors,
known-answer tests, the committed fixture made by the reference itself, and —
when oracle/_ref is built — the reference's own translation units."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_2412_00291_b200 as svx
from oracle import bindings as ob
from tests.helpers import Golden

pytestmark = pytest.mark.skipif(not ob.oracle_available(), reason="oracle not built")


def L():
    lib = ob.olib()
    lib.svxo_project_point.argtypes = [C.POINTER(C.c_double), C.POINTER(svx.LidarModel),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_double)]
    lib.svxo_back_project.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(svx.LidarModel),
                                      C.POINTER(C.c_double)]
    lib.svxo_nonprojective_distance.restype = C.c_double
    lib.svxo_nonprojective_distance.argtypes = [C.c_double] * 4
    lib.svxo_observation_weight.restype = C.c_float
    lib.svxo_observation_weight.argtypes = [C.c_double, C.c_double, C.c_float]
    lib.svxo_truncate_distance.restype = C.c_float
    lib.svxo_truncate_distance.argtypes = [C.c_double, C.c_double]
    lib.svxo_world_to_voxel.argtypes = [C.POINTER(C.c_double), C.c_float, C.POINTER(C.c_int32)]
    lib.svxo_traverse.restype = C.c_uint64
    lib.svxo_traverse.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_float,
                                  C.c_void_p, C.c_uint64]
    lib.svxo_label_to_likelihood.argtypes = [C.c_int, C.c_float, C.c_int, C.c_float,
                                             C.POINTER(C.c_float)]
    lib.svxo_bayes.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int]
    return lib


def d3(*v):
    return (C.c_double * 3)(*v)


def w2v(p, vs):
    out = (C.c_int32 * 3)()
    L().svxo_world_to_voxel(d3(*p), vs, out)
    return tuple(out)


def project_point(p, model):
    u, v, r = C.c_int(), C.c_int(), C.c_double()
    ok = L().svxo_project_point(d3(*p), C.byref(model.c()), C.byref(u), C.byref(v), C.byref(r))
    return bool(ok), u.value, v.value, r.value


# --- golden vectors of proj/tests/test_voxel_store.cpp:15-34
def test_world_to_voxel_golden():
    assert w2v((1.0, 0.0, -0.5), 0.25) == (4, 0, -2)
    assert w2v((0.0, 0.0, 0.0), 0.25) == (0, 0, 0)
    assert w2v((0.125, 0.0, 0.0), 0.25) == (1, 0, 0)   # half rounds toward +inf
    assert w2v((-0.125, 0.0, 0.0), 0.25) == (0, 0, 0)
    rng = np.random.default_rng(7)
    vs = np.float32(0.25)
    for v in rng.integers(-1000000, 1000001, size=(2000, 3)):
        c = tuple(float(np.float64(vs) * int(x)) for x in v)
        assert w2v(c, 0.25) == tuple(int(x) for x in v)


# --- proj/tests/test_scan_projection.cpp
def test_projection_golden():
    m = svx.ProjectionModel.spinning(1024, 64, 22.5, 22.5)
    ok, u, v, r = project_point((1.0, 0.0, 0.0), m)
    assert ok and u == 512 and abs(r - 1.0) < 1e-12           # :25-32
    assert not project_point((0.0, 0.0, 5.0), m)[0]            # pole drops (:34-40)
    rng = np.random.default_rng(17)                            # round trip (:70-87)
    for _ in range(1000):
        u0, v0 = int(rng.integers(0, 1024)), int(rng.integers(0, 64))
        d = float(rng.uniform(0.5, 60.0))
        p = (C.c_double * 3)()
        L().svxo_back_project(u0, v0, d, C.byref(m.c()), p)
        ok, u1, v1, r1 = project_point(tuple(p), m)
        assert ok and (u1, v1) == (u0, v0) and abs(r1 - d) <= 1e-6


def test_project_cloud_golden():
    m = svx.ProjectionModel.spinning(1024, 64, 22.5, 22.5)
    pose = svx.pose_c()
    d, h, n, v, dr = ob.OracleMap.project(m, np.array([[5, 0, 0], [2, 0, 0]], np.float32), pose)
    ok, u, vv, r = project_point((2.0, 0.0, 0.0), m)
    assert d[vv * 1024 + u] == pytest.approx(2.0)              # nearer wins (:42-51)
    _, _, _, _, dr = ob.OracleMap.project(
        m, np.array([[0.1, 0, 0], [np.nan, 0, 0]], np.float32), pose)
    assert dr == 2                                             # dropped (:93-99)
    rng = np.random.default_rng(3)                             # order independence (:53-68)
    pts = np.stack([rng.uniform(-20, 20, 5000), rng.uniform(-20, 20, 5000),
                    rng.uniform(-20, 20, 5000) * 0.2], 1).astype(np.float32)
    a = ob.OracleMap.project(m, pts, pose)
    b = ob.OracleMap.project(m, pts[rng.permutation(5000)], pose)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    tp = svx.pose_c(np.eye(3), [0, 0, 2.0])                    # height = world z (:101-111)
    d, h, *_ = ob.OracleMap.project(m, np.array([[3, 0, -1]], np.float32), tp)
    ok, u, vv, _ = project_point((3.0, 0.0, -1.0), m)
    assert h[vv * 1024 + u] == pytest.approx(1.0)


# --- proj/tests/test_tsdf_integrator.cpp:54-144 and acceptance A9
def test_equation_kats():
    lib = L()
    th, al, psi = 30 * math.pi / 180, 20 * math.pi / 180, 0.1
    got = lib.svxo_nonprojective_distance(psi, th, al, 1e-2)
    assert abs(got - 0.1747660307326763) <= 1e-9
    assert lib.svxo_nonprojective_distance(-psi, th, al, 1e-2) == pytest.approx(-got, rel=1e-6)
    assert lib.svxo_nonprojective_distance(0.2, 0.0, 0.0, 1e-2) == pytest.approx(0.2)
    assert lib.svxo_nonprojective_distance(0.2, math.pi / 3, 0.0, 1e-2) == pytest.approx(0.1)
    assert lib.svxo_observation_weight(0.5, 0.5, 0.01) == pytest.approx(1.0)
    assert lib.svxo_observation_weight(0.0, 0.5, 0.01) == pytest.approx(0.5)
    assert lib.svxo_observation_weight(-0.5, 0.5, 0.01) == pytest.approx(0.01)
    assert lib.svxo_truncate_distance(0.5, 0.3) == pytest.approx(0.3)
    assert lib.svxo_truncate_distance(-0.5, 0.3) == pytest.approx(-0.3)


def dense_march(a, b, vs):
    """oracles::marched_voxels (proj/tests/oracles.hpp:109-120)."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    ln = np.linalg.norm(b - a)
    steps = max(2, int(ln / (vs / 64.0)))
    inv = 1.0 / float(np.float32(vs))
    t = np.arange(steps + 1) / steps
    p = a[None] + (b - a)[None] * t[:, None]
    return set(map(tuple, np.floor(p * inv + 0.5).astype(np.int64)))


def test_dda_covers_dense_march():                 # test_tsdf_integrator.cpp:146-164
    rng = np.random.default_rng(5)
    for _ in range(100):
        a, b = rng.uniform(-2, 2, 3), rng.uniform(-2, 2, 3)
        out = np.zeros((4096, 3), np.int32)
        n = L().svxo_traverse(d3(*a), d3(*b), 0.1, out.ctypes.data_as(C.c_void_p), 4096)
        visited = set(map(tuple, out[:n].tolist()))
        marched = dense_march(a, b, 0.1)
        assert marched <= visited
        assert len(visited) <= len(marched) + 6


def test_semantic_kats():                          # test_semantic_integrator.cpp:37-99
    lib = L()
    p = (C.c_float * 2)(0.5, 0.5)
    lib.svxo_bayes(p, (C.c_float * 2)(0.7, 0.3), 2)
    lib.svxo_bayes(p, (C.c_float * 2)(0.6, 0.4), 2)
    assert p[0] == pytest.approx(0.42 / 0.54, rel=1e-6) and p[1] == pytest.approx(0.12 / 0.54, rel=1e-6)
    like = (C.c_float * 4)()
    assert lib.svxo_label_to_likelihood(2, 0.7, 4, 1e-3, like) == 0
    assert list(like) == pytest.approx([0.1, 0.1, 0.7, 0.1], rel=1e-5)
    assert lib.svxo_label_to_likelihood(0, 1.5, 2, 1e-3, like) == 1   # invalid confidence
    assert lib.svxo_label_to_likelihood(0, 1.0, 3, 1e-3, like) == 0
    assert like[1] > 0 and like[2] > 0                                 # flooring


def test_oracle_matches_reference_fixture():
    """The C restatement reproduces the reference's own outputs byte for byte
    (fixture generated by tests/golden/make_golden.py from the reference)."""
    g = Golden()
    for mode in (svx.NON_PROJECTIVE, svx.PROJECTIVE):
        o = ob.OracleMap(g.cfg)
        for i in range(g.n):
            d, h, n, v, dr = ob.OracleMap.project(g.model, g.points(i), g.pose(i))
            if mode == svx.NON_PROJECTIVE:
                assert np.array_equal(d, g.d[f"depth{i}"]) and np.array_equal(h, g.d[f"height{i}"])
                assert np.array_equal(n, g.d[f"normals{i}"]) and np.array_equal(v, g.d[f"valid{i}"])
                assert dr == int(g.d[f"dropped{i}"])
            r = o.integrate(g.model, d, n, v, g.pose(i), svx.IntegratorConfig(mode=mode))
            s = o.integrate_labels(g.label_image(i), svx.SemanticConfig())
            assert (r.updated_voxels, r.new_blocks, s.updated_voxels) == \
                tuple(g.d[f"reports_m{mode}"][i])
        g.check_map(o.save_bytes(), mode)


needs_ref = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built here")


@needs_ref
@pytest.mark.parametrize("variant", ["default", "projective", "drop_unreliable", "no_bayes",
                                     "tensor", "confidence", "raycast", "trunc_range"])
def test_oracle_equals_reference_tus(variant):
    """Oracle vs the reference's own translation units on the tiny workload."""
    from paper_2412_00291_b200 import workload as W
    wl = W.make("tiny", 3)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 18)
    icfg = svx.IntegratorConfig()
    scfg = svx.SemanticConfig()
    if variant == "projective":
        icfg.mode = svx.PROJECTIVE
    if variant == "drop_unreliable":
        icfg.drop_unreliable = True
    if variant == "no_bayes":
        scfg.use_bayes = False
    if variant == "raycast":
        scfg.occlusion = svx.RAYCAST
    if variant == "trunc_range":
        icfg.truncation, icfg.max_range = 0.3, 12.0
    o, r = ob.OracleMap(cfg), ob.RefMap(cfg)
    rng = np.random.default_rng(1)
    for p, i in wl.scans():
        p = p.numpy()
        pose = wl.pose(i)
        a = ob.OracleMap.project(wl.model, p, pose)
        b = ob.RefMap.project(wl.model, p, pose)
        for x, y in zip(a[:4], b[:4]):
            assert np.array_equal(x, y)
        ra = o.integrate(wl.model, a[0], a[2], a[3], pose, icfg)
        rb = r.integrate(wl.model, b[0], b[2], b[3], pose, icfg)
        assert (ra.updated_voxels, ra.new_blocks) == (rb.updated_voxels, rb.new_blocks)
        for li in wl.label_images(i):
            if variant == "tensor":
                t = rng.uniform(0, 1, (li.height, li.width, 20)).astype(np.float32)
                li.prob_tensor = t
            if variant == "confidence":
                li.confidence = rng.uniform(0, 1, (li.height, li.width)).astype(np.float32)
            sa = o.integrate_labels(li, scfg)
            sb = r.integrate_labels(li, scfg)
            assert sa.updated_voxels == sb.updated_voxels
    assert o.save_bytes() == r.save_bytes()
    assert np.array_equal(o.take_dirty(0), r.take_dirty(0))
    assert np.array_equal(o.take_dirty(1), r.take_dirty(1))


@needs_ref
def test_capacity_error_semantics_match_reference():
    """CapacityError mid-frame: sorted-prefix allocation, no voxel updated
    (tsdf_integrator.cpp:160-168)."""
    from paper_2412_00291_b200 import workload as W
    wl = W.make("tiny", 1)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 300)
    o, r = ob.OracleMap(cfg), ob.RefMap(cfg)
    p, i = next(iter(wl.scans()))
    a = ob.OracleMap.project(wl.model, p.numpy(), wl.pose(i))
    with pytest.raises(ob.CheckerError) as e1:
        o.integrate(wl.model, a[0], a[2], a[3], wl.pose(i), svx.IntegratorConfig())
    with pytest.raises(ob.CheckerError) as e2:
        r.integrate(wl.model, a[0], a[2], a[3], wl.pose(i), svx.IntegratorConfig())
    assert e1.value.code == e2.value.code == 2
    assert o.save_bytes() == r.save_bytes()
    assert o.block_count() == r.block_count() == 300
