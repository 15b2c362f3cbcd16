"""GPU parity: the CUDA path (through the C-ABI) vs the oracle and the reference's
own outputs on identical inputs. Bit-exact for keys, counts, weights, semantic
probabilities and (so far observed) the whole SVOX1 image; D/g within 1e-5."""
import numpy as np
import pytest

import paper_2412_00291_b200 as svx
from oracle import bindings as ob
from paper_2412_00291_b200 import workload as W
from tests.helpers import Golden, compare_maps

pytestmark = pytest.mark.gpu


def _run_pair(wl, icfg, scfg=None, frames=None, labels=True, label_mut=None, max_blocks=1 << 20):
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, max_blocks)
    g = svx.VoxelStore(cfg, 0)
    o = ob.OracleMap(cfg)
    ti, si = svx.TsdfIntegrator(g, icfg), svx.SemanticIntegrator(g, scfg or svx.SemanticConfig())
    for p, i in wl.scans(frames=frames):
        p = p.numpy()
        pose = wl.pose(i)
        rg = ti.integrate_cloud(p, pose, wl.model)
        d, h, n, v, _ = ob.OracleMap.project(wl.model, p, pose)
        ro = o.integrate(wl.model, d, n, v, pose, icfg)
        assert (rg.updated_voxels, rg.new_blocks) == (ro.updated_voxels, ro.new_blocks)
        assert rg.frame == ro.frame
        if labels:
            for li in wl.label_images(i):
                if label_mut:
                    label_mut(li)
                a = si.integrate_labels(li)
                b = o.integrate_labels(li, scfg or svx.SemanticConfig())
                assert a.updated_voxels == b.updated_voxels
    return g, o


def test_golden_fixture_reference_outputs():
    """GPU reproduces the reference's own SVOX1 snapshot byte for byte."""
    gd = Golden()
    for mode in (svx.NON_PROJECTIVE, svx.PROJECTIVE):
        g = svx.VoxelStore(gd.cfg, 0)
        ti = svx.TsdfIntegrator(g, svx.IntegratorConfig(mode=mode))
        si = svx.SemanticIntegrator(g)
        for i in range(gd.n):
            img = svx.project_cloud(gd.points(i), gd.pose(i), gd.model, g)
            if mode == svx.NON_PROJECTIVE:
                assert np.array_equal(img.depth, gd.d[f"depth{i}"])
                assert np.array_equal(img.height, gd.d[f"height{i}"])
                assert np.array_equal(img.normals, gd.d[f"normals{i}"])
                assert np.array_equal(img.normal_valid, gd.d[f"valid{i}"])
                assert img.dropped == int(gd.d[f"dropped{i}"])
            r = ti.integrate_frame(img, gd.pose(i))
            s = si.integrate_labels(gd.label_image(i))
            assert (r.updated_voxels, r.new_blocks, s.updated_voxels) == \
                tuple(gd.d[f"reports_m{mode}"][i])
        gd.check_map(g.save_bytes(), mode)
        g.close()


@pytest.mark.parametrize("mode", [svx.NON_PROJECTIVE, svx.PROJECTIVE])
def test_tiny_sequence_both_modes(mode):
    g, o = _run_pair(W.make("tiny", 4), svx.IntegratorConfig(mode=mode))
    st = compare_maps(g.save_bytes(), o.save_bytes(), exact=(mode == svx.PROJECTIVE))
    assert st["blocks"] > 1000
    assert np.array_equal(g.take_dirty_blocks(0), o.take_dirty(0))
    assert np.array_equal(g.take_dirty_blocks(1), o.take_dirty(1))


def test_cfg2_frames_full_size():
    """Headline geometry (128 x 1024, 0.1 m) at full size, 2 frames."""
    g, o = _run_pair(W.make("cfg2", 2), svx.IntegratorConfig(), labels=True)
    st = compare_maps(g.save_bytes(), o.save_bytes())
    assert st["blocks"] > 5000


def test_cfg1_frame():
    g, o = _run_pair(W.make("cfg1", 1), svx.IntegratorConfig(), labels=False)
    compare_maps(g.save_bytes(), o.save_bytes())


@pytest.mark.parametrize("variant", ["drop_unreliable", "trunc_range", "no_bayes", "tensor",
                                     "confidence", "raycast"])
def test_config_variants(variant):
    icfg, scfg = svx.IntegratorConfig(), svx.SemanticConfig()
    mut = None
    rng = np.random.default_rng(2)
    if variant == "drop_unreliable":
        icfg.drop_unreliable = True
    if variant == "trunc_range":
        icfg.truncation, icfg.max_range, icfg.alpha_epsilon = 0.3, 12.0, 0.05
    if variant == "no_bayes":
        scfg.use_bayes = False
    if variant == "raycast":
        scfg.occlusion = svx.RAYCAST
    if variant == "tensor":
        def mut(li):
            li.prob_tensor = rng.uniform(0, 1, (li.height, li.width, 20)).astype(np.float32)
    if variant == "confidence":
        def mut(li):
            li.confidence = rng.uniform(0, 1, (li.height, li.width)).astype(np.float32)
    g, o = _run_pair(W.make("tiny", 3), icfg, scfg, label_mut=mut)
    compare_maps(g.save_bytes(), o.save_bytes())


def test_projection_edge_cases_bit_exact():
    """Ties (equal ranges), duplicates, NaN, below min range, pole, permutations."""
    m = svx.ProjectionModel.spinning(512, 32, 25.0, 25.0)
    rng = np.random.default_rng(9)
    pts = np.stack([rng.uniform(-20, 20, 20000), rng.uniform(-20, 20, 20000),
                    rng.uniform(-4, 4, 20000)], 1).astype(np.float32)
    # exact range ties inside one pixel: mirror points across the pixel-centre ray
    base = pts[:300].copy()
    tie = base.copy()
    tie[:, 2] = base[:, 2] * np.float32(1.0)
    pts = np.concatenate([pts, base, tie, base[::-1], [[0.1, 0, 0], [np.nan, 0, 0], [0, 0, 5]]]).astype(np.float32)
    g = svx.VoxelStore(svx.MapConfig(0.1, 0.5, 4), 0)
    pose = svx.pose_c(np.eye(3), [1.0, -2.0, 0.5])
    for perm in (np.arange(len(pts)), rng.permutation(len(pts))):
        img = svx.project_cloud(pts[perm], pose, m, g)
        d, h, n, v, dr = ob.OracleMap.project(m, pts, pose)
        assert np.array_equal(img.depth, d) and np.array_equal(img.height, h)
        assert np.array_equal(img.normals, n) and np.array_equal(img.normal_valid, v)
        assert img.dropped == dr


def test_exact_range_ties_resolve_lexicographically():
    # rows cover 59..119 deg polar in 7.5 deg steps: +-z around the horizon stay in row 4,
    # azimuth 0.05 rad stays in column 31; (x, y, +z) and (x, y, -z) have equal ranges
    m = svx.ProjectionModel.spinning(64, 8, 31.0, 29.0)
    a = np.array([[4.0, 0.2, 0.01], [4.0, 0.2, -0.01], [4.0, 0.2, 0.01]], np.float32)
    g = svx.VoxelStore(svx.MapConfig(0.1, 0.5, 2), 0)
    pose = svx.pose_c(np.eye(3), [0, 0, 1.0])
    for perm in ([0, 1, 2], [2, 1, 0], [1, 0, 2]):
        img = svx.project_cloud(a[perm], pose, m, g)
        d, h, *_ = ob.OracleMap.project(m, a, pose)
        assert np.array_equal(img.depth, d) and np.array_equal(img.height, h)


def test_capacity_error_matches_oracle():
    wl = W.make("tiny", 1)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 300)
    g = svx.VoxelStore(cfg, 0)
    o = ob.OracleMap(cfg)
    p, i = next(iter(wl.scans()))
    p = p.numpy()
    with pytest.raises(svx.CapacityError):
        svx.TsdfIntegrator(g).integrate_cloud(p, wl.pose(i), wl.model)
    d, h, n, v, _ = ob.OracleMap.project(wl.model, p, wl.pose(i))
    with pytest.raises(ob.CheckerError):
        o.integrate(wl.model, d, n, v, wl.pose(i), svx.IntegratorConfig())
    assert g.block_count() == 300
    assert g.save_bytes() == o.save_bytes()
    assert np.array_equal(g.take_dirty_blocks(0), o.take_dirty(0))


def test_sweep_sizes_cfg5():
    for W_ in (80, 640):
        g, o = _run_pair(W.make(f"cfg5-{W_}", 2), svx.IntegratorConfig(), labels=False)
        compare_maps(g.save_bytes(), o.save_bytes())


def test_sweep_max_size_cfg5():
    """The largest scan of the cfg5 sweep (16384 x 128 = 2.1M pixels, every ray hits)."""
    g, o = _run_pair(W.make("cfg5-16384", 1), svx.IntegratorConfig(), labels=False, max_blocks=1 << 21)
    st = compare_maps(g.save_bytes(), o.save_bytes())
    assert st["blocks"] > 1000


def test_sensor_next_to_a_wall_many_rays_per_voxel():
    """Returns at 0.4-2 m (a sensor 0.5 m from a wall, a 4096-column scan): thousands of rays
    visit the same voxels and many own pixels fall outside the vertical field of view, so
    the fallback path orders long visit lists (sorted records, O(records)). One call per
    frame and one batched call both equal the oracle."""
    import torch
    wl = W.make("cfg5-4096", 3)
    wl.poses = [W.yaw_pose(14.5, 0.0, 0.5, 0.0), W.yaw_pose(14.4, 0.2, 0.6, 0.4), W.yaw_pose(14.45, -0.3, 0.4, -0.3)]
    g, o = _run_pair(wl, svx.IntegratorConfig(), labels=False)
    compare_maps(g.save_bytes(), o.save_bytes())
    b = svx.VoxelStore(svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20), 0)
    chunks = [p for p, _ in wl.scans()]
    offs = np.zeros(len(chunks) + 1, np.uint64)
    offs[1:] = np.cumsum([c.shape[0] for c in chunks])
    pts = torch.cat(chunks).contiguous().cuda()
    reps = b.integrate_clouds_device(wl.model, pts.data_ptr(), offs, 3, [wl.pose(i) for i in range(3)],
                                     svx.IntegratorConfig())
    assert b.save_bytes() == g.save_bytes()
    assert all(r.updated_voxels > 0 for r in reps)


def test_batched_paths_match_per_frame():
    """The batched entry points (clouds resident in HBM; clouds in pinned host memory,
    staged through the ingest ring) produce the same map, reports and dirty lists as
    one call per frame."""
    import torch
    wl = W.make("cfg2", 12)
    scans = [p.numpy() for p, _ in wl.scans()]
    poses = [wl.pose(i) for i in range(len(scans))]
    offs = np.zeros(len(scans) + 1, np.uint64)
    offs[1:] = np.cumsum([s.shape[0] for s in scans])
    flat = np.ascontiguousarray(np.concatenate(scans).astype(np.float32))
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
    icfg = svx.IntegratorConfig()

    ref = svx.VoxelStore(cfg, 0)
    ti = svx.TsdfIntegrator(ref, icfg)
    want = [ti.integrate_cloud(s, p, wl.model) for s, p in zip(scans, poses)]
    want_map = ref.save_bytes()
    want_dirty = np.asarray(ref.take_dirty_blocks(0))
    assert len(want_dirty) > 1000

    dev = torch.from_numpy(flat).cuda()
    host = torch.from_numpy(flat).pin_memory()
    import os
    for how in ("device", "host", "host_split", "device_resume"):
        if how == "device_resume":  # tiny record buffer and pool headroom: abort + resume
            os.environ["SVX_TEST_REC_CAP"], os.environ["SVX_TEST_POOL_HEAD"] = "256", "16"
        try:
            st = svx.VoxelStore(cfg, 0)
        finally:
            os.environ.pop("SVX_TEST_REC_CAP", None)
            os.environ.pop("SVX_TEST_POOL_HEAD", None)
        st.profile_enable(True)
        if how.startswith("device"):
            got = st.integrate_clouds_device(wl.model, dev.data_ptr(), offs, 3, poses, icfg)
        elif how == "host":
            got = st.integrate_clouds_host(wl.model, host.data_ptr(), offs, 3, poses, icfg)
        else:  # two calls: frame numbering and state continue across batches
            got = st.integrate_clouds_host(wl.model, host.data_ptr(), offs[:6], 3, poses[:5], icfg)
            got += st.integrate_clouds_host(wl.model, host.data_ptr(), offs[5:], 3, poses[5:], icfg)
        assert [(r.frame, r.updated_voxels, r.new_blocks) for r in got] == \
            [(r.frame, r.updated_voxels, r.new_blocks) for r in want], how
        assert st.save_bytes() == want_map, how
        assert np.array_equal(np.asarray(st.take_dirty_blocks(0)), want_dirty), how
        aborts = st.profile_read().as_dict()["aborts"]
        if how == "device_resume":
            assert aborts.get("records", 0) >= 1, aborts
        st.close()
    ref.close()


@pytest.mark.parametrize("variant", ["plain", "conf", "tensor"])
def test_label_batches_match_single_calls(variant):
    """svx_integrate_labels_batch (host and device inputs) == one integrate_labels
    call per image: same reports, same map bytes."""
    import torch
    wl = W.make("tiny", 3)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 16)
    rng = np.random.default_rng(5)

    def images(i):
        out = wl.label_images(i)
        for li in out:
            P = li.width * li.height
            if variant == "conf":
                li.confidence = rng.uniform(0.3, 1.0, P).astype(np.float32)
            if variant == "tensor":
                t = rng.uniform(0.0, 1.0, (P, wl.num_labels)).astype(np.float32)
                li.prob_tensor = t / t.sum(1, keepdims=True)
        return out

    imgs = {i: images(i) for i in range(3)}
    maps, reps = [], []
    for how in ("single", "host", "device"):
        st = svx.VoxelStore(cfg, 0)
        ti, si = svx.TsdfIntegrator(st, svx.IntegratorConfig()), svx.SemanticIntegrator(st)
        rr = []
        for p, i in wl.scans():
            ti.integrate_cloud(p.numpy(), wl.pose(i), wl.model)
            if how == "single":
                rr += [si.integrate_labels(li) for li in imgs[i]]
            elif how == "host":
                rr += si.integrate_labels_batch(imgs[i])
            else:
                dev = []
                for li in imgs[i]:
                    d = svx.LabelImage(li.width, li.height,
                                       torch.from_numpy(np.asarray(li.labels).view(np.int16).copy()).cuda(),
                                       li.fx, li.fy, li.cx, li.cy, li.pose, max_depth=li.max_depth)
                    if li.confidence is not None:
                        d.confidence = torch.from_numpy(li.confidence).cuda()
                    if li.prob_tensor is not None:
                        d.prob_tensor = torch.from_numpy(li.prob_tensor).cuda()
                    dev.append(d)
                torch.cuda.synchronize()
                rr += si.integrate_labels_batch(dev, on_device=True)
        maps.append(st.save_bytes())
        reps.append([(r.frame, r.updated_voxels) for r in rr])
        st.close()
    assert reps[0][-1][1] > 0
    assert reps[1] == reps[0] and reps[2] == reps[0]
    assert maps[1] == maps[0] and maps[2] == maps[0]


def test_key_sharded_maps_union_equals_unsharded():
    """two key shards (svx_map_set_shard, world 2) integrate the same
    scans and label images; they hold disjoint block sets, their per-frame reports sum
    to the unsharded map's, and their union is the unsharded map block for block."""
    from oracle.bindings import parse_svox1
    wl = W.make("tiny", 3)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 18)
    maps = []
    for shard in (None, (0, 2), (1, 2)):
        g = svx.VoxelStore(cfg, 0)
        if shard:
            g.set_shard(*shard)
        ti, si = svx.TsdfIntegrator(g, svx.IntegratorConfig()), svx.SemanticIntegrator(g)
        reps = []
        for p, i in wl.scans():
            r = ti.integrate_cloud(p.numpy(), wl.pose(i), wl.model)
            s = [si.integrate_labels(li).updated_voxels for li in wl.label_images(i)]
            reps.append((r.updated_voxels, r.new_blocks, sum(s)))
        maps.append((g, np.array(reps)))
    full, s0, s1 = maps
    assert np.array_equal(s0[1] + s1[1], full[1])
    _, kf, tf, sf = parse_svox1(full[0].save_bytes())
    parts = [parse_svox1(m.save_bytes()) for m, _ in (s0, s1)]
    assert len(parts[0][1]) > 0 and len(parts[1][1]) > 0
    keys = np.concatenate([p[1] for p in parts])
    tsdf = np.concatenate([p[2] for p in parts])
    has = np.concatenate([[i in p[3] for i in range(len(p[1]))] for p in parts])
    order = np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))
    assert np.array_equal(keys[order], kf)
    assert tsdf[order].tobytes() == tf.tobytes()
    assert np.array_equal(has[order], np.array([i in sf for i in range(len(kf))]))
    sems = [p[3][i] for p in parts for i in range(len(p[1])) if i in p[3]]
    sem_order = [j for j in order if has[j]]
    idx = {j: n for n, j in enumerate([j for j in range(len(keys)) if has[j]])}
    for n_full, j in enumerate(sem_order):
        assert np.array_equal(sems[idx[j]], sf[sorted(sf)[n_full]])
    for g, _ in maps:
        g.close()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_sharded_union_equals_unsharded(world):
    """The multi-GPU data plane (exchange mode, paper_2412_00291_b200.dist), every rank
    emulated in one process on one GPU: each rank casts its share of the rays, visits of
    other ranks' blocks are exchanged, each rank folds its own blocks. The ranks' block
    sets are disjoint, their reports sum to the unsharded map's, and their union is the
    unsharded map byte for byte (24 cfg2 frames: two groups)."""
    import torch
    from oracle.bindings import parse_svox1
    from paper_2412_00291_b200 import dist as sdist
    wl = W.make("cfg2", 24)
    scans = [p for p, _ in wl.scans(device=torch.device("cuda", 0))]
    offs = np.zeros(len(scans) + 1, np.uint64)
    offs[1:] = np.cumsum([s.shape[0] for s in scans])
    pts = torch.cat(scans).contiguous()
    poses = [wl.pose(i) for i in range(len(scans))]
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
    icfg = svx.IntegratorConfig()
    full = svx.VoxelStore(cfg, 0)
    want = full.integrate_clouds_device(wl.model, pts.data_ptr(), offs, 3, poses, icfg)
    stores = []
    for r in range(world):
        st = svx.VoxelStore(cfg, 0)
        st.set_shard(r, world)
        stores.append(st)
    reps = sdist.emulate_sharded(stores, wl.model, pts.data_ptr(), offs, 3, poses, icfg)
    for f in range(len(poses)):
        assert sum(reps[r][f].updated_voxels for r in range(world)) == want[f].updated_voxels
        assert sum(reps[r][f].new_blocks for r in range(world)) == want[f].new_blocks
        assert all(reps[r][f].frame == want[f].frame for r in range(world))
    _, kf, tf, _ = parse_svox1(full.save_bytes())
    parts = [parse_svox1(st.save_bytes()) for st in stores]
    assert all(len(p[1]) > 0 for p in parts)
    keys = np.concatenate([p[1] for p in parts])
    tsdf = np.concatenate([p[2] for p in parts])
    order = np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))
    assert len(keys) == len(kf)
    assert np.array_equal(keys[order], kf)
    assert tsdf[order].tobytes() == tf.tobytes()
    for st in stores + [full]:
        st.close()


@pytest.mark.parametrize("how", ["device", "host", "confidence"])
def test_clouds_labels_batch_matches_per_frame(how):
    """svx_integrate_clouds_labels (frame groups with each frame's label pass right after
    its fold) == one integrate_cloud + one integrate_labels batch per frame: same TSDF and
    label reports, same map bytes (cfg3 geometry, 6 cameras, 20 frames = two groups).
    With confidence maps the batch alternates frame by frame."""
    import torch
    wl = W.make("cfg3", 20)
    dev = torch.device("cuda", 0)
    scans = [p for p, _ in wl.scans(device=dev)]
    offs = np.zeros(len(scans) + 1, np.uint64)
    offs[1:] = np.cumsum([s.shape[0] for s in scans])
    pts = torch.cat(scans).contiguous()
    poses = [wl.pose(i) for i in range(len(scans))]
    frame_imgs = [wl.label_images(i, device=dev) for i in range(len(scans))]
    if how == "confidence":
        rng = np.random.default_rng(3)
        for f in frame_imgs:
            for li in f:
                li.confidence = rng.uniform(0.2, 1.0, li.width * li.height).astype(np.float32)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
    icfg, scfg = svx.IntegratorConfig(), svx.SemanticConfig()
    ref = svx.VoxelStore(cfg, 0)
    ti, si = svx.TsdfIntegrator(ref, icfg), svx.SemanticIntegrator(ref, scfg)
    want_t, want_l = [], []
    for i, s in enumerate(scans):
        want_t.append(ti.integrate_cloud(s.cpu().numpy(), poses[i], wl.model))
        want_l += si.integrate_labels_batch(frame_imgs[i])
    st = svx.VoxelStore(cfg, 0)
    if how == "device":
        dimgs = [[svx.LabelImage(li.width, li.height,
                                 torch.from_numpy(np.asarray(li.labels).view(np.int16).copy()).to(dev),
                                 li.fx, li.fy, li.cx, li.cy, li.pose, max_depth=li.max_depth) for li in f]
                 for f in frame_imgs]
        torch.cuda.synchronize()
        got_t, got_l = svx.integrate_clouds_labels(st, wl.model, pts.data_ptr(), offs, 3, poses, icfg, dimgs,
                                                   scfg, points_on_device=True, labels_on_device=True)
    else:
        host = pts.cpu().pin_memory()
        got_t, got_l = svx.integrate_clouds_labels(st, wl.model, host.data_ptr(), offs, 3, poses, icfg,
                                                   frame_imgs, scfg, points_on_device=False)
    assert [(r.frame, r.updated_voxels, r.new_blocks) for r in got_t] == \
        [(r.frame, r.updated_voxels, r.new_blocks) for r in want_t]
    assert [(r.frame, r.updated_voxels) for r in got_l] == [(r.frame, r.updated_voxels) for r in want_l]
    assert sum(r.updated_voxels for r in got_l) > 100000
    assert st.save_bytes() == ref.save_bytes()
    assert np.array_equal(st.take_dirty_blocks(1), ref.take_dirty_blocks(1))
    st.close()
    ref.close()


def test_semantic_eligibility_after_host_writes_and_load(tmp_path):
    """The semantic pass's cached per-voxel pre-tests (W > 0, D >= -tau/2) stay exact
    across TSDF writes from the host (block writes that flip voxels across both tests) and
    an SVOX1 load: GPU and oracle apply the same writes and label images."""
    wl = W.make("tiny", 4)
    g, o = _run_pair(wl, svx.IntegratorConfig(), frames=[0, 1])
    keys = np.asarray(g.block_coords_sorted())[:6]
    rng = np.random.default_rng(7)
    for b in keys:
        b = tuple(int(x) for x in b)
        t, _ = g.read_block(b)
        t = t.copy()
        sel = rng.random(512) < 0.3
        t["weight"][sel] = np.where(rng.random(sel.sum()) < 0.5, 0.0, 2.0).astype(np.float32)
        t["distance"][sel] = rng.uniform(-0.5, 0.5, sel.sum()).astype(np.float32)
        g.write_block(b, t)
        o.write_block(b, t)
    si = svx.SemanticIntegrator(g)
    for li in wl.label_images(2):
        assert si.integrate_labels(li).updated_voxels == o.integrate_labels(li, svx.SemanticConfig()).updated_voxels
    compare_maps(g.save_bytes(), o.save_bytes())
    # round trip through SVOX1, then more TSDF frames and label images on the loaded map
    path = tmp_path / "m.svox"
    g.save(str(path))
    h = svx.VoxelStore.load(str(path), 0)
    ti, sh = svx.TsdfIntegrator(h, svx.IntegratorConfig()), svx.SemanticIntegrator(h)
    oi = o
    for p, i in wl.scans(frames=[2, 3]):
        p = p.numpy()
        ti.integrate_cloud(p, wl.pose(i), wl.model)
        d, hh, n, v, _ = ob.OracleMap.project(wl.model, p, wl.pose(i))
        oi.integrate(wl.model, d, n, v, wl.pose(i), svx.IntegratorConfig())
        for li in wl.label_images(i):
            assert sh.integrate_labels(li).updated_voxels == \
                oi.integrate_labels(li, svx.SemanticConfig()).updated_voxels
    compare_maps(h.save_bytes(), oi.save_bytes())
