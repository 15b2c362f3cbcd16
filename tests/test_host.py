"""CPU: workload generator sanity and the multi-process (gloo, world 2) key
sharding logic used by bench.py's multi-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2412_00291_b200 as svx
from paper_2412_00291_b200 import workload as W


def test_workload_scan_shape_and_range():
    wl = W.make("tiny", 2)
    scans = list(wl.scans())
    assert len(scans) == 2
    for p, i in scans:
        assert p.dtype == torch.float32 and p.shape[1] == 3
        r = p.double().norm(dim=1)
        assert float(r.min()) >= wl.model.min_range
        assert 0.5 * wl.model.width * wl.model.height_px < p.shape[0] <= wl.model.width * wl.model.height_px


def test_workload_points_sit_on_pixel_centres():
    # one return per pixel-centre ray (synthetic.cpp:113-139): projecting the
    # points back hits distinct pixels far from pixel boundaries
    wl = W.make("tiny", 1)
    p, _ = next(iter(wl.scans()))
    p = p.double().numpy()
    az = np.arctan2(p[:, 1], p[:, 0])
    uf = (np.pi - az) / wl.model.delta_phi
    frac = uf - np.floor(uf)
    assert np.all(np.abs(frac - 0.5) < 0.01)


def test_workload_configs_exist():
    for name in ("cfg1", "cfg2", "cfg3", "cfg5-320"):
        wl = W.make(name, 2)
        assert len(wl.poses) == 2 and wl.num_labels == 20
    assert W.make("cfg2", 3).model.width == 1024 and W.make("cfg2", 3).model.height_px == 128
    assert W.make("cfg3", 1).voxel_size == 0.05 and len(W.make("cfg3", 1).cams) == 6


def test_label_images_render():
    wl = W.make("tiny", 1)
    (li,) = wl.label_images(0)
    assert li.labels.shape == (li.height, li.width) and li.labels.dtype == np.uint16
    assert li.labels.max() < 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0 is the ingest: it broadcasts the scan (bench.py's multi-GPU path)
    wl = W.make("tiny", 1)
    if rank == 0:
        p, _ = next(iter(wl.scans()))
        n = torch.tensor([p.shape[0]])
    else:
        n = torch.tensor([0])
    dist.broadcast(n, 0)
    buf = p if rank == 0 else torch.empty((int(n), 3), dtype=torch.float32)
    dist.broadcast(buf, 0)
    # every rank sees the same block set and keeps only the blocks it owns
    rng = np.random.default_rng(11)
    keys = rng.integers(-3000, 3000, size=(5000, 3))
    mine = [tuple(k) for k in keys if svx.block_owner(k, world) == rank]
    out = [None] * world
    dist.all_gather_object(out, (mine, float(buf.sum())))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_key_sharding_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    shards = [set(o[0]) for o in out]
    assert shards[0].isdisjoint(shards[1])
    rng = np.random.default_rng(11)
    keys = {tuple(k) for k in rng.integers(-3000, 3000, size=(5000, 3))}
    assert shards[0] | shards[1] == keys
    assert out[0][1] == out[1][1]  # both ranks received the identical scan


def _exchange_worker(rank, world, port, q):
    """dist.exchange (the all-to-all of the multi-GPU data plane) with gloo on the CPU:
    16-byte entries packed by destination; each rank must receive exactly the entries
    addressed to it, in source-rank order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_00291_b200 import dist as sdist
    rng = np.random.default_rng(100 + rank)
    # visit entries of random blocks: (key lo, key hi, src << 16 | seq, dest), routed by owner
    keys = rng.integers(-3000, 3000, size=(int(rng.integers(0, 400)), 3))
    dests = np.array([svx.block_owner(k, world) for k in keys], np.int64)
    order = np.argsort(dests, kind="stable")
    ent = np.zeros((len(keys), 4), np.uint32)
    ent[:, 0] = keys[order, 0].astype(np.uint32)
    ent[:, 1] = keys[order, 1].astype(np.uint32)
    ent[:, 2] = (rank << 16) | np.arange(len(keys), dtype=np.uint32)
    ent[:, 3] = dests[order].astype(np.uint32)
    counts = np.bincount(dests, minlength=world)
    meta = np.zeros((world, 17), np.int64)
    meta[:, 0] = counts
    meta[:, 1] = rank * 1000 + np.arange(world)  # per-frame voxel bits ride along
    send = torch.from_numpy(ent.view(np.uint8).reshape(-1).copy())
    recv, rmeta = sdist.exchange(send, meta)
    got = recv.numpy().view(np.uint32).reshape(-1, 4)
    assert np.array_equal(rmeta[:, 1], np.arange(world) * 1000 + rank)
    out = [None] * world
    dist.all_gather_object(out, (ent, got))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_exchange_all_to_all_gloo():
    for world in (2, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        out = q.get(timeout=240)
        for p in procs:
            p.join(timeout=60)
        sent = [o[0] for o in out]
        for d in range(world):
            got = out[d][1]
            want = np.concatenate([s[s[:, 3] == d] for s in sent]) if sent else np.zeros((0, 4), np.uint32)
            assert np.array_equal(got, want), (world, d)
            assert np.all(got[:, 3] == d)


def test_integrators_mirror_the_reference_methods():
    # both integrators expose the reference's take_dirty_blocks (tsdf_integrator.hpp:84,
    # semantic_integrator.hpp:59) plus their integrate entry points
    for cls, names in ((svx.TsdfIntegrator, ("integrate_frame", "take_dirty_blocks")),
                       (svx.SemanticIntegrator, ("integrate_labels", "integrate_labels_batch",
                                                 "take_dirty_blocks"))):
        for n in names:
            assert callable(getattr(cls, n, None)), (cls.__name__, n)


def test_cfg5_trajectory_stays_inside_the_room():
    # the sweep runs 3 passes of up to 64 scans: every pose stays clear of the room's walls
    # (|x|, |y| < 15 m), so no scan starts inside a wall
    wl = W.make("cfg5-80", 400)
    xs = np.array([wl.poses[i][1][0] for i in range(400)])
    ys = np.array([wl.poses[i][1][1] for i in range(400)])
    assert xs.min() >= -6.0 and xs.max() <= 10.0 and np.abs(ys).max() < 15.0
    # the first scans are the ones the parity tests use
    assert tuple(wl.poses[0][1][:2]) == (-6.0, 0.0) and tuple(wl.poses[1][1][:2]) == (-5.75, 0.0)
