#!/usr/bin/env python
"""Benchmark: points integrated/sec on BASELINE.json configs[1] (cfg2).

cfg2 = synthetic 128-beam LiDAR (1024 x 128, +-22.5 deg, OS1-128 geometry),
0.1 m voxels, tau = 0.5 m, 20 classes, 1000 scans along a 500 m street canyon.
One STEP = one pass of the hot path (project_cloud + compute_normal_image +
TsdfIntegrator::integrate_frame, i.e. the per-frame body of cmd_integrate,
proj/tools/semvox_main.cpp:122-124) over `--scans-per-step` consecutive scans
(default 100, so W=3 + K=7 steps = the 1000-scan sequence). Every step consumes
fresh scans (157 MB of points per step > 126 MB L2) on a map that keeps growing
(> 1 GB), so no step is served from L2.

Legs (one JSON line, printed by rank 0):
  value        device-resident scans, svx_integrate_clouds_device, CUDA events on
               the map stream, max over ranks
  e2e          the C-ABI call a user makes (svx_integrate_clouds) with the step's
               points in HOST pinned memory: H2D (overlapped with integration on a copy
               stream) + report D2H inside the timed region
  roofline     dominant kernel group, algorithmic bytes / event time
  cpu_baseline the reference's own code (oracle/_ref/libsemvox_ref.so, built from
               /root/reference) on the host cores, on a bounded sample of cfg2
--impl reference   only the reference CPU arm (rank 0), same metric and config.

Multi-GPU (torchrun): the map is key-sharded (owner = hash(block) mod N); rank 0
holds the scans and broadcasts each step's points with one NCCL call; every rank
integrates the blocks it owns. `value` counts each input point once.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points integrated/sec (and voxel updates/sec) at 1/2/4/8 B200; % HBM roofline"
UNIT = "points/s"
WORKLOAD = ("cfg2: synthetic 128-beam LiDAR (1024x128, +-22.5 deg), 0.1 m voxels, tau 0.5 m, "
            "20 classes, 1000 scans at 0.5 m spacing (street canyon), band-only TSDF "
            "(non-projective, the reference's default)")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons via NVML, sampled between timed steps.

    (A background `nvidia-smi -lms 200` stalls the launch stream for milliseconds
    per poll on these hosts, so sampling is done in-process at step boundaries:
    inside the overall timed region, outside each step's CUDA-event bracket.)"""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, torch_device):
        self.sm, self.mx, self.reasons = [], None, set()
        self.h = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(torch_device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)

    def sample(self):
        if self.h is None:
            return
        try:
            self.sm.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
            bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for b, n in self.REASONS.items():
                if bits & b:
                    self.reasons.add(n)
        except Exception:  # noqa: BLE001
            pass

    def result(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "method": "NVML at step boundaries inside the timed region"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ reference arm

def run_reference(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref/libsemvox_ref.so)."""
    if rank != 0:
        return 0
    nproc = os.cpu_count() or 1
    os.environ["SEMVOX_THREADS"] = str(nproc)  # read once by worker_count()
    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import workload as W
    from oracle.bindings import RefMap, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libsemvox_ref.so not built"}))
        return 0
    spp = args.ref_scans_per_step
    n = (args.warmup + args.steps) * spp
    wl = W.make(args.workload, max(n + args.ref_offset, 10))
    frames = list(range(args.ref_offset, args.ref_offset + n))
    scans = {i: p.numpy() for p, i in wl.scans(device="cpu", frames=frames)}
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 22)
    icfg = svx.IntegratorConfig()
    ref = RefMap(cfg)
    pts = wall = upd = 0.0
    step_ms = []
    for s in range(args.warmup + args.steps):
        sp = sw = su = 0.0
        for i in frames[s * spp:(s + 1) * spp]:
            rep, ms = ref.integrate_cloud(wl.model, scans[i], wl.pose(i), icfg)
            sp += len(scans[i])
            sw += ms
            su += rep.updated_voxels
        if s >= args.warmup:
            pts += sp
            wall += sw
            upd += su
            step_ms.append(sw)
    value = pts / (wall / 1e3)
    sample = (f"{args.steps} steps x {spp} scans of {args.workload} (frames "
              f"{frames[args.warmup * spp]}..{frames[-1]} after {args.warmup * spp} warm-up "
              f"scans), project_cloud + compute_normal_image + integrate_frame, "
              f"SEMVOX_THREADS={nproc}")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": WORKLOAD, "scans_per_step": spp, "parallelism": "cpu threads"},
           "voxel_updates_per_s": upd / (wall / 1e3),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def cpu_baseline(args, wl, scans_host):
    """Reference CPU path on the box's host cores on a bounded sample (rank 0, N=1)."""
    nproc = os.cpu_count() or 1
    os.environ["SEMVOX_THREADS"] = str(nproc)
    import paper_2412_00291_b200 as svx
    from oracle.bindings import RefMap, ref_available
    if not ref_available():
        return {"value": None, "unit": UNIT, "cores": nproc, "kind": "reference",
                "sample": "unavailable: oracle/_ref/libsemvox_ref.so not built"}
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 22)
    ref = RefMap(cfg)
    icfg = svx.IntegratorConfig()
    keys = sorted(scans_host)
    pts = wall = 0.0
    used = []
    t_start = time.time()
    for j, i in enumerate(keys):
        rep, ms = ref.integrate_cloud(wl.model, scans_host[i], wl.pose(i), icfg)
        if j == 0:
            continue  # first frame on an empty map: warm start, not timed
        pts += len(scans_host[i])
        wall += ms
        used.append(i)
        if time.time() - t_start > args.cpu_seconds or len(used) >= args.cpu_max_scans:
            break
    return {"value": pts / (wall / 1e3), "unit": UNIT, "cores": nproc, "kind": "reference",
            "sample": (f"{len(used)} consecutive {args.workload} scans (frames {used[0]}..{used[-1]}, "
                       f"{int(pts)} points, {wall / 1e3:.1f} s) after 1 untimed warm-start scan, "
                       f"project_cloud + compute_normal_image + integrate_frame, reference's own "
                       f"code at -O3, SEMVOX_THREADS={nproc}")}


# ------------------------------------------------------------------ GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--scans-per-step", type=int, default=100)
    ap.add_argument("--ref-scans-per-step", type=int, default=2)
    ap.add_argument("--ref-offset", type=int, default=300)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--cpu-max-scans", type=int, default=40)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-json", default="")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import workload as W

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    spp = args.scans_per_step
    n_frames = (args.warmup + args.steps) * spp
    wl = W.make(args.workload, n_frames)
    if wl.scene is not None and n_frames * 0.5 + 60 > 560:
        wl.scene = W.street_canyon(length=n_frames * 0.5 + 60)
    dev = torch.device("cuda", local)

    # scans: generated on the GPU (rank 0 only when sharded: it is the ingest GPU)
    counts, chunks = [], []
    if rank == 0:
        for p, i in wl.scans(device=dev):
            chunks.append(p)
            counts.append(p.shape[0])
    if world > 1:
        ct = torch.tensor(counts if rank == 0 else [0] * n_frames, dtype=torch.int64, device=dev)
        dist.broadcast(ct, 0)
        counts = ct.cpu().tolist()
    offsets = np.zeros(n_frames + 1, np.uint64)
    offsets[1:] = np.cumsum(counts)
    if rank == 0:
        pts_all = torch.cat(chunks).contiguous()
        del chunks
    else:
        pts_all = torch.empty((int(offsets[-1]), 3), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
    icfg = svx.IntegratorConfig()
    poses = [wl.pose(i) for i in range(n_frames)]

    def make_store():
        st = svx.VoxelStore(cfg, device=local)
        st.set_shard(rank, world)
        # diagnostic: one rank's share of an N-way key shard on a single GPU
        # (SVX_SIM_SHARD="r,N"), for per-rank cost estimates without N GPUs
        sim = os.environ.get("SVX_SIM_SHARD")
        if sim and world == 1:
            st.set_shard(*[int(x) for x in sim.split(",")])
        return st

    def run_leg(store, host_pts=None, clocks=None):
        """Returns (per-step ms (max over ranks), points, updates, launches, profile)."""
        ext = torch.cuda.ExternalStream(store.stream_ptr(), device=dev)
        step_ms, pts_t, upd_t = [], 0, 0
        launches0 = None
        warm_prof = None
        for s in range(args.warmup + args.steps):
            if s == 0:
                store.profile_enable(True)  # all kernel groups during warm-up
            if s == args.warmup:
                # time only the dominant group inside the timed region (2 events/frame)
                warm_prof = store.profile_read().as_dict()
                dom = max(warm_prof["ms"], key=warm_prof["ms"].get) if warm_prof["ms"] else "fold"
                store.profile_enable(1 << svx.K_NAMES.index(dom))
                launches0 = svx.kernel_launches()
                if clocks:
                    clocks.sample()
            f0, f1 = s * spp, (s + 1) * spp
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            upd = 0
            a, b = int(offsets[f0]), int(offsets[f1])
            rel = offsets[f0:f1 + 1] - offsets[f0]
            if world > 1:
                # rank 0 holds the scans (host or HBM); one NCCL broadcast of the step's
                # points, then every rank integrates the blocks it owns
                if host_pts is not None and rank == 0:
                    pts_all[a:b].copy_(host_pts[a:b], non_blocking=True)
                dist.broadcast(pts_all[a:b], 0)
                torch.cuda.current_stream().synchronize()
            if host_pts is not None and world == 1:
                reps = store.integrate_clouds_host(wl.model, host_pts.data_ptr() + a * 12, rel, 3,
                                                   poses[f0:f1], icfg)
            else:
                reps = store.integrate_clouds_device(wl.model, pts_all.data_ptr() + a * 12, rel, 3,
                                                     poses[f0:f1], icfg)
            upd = sum(r.updated_voxels for r in reps)
            e1.record(ext)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            if clocks and s >= args.warmup:
                clocks.sample()
            if world > 1:
                t = torch.tensor([ms, float(upd)], dtype=torch.float64, device=dev)
                tm = t.clone()
                dist.all_reduce(tm[:1], op=dist.ReduceOp.MAX)
                dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
                ms, upd = float(tm[0]), float(t[1])
            if s >= args.warmup:
                step_ms.append(ms)
                pts_t += int(offsets[f1] - offsets[f0])
                upd_t += upd
        launches = svx.kernel_launches() - launches0
        prof = store.profile_read()
        return step_ms, pts_t, upd_t, launches, prof, warm_prof

    # ---- leg 1: device-resident scans
    store = make_store()
    clocks = ClockSampler(dev) if rank == 0 else None
    step_ms, pts_t, upd_t, launches, prof, warm_prof = run_leg(store, clocks=clocks)
    clk = clocks.result() if clocks else None
    total_s = sum(step_ms) / 1e3
    value = pts_t / total_s
    pd = prof.as_dict()
    blocks_final = store.block_count()
    store.close()

    # ---- roofline: algorithmic bytes per kernel group
    peak, peak_src = peaks()
    # compulsory traffic per kernel group (per-scan intermediates excluded, L2-resident)
    alg = {
        "project": 12.0 * prof.points,                   # f32 xyz in
        # hash key + value + touched list per touched block, zero-fill of new blocks,
        # touched-voxel list entry (8 B) per updated voxel
        "raycast": 16.0 * prof.touched_blocks + 10240.0 * prof.new_blocks + 8.0 * prof.updated_voxels,
        "fold": 40.0 * prof.updated_voxels,              # voxel read + write (20 B each)
        "fallback": 0.0,                                 # counted in fold's updated voxels
    }
    ms_k = {k: v for k, v in pd["ms"].items()}
    dom = max(ms_k, key=ms_k.get) if ms_k else "fold"
    dom_ms = ms_k.get(dom, 0.0)
    dom_launches = pd["launches"].get(dom, 1)
    achieved = (alg.get(dom, 0.0) / (dom_ms / 1e3) / 1e9) if dom_ms else 0.0
    B_total = sum(alg.values())
    # measured DRAM traffic per launch of the dominant kernel (ncu --set full capture of
    # this build, committed as profiles/ncu_frame_kernels.json by scripts/ncu_summary.py)
    traffic, traffic_src = None, None
    kmap = {"raycast": ["k_raycast_band"], "fold": ["k_fold"], "fallback": ["k_fb_fold"],
            "project": ["k_project_points<float>", "k_finish_pixels<float>"]}
    try:
        nk = json.load(open(os.path.join(ROOT, "profiles", "ncu_frame_kernels.json")))
        traffic = sum(nk["kernels"][k]["dram_bytes_per_launch"] for k in kmap[dom])
        traffic_src = "profiles/ncu_frame_kernels.json (" + nk["report"] + ")"
    except Exception:  # noqa: BLE001
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": dom,
                "kernel_ms_per_launch": dom_ms / max(dom_launches, 1),
                "alg_bytes_per_launch": alg.get(dom, 0.0) / max(dom_launches, 1),
                "peak_source": peak_src,
                "pipeline": {"alg_bytes_per_frame": B_total / max(prof.frames, 1),
                             "achieved": B_total / total_s / 1e9,
                             "frac": B_total / total_s / 1e9 / peak},
                "timed_kernel_ms": ms_k,
                "warmup_kernel_us_per_frame": {
                    k: 1e3 * v / max(warm_prof["frames"], 1) for k, v in warm_prof["ms"].items()}
                if warm_prof else None}

    # ---- leg 2: end to end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        host_pts = None
        if rank == 0:
            host_pts = pts_all.cpu().pin_memory()
        store = make_store()
        s2, p2, u2, _, prof2, _ = run_leg(store, host_pts=host_pts if rank == 0 else torch.empty(0))
        store.close()
        e2e = {"value": p2 / (sum(s2) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(12 * p2 / args.steps),
               "d2h_bytes_per_step": int(32 * spp + 4 * 32),  # frame reports + counters
               "api": "svx_integrate_clouds (points in pinned host memory, staged H2D overlapped "
                      "with integration)"}

    # ---- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        off = min(args.ref_offset, n_frames // 2)
        sample = list(range(off, min(off + args.cpu_max_scans + 1, n_frames)))
        scans_host = {i: pts_all[int(offsets[i]):int(offsets[i + 1])].cpu().numpy() for i in sample}
        cpu = cpu_baseline(args, wl, scans_host)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": float(np.mean(step_ms)), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic",
               "config": {"workload": WORKLOAD, "scans_per_step": spp,
                          "points_per_step": pts_t / args.steps,
                          "l2": "inputs > L2: ~157 MB of fresh scans per step; map state > 1 GB",
                          "parallelism": f"key-sharded map x{world}" if world > 1 else "1 GPU",
                          "map_blocks": blocks_final},
               "voxel_updates_per_s": upd_t / total_s,
               "rays_per_s": prof.rays / total_s,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(launches), "clocks": clk, "profile": pd}
        print(json.dumps(out))
        if args.profile_json:
            json.dump(out, open(args.profile_json, "w"), indent=1)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
