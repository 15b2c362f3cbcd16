#!/usr/bin/env python
"""Benchmark: points integrated/sec (BASELINE.json metric) on the BASELINE.json configs.

Default (what the driver runs): cfg2 = BASELINE.json configs[1], synthetic 128-beam LiDAR
(1024 x 128, +-22.5 deg, OS1-128 geometry), 0.1 m voxels, tau = 0.5 m, 20 classes, a
street canyon. One STEP = one pass of the hot path (project_cloud + compute_normal_image +
TsdfIntegrator::integrate_frame: the per-frame body of cmd_integrate,
proj/tools/semvox_main.cpp:122-124) over `--scans-per-step` consecutive scans (default 100;
W = 3 + K = 7 steps = a 1000-scan sequence). Every step consumes fresh scans (150 MB of
points > 126 MB L2) on a map that keeps growing (> 1 GB), so no step is served from L2.

Legs (one JSON line, printed by rank 0):
  value        scans resident in HBM, svx_integrate_clouds_device (frame groups of 16),
               CUDA events on the map stream, max over ranks
  e2e          the C-ABI call a user makes (svx_integrate_clouds) with the step's points in
               pinned HOST memory: H2D (overlapped with integration on a copy stream) +
               report D2H inside the timed region
  roofline     dominant kernel group: SURVEY.md 8(d) algorithmic bytes / its event time
  cpu_baseline the reference's own code (oracle/_ref/libsemvox_ref.so, built from
               /root/reference) on the host cores, on a bounded sample of the workload
  parity       after timing: the same sample of frames through a fresh GPU map (the timed
               entry point) and through the reference's own code: SVOX1 images compared
--impl reference   only the reference CPU arm (rank 0), same metric and config.

Other workloads (builder runs; same contract line):
  --workload cfg1 | cfg3 | cfg4 | cfg5-<W>   (cfg3 adds 6 x 1280x720 label images per frame)
  --carve      the occupancy extension with free-space carving (configs[1] "with ray
               free-space carving"; parity against the project's own C oracle: unpinned)
  --sweep      cfg5: W in 80..16384 at 128 rows, geometry and geometry + semantics, one
               JSON line per point, then a summary line

Multi-GPU (--gpus N; relaunches itself under torch.distributed.run when WORLD_SIZE is
unset): the map is key-sharded (owner = hash(block) mod N); see DESIGN.md
section 6 for the data plane. `value` counts each input point once.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points integrated/sec (and voxel updates/sec) at 1/2/4/8 B200; % HBM roofline"
UNIT = "points/s"
DESC = {
    "cfg1": "cfg1: synthetic 64-beam LiDAR (2048x64, +2/-24.8 deg), 0.2 m voxels, tau 1.0 m, 20 classes",
    "cfg2": "cfg2: synthetic 128-beam LiDAR (1024x128, +-22.5 deg), 0.1 m voxels, tau 0.5 m, 20 classes",
    "cfg3": "cfg3: cfg2 LiDAR at 0.05 m voxels, tau 0.25 m + 6 x 1280x720 semantic label images per frame, "
            "20 classes",
    "cfg4": "cfg4: city scale, 128-beam LiDAR (1024x128), 0.1 m voxels, tau 0.5 m, 2 km trajectory",
    "cfg5": "cfg5: points-per-scan sweep, spinning(W, 128, +-22.5 deg) in a closed room, 0.1 m voxels",
}


def describe(workload, frames, spacing=0.5):
    base = DESC.get(workload.split("-")[0], workload)
    if workload.startswith("cfg5-"):
        base += f", W={workload.split('-')[1]}"
    return (f"{base}; {frames} consecutive scans at {spacing} m spacing, band-only TSDF (non-projective, "
            f"the reference's default)")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return "unknown"


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


def relaunch_if_needed(args):
    """`--gpus N` without a launcher: re-exec under torch.distributed.run with N ranks."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus and args.gpus != 1:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


def sha16(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


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
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsemvox_ref.so not built"}))
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
              f"SEMVOX_THREADS={nproc}, CPU: {cpu_model()}")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": describe(args.workload, n), "scans_per_step": spp,
                      "parallelism": "cpu threads"},
           "voxel_updates_per_s": upd / (wall / 1e3),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def cpu_and_parity(args, wl, scans_host, integrate_gpu):
    """Reference CPU path on the host cores on a bounded sample (rank 0, N = 1), and the
    parity check of the benchmarked entry point on the same sample: the sample's frames
    through a fresh GPU map (`integrate_gpu(store, frames)`, the timed call) and through
    the reference's own code, both from an empty map; SVOX1 images and reports compared."""
    nproc = os.cpu_count() or 1
    os.environ["SEMVOX_THREADS"] = str(nproc)
    import paper_2412_00291_b200 as svx
    from oracle.bindings import RefMap, ref_available
    if not ref_available():
        return ({"value": None, "unit": UNIT, "cores": nproc, "kind": "reference",
                 "sample": "unavailable: oracle/_ref/libsemvox_ref.so not built"},
                {"checked": False, "why": "oracle/_ref not built"})
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 22)
    ref = RefMap(cfg)
    icfg = svx.IntegratorConfig()
    keys = sorted(scans_host)
    pts = wall = 0.0
    used, ref_reps = [], []
    t_start = time.time()
    for j, i in enumerate(keys):
        rep, ms = ref.integrate_cloud(wl.model, scans_host[i], wl.pose(i), icfg)
        ref_reps.append((rep.updated_voxels, rep.new_blocks))
        if j == 0:
            continue  # first frame on an empty map: warm start, not timed
        pts += len(scans_host[i])
        wall += ms
        used.append(i)
        if time.time() - t_start > args.cpu_seconds or len(used) >= args.cpu_max_scans:
            break
    frames = keys[:len(used) + 1]
    cpu = {"value": pts / (wall / 1e3), "unit": UNIT, "cores": nproc, "kind": "reference",
           "sample": (f"{len(used)} consecutive {args.workload} scans (frames {used[0]}..{used[-1]}, "
                      f"{int(pts)} points, {wall / 1e3:.1f} s) after 1 untimed warm-start scan, "
                      f"project_cloud + compute_normal_image + integrate_frame, reference's own "
                      f"code at -O3, SEMVOX_THREADS={nproc}"),
           "cpu_model": cpu_model()}
    g = svx.VoxelStore(svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21), 0)
    reps = integrate_gpu(g, frames)
    a, b = g.save_bytes(), ref.save_bytes()
    par = {"frames": len(frames), "first_frame": frames[0],
           "entry_point": "svx_integrate_clouds_device (the timed call), one batch",
           "reports_equal": [(r.updated_voxels, r.new_blocks) for r in reps] == ref_reps[:len(frames)],
           "svox1_equal": a == b, "svox1_sha256_16": sha16(a), "reference_sha256_16": sha16(b),
           "blocks": g.block_count()}
    g.close()
    return cpu, par


# ------------------------------------------------------------------ GPU arm: TSDF streams

def run_tsdf(args, world, rank, local):
    """cfg1 / cfg2 / cfg4 / cfg5-<W>: a stream of scans, TSDF only."""
    import torch
    import torch.distributed as dist

    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import dist as sdist
    from paper_2412_00291_b200 import workload as W

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    spp = args.scans_per_step
    n_frames = (args.warmup + args.steps) * spp
    wl = W.make(args.workload, n_frames)
    if args.workload in ("cfg1", "cfg2") and n_frames * (0.5 if args.workload == "cfg2" else 1.0) + 60 > 560:
        wl.scene = W.street_canyon(length=n_frames * (0.5 if args.workload == "cfg2" else 1.0) + 60)
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

    max_blocks = (1 << 22) if args.workload == "cfg4" else (1 << 21)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, max_blocks)
    icfg = svx.IntegratorConfig()
    poses = [wl.pose(i) for i in range(n_frames)]

    def make_store():
        st = svx.VoxelStore(cfg, device=local)
        # the pool mapped before the timed steps (cfg4's city map reaches ~944k blocks)
        st.reserve((1 << 20) if args.workload == "cfg4" else (1 << 17))
        if world > 1:
            st.set_shard(rank, world)
        return st

    def run_leg(store, host_pts=None, clocks=None):
        """Returns (per-step ms (max over ranks), points, updates, launches, profile)."""
        ext = torch.cuda.ExternalStream(store.stream_ptr(), device=dev)
        step_ms, pts_t, upd_t = [], 0, 0
        launches0 = None
        warm_prof = None
        for s in range(args.warmup + args.steps):
            if s == max(args.warmup - 1, 0):
                store.profile_read()  # (discarded: one-time buffer sizing of the first steps)
                store.profile_enable(True)  # all kernel groups during the last warm-up step
            if s == args.warmup:
                # time only the dominant group inside the timed region (2 events per group);
                # the groups with SURVEY 8(d) bytes (the fallback's voxels count in the fold's)
                warm_prof = store.profile_read().as_dict()
                cand = {k: v for k, v in warm_prof["ms"].items() if k in ("project", "raycast", "fold")}
                dom = max(cand, key=cand.get) if cand else "fold"
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
            a, b = int(offsets[f0]), int(offsets[f1])
            rel = offsets[f0:f1 + 1] - offsets[f0]
            if world > 1:
                # rank 0 holds the scans (host or HBM); one NCCL broadcast of the step's
                # points, then every rank integrates the blocks it owns
                if host_pts is not None and rank == 0:
                    pts_all[a:b].copy_(host_pts[a:b], non_blocking=True)
                dist.broadcast(pts_all[a:b], 0)
                torch.cuda.current_stream().synchronize()
            if world > 1:
                # exchange mode: each rank casts its share of the rays, one all-to-all of
                # the visits per frame group, each rank folds the blocks it owns
                reps = sdist.integrate_sharded(store, wl.model, pts_all.data_ptr() + a * 12, rel, 3,
                                               poses[f0:f1], icfg)
            elif host_pts is not None:
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

    # ---- roofline: compulsory bytes per kernel group; per-frame
    # intermediates (pixel cache, visit masks, voxel lists, fallback records) excluded
    peak, peak_src = peaks()
    alg = {
        "project": 12.0 * prof.points,                                    # f32 xyz in
        "raycast": 16.0 * prof.touched_blocks + 10240.0 * prof.new_blocks,  # hash + zero-fill
        "fold": 40.0 * prof.updated_voxels,                               # voxel read + write
        "fallback": 0.0,                                                  # in fold's voxels
    }
    intermediates = {"voxel_lists": 4.0 * prof.updated_voxels, "pixel_cache": 48.0 * prof.rays}
    ms_k = dict(pd["ms"])
    dom = max(ms_k, key=ms_k.get) if ms_k else "fold"
    dom_ms = ms_k.get(dom, 0.0)
    # launches of the timed group: k_fold runs once per frame (a profiling mark spans a
    # frame group), the other kernels once per group
    dom_launches = max(prof.frames if dom == "fold" else pd["launches"].get(dom, 1), 1)
    achieved = (alg.get(dom, 0.0) / (dom_ms / 1e3) / 1e9) if dom_ms else 0.0
    B_total = sum(alg.values())
    traffic, traffic_src = None, None
    kmap = {"raycast": ["k_band"], "fold": ["k_fold"], "fallback": ["k_fb_runs"],
            "project": ["k_project_points<float>", "k_finish_pixels<float>"]}
    try:
        nk = json.load(open(os.path.join(ROOT, "profiles", "ncu_frame_kernels.json")))
        per_frame = {k: nk["kernels"][k]["dram_bytes_per_launch"] / nk["kernels"][k].get("frames_per_launch", 1)
                     for k in kmap[dom] if k in nk["kernels"]}
        if per_frame:
            traffic = sum(per_frame.values()) * prof.frames / dom_launches
            traffic_src = ("profiles/ncu_frame_kernels.json (" + nk["report"] + "), DRAM bytes per frame x "
                           "frames per launch")
    except Exception:  # noqa: BLE001
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": dom, "kernel_ms_per_launch": dom_ms / dom_launches,
                "alg_bytes_per_launch": alg.get(dom, 0.0) / dom_launches,
                "frames_per_launch": prof.frames / dom_launches,
                "alg_bytes_formula": "SURVEY 8(d): 12 N_in + 16 B_touched + 10240 B_new + 40 U_t",
                "peak_source": peak_src,
                "pipeline": {"alg_bytes_per_frame": B_total / max(prof.frames, 1),
                             "achieved": B_total / total_s / 1e9,
                             "frac": B_total / total_s / 1e9 / peak},
                "intermediate_bytes_per_frame": {k: v / max(prof.frames, 1) for k, v in intermediates.items()},
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

    # ---- CPU baseline + parity (rank 0, N=1)
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        off = min(args.ref_offset, n_frames // 2)
        sample = list(range(off, min(off + args.cpu_max_scans + 1, n_frames)))
        scans_host = {i: pts_all[int(offsets[i]):int(offsets[i + 1])].cpu().numpy() for i in sample}

        def gpu_frames(st, frames):
            f0, f1 = frames[0], frames[-1] + 1
            rel = offsets[f0:f1 + 1] - offsets[f0]
            return st.integrate_clouds_device(wl.model, pts_all.data_ptr() + int(offsets[f0]) * 12, rel, 3,
                                              poses[f0:f1], icfg)
        cpu, parity = cpu_and_parity(args, wl, scans_host, gpu_frames)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": float(np.mean(step_ms)), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic",
               "config": {"workload": describe(args.workload, n_frames), "frames_total": n_frames,
                          "scans_per_step": spp, "points_per_step": pts_t / args.steps,
                          "l2": "inputs > L2: ~150 MB of fresh scans per step; map state > 1 GB",
                          "parallelism": (f"key-sharded map x{world}, ray tiles round robin, one NCCL "
                                          f"all-to-all of visits per 16-frame group") if world > 1 else "1 GPU",
                          "map_blocks": blocks_final},
               "voxel_updates_per_s": upd_t / total_s,
               "rays_per_s": prof.rays / total_s,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
               "gpu_launches": int(launches), "clocks": clk, "profile": pd}
        if args.workload == "cfg4":  # A4-style scale independence: late vs early step cost
            out["scale_independence"] = {"first_step_ms": step_ms[0], "last_step_ms": step_ms[-1],
                                         "late_over_early": step_ms[-1] / step_ms[0]}
        print(json.dumps(out))
        if args.profile_json:
            json.dump(out, open(args.profile_json, "w"), indent=1)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ GPU arm: cfg3 (TSDF + labels)

def run_cfg3(args, world, rank, local):
    """cfg3: per frame one TSDF frame + its 6 label images (svx_integrate_labels_batch)."""
    import torch

    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import workload as W
    if world > 1:
        raise SystemExit("bench.py --workload cfg3 runs on one GPU (the semantic pass is per shard)")
    torch.cuda.set_device(local)
    spp = args.scans_per_step
    n_frames = (args.warmup + args.steps) * spp
    wl = W.make("cfg3", n_frames)
    dev = torch.device("cuda", local)
    scans = {i: p.cpu().numpy() for p, i in wl.scans(device=dev)}
    labels = {i: wl.label_images(i, device=dev) for i in range(n_frames)}
    offs = np.zeros(n_frames + 1, np.uint64)
    offs[1:] = np.cumsum([len(scans[i]) for i in range(n_frames)])
    flat = np.ascontiguousarray(np.concatenate([scans[i] for i in range(n_frames)]).astype(np.float32))
    pts_dev = torch.from_numpy(flat).to(dev)
    pts_host = torch.from_numpy(flat).pin_memory()

    def dev_images(i):
        return [svx.LabelImage(li.width, li.height,
                               torch.from_numpy(np.asarray(li.labels).view(np.int16).copy()).to(dev),
                               li.fx, li.fy, li.cx, li.cy, li.pose, max_depth=li.max_depth) for li in labels[i]]

    def pinned_images(i):
        out = []
        for li in labels[i]:
            t = torch.from_numpy(np.asarray(li.labels).view(np.int16).copy()).pin_memory()
            out.append(svx.LabelImage(li.width, li.height, t.numpy().view(np.uint16), li.fx, li.fy, li.cx,
                                      li.cy, li.pose, max_depth=li.max_depth))
        return out

    lab_dev = {i: dev_images(i) for i in range(n_frames)}
    lab_pin = {i: pinned_images(i) for i in range(n_frames)}
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
    icfg = svx.IntegratorConfig()
    torch.cuda.synchronize()

    scfg = svx.SemanticConfig()

    def leg(device_resident, clocks=None):
        st = svx.VoxelStore(cfg, local)
        if not os.environ.get("SVX_BENCH_NO_RESERVE"):
            st.reserve(1 << 17, 1 << 17)  # TSDF pool + semantic layers mapped before the timed steps
        ext = torch.cuda.ExternalStream(st.stream_ptr(), device=dev)
        step_ms, pts, upd = [], 0, 0
        launches0 = 0
        for s in range(args.warmup + args.steps):
            if s == 0:
                st.profile_enable(True)
            if s == args.warmup:
                launches0 = svx.kernel_launches()
                warm = st.profile_read().as_dict()
                st.profile_enable(True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            # the whole step in one call: TSDF frame groups, each frame's 6 label images
            # right after its fold (svx_integrate_clouds_labels)
            f0, f1 = s * spp, (s + 1) * spp
            rel = offs[f0:f1 + 1] - offs[f0]
            src = pts_dev if device_resident else pts_host
            tr, lr = svx.integrate_clouds_labels(
                st, wl.model, src.data_ptr() + 12 * int(offs[f0]), rel, 3, [wl.pose(i) for i in range(f0, f1)],
                icfg, [lab_dev[i] if device_resident else lab_pin[i] for i in range(f0, f1)], scfg,
                points_on_device=device_resident, labels_on_device=device_resident)
            su = sum(r.updated_voxels for r in tr) + sum(r.updated_voxels for r in lr)
            sp = int(offs[f1] - offs[f0])
            e1.record(ext)
            e1.synchronize()
            if clocks and s >= args.warmup:
                clocks.sample()
            if s >= args.warmup:
                step_ms.append(e0.elapsed_time(e1))
                pts += sp
                upd += su
        prof = st.profile_read().as_dict()
        launches = svx.kernel_launches() - launches0
        blocks = st.block_count()
        st.close()
        return step_ms, pts, upd, prof, launches, blocks, warm

    clocks = ClockSampler(dev)
    step_ms, pts, upd, prof, launches, blocks, warm = leg(True, clocks)
    total_s = sum(step_ms) / 1e3
    value = pts / total_s
    e2e = None
    if not args.no_e2e:
        s2, p2, _, _, _, _, _ = leg(False)
        e2e = {"value": p2 / (sum(s2) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(12 * p2 / args.steps + spp * sum(2 * li.width * li.height
                                                                           for li in labels[0])),
               "d2h_bytes_per_step": int(spp * 7 * 32),
               "api": "svx_integrate_clouds_labels (pinned host points and label images)"}
    peak, peak_src = peaks()
    nf = max(prof["frames"], 1)
    # SURVEY 8(d) bytes: geometry terms + semantic terms (2 B/label pixel, 8 B per frustum
    # voxel read (C_s ~ candidates x 512), 8K B per updated voxel, 2048K per new layer)
    K = wl.num_labels
    b_geo = 12.0 * prof["points"] + 16.0 * prof["touched_blocks"] + 10240.0 * prof["new_blocks"] + \
        40.0 * prof["updated_voxels"]
    b_sem = 2.0 * 1280 * 720 * prof["sem_images"] + 8.0 * 512 * prof["sem_candidates"] + \
        8.0 * K * prof["sem_updated"] + 2048.0 * K * prof["sem_new_layers"]
    ms_k = prof["ms"]
    dom = max(ms_k, key=ms_k.get)
    bytes_k = {"fold": 40.0 * prof["updated_voxels"],
               "raycast": 16.0 * prof["touched_blocks"] + 10240.0 * prof["new_blocks"],
               "sem_update": 8.0 * 512 * prof["sem_candidates"] + 8.0 * K * prof["sem_updated"] +
               2048.0 * K * prof["sem_new_layers"] + 2.0 * 1280 * 720 * prof["sem_images"],
               "sem_cull": 8.0 * prof["sem_candidates"], "project": 12.0 * prof["points"], "fallback": 0.0}
    ach = bytes_k.get(dom, 0.0) / (ms_k[dom] / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "kernel": dom, "peak_source": peak_src,
                "kernel_us_per_frame": {k: 1e3 * v / nf for k, v in ms_k.items()},
                "pipeline": {"alg_bytes_per_frame": (b_geo + b_sem) / nf,
                             "achieved": (b_geo + b_sem) / total_s / 1e9,
                             "frac": (b_geo + b_sem) / total_s / 1e9 / peak}}
    cpu = parity = None
    if not args.no_cpu:
        from oracle.bindings import RefMap, ref_available
        if ref_available():
            nproc = os.cpu_count() or 1
            os.environ["SEMVOX_THREADS"] = str(nproc)
            ref = RefMap(cfg)
            g = svx.VoxelStore(cfg, local)
            gi = svx.SemanticIntegrator(g)
            scfg = svx.SemanticConfig()
            wall = cpts = 0.0
            ok = True
            n_cpu = min(args.cfg3_cpu_frames, n_frames)
            for i in range(n_cpu):
                t0 = time.perf_counter()
                rb, _ = ref.integrate_cloud(wl.model, scans[i], wl.pose(i), icfg)
                sb = [ref.integrate_labels(li, scfg).updated_voxels for li in labels[i]]
                dt = time.perf_counter() - t0
                if i >= 1:
                    wall += dt
                    cpts += len(scans[i])
                ra = g.integrate_clouds_device(wl.model, pts_dev.data_ptr() + 12 * int(offs[i]),
                                               offs[i:i + 2] - offs[i], 3, [wl.pose(i)], icfg)[0]
                sa = [x.updated_voxels for x in gi.integrate_labels_batch(lab_dev[i], on_device=True)]
                ok &= (ra.updated_voxels, ra.new_blocks, sa) == (rb.updated_voxels, rb.new_blocks, sb)
            a, b = g.save_bytes(), ref.save_bytes()
            g.close()
            cpu = {"value": cpts / wall, "unit": UNIT, "cores": nproc, "kind": "reference",
                   "sample": f"{n_cpu - 1} cfg3 frames after 1 warm-start frame, integrate_cloud + 6 x "
                             f"integrate_labels, SEMVOX_THREADS={nproc}", "cpu_model": cpu_model()}
            parity = {"frames": n_cpu, "reports_equal": bool(ok), "svox1_equal": a == b,
                      "svox1_sha256_16": sha16(a), "reference_sha256_16": sha16(b)}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": describe("cfg3", n_frames), "frames_total": n_frames, "scans_per_step": spp,
                      "label_images_per_frame": 6, "parallelism": "1 GPU", "map_blocks": blocks},
           "voxel_updates_per_s": upd / total_s, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
           "parity": parity, "gpu_launches": int(launches), "clocks": clocks.result(), "profile": prof}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ GPU arm: carving

def run_carve(args, world, rank, local):
    """configs[1] "with ray free-space carving": the occupancy extension on cfg2 scans."""
    import torch

    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import workload as W
    if world > 1:
        raise SystemExit("bench.py --carve runs on one GPU")
    torch.cuda.set_device(local)
    spp = args.scans_per_step
    n_frames = (args.warmup + args.steps) * spp
    wl = W.make("cfg2", n_frames)
    if n_frames * 0.5 + 60 > 560:
        wl.scene = W.street_canyon(length=n_frames * 0.5 + 60)
    dev = torch.device("cuda", local)
    chunks = [p for p, _ in wl.scans(device=dev)]
    counts = [c.shape[0] for c in chunks]
    offs = np.zeros(n_frames + 1, np.uint64)
    offs[1:] = np.cumsum(counts)
    pts = torch.cat(chunks).contiguous()
    del chunks
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    lab = torch.randint(0, wl.num_labels, (pts.shape[0],), generator=gen, device=dev, dtype=torch.int32).to(torch.int16)
    conf = (0.3 + 0.7 * torch.rand(pts.shape[0], generator=gen, device=dev)).to(torch.float32)
    poses = [wl.pose(i) for i in range(n_frames)]
    ocfg = svx.OccupancyConfig(voxel_size=wl.voxel_size, num_labels=wl.num_labels, max_blocks=1 << 22,
                               max_range=70.0)

    def leg(device_resident, clocks=None):
        occ = svx.OccupancyMap(ocfg)
        occ.reserve(1 << 19, 1 << 17)
        ext = torch.cuda.ExternalStream(occ.stream_ptr(), device=dev)
        hp = hl = hc = None
        if not device_resident:
            hp, hl, hc = pts.cpu().pin_memory(), lab.cpu().pin_memory(), conf.cpu().pin_memory()
        step_ms, n_pts = [], 0
        for s in range(args.warmup + args.steps):
            f0, f1 = s * spp, (s + 1) * spp
            a = int(offs[f0])
            rel = offs[f0:f1 + 1] - offs[f0]
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            if device_resident:
                occ.integrate_batch_device(pts.data_ptr() + 12 * a, rel, 3, poses[f0:f1],
                                           lab.data_ptr() + 2 * a, conf.data_ptr() + 4 * a)
            else:
                occ.integrate_batch_host(hp.data_ptr() + 12 * a, rel, 3, poses[f0:f1],
                                         hl.data_ptr() + 2 * a, hc.data_ptr() + 4 * a)
            e1.record(ext)
            e1.synchronize()
            if clocks and s >= args.warmup:
                clocks.sample()
            if s >= args.warmup:
                step_ms.append(e0.elapsed_time(e1))
                n_pts += int(offs[f1] - offs[f0])
        blocks = occ.block_count()
        occ.close()
        return step_ms, n_pts, blocks

    launches0 = svx.kernel_launches()
    clocks = ClockSampler(dev)
    step_ms, n_pts, blocks = leg(True, clocks)
    launches = svx.kernel_launches() - launches0
    value = n_pts / (sum(step_ms) / 1e3)
    e2e = None
    if not args.no_e2e:
        s2, p2, _ = leg(False)
        e2e = {"value": p2 / (sum(s2) / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(18 * p2 / args.steps),
               "d2h_bytes_per_step": int(spp * 32),
               "api": "svx_occ_integrate_batch (pinned host points, labels, confidences)"}
    cpu = parity = None
    if not args.no_cpu:
        from oracle import bindings as ob
        o = ob.OracleOcc(ocfg)
        g = svx.OccupancyMap(ocfg)
        wall = cp = 0.0
        n = args.carve_cpu_scans
        for i in range(n):
            a, b = int(offs[i]), int(offs[i + 1])
            p_h = pts[a:b].cpu().numpy()
            l_h = lab[a:b].cpu().numpy().view(np.uint16)
            c_h = conf[a:b].cpu().numpy()
            t0 = time.perf_counter()
            o.integrate(p_h, poses[i], l_h, c_h)
            wall += time.perf_counter() - t0
            cp += b - a
            g.integrate(p_h, poses[i], l_h, c_h)
        ga, ob_ = g.save_bytes(), o.save_bytes()
        g.close()
        cpu = {"value": cp / wall, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{n} cfg2 scans with carving to 70 m, the project's own serial C oracle "
                         f"(svx_oracle.c; the reference has no carving code)", "cpu_model": cpu_model()}
        parity = {"frames": n, "socc1_equal": ga == ob_, "pinned": False,
                  "note": "parity unpinned: the reference declines carving (SPEC.md:255); checked "
                          "against the project's own C oracle"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": "cfg2 scans with ray free-space carving (occupancy extension: log-odds, "
                                  f"hit/miss counters, u32 class histograms), max range 70 m; {n_frames} scans",
                      "frames_total": n_frames, "scans_per_step": spp, "parallelism": "1 GPU",
                      "map_blocks": blocks},
           "roofline": None, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
           "gpu_launches": int(launches), "clocks": clocks.result()}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ multi-GPU emulation

def run_emulated(args):
    """The multi-GPU data plane with N ranks emulated on ONE GPU (dist.emulate_sharded: the
    ranks' calls run one after another, the all-to-all is a device copy). Per frame group
    the cost of rank r is its xbegin + xend time; an N-GPU step would take the max over
    ranks plus the all-to-all of the visit entries (estimated at the measured 770 GB/s
    NVLink peer bandwidth, B200_PROFILING.md). Not a measured multi-GPU number: the
    per-rank cost model behind DESIGN.md section 6's scaling estimate."""
    import torch

    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import dist as sdist
    from paper_2412_00291_b200 import workload as W
    dev = torch.device("cuda", 0)
    spp = args.scans_per_step
    n_frames = (args.warmup + args.steps) * spp
    wl = W.make(args.workload, n_frames)
    if args.workload == "cfg2" and n_frames * 0.5 + 60 > 560:
        wl.scene = W.street_canyon(length=n_frames * 0.5 + 60)
    chunks = [p for p, _ in wl.scans(device=dev)]
    offs = np.zeros(n_frames + 1, np.uint64)
    offs[1:] = np.cumsum([c.shape[0] for c in chunks])
    pts = torch.cat(chunks).contiguous()
    del chunks
    poses = [wl.pose(i) for i in range(n_frames)]
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
    icfg = svx.IntegratorConfig()
    out = {"emulated": True, "workload": describe(args.workload, n_frames), "scans_per_step": spp, "ranks": {}}
    for N in args.emulate_ranks:
        stores = []
        for r in range(N):
            st = svx.VoxelStore(cfg, 0)
            st.reserve(1 << 18)  # pool mapped before timing (no background mapping threads meanwhile)
            if N > 1:
                st.set_shard(r, N)
            stores.append(st)
        step_max, step_sum, xbytes, pts_t = [], [], [], 0
        for s in range(args.warmup + args.steps):
            f0, f1 = s * spp, (s + 1) * spp
            rel = offs[f0:f1 + 1] - offs[f0]
            timers = []
            if N > 1:
                sdist.emulate_sharded(stores, wl.model, pts.data_ptr() + int(offs[f0]) * 12, rel, 3, poses[f0:f1],
                                      icfg, timers=timers)
                tmax = sum(max(b + e for b, e in zip(t["xbegin_ms"], t["xend_ms"])) for t in timers)
                if os.environ.get("SVX_EMU_DEBUG"):
                    print(json.dumps({"N": N, "step": s, "groups": [[round(b, 2) for b in t["xbegin_ms"]] +
                                                                  [round(e, 2) for e in t["xend_ms"]] for t in timers]}),
                          file=sys.stderr, flush=True)
                tsum = sum(sum(t["xbegin_ms"]) + sum(t["xend_ms"]) for t in timers)
                ent = sum(sum(t["entries"]) for t in timers)
            else:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                stores[0].integrate_clouds_device(wl.model, pts.data_ptr() + int(offs[f0]) * 12, rel, 3,
                                                  poses[f0:f1], icfg)
                tmax = tsum = (time.perf_counter() - t0) * 1e3
                ent = 0
            if s >= args.warmup:
                step_max.append(tmax)
                step_sum.append(tsum)
                xbytes.append(16 * ent)
                pts_t += int(offs[f1] - offs[f0])
        # all-to-all: each rank sends/receives ~1/N of the entries; time at 770 GB/s per
        # direction per GPU (measured peer copy), per step
        xchg_ms = [b / N / 770e9 * 1e3 for b in xbytes]
        t_step = [a + x for a, x in zip(step_max, xchg_ms)]
        # the median step: a rank's one-time buffer growth (a host synchronisation inside one
        # call) lands in a single step; the mean keeps it for reference
        n_t = len(t_step)
        out["ranks"][N] = {"max_rank_ms_per_step": float(np.median(step_max)),
                           "max_rank_ms_per_step_mean": float(np.mean(step_max)),
                           "all_ranks_ms_per_step": float(np.median(step_sum)),
                           "exchange_bytes_per_step": float(np.mean(xbytes)),
                           "exchange_ms_per_step_est": float(np.mean(xchg_ms)),
                           "points_per_s_est": (pts_t / n_t) / (float(np.median(t_step)) / 1e3),
                           "blocks_per_rank": [st.block_count() for st in stores]}
        for st in stores:
            st.close()
    base = out["ranks"].get(1, {}).get("points_per_s_est")
    if base:
        for N, r in out["ranks"].items():
            r["speedup_vs_1"] = r["points_per_s_est"] / base
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ cfg5 sweep

def run_sweep(args):
    """cfg5: W in 80..16384 (P = 10k..2.1M points per scan), geometry only and geometry +
    one 1280x720 label image per scan; points/s and the SURVEY 8(d) pipeline fraction per
    point of the sweep, so the fixed per-frame cost shows where it dominates."""
    import torch

    import paper_2412_00291_b200 as svx
    from paper_2412_00291_b200 import workload as W
    dev = torch.device("cuda", 0)
    peak, _ = peaks()
    rows = []
    for Wd in args.sweep_widths:
        n = args.sweep_scans
        wl = W.make(f"cfg5-{Wd}", 3 * n + 8)
        wl.cams = [(W._forward_cam(0), np.zeros(3), 1280, 720, 640.0, 640.0, 640.0, 360.0)]
        chunks = [p for p, _ in wl.scans(device=dev)]
        offs = np.zeros(len(chunks) + 1, np.uint64)
        offs[1:] = np.cumsum([c.shape[0] for c in chunks])
        pts = torch.cat(chunks).contiguous()
        poses = [wl.pose(i) for i in range(len(chunks))]
        labs = {i: [svx.LabelImage(li.width, li.height,
                                   torch.from_numpy(np.asarray(li.labels).view(np.int16).copy()).to(dev),
                                   li.fx, li.fy, li.cx, li.cy, li.pose, max_depth=li.max_depth)
                    for li in wl.label_images(i, device=dev)] for i in range(len(chunks))}
        for sem in (False, True):
            st = svx.VoxelStore(svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21), 0)
            ext = torch.cuda.ExternalStream(st.stream_ptr(), device=dev)
            icfg = svx.IntegratorConfig()
            st.reserve(1 << 20, (1 << 18) if sem else 0)  # pool mapped before the timed passes
            # warm-up: the first 8 scans
            rel = offs[:9] - offs[0]
            st.integrate_clouds_device(wl.model, pts.data_ptr(), rel, 3, poses[:8], icfg)
            def one_pass(first):
                """Scans first..first + n in one call (frame groups; with semantics each TSDF
                frame's label image right after its fold, svx_integrate_clouds_labels);
                device time of the pass."""
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(ext)
                rel = offs[first:first + n + 1] - offs[first]
                if sem:
                    svx.integrate_clouds_labels(st, wl.model, pts.data_ptr() + 12 * int(offs[first]), rel, 3,
                                                poses[first:first + n], icfg,
                                                [labs[i] for i in range(first, first + n)],
                                                labels_on_device=True)
                else:
                    st.integrate_clouds_device(wl.model, pts.data_ptr() + 12 * int(offs[first]), rel, 3,
                                               poses[first:first + n], icfg)
                e1.record(ext)
                e1.synchronize()
                return e0.elapsed_time(e1)
            one_pass(8)                           # warm-up pass: buffers sized, pool mapped ahead
            st.profile_enable(False)              # (resets the counters; no kernel marks)
            ms = one_pass(8 + n)                  # timed: no profiling marks (PDL chains intact)
            hp = st.profile_read().as_dict()      # host-side work of the timed pass
            st.profile_enable(True)               # kernel breakdown: a third, profiled pass
            one_pass(8 + 2 * n)
            p = st.profile_read().as_dict()
            npts = int(offs[8 + 2 * n] - offs[8 + n])
            # SURVEY 8(d) bytes of the profiled pass, scaled to the timed pass's points
            npts_prof = int(offs[8 + 3 * n] - offs[8 + 2 * n])
            B = 12.0 * npts_prof + 16.0 * p["touched_blocks"] + 10240.0 * p["new_blocks"] + \
                40.0 * p["updated_voxels"]
            if sem:
                B += 2.0 * 1280 * 720 * p["sem_images"] + 8.0 * 512 * p["sem_candidates"] + \
                    8.0 * 20 * p["sem_updated"]
            B *= npts / max(npts_prof, 1)
            row = {"sweep": "cfg5", "W": Wd, "points_per_scan": npts / n, "semantics": sem, "scans": n,
                   "points_per_s": npts / (ms / 1e3), "ms_per_scan": ms / n,
                   "pipeline_frac": B / (ms / 1e3) / 1e9 / peak,
                   "kernel_us_per_scan": {k: 1e3 * v / n for k, v in p["ms"].items()},
                   "timed_pass_host": {k: hp[k] for k in ("host_enqueue_ms", "host_resume_ms", "host_map_ms",
                                                          "aborts")}}
            rows.append(row)
            print(json.dumps(row), flush=True)
            st.close()
    geo = [r for r in rows if not r["semantics"]]
    print(json.dumps({"metric": METRIC, "sweep": "cfg5 points-per-scan (geometry only)", "unit": UNIT,
                      "points_per_scan": [r["points_per_scan"] for r in geo],
                      "value": [r["points_per_s"] for r in geo],
                      "pipeline_frac": [r["pipeline_frac"] for r in geo]}))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--scans-per-step", type=int, default=None)
    ap.add_argument("--ref-scans-per-step", type=int, default=2)
    ap.add_argument("--ref-offset", type=int, default=300)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--cpu-max-scans", type=int, default=40)
    ap.add_argument("--cfg3-cpu-frames", type=int, default=4)
    ap.add_argument("--carve", action="store_true")
    ap.add_argument("--carve-cpu-scans", type=int, default=2)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--sweep-widths", type=int, nargs="*",
                    default=[80, 160, 320, 640, 1280, 2560, 5120, 10240, 16384])
    ap.add_argument("--sweep-scans", type=int, default=16,
                    help="scans per timed pass (16: x in 0..4 m of the room; from 64 on the passes "
                         "include the wall-adjacent stretch x ~ 8..10 m, fallback-bound)")
    ap.add_argument("--emulate-ranks", type=int, nargs="*", default=None,
                    help="emulate the multi-GPU data plane with these rank counts on one GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-json", default="")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.scans_per_step is None:
        args.scans_per_step = {"cfg3": 16, "cfg4": 400}.get(args.workload, 100)
    relaunch_if_needed(args)
    world, rank, local = dist_env()
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if args.sweep:
        return run_sweep(args) if rank == 0 else 0
    if args.emulate_ranks:
        return run_emulated(args) if rank == 0 else 0
    if args.carve:
        return run_carve(args, world, rank, local)
    if args.workload == "cfg3":
        return run_cfg3(args, world, rank, local)
    return run_tsdf(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
