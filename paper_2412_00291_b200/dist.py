"""Multi-GPU data plane (exchange mode), host side: one process per GPU, NCCL through
torch.distributed for the plumbing.

The map is key-sharded (owner(block) = mix64(key) mod N, svx_block_owner). Per frame
group (<= 16 clouds, the same clouds on every rank):

  1. svx_integrate_clouds_xbegin: every rank projects the group (replicated, 6 us per
     frame) and casts the rays of its share of the pixel tiles (round robin); visits of
     blocks another rank owns leave as 16-byte entries packed by destination;
  2. one all-to-all of those entries (all_to_all_single: counts, then payload);
  3. svx_integrate_clouds_xend: every rank applies what it received and folds its own
     blocks (own-pixel measurement, fallback ordered sums, accumulate-then-merge).

Every per-voxel result is computed by the voxel's owner from the same inputs in the same
order as on one GPU, so the union of the ranks' maps is the single-GPU map byte for byte
(tests/test_gpu_parity.py::test_exchange_sharded_union_equals_unsharded, emulated on one
GPU; tests/test_host.py covers the exchange routine with gloo on the CPU).
"""
from __future__ import annotations

import numpy as np

ENTRY_BYTES = 16


class _CudaBytes:
    """Zero-copy view of device memory as a torch uint8 tensor (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


def device_bytes(ptr: int, nbytes: int, device):
    import torch
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_CudaBytes(ptr, nbytes), device=device)


def exchange(send, meta, group=None):
    """All-to-all of variable-size entry lists.

    send: uint8 tensor of 16-byte entries packed by destination rank; meta[world][17]:
    per destination, the entry count then 16 per-frame voxel-bit counts. Returns (the
    uint8 tensor of the entries every rank sent to this one, in source-rank order; the
    senders' metadata rows for this rank, [world][17]). Works with any torch.distributed
    backend (gloo on the CPU, NCCL on the GPU)."""
    import torch
    import torch.distributed as dist
    meta = np.asarray(meta, np.int64)
    m = torch.as_tensor(meta.reshape(-1), device=send.device)
    rm = torch.empty_like(m)
    dist.all_to_all_single(rm, m, group=group)
    rmeta = rm.cpu().numpy().reshape(meta.shape)
    rcounts = [int(x) for x in rmeta[:, 0]]
    recv = torch.empty(sum(rcounts) * ENTRY_BYTES, dtype=torch.uint8, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=[n * ENTRY_BYTES for n in rcounts],
                           input_split_sizes=[int(n) * ENTRY_BYTES for n in meta[:, 0]], group=group)
    return recv, rmeta


def integrate_group(store, model, d_points_ptr, offsets, stride, poses, cfg, group=None):
    """One frame group on this rank: xbegin, all-to-all, xend. Returns this rank's reports."""
    import torch
    meta, ptr = store.xbegin(model, d_points_ptr, offsets, stride, poses, cfg)
    dev = torch.device("cuda", store.device)
    send = device_bytes(ptr, int(meta[:, 0].sum()) * ENTRY_BYTES, dev)
    recv, rmeta = exchange(send, meta, group)
    torch.cuda.current_stream(dev).synchronize()  # the map stream reads recv next
    return store.xend(recv.data_ptr() if recv.numel() else 0, rmeta)


def integrate_sharded(store, model, d_points_ptr, offsets, stride, poses, cfg, group_size=16, group=None):
    """A sequence of clouds (device memory, offsets per frame) on this rank, group by group."""
    offs = np.asarray(offsets, np.uint64)
    reps = []
    for a in range(0, len(poses), group_size):
        b = min(len(poses), a + group_size)
        rel = offs[a:b + 1] - offs[a]
        reps += integrate_group(store, model, d_points_ptr + int(offs[a]) * stride * 4, rel, stride, poses[a:b],
                                cfg, group)
    return reps


def emulate_sharded(stores, model, d_points_ptr, offsets, stride, poses, cfg, group_size=16, timers=None):
    """Every rank of a key-sharded set of maps in ONE process on ONE GPU (tests, per-rank
    cost measurement): the same calls as integrate_sharded, with the all-to-all done by
    device copies. Ranks run one after another (none waits on another). `timers`, when a
    list, receives per group and rank the host ms of (xbegin, xend) (each call ends with
    a stream synchronisation, so these are device-bound times)."""
    import torch
    world = len(stores)
    offs = np.asarray(offsets, np.uint64)
    reps = [[] for _ in range(world)]
    for a in range(0, len(poses), group_size):
        b = min(len(poses), a + group_size)
        rel = offs[a:b + 1] - offs[a]
        sends, metas, t_begin = [], [], []
        for st in stores:
            t0 = _now_ms()
            meta, ptr = st.xbegin(model, d_points_ptr + int(offs[a]) * stride * 4, rel, stride, poses[a:b], cfg)
            t_begin.append(_now_ms() - t0)
            dev = torch.device("cuda", st.device)
            sends.append(device_bytes(ptr, int(meta[:, 0].sum()) * ENTRY_BYTES, dev).clone())
            metas.append(meta.astype(np.int64))
        t_end = []
        for d, st in enumerate(stores):
            parts = []
            for r in range(world):
                o = int(metas[r][:d, 0].sum()) * ENTRY_BYTES
                parts.append(sends[r][o:o + int(metas[r][d, 0]) * ENTRY_BYTES])
            recv = torch.cat(parts)
            rmeta = np.stack([metas[r][d] for r in range(world)])
            torch.cuda.synchronize()
            t0 = _now_ms()
            reps[d] += st.xend(recv.data_ptr() if recv.numel() else 0, rmeta)
            t_end.append(_now_ms() - t0)
        if timers is not None:
            timers.append({"xbegin_ms": t_begin, "xend_ms": t_end,
                           "entries": [int(m[:, 0].sum()) for m in metas]})
    return reps


def _now_ms():
    import time
    return time.perf_counter() * 1e3
