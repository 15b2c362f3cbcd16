"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the two CPU checkers.

  OracleMap  oracle/_ref/libsvx_oracle.so  (plain-C restatement, svx_oracle.c)
  RefMap     oracle/_ref/libsemvox_ref.so  (the reference's own translation units,
                                            built from /root/reference by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module, and only as the checker / baseline, never as the
product path. Both expose the same methods so tests can compare either with the
GPU library on identical inputs.
"""
from __future__ import annotations

import ctypes as C
import os
import tempfile

import numpy as np

import paper_2412_00291_b200 as svx
from paper_2412_00291_b200 import (FrameReport, FrameReportC, IntegratorCfg, LabelImageC,
                                   LidarModel, MapCfg, PoseC, SemanticCfg, StatsC, TSDF_DTYPE)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_ref", "libsvx_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsemvox_ref.so")

_P = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


_olib = None
_rlib = None


def olib():
    global _olib
    if _olib is None:
        L = C.CDLL(ORACLE_SO)
        L.svxo_map_create.restype = _P
        L.svxo_map_create.argtypes = [C.POINTER(MapCfg), C.POINTER(C.c_int)]
        L.svxo_map_destroy.argtypes = [_P]
        L.svxo_project.argtypes = [C.POINTER(LidarModel), _P, C.c_uint64, C.c_int32,
                                   C.POINTER(PoseC), _P, _P, C.POINTER(C.c_uint64)]
        L.svxo_normals.argtypes = [C.POINTER(LidarModel), _P, _P, _P]
        L.svxo_integrate.argtypes = [_P, C.POINTER(LidarModel), _P, _P, _P, C.POINTER(PoseC),
                                     C.POINTER(IntegratorCfg), C.POINTER(FrameReportC)]
        L.svxo_integrate_labels.argtypes = [_P, C.POINTER(LabelImageC), C.POINTER(SemanticCfg),
                                            C.POINTER(FrameReportC)]
        L.svxo_save_mem.restype = C.c_uint64
        L.svxo_save_mem.argtypes = [_P, _P, C.c_uint64]
        L.svxo_block_count.restype = C.c_uint64
        L.svxo_block_count.argtypes = [_P]
        L.svxo_get_or_allocate_block.argtypes = [_P, C.POINTER(C.c_int32)]
        L.svxo_block_write.argtypes = [_P, C.POINTER(C.c_int32), _P, _P, C.c_int32]
        L.svxo_lookup.argtypes = [_P, C.POINTER(C.c_int32), _P, _P]
        L.svxo_observed.restype = C.c_uint64
        L.svxo_observed.argtypes = [_P]
        L.svxo_take_dirty.restype = C.c_uint64
        L.svxo_take_dirty.argtypes = [_P, C.c_int32, _P, C.c_uint64]
        L.svxo_mesh_extract.argtypes = [_P, C.c_float, C.c_int32, _P, C.c_uint64,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.svxo_mesh_read.argtypes = [_P, _P, _P, _P, _P]
        L.svxo_mesh_read.restype = None
        L.svxo_occ_create.argtypes = [C.POINTER(svx.OccCfgC)]
        L.svxo_occ_create.restype = _P
        L.svxo_occ_destroy.argtypes = [_P]
        L.svxo_occ_integrate.argtypes = [_P, _P, _P, _P, C.c_uint64, C.c_int32, C.POINTER(PoseC),
                                         C.POINTER(svx.OccReportC)]
        L.svxo_occ_integrate_depth.argtypes = [_P, _P, _P, _P, C.POINTER(svx.PinholeC), C.POINTER(PoseC),
                                               C.POINTER(svx.OccReportC)]
        L.svxo_occ_save_mem.argtypes = [_P, _P, C.c_uint64]
        L.svxo_occ_save_mem.restype = C.c_uint64
        L.svxo_last_error.restype = C.c_char_p
        _olib = L
    return _olib


def rlib():
    global _rlib
    if _rlib is None:
        L = C.CDLL(REF_SO)
        L.ref_map_create.restype = _P
        L.ref_map_create.argtypes = [C.POINTER(MapCfg)]
        L.ref_map_load.argtypes = [C.c_char_p]
        L.ref_map_load.restype = _P
        L.ref_map_destroy.argtypes = [_P]
        L.ref_project.argtypes = [C.POINTER(LidarModel), _P, C.c_uint64, C.c_int32,
                                  C.POINTER(PoseC), _P, _P, _P, _P, C.POINTER(C.c_uint64)]
        L.ref_integrate.argtypes = [_P, C.POINTER(LidarModel), _P, _P, _P, C.POINTER(PoseC),
                                    C.POINTER(IntegratorCfg), C.POINTER(FrameReportC)]
        L.ref_integrate_cloud.argtypes = [_P, C.POINTER(LidarModel), _P, C.c_uint64, C.c_int32,
                                          C.POINTER(PoseC), C.POINTER(IntegratorCfg),
                                          C.POINTER(FrameReportC), C.POINTER(C.c_double)]
        L.ref_integrate_labels.argtypes = [_P, C.POINTER(LabelImageC), C.POINTER(SemanticCfg),
                                           C.POINTER(FrameReportC)]
        L.ref_save.argtypes = [_P, C.c_char_p]
        L.ref_block_count.restype = C.c_uint64
        L.ref_block_count.argtypes = [_P]
        L.ref_stats.argtypes = [_P, C.POINTER(StatsC)]
        L.ref_get_or_allocate_block.argtypes = [_P, C.POINTER(C.c_int32)]
        L.ref_block_write.argtypes = [_P, C.POINTER(C.c_int32), _P, _P, C.c_int32]
        L.ref_lookup.argtypes = [_P, _P, C.c_uint64, _P, _P, _P]
        L.ref_take_dirty.restype = C.c_uint64
        L.ref_take_dirty.argtypes = [_P, C.c_int32, _P, C.c_uint64]
        L.ref_mesh_extract.argtypes = [_P, C.c_float, C.c_int32, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]
        L.ref_mesh_incremental.argtypes = [_P, C.c_float, C.c_int32, _P, C.c_uint64,
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _P,
                                           C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_mesh_read.argtypes = [_P, _P, _P, _P, _P]
        L.ref_mesh_read.restype = None
        L.ref_last_error.restype = C.c_char_p
        L.ref_worker_count.restype = C.c_int
        L.ref_lidar_spinning.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                         C.POINTER(LidarModel)]
        _rlib = L
    return _rlib


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _label_c(img, K):
    P = img.width * img.height
    lbl = np.ascontiguousarray(np.asarray(img.labels, np.uint16).reshape(-1))
    conf = None if img.confidence is None else np.ascontiguousarray(
        np.asarray(img.confidence, np.float32).reshape(-1))
    ten = None
    if img.prob_tensor is not None and np.asarray(img.prob_tensor).size == P * K:
        ten = np.ascontiguousarray(np.asarray(img.prob_tensor, np.float32).reshape(-1))
    from paper_2412_00291_b200 import Pose, pose_c
    pc = img.pose if isinstance(img.pose, PoseC) else (
        img.pose.c() if isinstance(img.pose, Pose) else pose_c(img.pose))
    li = LabelImageC(img.width, img.height, lbl.ctypes.data_as(C.POINTER(C.c_uint16)),
                     None if conf is None else conf.ctypes.data_as(C.POINTER(C.c_float)),
                     None if ten is None else ten.ctypes.data_as(C.POINTER(C.c_float)),
                     img.fx, img.fy, img.cx, img.cy, pc, img.max_depth)
    return li, (lbl, conf, ten)


class _Base:
    K: int

    def project(self, model, points, pose):
        """-> (depth, height, normals[P,3], valid[P], dropped)"""
        raise NotImplementedError


class OracleMap(_Base):
    """The plain-C restatement (serial)."""

    def __init__(self, cfg):
        st = C.c_int()
        self.cfg = cfg
        self.K = cfg.num_labels
        self.h = olib().svxo_map_create(C.byref(cfg.c()), C.byref(st))
        if not self.h:
            raise CheckerError(st.value, olib().svxo_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            olib().svxo_map_destroy(self.h)
            self.h = None

    @staticmethod
    def project(model, points, pose):
        a = np.ascontiguousarray(np.asarray(points, np.float32))
        P = model.width * model.height_px
        d = np.zeros(P, np.float32)
        h = np.zeros(P, np.float32)
        n = np.zeros((P, 3), np.float32)
        v = np.zeros(P, np.uint8)
        dropped = C.c_uint64()
        st = olib().svxo_project(C.byref(model.c()), _ptr(a), a.shape[0], a.shape[1],
                                 C.byref(pose), _ptr(d), _ptr(h), C.byref(dropped))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())
        olib().svxo_normals(C.byref(model.c()), _ptr(d), _ptr(n), _ptr(v))
        return d, h, n, v, int(dropped.value)

    @staticmethod
    def normals(model, depth):
        P = model.width * model.height_px
        n = np.zeros((P, 3), np.float32)
        v = np.zeros(P, np.uint8)
        olib().svxo_normals(C.byref(model.c()), _ptr(np.ascontiguousarray(depth, np.float32)),
                            _ptr(n), _ptr(v))
        return n, v

    def integrate(self, model, depth, normals, valid, pose, icfg):
        rep = FrameReportC()
        st = olib().svxo_integrate(self.h, C.byref(model.c()),
                                   _ptr(np.ascontiguousarray(depth, np.float32)),
                                   _ptr(None if normals is None else np.ascontiguousarray(normals, np.float32)),
                                   _ptr(None if valid is None else np.ascontiguousarray(valid, np.uint8)),
                                   C.byref(pose), C.byref(icfg.c()), C.byref(rep))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())
        return FrameReport.of(rep)

    def integrate_cloud(self, model, points, pose, icfg):
        d, h, n, v, _ = self.project(model, points, pose)
        return self.integrate(model, d, n, v, pose, icfg)

    def integrate_labels(self, img, scfg):
        li, keep = _label_c(img, self.K)
        rep = FrameReportC()
        st = olib().svxo_integrate_labels(self.h, C.byref(li), C.byref(scfg.c()), C.byref(rep))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())
        return FrameReport.of(rep)

    def save_bytes(self) -> bytes:
        n = olib().svxo_save_mem(self.h, None, 0)
        buf = np.zeros(n, np.uint8)
        olib().svxo_save_mem(self.h, _ptr(buf), n)
        return buf.tobytes()

    def block_count(self):
        return int(olib().svxo_block_count(self.h))

    def observed(self):
        return int(olib().svxo_observed(self.h))

    def get_or_allocate_block(self, b):
        st = olib().svxo_get_or_allocate_block(self.h, (C.c_int32 * 3)(*b))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())

    def write_block(self, b, tsdf, sem=None, has_sem=False):
        t = np.ascontiguousarray(tsdf, TSDF_DTYPE)
        s = None if sem is None else np.ascontiguousarray(sem, np.float32)
        st = olib().svxo_block_write(self.h, (C.c_int32 * 3)(*b), _ptr(t), _ptr(s),
                                     int(has_sem or sem is not None))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())

    def extract_mesh(self, min_weight=1e-4, reserved=-1, blocks=None):
        """extract_mesh restated (svx_oracle.c) -> (vertices, normals, labels, faces)."""
        nv, nf = C.c_uint64(), C.c_uint64()
        b = None if blocks is None else np.ascontiguousarray(np.asarray(blocks, np.int32).reshape(-1, 3))
        olib().svxo_mesh_extract(self.h, min_weight, reserved, _ptr(b), 0 if b is None else b.shape[0],
                                 C.byref(nv), C.byref(nf))
        return _mesh_arrays(olib().svxo_mesh_read, self.h, nv.value, nf.value)

    def take_dirty(self, which):
        cap = max(self.block_count(), 1)  # unique dirty blocks <= allocated blocks
        out = np.zeros((cap, 3), np.int32)
        n = olib().svxo_take_dirty(self.h, which, _ptr(out), cap)
        return out[:n]


class RefMap(_Base):
    """The reference's own code (libsemvox_ref.so), multi-threaded per SEMVOX_THREADS."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.K = cfg.num_labels
        self.h = rlib().ref_map_create(C.byref(cfg.c()))
        if not self.h:
            raise CheckerError(1, rlib().ref_last_error().decode())

    @staticmethod
    def load(path, cfg):
        """VoxelStore::load of an SVOX1 file (the reference's own reader)."""
        m = RefMap.__new__(RefMap)
        m.cfg, m.K = cfg, cfg.num_labels
        m.h = rlib().ref_map_load(str(path).encode())
        if not m.h:
            raise CheckerError(3, rlib().ref_last_error().decode())
        return m

    def __del__(self):
        if getattr(self, "h", None):
            try:
                rlib().ref_map_destroy(self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    @staticmethod
    def project(model, points, pose):
        a = np.ascontiguousarray(np.asarray(points, np.float32))
        P = model.width * model.height_px
        d = np.zeros(P, np.float32)
        h = np.zeros(P, np.float32)
        n = np.zeros((P, 3), np.float32)
        v = np.zeros(P, np.uint8)
        dropped = C.c_uint64()
        st = rlib().ref_project(C.byref(model.c()), _ptr(a), a.shape[0], a.shape[1],
                                C.byref(pose), _ptr(d), _ptr(h), _ptr(n), _ptr(v),
                                C.byref(dropped))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())
        return d, h, n, v, int(dropped.value)

    def integrate(self, model, depth, normals, valid, pose, icfg):
        rep = FrameReportC()
        st = rlib().ref_integrate(self.h, C.byref(model.c()),
                                  _ptr(np.ascontiguousarray(depth, np.float32)),
                                  _ptr(None if normals is None else np.ascontiguousarray(normals, np.float32)),
                                  _ptr(None if valid is None else np.ascontiguousarray(valid, np.uint8)),
                                  C.byref(pose), C.byref(icfg.c()), C.byref(rep))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())
        return FrameReport.of(rep)

    def integrate_cloud(self, model, points, pose, icfg):
        """Full per-frame body of cmd_integrate; returns (report, wall_ms)."""
        a = np.ascontiguousarray(np.asarray(points, np.float32))
        rep = FrameReportC()
        ms = C.c_double()
        st = rlib().ref_integrate_cloud(self.h, C.byref(model.c()), _ptr(a), a.shape[0],
                                        a.shape[1], C.byref(pose), C.byref(icfg.c()),
                                        C.byref(rep), C.byref(ms))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())
        return FrameReport.of(rep), ms.value

    def integrate_labels(self, img, scfg):
        li, keep = _label_c(img, self.K)
        rep = FrameReportC()
        st = rlib().ref_integrate_labels(self.h, C.byref(li), C.byref(scfg.c()), C.byref(rep))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())
        return FrameReport.of(rep)

    def save_bytes(self) -> bytes:
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "m.svox")
            st = rlib().ref_save(self.h, p.encode())
            if st:
                raise CheckerError(st, rlib().ref_last_error().decode())
            return open(p, "rb").read()

    def block_count(self):
        return int(rlib().ref_block_count(self.h))

    def observed(self):
        s = StatsC()
        rlib().ref_stats(self.h, C.byref(s))
        return int(s.observed_voxels)

    def get_or_allocate_block(self, b):
        st = rlib().ref_get_or_allocate_block(self.h, (C.c_int32 * 3)(*b))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())

    def write_block(self, b, tsdf, sem=None, has_sem=False):
        t = np.ascontiguousarray(tsdf, TSDF_DTYPE)
        s = None if sem is None else np.ascontiguousarray(sem, np.float32)
        st = rlib().ref_block_write(self.h, (C.c_int32 * 3)(*b), _ptr(t), _ptr(s),
                                    int(has_sem or sem is not None))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())

    def lookup(self, coords):
        v = np.ascontiguousarray(np.asarray(coords, np.int32).reshape(-1, 3))
        n = v.shape[0]
        t = np.zeros(n, TSDF_DTYPE)
        p = np.zeros((n, self.K), np.float32)
        f = np.zeros(n, np.uint8)
        rlib().ref_lookup(self.h, _ptr(v), n, _ptr(t), _ptr(p), _ptr(f))
        return f.astype(bool), t, p

    def take_dirty(self, which):
        cap = max(self.block_count(), 1)
        out = np.zeros((cap, 3), np.int32)
        n = rlib().ref_take_dirty(self.h, which, _ptr(out), cap)
        return out[:n]

    def extract_mesh(self, min_weight=1e-4, reserved=-1):
        """The reference's extract_mesh -> (vertices, normals, labels, faces)."""
        nv, nf = C.c_uint64(), C.c_uint64()
        st = rlib().ref_mesh_extract(self.h, min_weight, reserved, C.byref(nv), C.byref(nf))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())
        return _mesh_arrays(rlib().ref_mesh_read, self.h, nv.value, nf.value)

    def mesh_incremental(self, dirty, min_weight=1e-4, reserved=-1):
        """The reference's IncrementalMesher::update -> (mesh arrays, last_remeshed)."""
        d = np.ascontiguousarray(np.asarray(dirty, np.int32).reshape(-1, 3))
        nv, nf, nr = C.c_uint64(), C.c_uint64(), C.c_uint64()
        cap = 8 * d.shape[0] + 1
        rem = np.zeros((cap, 3), np.int32)
        st = rlib().ref_mesh_incremental(self.h, min_weight, reserved, _ptr(d), d.shape[0],
                                         C.byref(nv), C.byref(nf), _ptr(rem), cap, C.byref(nr))
        if st:
            raise CheckerError(st, rlib().ref_last_error().decode())
        return _mesh_arrays(rlib().ref_mesh_read, self.h, nv.value, nf.value), rem[:nr.value]


class OracleOcc:
    """Serial restatement of the occupancy extension (svx_oracle.c, parity unpinned)."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.h = olib().svxo_occ_create(C.byref(cfg.c()))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                olib().svxo_occ_destroy(self.h)
            except TypeError:
                pass
            self.h = None

    def integrate(self, points, pose, labels=None, conf=None):
        a = np.ascontiguousarray(np.asarray(points, np.float32))
        lb = None if labels is None else np.ascontiguousarray(labels, np.uint16)
        cf = None if conf is None else np.ascontiguousarray(conf, np.float32)
        rep = svx.OccReportC()
        st = olib().svxo_occ_integrate(self.h, _ptr(a), _ptr(lb), _ptr(cf), a.shape[0], a.shape[1],
                                       C.byref(pose), C.byref(rep))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())
        return rep

    def integrate_depth(self, depth, cam, pose, labels=None, conf=None):
        d = np.ascontiguousarray(np.asarray(depth, np.float32))
        lb = None if labels is None else np.ascontiguousarray(labels, np.uint16)
        cf = None if conf is None else np.ascontiguousarray(conf, np.float32)
        rep = svx.OccReportC()
        st = olib().svxo_occ_integrate_depth(self.h, _ptr(d), _ptr(lb), _ptr(cf), C.byref(cam),
                                             C.byref(pose), C.byref(rep))
        if st:
            raise CheckerError(st, olib().svxo_last_error().decode())
        return rep

    def save_bytes(self) -> bytes:
        n = olib().svxo_occ_save_mem(self.h, None, 0)
        buf = np.zeros(n, np.uint8)
        olib().svxo_occ_save_mem(self.h, _ptr(buf), n)
        return buf.tobytes()


def parse_socc1(buf: bytes):
    """SOCC1 (include/svx.h svx_occ_save_mem) -> (header, keys[n,3], L[n,512], hits, misses, hist dict)."""
    import struct
    if buf[:5] != b"SOCC1":
        raise ValueError("not SOCC1")
    vs, K, lh, lm, lmin, lmax = struct.unpack_from("<fIffff", buf, 5)
    (nb,) = struct.unpack_from("<Q", buf, 29)
    off = 37
    keys = np.zeros((nb, 3), np.int32)
    L = np.zeros((nb, 512), np.float32)
    hits = np.zeros((nb, 512), np.uint32)
    misses = np.zeros((nb, 512), np.uint32)
    hist = {}
    for i in range(nb):
        keys[i] = np.frombuffer(buf, np.int32, 3, off)
        off += 12
        L[i] = np.frombuffer(buf, np.float32, 512, off)
        hits[i] = np.frombuffer(buf, np.uint32, 512, off + 2048)
        misses[i] = np.frombuffer(buf, np.uint32, 512, off + 4096)
        off += 6144
        hs = buf[off]
        off += 1
        if hs:
            hist[i] = np.frombuffer(buf, np.uint32, 512 * K, off).reshape(512, K)
            off += 2048 * K
    return {"voxel_size": vs, "num_labels": K, "l": (lh, lm, lmin, lmax)}, keys, L, hits, misses, hist


def _mesh_arrays(read, h, nv, nf):
    v = np.zeros((nv, 3), np.float32)
    n = np.zeros((nv, 3), np.float32)
    lab = np.zeros(nv, np.uint8)
    f = np.zeros((nf, 3), np.uint32)
    read(h, _ptr(v), _ptr(n), _ptr(lab), _ptr(f))
    return v, n, lab, f


def parse_svox1(buf: bytes):
    """SVOX1 (voxel_store.cpp:101-130) -> (header dict, keys[n,3], tsdf[n,512], sem dict)."""
    import struct
    if buf[:5] != b"SVOX1":
        raise ValueError("not SVOX1")
    vs, tr, K = struct.unpack_from("<ffI", buf, 5)
    (nb,) = struct.unpack_from("<Q", buf, 17)
    off = 25
    keys = np.zeros((nb, 3), np.int32)
    tsdf = np.zeros((nb, 512), TSDF_DTYPE)
    sem = {}
    for i in range(nb):
        keys[i] = np.frombuffer(buf, np.int32, 3, off)
        off += 12
        tsdf[i] = np.frombuffer(buf, TSDF_DTYPE, 512, off)
        off += 512 * 20
        hs = buf[off]
        off += 1
        if hs:
            sem[i] = np.frombuffer(buf, np.float32, 512 * K, off).reshape(512, K)
            off += 512 * K * 4
    return {"voxel_size": vs, "truncation": tr, "num_labels": K}, keys, tsdf, sem
