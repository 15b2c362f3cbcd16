"""B200-native semvox voxel-integration hot path (arXiv 2412.00291).

Python host mirror of the reference C++ API (proj/include/semvox/*.hpp) over the
C-ABI in include/svx.h, backed by lib/libsvx_b200.so (sm_100a kernels). Same
names, argument meaning and error behaviour as the reference:

  reference (C++)                         here
  ------------------------------------   -------------------------------------
  MapConfig / VoxelStore                  MapConfig / VoxelStore
  ProjectionModel::spinning               ProjectionModel.spinning
  project_cloud / compute_normal_image    project_cloud / compute_normal_image
  TsdfIntegrator::integrate_frame         TsdfIntegrator.integrate_frame
  SemanticIntegrator::integrate_labels    SemanticIntegrator.integrate_labels
  CapacityError / DataError /             CapacityError / DataError /
  std::invalid_argument                   InvalidArgument (a ValueError)

There is no CPU fallback: importing works without a GPU (so the library can be
inspected), but every compute call goes to the CUDA library and fails loudly if
it is missing or no device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SVX_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("SVX_LIB") or os.path.join(_HERE, "lib", "libsvx_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "svx.h")

# ----------------------------------------------------------------- errors


class SvxError(RuntimeError):
    pass


class InvalidArgument(SvxError, ValueError):
    """std::invalid_argument"""


class CapacityError(SvxError):
    """semvox::CapacityError (types.hpp:20-22)"""


class DataError(SvxError):
    """semvox::DataError (types.hpp:25-27)"""


class CudaError(SvxError):
    pass


class NotFound(SvxError, KeyError):
    pass


_STATUS = {1: InvalidArgument, 2: CapacityError, 3: DataError, 4: CudaError, 5: NotFound}

# ---------------------------------------------------------------- structs


class MapCfg(C.Structure):
    _fields_ = [("voxel_size", C.c_float), ("truncation", C.c_float),
                ("num_labels", C.c_int32), ("max_blocks", C.c_uint32)]


class LidarModel(C.Structure):
    _fields_ = [("width", C.c_int32), ("height_px", C.c_int32), ("delta_phi", C.c_double),
                ("delta_theta", C.c_double), ("theta0", C.c_double), ("scale_f", C.c_double),
                ("offset_o", C.c_double), ("min_range", C.c_double)]


class PoseC(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class IntegratorCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("truncation", C.c_float), ("max_range", C.c_double),
                ("alpha_epsilon", C.c_double), ("min_weight_clamp", C.c_float),
                ("drop_unreliable", C.c_int32)]


class SemanticCfg(C.Structure):
    _fields_ = [("use_bayes", C.c_int32), ("likelihood_floor", C.c_float),
                ("default_confidence", C.c_float), ("occlusion", C.c_int32)]


class FrameReportC(C.Structure):
    _fields_ = [("frame", C.c_int32), ("updated_voxels", C.c_uint64),
                ("new_blocks", C.c_uint64), ("elapsed_ms", C.c_double)]


class LabelImageC(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("labels", C.POINTER(C.c_uint16)), ("confidence", C.POINTER(C.c_float)),
                ("prob_tensor", C.POINTER(C.c_float)), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("pose", PoseC),
                ("max_depth", C.c_double)]


class StatsC(C.Structure):
    _fields_ = [("allocated_blocks", C.c_uint64), ("observed_voxels", C.c_uint64),
                ("memory_bytes", C.c_uint64)]


K_NAMES = ["project", "raycast", "fold", "fallback", "sem_cull", "sem_update", "compact", "k7"]


class ProfileC(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_uint64 * 8), ("frames", C.c_uint64),
                ("points", C.c_uint64), ("rays", C.c_uint64), ("touched_blocks", C.c_uint64),
                ("new_blocks", C.c_uint64), ("updated_voxels", C.c_uint64),
                ("fallback_voxels", C.c_uint64), ("sem_images", C.c_uint64),
                ("sem_candidates", C.c_uint64), ("sem_updated", C.c_uint64),
                ("sem_new_layers", C.c_uint64), ("host_enqueue_ms", C.c_double),
                ("host_resume_ms", C.c_double), ("host_map_ms", C.c_double),
                ("aborts", C.c_uint64 * 8)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("ms", "launches", "aborts")}
        names = ["pool", "capacity", "key", "hash", "records", "exchange", "voxel_list", "b7"]
        d["aborts"] = {names[i]: self.aborts[i] for i in range(8) if self.aborts[i]}
        d["ms"] = {K_NAMES[i]: self.ms[i] for i in range(8) if self.launches[i]}
        d["launches"] = {K_NAMES[i]: self.launches[i] for i in range(8) if self.launches[i]}
        return d


XMETA = 17  # exchange-mode metadata per destination: entries, voxel bits of frames 0..15
TSDF_DTYPE = np.dtype([("distance", "<f4"), ("weight", "<f4"), ("gradient", "<f4", (3,))])
BLOCK_VOXELS = 512

# ------------------------------------------------------------------ loading

_lib: Optional[C.CDLL] = None


class OccCfgC(C.Structure):
    _fields_ = [("voxel_size", C.c_float), ("num_labels", C.c_int32), ("max_blocks", C.c_uint32),
                ("l_hit", C.c_float), ("l_miss", C.c_float), ("l_min", C.c_float),
                ("l_max", C.c_float), ("min_range", C.c_double), ("max_range", C.c_double),
                ("carve", C.c_int32)]


class PinholeC(C.Structure):
    """svx_pinhole: a pinhole depth camera (x right, y down, z forward)."""
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("max_depth", C.c_double)]


class OccReportC(C.Structure):
    _fields_ = [("frame", C.c_int32), ("points", C.c_uint64), ("rays", C.c_uint64),
                ("hit_voxels", C.c_uint64), ("miss_voxels", C.c_uint64),
                ("new_blocks", C.c_uint64), ("elapsed_ms", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def _sig(lib: C.CDLL) -> None:
    P = C.c_void_p
    S = C.c_int
    f = {
        "svx_last_error": (C.c_size_t, [C.c_char_p, C.c_size_t]),
        "svx_status_name": (C.c_char_p, [C.c_int]),
        "svx_kernel_launches": (C.c_uint64, []),
        "svx_map_create": (S, [C.POINTER(MapCfg), C.c_int, C.POINTER(P)]),
        "svx_map_destroy": (S, [P]),
        "svx_map_config": (S, [P, C.POINTER(MapCfg)]),
        "svx_map_get_stream": (S, [P, C.POINTER(P)]),
        "svx_get_or_allocate_block": (S, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "svx_has_block": (S, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "svx_block_count": (S, [P, C.POINTER(C.c_uint64)]),
        "svx_block_keys_sorted": (S, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "svx_block_read": (S, [P, C.POINTER(C.c_int32), P, P, C.POINTER(C.c_int32)]),
        "svx_blocks_read": (S, [P, P, C.c_uint64, P, P, P]),
        "svx_block_write": (S, [P, C.POINTER(C.c_int32), P, P, C.c_int32]),
        "svx_lookup": (S, [P, P, C.c_uint64, P, P, P]),
        "svx_stats_get": (S, [P, C.POINTER(StatsC)]),
        "svx_save": (S, [P, C.c_char_p]),
        "svx_save_mem": (S, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "svx_load": (S, [C.c_char_p, C.c_int, C.c_uint32, C.POINTER(P)]),
        "svx_take_dirty_blocks": (S, [P, C.c_int32, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "svx_scan_create": (S, [P, C.POINTER(LidarModel), C.POINTER(P)]),
        "svx_scan_destroy": (S, [P]),
        "svx_project": (S, [P, P, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(PoseC)]),
        "svx_project_f64": (S, [P, P, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(PoseC)]),
        "svx_compute_normals": (S, [P]),
        "svx_scan_upload": (S, [P, P, P, P, P]),
        "svx_scan_download": (S, [P, P, P, P, P, C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]),
        "svx_integrate_scan": (S, [P, P, C.POINTER(PoseC), C.POINTER(IntegratorCfg),
                                   C.POINTER(FrameReportC)]),
        "svx_integrate_cloud": (S, [P, P, P, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(PoseC),
                                    C.POINTER(IntegratorCfg), C.POINTER(FrameReportC)]),
        "svx_integrate_clouds_device": (S, [P, P, P, P, C.c_int32, P, C.c_int32,
                                            C.POINTER(IntegratorCfg), P]),
        "svx_integrate_clouds": (S, [P, P, P, P, C.c_int32, P, C.c_int32,
                                     C.POINTER(IntegratorCfg), P]),
        "svx_integrate_clouds_labels": (S, [P, P, P, P, C.c_int32, C.c_int32, P, C.c_int32,
                                            C.POINTER(IntegratorCfg), P, P, C.c_int32, C.POINTER(SemanticCfg),
                                            P, P]),
        "svx_integrate_clouds_xbegin": (S, [P, P, P, P, C.c_int32, P, C.c_int32, C.POINTER(IntegratorCfg),
                                            P, C.POINTER(P)]),
        "svx_integrate_clouds_xend": (S, [P, P, P, P]),
        "svx_integrate_labels_batch": (S, [P, P, C.c_int32, C.c_int32, C.POINTER(SemanticCfg), P]),
        "svx_integrate_labels": (S, [P, C.POINTER(LabelImageC), C.POINTER(SemanticCfg),
                                     C.POINTER(FrameReportC)]),
        "svx_default_integrator_cfg": (None, [C.POINTER(IntegratorCfg)]),
        "svx_default_semantic_cfg": (None, [C.POINTER(SemanticCfg)]),
        "svx_lidar_spinning": (S, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                   C.POINTER(LidarModel)]),
        "svx_map_set_shard": (S, [P, C.c_int32, C.c_int32]),
        "svx_profile_enable": (S, [P, C.c_int32]),
        "svx_profile_read": (S, [P, C.POINTER(ProfileC)]),
        "svx_block_owner": (C.c_int32, [C.POINTER(C.c_int32), C.c_int32]),
        "svx_has_blocks": (S, [P, P, C.c_uint64, P]),
        "svx_map_reserve": (S, [P, C.c_uint64, C.c_uint64]),
        "svx_mesh_extract": (S, [P, C.c_float, C.c_int32, P, C.c_uint64, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]),
        "svx_mesh_read": (S, [P, P, P, P, P]),
        "svx_mesh_device": (S, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
        "svx_default_occ_cfg": (None, [C.POINTER(OccCfgC)]),
        "svx_occ_create": (S, [C.POINTER(OccCfgC), C.c_int, C.POINTER(P)]),
        "svx_occ_destroy": (S, [P]),
        "svx_occ_get_stream": (S, [P, C.POINTER(P)]),
        "svx_occ_set_shard": (S, [P, C.c_int32, C.c_int32]),
        "svx_occ_reserve": (S, [P, C.c_uint64, C.c_uint64]),
        "svx_occ_integrate_depth": (S, [P, P, P, P, C.POINTER(PinholeC), C.POINTER(PoseC), C.c_int32,
                                        C.c_int32, C.POINTER(OccReportC)]),
        "svx_occ_integrate": (S, [P, P, P, P, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(PoseC),
                                  C.POINTER(OccReportC)]),
        "svx_occ_integrate_batch": (S, [P, P, P, P, P, C.c_int32, C.c_int32, P, C.c_int32, P]),
        "svx_occ_lookup": (S, [P, P, C.c_uint64, P, P, P, P, P, P]),
        "svx_occ_block_count": (S, [P, C.POINTER(C.c_uint64)]),
        "svx_occ_save_mem": (S, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
    }
    for name, (res, args) in f.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    """The CUDA library. Raises if it was not built (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2412_00291_b200/csrc)")
        _lib = C.CDLL(LIB_PATH)
        _sig(_lib)
    return _lib


def declared_symbols() -> list[str]:
    """Function names declared in include/svx.h (the drop-in boundary)."""
    import re
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:svx_status|size_t|const char\*|uint64_t|void|int32_t)"
                                 r"\s+(svx_\w+)\s*\(", text, re.M)))


def _check(status: int) -> None:
    if status == 0:
        return
    buf = C.create_string_buffer(1024)
    lib().svx_last_error(buf, 1024)
    raise _STATUS.get(status, SvxError)(buf.value.decode(errors="replace"))


def kernel_launches() -> int:
    return int(lib().svx_kernel_launches())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _i3(b) -> C.Array:
    return (C.c_int32 * 3)(*[int(x) for x in b])

# ------------------------------------------------------------------ config


@dataclass
class MapConfig:
    """semvox::MapConfig (types.hpp:97-112)."""
    voxel_size: float = 0.25
    truncation: float = 1.25
    num_labels: int = 2
    max_blocks: int = 1 << 20

    def c(self) -> MapCfg:
        return MapCfg(self.voxel_size, self.truncation, self.num_labels, self.max_blocks)


@dataclass
class ProjectionModel:
    """semvox::ProjectionModel (scan_projection.hpp:16-38)."""
    width: int = 1024
    height_px: int = 64
    delta_phi: float = 2.0 * np.pi / 1024
    delta_theta: float = 0.0
    theta0: float = 0.0
    scale_f: float = 256.0
    offset_o: float = 0.0
    min_range: float = 0.3

    @staticmethod
    def spinning(width: int, height_px: int, fov_up_deg: float, fov_down_deg: float
                 ) -> "ProjectionModel":
        # ProjectionModel::spinning (scan_projection.cpp:9-19), same double arithmetic
        pi = 3.141592653589793
        m = ProjectionModel(width=width, height_px=height_px)
        m.delta_phi = 2.0 * pi / width
        m.theta0 = (90.0 - fov_up_deg) * pi / 180.0
        m.delta_theta = (fov_up_deg + fov_down_deg) * pi / 180.0 / height_px
        m.validate()
        return m

    def validate(self) -> None:
        if self.width <= 0 or self.height_px <= 0:
            raise InvalidArgument("projection model: empty image")
        if abs(self.width * self.delta_phi - 2.0 * np.pi) > 1e-6:
            raise InvalidArgument("projection model: width * delta_phi must equal 2*pi")
        if not self.delta_theta > 0.0:
            raise InvalidArgument("projection model: delta_theta must be > 0")

    def c(self) -> LidarModel:
        return LidarModel(self.width, self.height_px, self.delta_phi, self.delta_theta,
                          self.theta0, self.scale_f, self.offset_o, self.min_range)

    def key(self) -> tuple:
        return (self.width, self.height_px, self.delta_phi, self.delta_theta, self.theta0,
                self.min_range)


PROJECTIVE, NON_PROJECTIVE = 0, 1
SURROGATE, RAYCAST = 0, 1


@dataclass
class IntegratorConfig:
    """semvox::IntegratorConfig (tsdf_integrator.hpp:14-23)."""
    mode: int = NON_PROJECTIVE
    truncation: float = 0.0
    max_range: float = 70.0
    alpha_epsilon: float = 1e-2
    min_weight_clamp: float = 0.01
    drop_unreliable: bool = False

    def c(self) -> IntegratorCfg:
        return IntegratorCfg(self.mode, self.truncation, self.max_range, self.alpha_epsilon,
                             self.min_weight_clamp, int(self.drop_unreliable))


@dataclass
class SemanticConfig:
    """semvox::SemanticConfig (semantic_integrator.hpp:31-38)."""
    use_bayes: bool = True
    likelihood_floor: float = 1e-3
    default_confidence: float = 0.9
    occlusion: int = SURROGATE

    def c(self) -> SemanticCfg:
        return SemanticCfg(int(self.use_bayes), self.likelihood_floor, self.default_confidence,
                           self.occlusion)


@dataclass
class FrameReport:
    """semvox::FrameReport (tsdf_integrator.hpp:25-32)."""
    frame: int = -1
    updated_voxels: int = 0
    new_blocks: int = 0
    elapsed_ms: float = 0.0

    def json_line(self) -> str:
        # FrameReport::json_line (tsdf_integrator.cpp:12-18)
        return ('{"frame":%d,"updated_voxels":%d,"new_blocks":%d,"elapsed_ms":%.3f}'
                % (self.frame, self.updated_voxels, self.new_blocks, self.elapsed_ms))

    @staticmethod
    def of(r: FrameReportC) -> "FrameReport":
        return FrameReport(r.frame, r.updated_voxels, r.new_blocks, r.elapsed_ms)


def pose_c(R=None, t=None) -> PoseC:
    """(R 3x3, t 3) -> svx_pose. A 4x4 matrix may be passed as R."""
    R = np.eye(3) if R is None else np.asarray(R, dtype=np.float64)
    if R.shape == (4, 4):
        R, t = R[:3, :3], R[:3, 3]
    t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64)
    p = PoseC()
    p.R[:] = [float(x) for x in R.reshape(9)]
    p.t[:] = [float(x) for x in t.reshape(3)]
    return p


@dataclass
class Pose:
    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def c(self) -> PoseC:
        return pose_c(self.R, self.t)

# -------------------------------------------------------------- the store


class VoxelStore:
    """semvox::VoxelStore (voxel_store.hpp:49-103), resident in HBM on `device`."""

    def __init__(self, cfg: MapConfig = None, device: int = 0, _handle=None):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
            c = MapCfg()
            _check(lib().svx_map_config(self._h, C.byref(c)))
            self.cfg = MapConfig(c.voxel_size, c.truncation, c.num_labels, c.max_blocks)
        else:
            self.cfg = cfg or MapConfig()
            _check(lib().svx_map_create(C.byref(self.cfg.c()), device, C.byref(self._h)))
        self.device = device
        self._scans: dict = {}
        self._world = 1

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            for s in self._scans.values():
                lib().svx_scan_destroy(s)
            self._scans.clear()
            _check(lib().svx_map_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def config(self) -> MapConfig:
        return self.cfg

    @property
    def handle(self):
        return self._h

    def stream_ptr(self) -> int:
        s = C.c_void_p()
        _check(lib().svx_map_get_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def scan(self, model: ProjectionModel):
        """Device ScanImages buffers for `model` (cached per model)."""
        k = model.key()
        if k not in self._scans:
            s = C.c_void_p()
            _check(lib().svx_scan_create(self._h, C.byref(model.c()), C.byref(s)))
            self._scans[k] = s
        return self._scans[k]

    def set_shard(self, rank: int, world: int) -> None:
        _check(lib().svx_map_set_shard(self._h, rank, world))
        self._world = world

    def profile_enable(self, on: bool = True) -> None:
        _check(lib().svx_profile_enable(self._h, int(on)))

    def profile_read(self) -> ProfileC:
        p = ProfileC()
        _check(lib().svx_profile_read(self._h, C.byref(p)))
        return p

    def integrate_clouds_device(self, model: ProjectionModel, d_points_ptr: int,
                                offsets: np.ndarray, stride: int, poses: list,
                                cfg: "IntegratorConfig") -> list:
        """A sequence of clouds already in HBM (device pointer), one call."""
        n = len(poses)
        offs = np.ascontiguousarray(np.asarray(offsets, np.uint64))
        parr = (PoseC * n)(*poses)
        reps = (FrameReportC * n)()
        _check(lib().svx_integrate_clouds_device(self._h, self.scan(model), C.c_void_p(d_points_ptr),
                                                 _ptr(offs), stride, C.cast(parr, C.c_void_p), n,
                                                 C.byref(cfg.c()), C.cast(reps, C.c_void_p)))
        return [FrameReport.of(r) for r in reps]

    def integrate_clouds_host(self, model: ProjectionModel, points_ptr: int, offsets: np.ndarray,
                              stride: int, poses: list, cfg: "IntegratorConfig") -> list:
        """A sequence of clouds in host memory (pointer; pinned memory overlaps the
        copies with the integration), one call."""
        n = len(poses)
        offs = np.ascontiguousarray(np.asarray(offsets, np.uint64))
        parr = (PoseC * n)(*poses)
        reps = (FrameReportC * n)()
        _check(lib().svx_integrate_clouds(self._h, self.scan(model), C.c_void_p(points_ptr), _ptr(offs),
                                          stride, C.cast(parr, C.c_void_p), n, C.byref(cfg.c()),
                                          C.cast(reps, C.c_void_p)))
        return [FrameReport.of(r) for r in reps]

    # ---- multi-GPU data plane (exchange mode): see paper_2412_00291_b200.dist
    def xbegin(self, model: ProjectionModel, d_points_ptr: int, offsets: np.ndarray, stride: int,
               poses: list, cfg: "IntegratorConfig"):
        """svx_integrate_clouds_xbegin: one group (<= 16 clouds in HBM) on a key-sharded map.
        Returns (send_meta[world][17]: entries, then voxel bits per frame, per destination;
        device pointer of the 16-byte entries packed by destination)."""
        n = len(poses)
        offs = np.ascontiguousarray(np.asarray(offsets, np.uint64))
        parr = (PoseC * n)(*poses)
        meta = np.zeros((self._world, XMETA), np.uint64)
        ptr = C.c_void_p()
        _check(lib().svx_integrate_clouds_xbegin(self._h, self.scan(model), C.c_void_p(d_points_ptr), _ptr(offs),
                                                 stride, C.cast(parr, C.c_void_p), n, C.byref(cfg.c()),
                                                 _ptr(meta), C.byref(ptr)))
        self._xn = n
        return meta, int(ptr.value or 0)

    def xend(self, d_recv_ptr: int, recv_meta: np.ndarray) -> list:
        """svx_integrate_clouds_xend: the entries received from all ranks (device pointer,
        source-rank order) and their senders' metadata rows for this rank ([world][17])."""
        rm = np.ascontiguousarray(np.asarray(recv_meta, np.uint64).reshape(self._world, XMETA))
        reps = (FrameReportC * self._xn)()
        _check(lib().svx_integrate_clouds_xend(self._h, C.c_void_p(d_recv_ptr or None), _ptr(rm),
                                               C.cast(reps, C.c_void_p)))
        return [FrameReport.of(r) for r in reps]

    def get_or_allocate_block(self, bc) -> bool:
        nw = C.c_int32()
        _check(lib().svx_get_or_allocate_block(self._h, _i3(bc), C.byref(nw)))
        return bool(nw.value)

    def find_block(self, bc) -> bool:
        f = C.c_int32()
        _check(lib().svx_has_block(self._h, _i3(bc), C.byref(f)))
        return bool(f.value)

    def block_count(self) -> int:
        n = C.c_uint64()
        _check(lib().svx_block_count(self._h, C.byref(n)))
        return int(n.value)

    def block_coords_sorted(self) -> np.ndarray:
        n = C.c_uint64()
        _check(lib().svx_block_keys_sorted(self._h, None, 0, C.byref(n)))
        out = np.zeros((n.value, 3), dtype=np.int32)
        _check(lib().svx_block_keys_sorted(self._h, _ptr(out), n.value, C.byref(n)))
        return out

    def read_block(self, bc):
        """(tsdf[512] structured array, semantics [512,K] or None)."""
        t = np.zeros(BLOCK_VOXELS, dtype=TSDF_DTYPE)
        s = np.zeros((BLOCK_VOXELS, self.cfg.num_labels), dtype=np.float32)
        hs = C.c_int32()
        _check(lib().svx_block_read(self._h, _i3(bc), _ptr(t), _ptr(s), C.byref(hs)))
        return t, (s if hs.value else None)

    def write_block(self, bc, tsdf: np.ndarray, semantics: Optional[np.ndarray] = None,
                    ensure_semantics: bool = False) -> None:
        t = np.ascontiguousarray(tsdf, dtype=TSDF_DTYPE)
        s = None if semantics is None else np.ascontiguousarray(semantics, dtype=np.float32)
        hs = int(ensure_semantics or semantics is not None)
        _check(lib().svx_block_write(self._h, _i3(bc), _ptr(t), _ptr(s), hs))

    def lookup_voxels(self, coords, with_probs: bool = True):
        """Batched VoxelStore::lookup_voxel: (found[n], tsdf[n], probs[n,K])."""
        v = np.ascontiguousarray(np.asarray(coords, dtype=np.int32).reshape(-1, 3))
        n = v.shape[0]
        t = np.zeros(n, dtype=TSDF_DTYPE)
        p = np.zeros((n, self.cfg.num_labels), dtype=np.float32) if with_probs else None
        f = np.zeros(n, dtype=np.uint8)
        if n:
            _check(lib().svx_lookup(self._h, _ptr(v), n, _ptr(t), _ptr(p), _ptr(f)))
        return f.astype(bool), t, p

    def lookup_voxel(self, vc):
        f, t, p = self.lookup_voxels([vc])
        if not f[0]:
            return None
        return t[0], p[0]

    def stats(self) -> StatsC:
        s = StatsC()
        _check(lib().svx_stats_get(self._h, C.byref(s)))
        return s

    def save(self, path: str) -> None:
        _check(lib().svx_save(self._h, str(path).encode()))

    def save_bytes(self) -> bytes:
        n = C.c_uint64()
        _check(lib().svx_save_mem(self._h, None, 0, C.byref(n)))
        buf = np.zeros(n.value, dtype=np.uint8)
        _check(lib().svx_save_mem(self._h, _ptr(buf), n.value, C.byref(n)))
        return buf.tobytes()

    @staticmethod
    def load(path: str, device: int = 0, max_blocks: int = 0) -> "VoxelStore":
        h = C.c_void_p()
        _check(lib().svx_load(str(path).encode(), device, max_blocks, C.byref(h)))
        return VoxelStore(device=device, _handle=h)

    def reserve(self, blocks: int, layers: int = 0) -> None:
        """Map pool memory for `blocks` TSDF blocks / `layers` semantic layers up front."""
        _check(lib().svx_map_reserve(self._h, blocks, layers))

    def has_blocks(self, coords) -> np.ndarray:
        """find_block(b) != nullptr for many blocks at once."""
        b = np.ascontiguousarray(np.asarray(coords, dtype=np.int32).reshape(-1, 3))
        f = np.zeros(b.shape[0], dtype=np.uint8)
        if b.shape[0]:
            _check(lib().svx_has_blocks(self._h, _ptr(b), b.shape[0], _ptr(f)))
        return f.astype(bool)

    def take_dirty_blocks(self, which: int) -> np.ndarray:
        n = C.c_uint64()
        _check(lib().svx_take_dirty_blocks(self._h, which, None, 0, C.byref(n)))
        out = np.zeros((n.value, 3), dtype=np.int32)
        _check(lib().svx_take_dirty_blocks(self._h, which, _ptr(out), n.value, C.byref(n)))
        return out

# ----------------------------------------------------------- preprocessing


@dataclass
class ScanImages:
    """semvox::ScanImages (scan_projection.hpp:44-58) mirrored to host."""
    model: ProjectionModel
    depth: np.ndarray
    height: np.ndarray
    normals: Optional[np.ndarray] = None
    normal_valid: Optional[np.ndarray] = None
    dropped: int = 0

    @property
    def width(self):
        return self.model.width

    @property
    def height_px(self):
        return self.model.height_px

    def has_normals(self) -> bool:
        return self.normals is not None


def _as_points(points) -> tuple[np.ndarray, int]:
    a = np.ascontiguousarray(np.asarray(points, dtype=np.float32))
    if a.ndim != 2 or a.shape[1] not in (3, 4):
        raise InvalidArgument("points must be (n, 3) or (n, 4) float32")
    return a, a.shape[1]


def _download(store: VoxelStore, model: ProjectionModel, normals: bool = True) -> ScanImages:
    s = store.scan(model)
    P = model.width * model.height_px
    d = np.zeros(P, np.float32)
    h = np.zeros(P, np.float32)
    n = np.zeros((P, 3), np.float32)
    v = np.zeros(P, np.uint8)
    dropped = C.c_uint64()
    hn = C.c_int32()
    _check(lib().svx_scan_download(s, _ptr(d), _ptr(h), _ptr(n), _ptr(v), C.byref(dropped),
                                   C.byref(hn)))
    img = ScanImages(model, d, h, None, None, int(dropped.value))
    if normals and hn.value:
        img.normals, img.normal_valid = n, v
    return img


def project_cloud(points, pose, model: ProjectionModel, store: VoxelStore,
                  with_normals: bool = True) -> ScanImages:
    """project_cloud (+ compute_normal_image) on the device of `store`."""
    a, stride = _as_points(points)
    pc = pose if isinstance(pose, PoseC) else (pose.c() if isinstance(pose, Pose) else pose_c(pose))
    s = store.scan(model)
    _check(lib().svx_project(s, _ptr(a), a.shape[0], stride, 0, C.byref(pc)))
    return _download(store, model, normals=with_normals)


def compute_normal_image(img: ScanImages, store: VoxelStore) -> ScanImages:
    s = store.scan(img.model)
    _check(lib().svx_scan_upload(s, _ptr(np.ascontiguousarray(img.depth, np.float32)),
                                 _ptr(np.ascontiguousarray(img.height, np.float32)), None, None))
    _check(lib().svx_compute_normals(s))
    out = _download(store, img.model)
    img.normals, img.normal_valid = out.normals, out.normal_valid
    return img

# -------------------------------------------------------------- integrators


class TsdfIntegrator:
    """semvox::TsdfIntegrator (tsdf_integrator.hpp:75-91)."""

    def __init__(self, store: VoxelStore, cfg: IntegratorConfig = None):
        self.store = store
        self.cfg = cfg or IntegratorConfig()
        if not self.cfg.alpha_epsilon > 0.0:
            raise InvalidArgument("alpha_epsilon must be > 0")

    def integrate_frame(self, images: ScanImages, pose) -> FrameReport:
        s = self.store.scan(images.model)
        nrm = None if images.normals is None else np.ascontiguousarray(images.normals, np.float32)
        val = None if images.normal_valid is None else np.ascontiguousarray(images.normal_valid,
                                                                           np.uint8)
        _check(lib().svx_scan_upload(s, _ptr(np.ascontiguousarray(images.depth, np.float32)),
                                     None, _ptr(nrm), _ptr(val)))
        rep = FrameReportC()
        pc = pose if isinstance(pose, PoseC) else (pose.c() if isinstance(pose, Pose) else pose_c(pose))
        _check(lib().svx_integrate_scan(self.store.handle, s, C.byref(pc), C.byref(self.cfg.c()),
                                        C.byref(rep)))
        return FrameReport.of(rep)

    def integrate_cloud(self, points, pose, model: ProjectionModel) -> FrameReport:
        """project_cloud + compute_normal_image + integrate_frame in one device call."""
        a, stride = _as_points(points)
        pc = pose if isinstance(pose, PoseC) else (pose.c() if isinstance(pose, Pose) else pose_c(pose))
        s = self.store.scan(model)
        rep = FrameReportC()
        _check(lib().svx_integrate_cloud(self.store.handle, s, _ptr(a), a.shape[0], stride, 0,
                                         C.byref(pc), C.byref(self.cfg.c()), C.byref(rep)))
        return FrameReport.of(rep)

    def integrate_cloud_device(self, points, pose, model: ProjectionModel) -> FrameReport:
        """Same as integrate_cloud for a CUDA tensor (n, 3|4) float32 already in HBM.
        The caller orders the tensor's producer before this call (synchronous API)."""
        n, stride = int(points.shape[0]), int(points.shape[1])
        pc = pose if isinstance(pose, PoseC) else (pose.c() if isinstance(pose, Pose) else pose_c(pose))
        s = self.store.scan(model)
        rep = FrameReportC()
        _check(lib().svx_integrate_cloud(self.store.handle, s, C.c_void_p(points.data_ptr()), n,
                                         stride, 1, C.byref(pc), C.byref(self.cfg.c()),
                                         C.byref(rep)))
        return FrameReport.of(rep)

    def take_dirty_blocks(self) -> np.ndarray:
        return self.store.take_dirty_blocks(0)


@dataclass
class LabelImage:
    """semvox::LabelImage (semantic_integrator.hpp:14-26)."""
    width: int
    height: int
    labels: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    pose: object = None
    confidence: Optional[np.ndarray] = None
    prob_tensor: Optional[np.ndarray] = None
    max_depth: float = 30.0


class SemanticIntegrator:
    """semvox::SemanticIntegrator (semantic_integrator.hpp:50-63)."""

    def __init__(self, store: VoxelStore, cfg: SemanticConfig = None):
        self.store = store
        self.cfg = cfg or SemanticConfig()

    def integrate_labels(self, img: LabelImage) -> FrameReport:
        K = self.store.cfg.num_labels
        P = img.width * img.height
        lbl = np.ascontiguousarray(np.asarray(img.labels, np.uint16).reshape(-1))
        if lbl.size != P:
            raise InvalidArgument("labels size mismatch")
        conf = None
        if img.confidence is not None and np.asarray(img.confidence).size == P:
            conf = np.ascontiguousarray(np.asarray(img.confidence, np.float32).reshape(-1))
        ten = None
        if img.prob_tensor is not None and np.asarray(img.prob_tensor).size == P * K:
            ten = np.ascontiguousarray(np.asarray(img.prob_tensor, np.float32).reshape(-1))
        pc = img.pose if isinstance(img.pose, PoseC) else (
            img.pose.c() if isinstance(img.pose, Pose) else pose_c(img.pose))
        li = LabelImageC(img.width, img.height, lbl.ctypes.data_as(C.POINTER(C.c_uint16)),
                         None if conf is None else conf.ctypes.data_as(C.POINTER(C.c_float)),
                         None if ten is None else ten.ctypes.data_as(C.POINTER(C.c_float)),
                         img.fx, img.fy, img.cx, img.cy, pc, img.max_depth)
        rep = FrameReportC()
        _check(lib().svx_integrate_labels(self.store.handle, C.byref(li), C.byref(self.cfg.c()),
                                          C.byref(rep)))
        return FrameReport.of(rep)

    def integrate_labels_batch(self, imgs: list, on_device: bool = False) -> list:
        """Several label images in order with one synchronisation
        (svx_integrate_labels_batch). With on_device, labels / confidence /
        prob_tensor are CUDA tensors (or device pointers) holding the same bytes."""
        K = self.store.cfg.num_labels
        n = len(imgs)
        arr = (LabelImageC * n)()
        keep = []

        def addr(x, dtype):
            if x is None:
                return None
            if on_device:
                return C.c_void_p(x if isinstance(x, int) else x.data_ptr())
            a = np.ascontiguousarray(np.asarray(x, dtype).reshape(-1))
            keep.append(a)
            return C.c_void_p(a.ctypes.data)

        for i, img in enumerate(imgs):
            P = img.width * img.height
            conf = img.confidence if (img.confidence is not None and (
                on_device or np.asarray(img.confidence).size == P)) else None
            ten = img.prob_tensor if (img.prob_tensor is not None and (
                on_device or np.asarray(img.prob_tensor).size == P * K)) else None
            pc = img.pose if isinstance(img.pose, PoseC) else (
                img.pose.c() if isinstance(img.pose, Pose) else pose_c(img.pose))
            arr[i] = LabelImageC(img.width, img.height,
                                 C.cast(addr(img.labels, np.uint16), C.POINTER(C.c_uint16)),
                                 C.cast(addr(conf, np.float32), C.POINTER(C.c_float)),
                                 C.cast(addr(ten, np.float32), C.POINTER(C.c_float)),
                                 img.fx, img.fy, img.cx, img.cy, pc, img.max_depth)
        reps = (FrameReportC * n)()
        _check(lib().svx_integrate_labels_batch(self.store.handle, C.cast(arr, C.c_void_p), n,
                                                int(on_device), C.byref(self.cfg.c()),
                                                C.cast(reps, C.c_void_p)))
        return [FrameReport.of(r) for r in reps]

    def label_array(self, imgs: list, on_device: bool = False):
        """(LabelImageC array, buffers to keep alive) for the C-ABI."""
        K = self.store.cfg.num_labels
        n = len(imgs)
        arr = (LabelImageC * max(n, 1))()
        keep = []

        def addr(x, dtype):
            if x is None:
                return None
            if on_device:
                return C.c_void_p(x if isinstance(x, int) else x.data_ptr())
            a = np.ascontiguousarray(np.asarray(x, dtype).reshape(-1))
            keep.append(a)
            return C.c_void_p(a.ctypes.data)

        for i, img in enumerate(imgs):
            P = img.width * img.height
            conf = img.confidence if (img.confidence is not None and (
                on_device or np.asarray(img.confidence).size == P)) else None
            ten = img.prob_tensor if (img.prob_tensor is not None and (
                on_device or np.asarray(img.prob_tensor).size == P * K)) else None
            pc = img.pose if isinstance(img.pose, PoseC) else (
                img.pose.c() if isinstance(img.pose, Pose) else pose_c(img.pose))
            arr[i] = LabelImageC(img.width, img.height,
                                 C.cast(addr(img.labels, np.uint16), C.POINTER(C.c_uint16)),
                                 C.cast(addr(conf, np.float32), C.POINTER(C.c_float)),
                                 C.cast(addr(ten, np.float32), C.POINTER(C.c_float)),
                                 img.fx, img.fy, img.cx, img.cy, pc, img.max_depth)
        return arr, keep

    def take_dirty_blocks(self) -> np.ndarray:
        return self.store.take_dirty_blocks(1)


def integrate_clouds_labels(store: "VoxelStore", model: ProjectionModel, points_ptr: int, offsets,
                            stride: int, poses: list, icfg: "IntegratorConfig", frame_images: list,
                            scfg: "SemanticConfig" = None, points_on_device: bool = True,
                            labels_on_device: bool = False):
    """svx_integrate_clouds_labels: cmd_integrate's per-frame body over a sequence (the
    TSDF frame, then its label images frame_images[f]) in frame groups. Returns (TSDF
    reports, label reports)."""
    scfg = scfg or SemanticConfig()
    n = len(poses)
    imgs = [li for f in frame_images for li in f]
    img_off = np.zeros(n + 1, np.int32)
    img_off[1:] = np.cumsum([len(f) for f in frame_images])
    arr, keep = SemanticIntegrator(store, scfg).label_array(imgs, labels_on_device)
    offs = np.ascontiguousarray(np.asarray(offsets, np.uint64))
    parr = (PoseC * n)(*poses)
    reps = (FrameReportC * n)()
    lreps = (FrameReportC * max(len(imgs), 1))()
    _check(lib().svx_integrate_clouds_labels(store.handle, store.scan(model), C.c_void_p(points_ptr), _ptr(offs),
                                             stride, int(points_on_device), C.cast(parr, C.c_void_p), n,
                                             C.byref(icfg.c()), C.cast(arr, C.c_void_p), _ptr(img_off),
                                             int(labels_on_device), C.byref(scfg.c()), C.cast(reps, C.c_void_p),
                                             C.cast(lreps, C.c_void_p)))
    del keep
    return [FrameReport.of(r) for r in reps], [FrameReport.of(lreps[i]) for i in range(len(imgs))]


# ------------------------------------------------------------------ mesh

DEFAULT_MESH_MIN_WEIGHT = 1e-4  # kDefaultMeshMinWeight, mesh.hpp:32
UNLABELED = 255                 # kUnlabeled, types.hpp:32


@dataclass
class LabeledMesh:
    """semvox::LabeledMesh (mesh.hpp:11-21) as numpy arrays."""
    vertices: np.ndarray        # [V,3] f32
    faces: np.ndarray           # [F,3] u32
    vertex_labels: np.ndarray   # [V] u8, 255 = unlabeled
    vertex_normals: np.ndarray  # [V,3] f32
    vertex_colors: Optional[np.ndarray] = None  # [V,3] u8 when a label colour table is given

    def vertex_count(self) -> int:
        return int(self.vertices.shape[0])

    def empty(self) -> bool:
        return self.faces.shape[0] == 0


def _reserved_unlabeled(label_names) -> int:
    """reserved_unlabeled_id (mesh.cpp:218-222): a trailing "unlabeled" class."""
    if label_names and label_names[-1] == "unlabeled":
        return len(label_names) - 1
    return -1


def _read_mesh(store: "VoxelStore", nv: int, nf: int, colors) -> LabeledMesh:
    v = np.empty((nv, 3), np.float32)
    n = np.empty((nv, 3), np.float32)
    lab = np.empty(nv, np.uint8)
    f = np.empty((nf, 3), np.uint32)
    _check(lib().svx_mesh_read(store.handle, _ptr(v), _ptr(n), _ptr(lab), _ptr(f)))
    col = None
    if colors is not None:  # LabelSet::color_of_label; gray (128) for unlabeled
        table = np.full((256, 3), 128, np.uint8)
        c = np.asarray(colors, np.uint8).reshape(-1, 3)
        table[:min(len(c), 255)] = c[:255]
        col = table[lab]
    return LabeledMesh(v, f, lab, n, col)


def extract_mesh(store: "VoxelStore", min_weight: float = DEFAULT_MESH_MIN_WEIGHT,
                 label_names=None, label_colors=None, blocks=None) -> LabeledMesh:
    """extract_mesh (mesh.cpp:224-229) on the device; `blocks` restricts the cells to
    those based in the given blocks (None = every allocated block)."""
    nv, nf = C.c_uint64(), C.c_uint64()
    b = None if blocks is None else np.ascontiguousarray(np.asarray(blocks, np.int32).reshape(-1, 3))
    _check(lib().svx_mesh_extract(store.handle, float(min_weight), _reserved_unlabeled(label_names),
                                  _ptr(b), 0 if b is None else b.shape[0], C.byref(nv), C.byref(nf)))
    return _read_mesh(store, nv.value, nf.value, label_colors)


class IncrementalMesher:
    """IncrementalMesher (mesh.hpp:37-63, mesh.cpp:231-287): keeps the set of meshed
    blocks; update() adds the blocks a dirty set affects (D - {0,1}^3) that exist and
    drops those that do not, then re-meshes the set on the device. The stitched mesh
    equals extract_mesh over the set, which is what the reference guarantees for
    blocks that were reported dirty whenever they changed."""

    def __init__(self, min_weight: float = DEFAULT_MESH_MIN_WEIGHT, label_names=None,
                 label_colors=None):
        self.min_weight = min_weight
        self.label_names = label_names
        self.label_colors = label_colors
        self._cache: set = set()
        self.last_remeshed = np.zeros((0, 3), np.int32)
        self.mesh = LabeledMesh(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.uint32),
                                np.zeros(0, np.uint8), np.zeros((0, 3), np.float32))

    def update(self, store: "VoxelStore", dirty) -> LabeledMesh:
        d = np.asarray(dirty, np.int32).reshape(-1, 3)
        off = np.array([(x, y, z) for z in (-1, 0) for y in (-1, 0) for x in (-1, 0)], np.int32)
        aff = np.unique((d[:, None, :] + off[None]).reshape(-1, 3), axis=0) if len(d) else d
        present = store.has_blocks(aff)
        for bc, ok in zip(map(tuple, aff.tolist()), present):
            if ok:
                self._cache.add(bc)
            else:
                self._cache.discard(bc)
        self.last_remeshed = aff[present]
        if not self._cache:
            self.mesh = LabeledMesh(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.uint32),
                                    np.zeros(0, np.uint8), np.zeros((0, 3), np.float32))
            return self.mesh
        blocks = np.array(sorted(self._cache), np.int32)
        self.mesh = extract_mesh(store, self.min_weight, self.label_names, self.label_colors, blocks)
        return self.mesh


# ------------------------------------------------------- occupancy extension


@dataclass
class OccupancyConfig:
    """svx_occ_cfg (include/svx.h): free-space carving + log-odds + hit/miss counters +
    integer class histograms. No reference implementation (parity unpinned)."""
    voxel_size: float = 0.1
    num_labels: int = 20
    max_blocks: int = 1 << 20
    l_hit: float = 0.85
    l_miss: float = -0.4
    l_min: float = -2.0
    l_max: float = 3.5
    min_range: float = 0.3
    max_range: float = 70.0
    carve: bool = True

    def c(self) -> OccCfgC:
        return OccCfgC(self.voxel_size, self.num_labels, self.max_blocks, self.l_hit, self.l_miss,
                       self.l_min, self.l_max, self.min_range, self.max_range, int(self.carve))


class OccupancyMap:
    """Device occupancy map (svx_occ_*)."""

    def __init__(self, cfg: OccupancyConfig = None, device: int = 0):
        self.cfg = cfg or OccupancyConfig()
        self.device = device
        h = C.c_void_p()
        _check(lib().svx_occ_create(C.byref(self.cfg.c()), device, C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().svx_occ_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def handle(self):
        return self._h

    def set_shard(self, rank: int, world: int) -> None:
        _check(lib().svx_occ_set_shard(self._h, rank, world))

    def reserve(self, blocks: int, layers: int = 0) -> None:
        """Map pool memory for `blocks` blocks / `layers` histogram layers up front."""
        _check(lib().svx_occ_reserve(self._h, blocks, layers))

    def integrate(self, points, pose, labels=None, conf=None) -> OccReportC:
        p, stride = _as_points(points)
        n = p.shape[0]
        lb = None if labels is None else np.ascontiguousarray(labels, np.uint16)
        cf = None if conf is None else np.ascontiguousarray(conf, np.float32)
        rep = OccReportC()
        _check(lib().svx_occ_integrate(self._h, _ptr(p), _ptr(lb), _ptr(cf), n, stride, 0,
                                       C.byref(pose), C.byref(rep)))
        return rep

    def integrate_depth(self, depths, cams, poses, labels=None, conf=None) -> list:
        """Pinhole depth images (host arrays): depths[i] is (height, width) f32 metres,
        cams[i] a PinholeC, poses[i] camera->world; labels / conf per pixel or None.
        Each image is one scan (svx.h svx_occ_integrate_depth)."""
        if len(depths) != len(cams) or len(depths) != len(poses):
            raise InvalidArgument("depths, cams and poses must have the same length")
        for d, c in zip(depths, cams):
            if np.shape(d) != (c.height, c.width):
                raise InvalidArgument("depth image shape must be (height, width) of its camera")
        cat = lambda xs, t: None if xs is None else np.ascontiguousarray(  # noqa: E731
            np.concatenate([np.asarray(x, t).reshape(-1) for x in xs]))
        d = cat(depths, np.float32) if len(depths) else np.zeros(0, np.float32)
        lb, cf = cat(labels, np.uint16), cat(conf, np.float32)
        n = len(depths)
        ca, pa, reps = (PinholeC * max(n, 1))(*cams), (PoseC * max(n, 1))(*poses), (OccReportC * max(n, 1))()
        _check(lib().svx_occ_integrate_depth(self._h, _ptr(d), _ptr(lb), _ptr(cf), ca, pa, n, 0, reps))
        return list(reps)[:n]

    def integrate_depth_device(self, d_depth_ptr: int, cams, poses, d_labels_ptr: int = 0,
                               d_conf_ptr: int = 0) -> list:
        """Depth images already in HBM (concatenated, row-major)."""
        n = len(cams)
        ca, pa, reps = (PinholeC * max(n, 1))(*cams), (PoseC * max(n, 1))(*poses), (OccReportC * max(n, 1))()
        _check(lib().svx_occ_integrate_depth(self._h, C.c_void_p(d_depth_ptr), C.c_void_p(d_labels_ptr or None),
                                             C.c_void_p(d_conf_ptr or None), ca, pa, n, 1, reps))
        return list(reps)[:n]

    def integrate_batch_device(self, d_points_ptr: int, offsets: np.ndarray, stride: int, poses,
                               d_labels_ptr: int = 0, d_conf_ptr: int = 0) -> list:
        """Scans already in HBM (device pointers, e.g. torch tensor .data_ptr())."""
        return self._batch(d_points_ptr, offsets, stride, poses, d_labels_ptr, d_conf_ptr, 1)

    def integrate_batch_host(self, points_ptr: int, offsets: np.ndarray, stride: int, poses,
                             labels_ptr: int = 0, conf_ptr: int = 0) -> list:
        """Scans in host memory (pinned for overlap): copied inside the call."""
        return self._batch(points_ptr, offsets, stride, poses, labels_ptr, conf_ptr, 0)

    def _batch(self, pts, offsets, stride, poses, labels, conf, on_device) -> list:
        offs = np.ascontiguousarray(offsets, np.uint64)
        nf = len(offs) - 1
        pa = (PoseC * nf)(*poses)
        reps = (OccReportC * nf)()
        _check(lib().svx_occ_integrate_batch(self._h, C.c_void_p(pts), C.c_void_p(labels or None),
                                             C.c_void_p(conf or None), _ptr(offs), stride, on_device,
                                             pa, nf, reps))
        return list(reps)

    def stream_ptr(self) -> int:
        p = C.c_void_p()
        _check(lib().svx_occ_get_stream(self._h, C.byref(p)))
        return p.value or 0

    def lookup(self, coords) -> dict:
        v = np.ascontiguousarray(np.asarray(coords, np.int32).reshape(-1, 3))
        n, K = v.shape[0], self.cfg.num_labels
        out = {"log_odds": np.zeros(n, np.float32), "hits": np.zeros(n, np.uint32),
               "misses": np.zeros(n, np.uint32), "hist": np.zeros((n, K), np.uint32),
               "label": np.zeros(n, np.int32), "found": np.zeros(n, np.uint8)}
        if n:
            _check(lib().svx_occ_lookup(self._h, _ptr(v), n, _ptr(out["log_odds"]), _ptr(out["hits"]),
                                        _ptr(out["misses"]), _ptr(out["hist"]), _ptr(out["label"]),
                                        _ptr(out["found"])))
        out["found"] = out["found"].astype(bool)
        return out

    def block_count(self) -> int:
        n = C.c_uint64()
        _check(lib().svx_occ_block_count(self._h, C.byref(n)))
        return int(n.value)

    def save_bytes(self) -> bytes:
        n = C.c_uint64()
        _check(lib().svx_occ_save_mem(self._h, None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        _check(lib().svx_occ_save_mem(self._h, _ptr(buf), n.value, C.byref(n)))
        return buf.tobytes()


def block_owner(bc, world: int) -> int:
    return int(lib().svx_block_owner(_i3(bc), world))


__all__ = [
    "MapConfig", "ProjectionModel", "IntegratorConfig", "SemanticConfig", "FrameReport",
    "VoxelStore", "ScanImages", "project_cloud", "compute_normal_image", "TsdfIntegrator",
    "SemanticIntegrator", "LabelImage", "Pose", "pose_c", "CapacityError", "DataError",
    "InvalidArgument", "CudaError", "NotFound", "PROJECTIVE", "NON_PROJECTIVE", "SURROGATE",
    "RAYCAST", "TSDF_DTYPE", "lib", "declared_symbols", "kernel_launches", "block_owner",
    "OccupancyConfig", "OccupancyMap", "LabeledMesh", "extract_mesh", "IncrementalMesher", "DEFAULT_MESH_MIN_WEIGHT", "UNLABELED",
]
