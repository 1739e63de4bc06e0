"""Device-resident occupancy mapping and exact distance fields.

Drop-in counterpart of vp/mapping.py.  The grid state lives in HBM
(``log_odds`` f64, ``observed`` u8 and a packed 1-bit occupancy mask kept in
sync by the fusion kernel), every update and transform is a libvpb200 kernel,
and host copies are made only when a caller asks for numpy arrays.

Layout: dense C-order ``x * (Ny*Nz) + y * Nz + z`` (vp/mapping.py:3-4); the
occupancy mask packs z into 32-bit words per (x, y) line.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field as dc_field
from enum import IntEnum

import numpy as np
import torch

from . import _device as D
from ._lib import VpbCamera, VpbField, VpbGrid, VpbJournal, VpbMapParams, check, fill, i64x3, load
from .errors import FrameMismatch, VolumeOutOfBounds
from .geometry import RigidTransform

INF_SENTINEL = 1e20  # vp/mapping.py:32 (kept for API parity; the GPU EDT uses exact ints)
DEFAULT_MASK_PAD = 0.01  # vp/mapping.py:383


class VoxelState(IntEnum):
    UNKNOWN = 0
    FREE = 1
    OCCUPIED = 2


@dataclass(frozen=True)
class MapParams:
    """vp/mapping.py:41-50."""

    l_hit: float = 0.85
    l_miss: float = -0.4
    l_min: float = -2.0
    l_max: float = 3.5
    l_occ_threshold: float = 1.0
    tau_factor: float = 2.5


@dataclass(frozen=True)
class VoxelBox:
    """Half-open voxel index box [lo, hi) (vp/mapping.py:53-73)."""

    lo: tuple[int, int, int]
    hi: tuple[int, int, int]

    def __post_init__(self):
        lo = tuple(int(v) for v in self.lo)
        hi = tuple(int(v) for v in self.hi)
        if any(h <= l for l, h in zip(lo, hi)):
            raise ValueError(f"empty voxel box lo={lo} hi={hi}")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(h - l for l, h in zip(self.lo, self.hi))

    def slices(self):
        return tuple(slice(l, h) for l, h in zip(self.lo, self.hi))

    def native(self):
        """(lo, shape) as cached int64[3] ctypes arrays."""
        n = self.__dict__.get("_native")
        if n is None:
            n = (i64x3(self.lo), i64x3(self.shape))
            object.__setattr__(self, "_native", n)
        return n


class VoxelGrid:
    """Dense occupancy grid in device memory (vp/mapping.py:76-140).

    ``log_odds`` / ``observed`` are CUDA tensors.  Reading the ``log_odds``
    property hands out a writable tensor, so the packed occupancy mask is
    re-derived before the next transform; the mapper pipeline uses the
    internal tensors and keeps the mask current from inside the fusion kernel.
    """

    def __init__(self, origin, voxel_size: float, dims, params: MapParams | None = None, device=None):
        origin = np.asarray(origin, dtype=float).reshape(3)
        dims = tuple(int(d) for d in dims)
        if any(d < 1 for d in dims):
            raise ValueError(f"grid dims must be >= 1, got {dims}")
        if voxel_size <= 0.0:
            raise ValueError(f"voxel size must be positive, got {voxel_size}")
        self.device = D.device(device)
        self.origin = origin
        self.voxel_size = float(voxel_size)
        self.dims = dims
        self.params = params or MapParams()
        self._log_odds = torch.zeros(dims, dtype=torch.float64, device=self.device)
        self._observed = torch.zeros(dims, dtype=torch.uint8, device=self.device)
        words = int(load().vpb_occ_words(i64x3(dims)))
        self._occ_bits = torch.zeros(words, dtype=torch.int32, device=self.device)
        self._bits_valid = True
        self._frozen = False
        self._native = None  # cached VpbGrid (device pointers are stable until a tensor is replaced)
        self._native_params = None
        self._snaps: list = []  # weakrefs to the live (unmaterialised) snapshots of this grid
        self._journal = None

    # -- state access -------------------------------------------------------
    @property
    def log_odds(self) -> torch.Tensor:
        if not self._frozen:
            self._detach_snapshots()  # the caller may write through this handle
            self._bits_valid = False
        return self._log_odds

    @log_odds.setter
    def log_odds(self, value) -> None:
        if self._frozen:
            raise ValueError("cannot modify a frozen grid snapshot")
        self._detach_snapshots()
        self._log_odds = torch.as_tensor(value, dtype=torch.float64, device=self.device).reshape(self.dims).contiguous()
        self._bits_valid = False
        self._native = None

    @property
    def observed(self) -> torch.Tensor:
        if not self._frozen:
            self._detach_snapshots()  # a writable view
        return self._observed.view(torch.bool)

    def log_odds_host(self) -> np.ndarray:
        return self._log_odds.cpu().numpy()

    def observed_host(self) -> np.ndarray:
        return self._observed.cpu().numpy().astype(bool)

    def set_log_odds(self, values) -> None:
        """Overwrite the whole log-odds grid from host or device data."""
        self.log_odds = values

    def mark_occupied(self, mask, value: float | None = None) -> None:
        """log_odds[mask] = value (default l_max), like `grid.log_odds[occ] = l_max`."""
        if self._frozen:
            raise ValueError("cannot modify a frozen grid snapshot")
        self._detach_snapshots()
        m = torch.as_tensor(np.asarray(mask, dtype=bool) if not torch.is_tensor(mask) else mask,
                            device=self.device)
        self._log_odds[m] = self.params.l_max if value is None else float(value)
        self._bits_valid = False

    @property
    def tau(self) -> float:
        return self.params.tau_factor * self.voxel_size

    def full_box(self) -> VoxelBox:
        fb = self.__dict__.get("_full_box")
        if fb is None:  # (VoxelBox is frozen: one shared instance caches its native views)
            fb = self.__dict__["_full_box"] = VoxelBox((0, 0, 0), self.dims)
        return fb

    def voxel_center(self, index) -> np.ndarray:
        return self.origin + (np.asarray(index, dtype=float) + 0.5) * self.voxel_size

    def world_to_voxel(self, point) -> np.ndarray:
        return np.floor((np.asarray(point, dtype=float) - self.origin) / self.voxel_size).astype(np.int64)

    def occupied_mask(self) -> torch.Tensor:
        return self._log_odds >= self.params.l_occ_threshold

    def states(self) -> torch.Tensor:
        """VoxelState per voxel (vp/mapping.py:116-123)."""
        occ = self.occupied_mask()
        free = self.observed & (self._log_odds <= 0.0) & ~occ
        out = torch.zeros(self.dims, dtype=torch.int8, device=self.device)
        out[free] = int(VoxelState.FREE)
        out[occ] = int(VoxelState.OCCUPIED)
        return out

    def freeze(self) -> "VoxelGrid":
        """Immutable snapshot (vp/mapping.py:125-133) in O(1): a copy-on-write
        view.  While it is alive, every fusion into this grid journals the
        words it modifies (old values, on the device); the snapshot's own
        state is materialised -- clone of the live grid + the undo records,
        newest update first -- only if it is ever read.  A snapshot that is
        dropped unread (the planner reads only the field) never costs a copy."""
        if self._frozen:
            return self
        snap = SnapshotGrid(self)
        self._snaps.append(weakref.ref(snap))
        return snap

    # -- copy-on-write snapshots ------------------------------------------------
    def _live_snaps(self) -> list:
        live = [r() for r in self._snaps]
        live = [g for g in live if g is not None and g._state is None]
        self._snaps = [weakref.ref(g) for g in live]
        return live

    def _detach_snapshots(self) -> None:
        """Before an unjournaled in-place change: give every live snapshot its own state."""
        for g in self._live_snaps():
            g._materialize()
        self._snaps = []
        if self._journal is not None:
            self._journal.reset()

    def _journal_for_update(self, box: "VoxelBox"):
        """The journal struct for the next fusion (None if no snapshot is alive)."""
        live = self._live_snaps()
        j = self._journal
        if not live:
            if j is not None:
                j.reset()
            return None
        if j is None:
            j = self._journal = _Journal(self)
        if min(g._seg for g in live) == j.nseg:  # nothing journaled so far is still needed
            j.reset()
            for g in live:
                g._seg = 0
        words = box.shape[0] * box.shape[1] * ((box.hi[2] - 1) // 32 - box.lo[2] // 32 + 1)
        if j.nseg == _Journal.MAX_SEG:  # a snapshot outlived too many updates: give it its own state
            self._detach_snapshots()
            return None
        return j.begin_segment(words)

    def validate_box(self, box: VoxelBox) -> None:
        for axis in range(3):
            if box.lo[axis] < 0 or box.hi[axis] > self.dims[axis]:
                raise VolumeOutOfBounds(f"volume {box.lo}..{box.hi} exceeds grid dims {self.dims}")

    # -- native views ---------------------------------------------------------
    def _struct(self) -> VpbGrid:
        if self._native is not None:
            return self._native
        g = VpbGrid()
        g.log_odds = D.ptr(self._log_odds)
        g.observed = D.ptr(self._observed)
        g.occ_bits = D.ptr(self._occ_bits)
        g.dims = i64x3(self.dims)
        fill(g.origin, self.origin)
        g.voxel = self.voxel_size
        self._native = g
        return g

    def _ensure_bits(self) -> None:
        if not self._bits_valid:
            g = self._struct()
            check(load().vpb_occ_bits_from_log_odds(g, self.params.l_occ_threshold, D.stream(self.device)),
                  "occupancy mask")
            self._bits_valid = True


class _Journal:
    """Undo records of one live grid (include/vpb200.h vpb_journal): device
    buffers grown on demand, one segment per journaled update."""

    MAX_SEG = 16
    RECORD_BYTES = 8 + 32 * 8 + 32 + 4

    def __init__(self, grid: VoxelGrid):
        self.dev = grid.device
        self.cap = 0
        self.bound = 0  # host upper bound of the records written (one per box word per update)
        self.nseg = 0
        self.count = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.starts = torch.zeros(self.MAX_SEG, dtype=torch.int64, device=self.dev)
        self.idx = self.lo = self.ob = self.occ = None
        self._struct = None
        self._pending_reset = False

    def reset(self) -> None:
        # the record count is zeroed on the device by the next journaled
        # update itself (vpb_journal.reset), not by a launch of its own
        if self.nseg or self.bound:
            self._pending_reset = True
        self.nseg = 0
        self.bound = 0

    def _grow(self, cap: int) -> None:
        new = (torch.empty(cap, dtype=torch.int64, device=self.dev),
               torch.empty(cap * 32, dtype=torch.float64, device=self.dev),
               torch.empty(cap * 32, dtype=torch.uint8, device=self.dev),
               torch.empty(cap, dtype=torch.int32, device=self.dev))
        if self.idx is not None and self.bound:
            keep = min(self.bound, self.cap)
            for a, b, k in zip(new, (self.idx, self.lo, self.ob, self.occ), (1, 32, 32, 1)):
                a[:keep * k].copy_(b[:keep * k])
        self.idx, self.lo, self.ob, self.occ = new
        self.cap = cap
        j = VpbJournal()
        j.idx, j.lo, j.ob, j.occ = (D.ptr(t) for t in new)
        j.count, j.overflow, j.capacity = D.ptr(self.count), D.ptr(self.overflow), cap
        j.starts = D.ptr(self.starts)
        self._struct = j

    def begin_segment(self, words: int) -> VpbJournal:
        if self.bound + words > self.cap:
            if self._pending_reset:  # (_grow keeps the first `bound` records, none after a reset)
                self.count.zero_()
                self._pending_reset = False
            self._grow(max(2 * self.cap, self.bound + words))
        # starts[nseg] = count (after the pending reset, if any), on the device
        # at the start of the update (vpb_journal.seg / reset)
        j = self._struct
        j.seg = self.nseg
        j.reset = 1 if self._pending_reset else 0
        self._pending_reset = False
        self.nseg += 1
        self.bound += words
        return j

    def restore_into(self, grid: "SnapshotGrid", first_seg: int) -> None:
        """Write the undo records of segments nseg-1 .. first_seg (newest first) into grid."""
        if first_seg >= self.nseg:
            return
        ends = torch.cat([self.starts[:self.nseg], self.count]).cpu().numpy()
        if int(self.overflow.item()):
            raise RuntimeError("snapshot journal overflow (sizing bug)")
        L = load()
        st = grid._struct()
        for k in range(self.nseg - 1, first_seg - 1, -1):
            check(L.vpb_journal_restore(st, self._struct, int(ends[k]), int(ends[k + 1]), D.stream(self.dev)),
                  "journal_restore")


class SnapshotGrid(VoxelGrid):
    """Frozen VoxelGrid produced by VoxelGrid.freeze(): reads materialise it."""

    def __init__(self, live: VoxelGrid):  # noqa: D401 - no VoxelGrid.__init__ (no allocation)
        self.device = live.device
        self.origin = live.origin.copy()
        self.voxel_size = live.voxel_size
        self.dims = live.dims
        self.params = live.params
        self._frozen = True
        self._native = None
        self._native_params = None
        self._snaps = []
        self._journal = None
        self._live = live
        self._seg = live._journal.nseg if live._journal is not None else 0
        self._bits_at_freeze = live._bits_valid
        self._state = None  # (log_odds, observed, occ_bits) once materialised

    def _materialize(self):
        if self._state is None:
            live = self._live
            state = (live._log_odds.clone(), live._observed.clone(), live._occ_bits.clone())
            self._state = state
            if live._journal is not None:
                live._journal.restore_into(self, self._seg)
            self._live = None
        return self._state

    @property
    def _log_odds(self):
        return self._materialize()[0]

    @property
    def _observed(self):
        return self._materialize()[1]

    @property
    def _occ_bits(self):
        return self._materialize()[2]

    @property
    def _bits_valid(self):
        return self._bits_at_freeze

    @_bits_valid.setter
    def _bits_valid(self, value):
        self._bits_at_freeze = value

    def _struct(self) -> VpbGrid:
        if self._state is None:  # restore needs the clone's pointers: materialise first
            self._materialize()
        return VoxelGrid._struct(self)


@dataclass(frozen=True)
class CameraModel:
    """Pinhole depth camera; pose maps camera to world (vp/mapping.py:143-166)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    d_min: float
    d_max: float
    pose: RigidTransform = dc_field(default_factory=RigidTransform.identity)

    def __post_init__(self):
        if self.fx <= 0.0 or self.fy <= 0.0:
            raise ValueError("focal lengths must be positive")
        if not 0.0 < self.d_min < self.d_max:
            raise ValueError(f"need 0 < d_min < d_max, got [{self.d_min}, {self.d_max}]")

    def world_to_camera(self):
        inv = self.pose.inverse()
        return inv.rotation.matrix, inv.translation

    def _struct(self) -> VpbCamera:
        cached = self.__dict__.get("_native")
        if cached is not None:
            return cached
        c = VpbCamera()
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        c.d_min, c.d_max = self.d_min, self.d_max
        c.width, c.height = int(self.width), int(self.height)
        fill(c.pose_r, self.pose.rotation.matrix)
        fill(c.pose_t, self.pose.translation)
        r, t = self.world_to_camera()
        fill(c.w2c_r, r)
        fill(c.w2c_t, t)
        object.__setattr__(self, "_native", c)  # frozen: the struct never changes
        return c


class DepthImage:
    """Row-major depth raster in meters; 0 or NaN = no return (vp/mapping.py:187-202).

    Accepts host (numpy) or device (torch CUDA) data; the device copy is made
    once and cached."""

    def __init__(self, data):
        if torch.is_tensor(data):
            if data.ndim != 2:
                raise ValueError(f"depth image must be 2-D, got shape {tuple(data.shape)}")
            self._dev = data.to(torch.float64).contiguous()
            self._host = None
        else:
            a = np.asarray(data, dtype=np.float64)
            if a.ndim != 2:
                raise ValueError(f"depth image must be 2-D, got shape {a.shape}")
            self._host = a
            self._dev = None

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host

    @property
    def shape(self):
        return tuple(self._dev.shape) if self._dev is not None else self._host.shape

    @property
    def height(self) -> int:
        return self.shape[0]

    @property
    def width(self) -> int:
        return self.shape[1]

    def device_tensor(self, dev: torch.device) -> torch.Tensor:
        if self._dev is None or self._dev.device != dev:
            src = self._host if self._host is not None else self._dev.cpu().numpy()
            self._dev = _upload_depth(np.ascontiguousarray(src), dev)
        return self._dev


# Depth frames reach the device through two pinned staging buffers per shape
# (ping-pong, each guarded by the event of its last copy): the H2D copy is
# asynchronous on the current stream instead of a pageable, host-blocking one.
_PINNED: dict = {}


def _upload_depth(src: np.ndarray, dev: torch.device) -> torch.Tensor:
    key = (src.shape, dev)
    slots = _PINNED.get(key)
    if slots is None:
        slots = _PINNED[key] = [[torch.empty(src.shape, dtype=torch.float64, pin_memory=True), None]
                                for _ in range(2)]
    slot = slots.pop(0)
    slots.append(slot)
    pin, ev = slot
    if ev is not None:
        ev.synchronize()  # the copy that last read this buffer is done
    src = np.ascontiguousarray(src, dtype=np.float64)
    out = torch.empty(src.shape, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    # host copy into the pinned slot + the async H2D in one native call (the
    # numpy copy + tensor copy_ pair cost ~25 us of host time per frame)
    check(load().vpb_stage_h2d(D.ptr(out), pin.data_ptr(), src.ctypes.data, src.nbytes, stream.cuda_stream),
          "depth upload")
    if ev is None:
        ev = slot[1] = torch.cuda.Event()
    ev.record(stream)
    return out


def _mask_arrays(mask):
    if mask is None:
        return np.zeros((0, 3)), np.zeros(0)
    centers = np.ascontiguousarray(mask[0], dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(mask[1], dtype=np.float64).reshape(-1)
    if centers.shape[0] != radii.shape[0]:
        raise ValueError("mask centers and radii disagree in count")
    return centers, radii


def _map_params(grid: VoxelGrid) -> VpbMapParams:
    if grid._native_params is None:
        p = grid.params
        grid._native_params = VpbMapParams(p.l_hit, p.l_miss, p.l_min, p.l_max, p.l_occ_threshold, grid.tau)
    return grid._native_params


def update_occupancy(grid: VoxelGrid, depth: DepthImage, cam: CameraModel, mask=None,
                     volume: VoxelBox | None = None, mask_pad: float = DEFAULT_MASK_PAD) -> VoxelGrid:
    """Fuse one depth image by voxel projection (vp/mapping.py:386-455).

    Same validation and errors as the reference; the masked-pixel test and
    the fusion run as two kernels on the current stream.  Mutates and
    returns ``grid``."""
    if grid._frozen:
        raise ValueError("cannot update a frozen grid snapshot")
    if not isinstance(depth, DepthImage):
        depth = DepthImage(depth)
    if tuple(depth.shape) != (cam.height, cam.width):
        raise FrameMismatch(f"depth image is {tuple(depth.shape)}, camera expects {(cam.height, cam.width)}")
    box = volume or grid.full_box()
    grid.validate_box(box)
    grid._ensure_bits()
    centers, radii = _mask_arrays(mask)
    dev = grid.device
    d_dev = depth.device_tensor(dev)
    scratch = D.Workspace.get(dev, "pixel_mask", int(load().vpb_pixel_scratch_bytes(cam.width, cam.height)),
                              zeroed=True)
    blo, bn = box.native()
    journal = grid._journal_for_update(box) if grid._snaps else None
    check(load().vpb_update_occupancy_journaled(
        grid._struct(), blo, bn, cam._struct(), D.ptr(d_dev),
        D.host_ptr(centers), D.host_ptr(radii), centers.shape[0], float(mask_pad),
        _map_params(grid), D.ptr(scratch), journal, D.stream(dev)), "update_occupancy")
    return grid


def masked_pixels(depth: DepthImage, cam: CameraModel, centers, radii, pad: float) -> torch.Tensor:
    """Device version of vp/mapping.py:357-380 (bool H x W tensor)."""
    centers, radii = _mask_arrays((centers, radii))
    dev = D.device()
    d_dev = depth.device_tensor(dev)
    out = torch.empty((cam.height, cam.width), dtype=torch.uint8, device=dev)
    check(load().vpb_masked_pixels(D.ptr(d_dev), cam._struct(), D.host_ptr(centers), D.host_ptr(radii),
                                   centers.shape[0], float(pad), D.ptr(out), D.stream(dev)), "masked_pixels")
    return out.view(torch.bool)


@dataclass(frozen=True, eq=False)
class DistanceField:
    """Squared voxel distances to the nearest occupied voxel over one box
    (vp/mapping.py:556-583).  ``sq_device`` is the f32 device tensor the
    planner reads (exact integers, +inf = no source in the volume); ``sq``
    is the float64 host copy the reference exposes, made on first access."""

    origin: np.ndarray
    voxel_size: float
    dims: tuple[int, int, int]
    volume: VoxelBox
    sq_device: torch.Tensor
    outside_default: float

    def __post_init__(self):
        if tuple(self.sq_device.shape) != self.volume.shape:
            raise ValueError(f"sq shape {tuple(self.sq_device.shape)} != volume shape {self.volume.shape}")
        o = np.asarray(self.origin, dtype=float).reshape(3).copy()
        o.flags.writeable = False
        object.__setattr__(self, "origin", o)
        object.__setattr__(self, "_sq_host", None)
        object.__setattr__(self, "_sq_ptr", self.sq_device.data_ptr())  # the per-step native call passes it

    @property
    def sq(self) -> np.ndarray:
        if self._sq_host is None:
            h = self.sq_device.to(torch.float64).cpu().numpy()
            h.flags.writeable = False
            object.__setattr__(self, "_sq_host", h)
        return self._sq_host

    def metric(self) -> np.ndarray:
        return self.voxel_size * np.sqrt(self.sq)

    def _struct(self) -> VpbField:
        f = VpbField()
        f.sq = D.ptr(self.sq_device)
        f.n = i64x3(self.volume.shape)
        f.lo = i64x3(self.volume.lo)
        fill(f.origin, self.origin)
        f.voxel = self.voxel_size
        f.outside_default = float(self.outside_default)
        return f


def edt_3d(grid: VoxelGrid, volume: VoxelBox | None = None, outside_default: float = 1.0,
           pass_order: tuple[str, str, str] = ("y", "x", "z")) -> DistanceField:
    """Exact squared EDT of the occupied voxels in ``volume`` (vp/mapping.py:586-613).

    The result is the exact squared distance and therefore independent of
    ``pass_order`` (validated for API parity)."""
    box = volume or grid.full_box()
    grid.validate_box(box)
    if pass_order != ("y", "x", "z") and sorted(pass_order) != ["x", "y", "z"]:
        raise ValueError(f"pass_order must permute x, y, z; got {pass_order}")
    grid._ensure_bits()
    dev = grid.device
    blo, n = box.native()
    L = load()
    ws_bytes = box.__dict__.get("_edt_ws_bytes")
    if ws_bytes is None:
        ws_bytes = int(L.vpb_edt3d_workspace_bytes(n))
        object.__setattr__(box, "_edt_ws_bytes", ws_bytes)
    ws = D.Workspace.get(dev, "edt", ws_bytes)
    out = torch.empty(box.shape, dtype=torch.float32, device=dev)
    check(L.vpb_edt3d(grid._struct(), blo, n, grid.params.l_occ_threshold, 1, D.ptr(out),
                      D.ptr(ws), ws.numel(), D.stream(dev)), "edt_3d")
    return DistanceField(grid.origin, grid.voxel_size, grid.dims, box, out, float(outside_default))


def query_distances(field: DistanceField, points) -> np.ndarray:
    """Batched vp/mapping.py:688-710 on the device (fp64, reference order)."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    dev = field.sq_device.device
    p_dev = torch.from_numpy(pts).to(dev)
    out = torch.empty(pts.shape[0], dtype=torch.float64, device=dev)
    check(load().vpb_query_distance(field._struct(), D.ptr(p_dev), pts.shape[0], D.ptr(out), D.stream(dev)),
          "query_distance")
    return out.cpu().numpy()


def query_distance(field: DistanceField, point) -> float:
    """Metric distance at a world point (vp/mapping.py:688-710)."""
    return float(query_distances(field, np.asarray(point, dtype=float).reshape(1, 3))[0])


@dataclass(frozen=True)
class MapSnapshot:
    grid: VoxelGrid
    field: DistanceField


def snapshot(grid: VoxelGrid, field: DistanceField) -> MapSnapshot:
    """vp/mapping.py:713-723."""
    return MapSnapshot(grid.freeze(), field)


class OccupancyMapper:
    """Single-writer pipeline update -> EDT -> publish (vp/mapping.py:726-767),
    with all state resident on the device."""

    def __init__(self, grid: VoxelGrid, cam: CameraModel, volume: VoxelBox | None = None,
                 outside_default: float = 1.0, mask_pad: float = DEFAULT_MASK_PAD):
        self.grid = grid
        self.cam = cam
        self.volume = volume or grid.full_box()
        grid.validate_box(self.volume)
        self.outside_default = float(outside_default)
        self.mask_pad = float(mask_pad)
        self._field: DistanceField | None = None

    def update(self, depth, mask=None) -> None:
        update_occupancy(self.grid, depth, self.cam, mask=mask, volume=self.volume, mask_pad=self.mask_pad)

    def recompute_edt(self) -> DistanceField:
        self._field = edt_3d(self.grid, self.volume, self.outside_default)
        return self._field

    def snapshot(self) -> MapSnapshot:
        if self._field is None:
            self.recompute_edt()
        return snapshot(self.grid, self._field)
