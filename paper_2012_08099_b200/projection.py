"""Discrete projections, API-compatible with the reference projection module
(projection.py:1-228) but computed by the CUDA projection pass.

Index maps (stored ``pixels[j, i]``), projection.py:7-14:
    XY (x, y)  L x M       YZ (y, z)  M x N       ZX (z, x)  N x L
    DIAG (x+z, y)  (L+N-1) x M
    ANTI (x-z, y)  stored at x-z+N-1, origin_offset N-1
Extension (orders 5-6): X2P (x+2z, y) and X2M (x-2z, y) stored at x-2z+2(N-1),
both (L+2N-2) x M -- available through ``project_extended``.
"""
from __future__ import annotations

import enum
import os
import threading
import warnings
from dataclasses import dataclass

import numpy as np

from .counters import OpCounters
from .volume import Volume


class Orientation(enum.Enum):
    XY = "xy"
    YZ = "yz"
    ZX = "zx"
    DIAG = "diag"
    ANTI = "anti"


#: (theta, phi) rotation angles, in radians, for each orientation tag (projection.py:39-45)
ANGLES = {
    Orientation.XY: (0.0, 0.0),
    Orientation.YZ: (0.0, np.pi / 2),
    Orientation.ZX: (np.pi / 2, 0.0),
    Orientation.DIAG: (np.pi / 4, 0.0),
    Orientation.ANTI: (-np.pi / 4, 0.0),
}

#: device image index of each tag (include/dpm_b200.h DPM_IMG_*)
IMAGE_INDEX = {Orientation.XY: 0, Orientation.YZ: 1, Orientation.ZX: 2,
               Orientation.DIAG: 3, Orientation.ANTI: 4}
EXTENDED_NAMES = ("xy", "yz", "zx", "diag", "anti", "x2p", "x2m")


@dataclass(frozen=True, eq=False)
class ProjectionImage:
    """2D integer accumulator image tagged with its orientation (projection.py:48-75).

    ``pixels[j, i]`` (int64, read-only) holds the ray sum at image coordinates
    (i, j); logical index 0 along i sits at ``origin_offset``.
    """

    orientation: Orientation | str
    pixels: np.ndarray
    origin_offset: int = 0

    def __post_init__(self):
        self.pixels.setflags(write=False)

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def mass(self) -> int:
        return int(self.pixels.sum())


@dataclass(frozen=True)
class ProjectionSet:
    """The five projections of one volume; all share the volume's mass."""

    xy: ProjectionImage
    yz: ProjectionImage
    zx: ProjectionImage
    diag: ProjectionImage
    anti: ProjectionImage

    def __getitem__(self, orientation: Orientation) -> ProjectionImage:
        return getattr(self, orientation.value)


def _device_images(volume, n_img: int) -> list[np.ndarray]:
    """Run the CUDA projection pass; widen the uint32 images to int64 numpy."""
    import torch

    from . import engine

    vox = _to_device(volume)
    imgs = engine.project(vox, n_img)
    torch.cuda.current_stream().synchronize()
    return [t[0].cpu().numpy().view(np.uint32).astype(np.int64) for t in imgs]


_TORCH_OF = {}   # numpy dtype -> torch dtype, filled on first use


def _torch_dtypes():
    import torch

    if not _TORCH_OF:
        _TORCH_OF.update({np.dtype("uint8"): torch.uint8, np.dtype("uint16"): torch.uint16})
    return _TORCH_OF


class _Uploader:
    """Host -> device copies of large pageable volumes: plane chunks are copied
    by a thread pool (numpy releases the GIL) into two pinned staging buffers
    while the other buffer's H2D runs on a copy stream -- ~2-3x the driver's
    pageable copy rate.  One per (device, calling thread) -- the staging
    buffers, the copy stream and its events are never shared between
    concurrent callers -- created lazily by ``_uploader()``."""

    CHUNK = int(os.environ.get("DPM_UPLOAD_CHUNK_MB", "256")) << 20   # 64 MB: 0.41-0.60 s per cfg5 volume, 256 MB: 0.35 s
    THREADS = int(os.environ.get("DPM_UPLOAD_THREADS", "8"))

    def __init__(self, device):
        import torch
        from concurrent.futures import ThreadPoolExecutor

        self.device = torch.device(device)
        self.stage = [torch.empty(self.CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        with torch.cuda.device(self.device):
            self.done = [torch.cuda.Event() for _ in range(2)]
            self.stream = torch.cuda.Stream(device=self.device)
        self.pool = ThreadPoolExecutor(self.THREADS)

    def upload(self, arr: np.ndarray):
        import torch

        n = arr.shape[0]
        plane = arr[0].nbytes if n else 1
        per = max(1, self.CHUNK // plane)
        if per * plane > self.CHUNK or plane > self.CHUNK:
            return None                                   # planes larger than a chunk: caller's fallback
        dev = torch.empty(arr.shape, dtype=_torch_dtypes()[arr.dtype], device=self.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        for k, z0 in enumerate(range(0, n, per)):
            z1 = min(n, z0 + per)
            i = k % 2
            self.done[i].synchronize()                    # this staging buffer's previous H2D finished
            view = self.stage[i][: (z1 - z0) * plane].numpy().view(arr.dtype).reshape((z1 - z0,) + arr.shape[1:])
            cuts = np.linspace(z0, z1, min(self.THREADS, z1 - z0) + 1).astype(int)
            list(self.pool.map(lambda ab: np.copyto(view[ab[0] - z0:ab[1] - z0], arr[ab[0]:ab[1]]),
                               zip(cuts[:-1], cuts[1:])))
            with torch.cuda.stream(self.stream):
                dev[z0:z1].copy_(self.stage[i][: (z1 - z0) * plane].view(dev.dtype).view(dev[z0:z1].shape),
                                 non_blocking=True)
                self.done[i].record(self.stream)
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return dev


_UPLOADERS: dict = {}
_UPLOADERS_LOCK = threading.Lock()


def _uploader():
    """This thread's uploader for the current CUDA device."""
    import torch

    key = (torch.cuda.current_device(), threading.get_ident())
    with _UPLOADERS_LOCK:
        up = _UPLOADERS.get(key)
        if up is None:
            up = _UPLOADERS[key] = _Uploader(torch.device("cuda", key[0]))
        return up


def _is_volume(volume) -> bool:
    """This package's Volume, or any object with the reference Volume's shape
    (a numpy ``voxels`` [z, y, x] array and ``dims``), e.g. a reference
    ``volmoments.Volume`` handed to the engine registered in the reference's
    ENGINES."""
    return isinstance(volume, Volume) or (isinstance(getattr(volume, "voxels", None), np.ndarray)
                                          and hasattr(volume, "dims"))


def _to_device(volume):
    import torch

    if _is_volume(volume):
        arr = np.ascontiguousarray(volume.voxels)
        if arr.nbytes >= (32 << 20) and arr.ndim == 3:
            dev = _uploader().upload(arr)
            if dev is not None:
                return dev
        with warnings.catch_warnings():   # read-only voxels are only read (copied to the device), never written
            warnings.simplefilter("ignore", UserWarning)
            host = torch.from_numpy(arr)
        return host.to("cuda", non_blocking=False)
    if isinstance(volume, torch.Tensor):
        if not volume.is_cuda:
            return volume.contiguous().to("cuda")
        return volume
    raise TypeError(f"expected Volume or torch.Tensor, got {type(volume).__name__}")


def _origin(orientation: Orientation, n: int) -> int:
    return n - 1 if orientation is Orientation.ANTI else 0


def _count(counters: OpCounters | None, n_images: int, voxels: int) -> None:
    # the pass is addition-only: P adds per voxel, zero multiplications (projection.py:184-185)
    if counters is not None:
        counters.additions += n_images * voxels


def project(volume: Volume, orientation: Orientation) -> ProjectionImage:
    """Project a volume along one orientation (projection.py:194-197)."""
    imgs = _device_images(volume, 5 if orientation is Orientation.ANTI else 4)
    n = volume.dims[2]
    return ProjectionImage(orientation, imgs[IMAGE_INDEX[orientation]], _origin(orientation, n))


def project_all(volume: Volume, counters: OpCounters | None = None) -> ProjectionSet:
    """All five projections in ONE streaming pass over the voxels (projection.py:200-203)."""
    imgs = _device_images(volume, 5)
    n = volume.dims[2]
    _count(counters, 5, volume.voxels.size)
    return ProjectionSet(*(ProjectionImage(o, imgs[IMAGE_INDEX[o]], _origin(o, n)) for o in Orientation))


def project_subset(volume: Volume, wanted: tuple[Orientation, ...],
                   counters: OpCounters | None = None) -> dict[Orientation, ProjectionImage]:
    """Single-pass projection of just the requested orientations (projection.py:206-210)."""
    need = 5 if Orientation.ANTI in wanted else 4
    imgs = _device_images(volume, need)
    n = volume.dims[2]
    _count(counters, len(wanted), volume.voxels.size)
    return {o: ProjectionImage(o, imgs[IMAGE_INDEX[o]], _origin(o, n)) for o in wanted}


def project_extended(volume: Volume) -> dict[str, ProjectionImage]:
    """All seven images of the order-6 method, keyed by name (xy ... x2m)."""
    imgs = _device_images(volume, 7)
    n = volume.dims[2]
    offs = {"anti": n - 1, "x2m": 2 * (n - 1)}
    return {name: ProjectionImage(name, imgs[k], offs.get(name, 0)) for k, name in enumerate(EXTENDED_NAMES)}


def write_pgm(image: ProjectionImage, path) -> None:
    """Dump an image as 16-bit binary PGM, rescaled to full range, with the
    scale factor in a comment line (projection.py:213-228)."""
    peak = int(image.pixels.max()) if image.pixels.size else 0
    scale = 65535.0 / peak if peak > 0 else 1.0
    scaled = np.round(image.pixels * scale).astype(">u2")
    tag = image.orientation.value if isinstance(image.orientation, Orientation) else str(image.orientation)
    header = f"P5\n# volmoments {tag} projection, scale={scale!r}\n{image.width} {image.height}\n65535\n"
    with open(path, "wb") as fh:
        fh.write(header.encode("ascii"))
        fh.write(scaled.tobytes())
