"""3D raw moments through the CUDA DPM pipeline, API-compatible with the
reference moments3d module (moments3d.py:27-278).

``dpm_moments`` keeps the reference signature and returns exact Python ints:
the device computes every 2D and 3D moment exactly in 128-bit integers
(paper_2012_08099_b200/csrc/moments2d.cu, derive3d.cu).  Orders 3..6 are
accepted (the reference accepts 3 and 4; 5 and 6 add the (x+-2z, y) images).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native as nat
from .counters import OpCounters
from .errors import InconsistencyError
from .volume import Volume


@dataclass(frozen=True)
class MomentTensor3:
    """Raw moments M[p][q][r] for p + q + r <= order, exact integers (moments3d.py:27-43)."""

    order: int
    values: dict[tuple[int, int, int], int]

    def __getitem__(self, pqr: tuple[int, int, int]) -> int:
        return self.values[pqr]

    def items(self):
        """(index, value) pairs in lexicographic (p, q, r) order."""
        return sorted(self.values.items())

    @property
    def mass(self) -> int:
        return self.values[(0, 0, 0)]

    def as_float64(self) -> np.ndarray:
        """Values in moment_indices order as fp64."""
        return np.array([float(self.values[k]) for k in moment_indices(self.order)], dtype=np.float64)


@lru_cache(maxsize=8)
def moment_indices(order: int) -> tuple[tuple[int, int, int], ...]:
    """All (p, q, r) with p + q + r <= order, lexicographically sorted (moments3d.py:46-54)."""
    return tuple((p, q, r) for p in range(order + 1) for q in range(order + 1 - p)
                 for r in range(order + 1 - p - q))


_STATUS_TEXT = (
    (nat.DPM_ST_DISAGREE, "projection routes disagree on a duplicated moment"),
    (nat.DPM_ST_NONEXACT, "an exact division left a remainder"),
    (nat.DPM_ST_MASS, "projection image masses disagree"),
)


def raise_status(status: int, where: str = "dpm") -> None:
    """Map the device status word to InconsistencyError (errors.py:8-15)."""
    if status:
        msgs = [t for bit, t in _STATUS_TEXT if status & bit]
        raise InconsistencyError(f"{where}: " + "; ".join(msgs) + f" (status {status})")


def _count(counters: OpCounters | None, order: int, dims) -> None:
    """Analytic tallies of the device method (see counters.py)."""
    if counters is None:
        return
    from .engine import num_images
    l, m, n = dims
    p = num_images(order)
    counters.additions += p * l * m * n                     # projection pass: P - 1 images + the profile
    widths = [l + n - 1, l + n - 1, l + 2 * n - 2, l + 2 * n - 2][: p - 3]
    t = {3: 1, 4: 2, 5: 2, 6: 3}[order]
    px = l * m + m * n + sum(widths) * m + (l + t * (n - 1))  # image pixels + profile cells
    counters.multiplications += (order + 1) * px              # row-power products
    counters.additions += (order + 1) * px


def dpm_moments(volume: Volume, order: int, counters: OpCounters | None = None,
                check_consistency: bool = True) -> MomentTensor3:
    """Projection-based engine on the GPU (moments3d.py:232-264).

    Pipeline: one streaming projection pass -> exact 2D moments of every image
    -> device epilogue (placement, duplicate-route checks, cross-axis solve).
    With ``check_consistency`` any failed check raises InconsistencyError.
    """
    import torch

    from . import engine
    from .projection import _to_device

    engine.check_order(order)
    vox = _to_device(volume)
    res = engine.moments(vox, order)
    torch.cuda.current_stream().synchronize()
    st = int(res.status[0].item())
    if check_consistency:
        raise_status(st)
    vals = engine.i128_to_ints(res.i128[0].cpu().numpy())
    dims = tuple(volume.dims) if hasattr(volume, "dims") else tuple(reversed(vox.shape[-3:]))
    _count(counters, order, dims)
    return MomentTensor3(order, dict(zip(moment_indices(order), vals)))


def dpm_moments_file(source, order: int, meta=None, chunk_planes: int = 64, counters: OpCounters | None = None,
                     check_consistency: bool = True) -> MomentTensor3:
    """``dpm_moments`` of a volume file streamed slab by slab (SURVEY.md §8(f)
    row 1): ``source`` is a raw path (with ``meta``, a ``VolumeMeta``), an
    NRRD path, or a ``Volume`` (e.g. memory-mapped).  The volume never has to
    fit in host or device memory; results are identical to ``dpm_moments``."""
    import torch

    from . import engine, volio
    from .streaming import FileStreamer

    engine.check_order(order)
    if isinstance(source, Volume):
        vol = source
    elif meta is not None:
        vol = volio.open_raw(source, meta)
    else:
        vol = volio.open_nrrd(source)
    l, m, n = vol.dims
    engine.check_envelope(l, m, n, nat.DPM_U8 if vol.bit_depth == 8 else nat.DPM_U16, order)
    fs = FileStreamer((n, m, l), vol.voxels.dtype, order, chunk_planes=chunk_planes)
    res = fs.moments(vol.voxels)
    torch.cuda.current_stream().synchronize()
    st = int(res.status[0].item())
    if check_consistency:
        raise_status(st)
    vals = engine.i128_to_ints(res.i128[0].cpu().numpy())
    _count(counters, order, vol.dims)
    return MomentTensor3(order, dict(zip(moment_indices(order), vals)))


def dpm_moments_batch(volumes, order: int, check_consistency: bool = True, offset: int = 0,
                      as_float: bool = False):
    """Moments of a batch of equally shaped volumes ([B, N, M, L] numpy or torch).

    Returns a list of MomentTensor3 (exact), or with ``as_float`` the [B, n3d]
    fp64 array.  The reference has no batch type; this is the config-4 entry.
    """
    import torch

    from . import engine

    engine.check_order(order)
    if isinstance(volumes, torch.Tensor):
        vox = volumes if volumes.is_cuda else volumes.to("cuda")
    else:
        arr = np.ascontiguousarray(volumes)
        if arr.ndim != 4:
            raise ValueError("batch must be [B, N, M, L]")
        from .projection import _uploader
        # large host batches: the threaded pinned-staging upload (volumes along the leading axis)
        vox = _uploader().upload(arr) if arr.nbytes >= (32 << 20) else None
        if vox is None:
            vox = torch.from_numpy(arr).to("cuda")
    if vox.dim() != 4:
        raise ValueError("batch must be [B, N, M, L]")
    res = engine.moments(vox, order, offset=offset)
    torch.cuda.current_stream().synchronize()
    status = res.status.cpu().numpy()
    if check_consistency:
        for b, st in enumerate(status.tolist()):
            raise_status(st, f"volume {b}")
    if as_float:
        return res.f64.cpu().numpy()
    i128 = res.i128.cpu().numpy()
    idx = moment_indices(order)
    return [MomentTensor3(order, dict(zip(idx, engine.i128_to_ints(i128[b])))) for b in range(i128.shape[0])]


def dpm_generic_moments(volume: Volume, order: int, counters: OpCounters | None = None,
                        check_consistency: bool = True) -> MomentTensor3:
    """A second, independent device route: the reference's image set (with the
    ZX image, no profile) built by the shape-generic brick kernel
    (``dpm_project_generic``) instead of the TMA streaming kernel, its 2D
    moments, and the epilogue placing M_{p,0,r} from ZX.  ``dpm_moments`` uses
    a different kernel AND a different set of projections (profile instead of
    ZX), so ``harness.verify_engines`` cross-checks two implementations the way
    the reference cross-checks its engines (moments3d.py:267-271,
    harness.py:101-120)."""
    import torch

    from . import engine
    from .projection import _to_device

    engine.check_order(order)
    vox = _to_device(volume)
    dims = tuple(volume.dims) if hasattr(volume, "dims") else tuple(reversed(vox.shape[-3:]))
    engine.check_envelope(dims[0], dims[1], dims[2], nat.DPM_U8 if vox.dtype == torch.uint8 else nat.DPM_U16,
                          order)
    imgs = engine.project(vox, engine.num_images(order), kernel="generic")
    acc = engine.moments2d_images(vox, imgs, order)
    res = engine.derive(acc, order, kind="images")
    torch.cuda.current_stream().synchronize()
    st = int(res.status[0].item())
    if check_consistency:
        raise_status(st, "dpm_generic")
    vals = engine.i128_to_ints(res.i128[0].cpu().numpy())
    _count(counters, order, dims)
    return MomentTensor3(order, dict(zip(moment_indices(order), vals)))


def _direct(volume: Volume, order: int, method: int, name: str, check_consistency: bool = True) -> MomentTensor3:
    """Exact Eq. 2 sums on the device (csrc/direct3d.cu, dpm_direct_moments)."""
    import ctypes

    import torch

    from . import engine
    from .projection import _to_device

    engine.check_order(order)
    vox = _to_device(volume)
    desc = engine.make_desc(vox)
    dims = tuple(volume.dims) if hasattr(volume, "dims") else tuple(reversed(vox.shape[-3:]))
    engine.check_envelope(dims[0], dims[1], dims[2], desc.dtype, order)
    lib = nat.lib()
    wsb = int(lib.dpm_direct_workspace_bytes(ctypes.byref(desc), order))
    ws = torch.empty(wsb, dtype=torch.uint8, device=vox.device)
    n3 = len(moment_indices(order))
    out = torch.empty((desc.B, n3, 2), dtype=torch.int64, device=vox.device)
    nat.check(lib.dpm_direct_moments(ctypes.byref(desc), vox.data_ptr(), order, method, ws.data_ptr(), wsb,
                                     out.data_ptr(), None, engine.stream_handle()), name)
    torch.cuda.current_stream().synchronize()
    vals = engine.i128_to_ints(out[0].cpu().numpy())
    return MomentTensor3(order, dict(zip(moment_indices(order), vals)))


def naive_moments(volume: Volume, order: int, counters: OpCounters | None = None,
                  check_consistency: bool = True) -> MomentTensor3:
    """Direct evaluation M[p][q][r] = sum V x^p y^q z^r (moments3d.py:78-139),
    exact, on the device: every voxel is multiplied by every in-plane monomial
    x^p y^q (csrc/direct3d.cu, NAIVE), the plane totals by z^r.  Counters are
    the reference's tallies for this method: per moment, one multiply and one
    add per voxel and per plane."""
    res = _direct(volume, order, nat.DPM_DIRECT_NAIVE, "naive_moments")
    if counters is not None:
        l, m, n = volume.dims
        k = len(moment_indices(order))
        counters.multiplications += k * (l * m * n + n)
        counters.additions += k * (l * m * n + n)
    return res


def factored_moments(volume: Volume, order: int, counters: OpCounters | None = None,
                     check_consistency: bool = True) -> MomentTensor3:
    """Row -> slice -> volume factored evaluation (moments3d.py:142-198),
    exact, on the device: per x-row the K + 1 sums V x^p, rows weighted by
    y^q per slice, slices by z^r (csrc/direct3d.cu, FACTORED).  Counters are
    the reference's tallies for this method."""
    res = _direct(volume, order, nat.DPM_DIRECT_FACTORED, "factored_moments")
    if counters is not None:
        l, m, n = volume.dims
        pq = (order + 1) * (order + 2) // 2
        k = len(moment_indices(order))
        counters.multiplications += order * l * m * n + pq * m * n + k * n
        counters.additions += (order + 1) * l * m * n + pq * m * n + k * n
    return res


ENGINES = {
    "naive": naive_moments,
    "factored": factored_moments,
    "dpm": dpm_moments,
    "dpm_generic": dpm_generic_moments,
}


def count_ops(engine: str, volume: Volume, order: int) -> OpCounters:
    """Run an engine with instrumentation and return its operation tallies (moments3d.py:274-278)."""
    counters = OpCounters()
    ENGINES[engine](volume, order, counters)
    return counters
