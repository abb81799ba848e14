"""Volume files: raw + sidecar header and the NRRD subset (reference
volume.py:55-194), plus memory-mapped opening for the streaming path.

``load_raw`` / ``load_nrrd`` / ``write_raw`` / ``meta_from_header_file`` /
``VolumeMeta`` keep the reference's names, arguments and ``FormatError``
behaviour.  ``open_raw`` / ``open_nrrd`` return the same ``Volume`` backed by
a read-only ``np.memmap`` instead of a byte copy, so a volume larger than host
memory can be fed plane-slab by plane-slab to the device
(``streaming.FileStreamer``).  Files are little-endian,
x fastest: voxel (x, y, z) at flat index x + L (y + M z) (volume.py:1-6).
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import FormatError
from .volume import Volume

_DEPTH_DTYPE = {8: np.dtype("<u1"), 16: np.dtype("<u2")}
# NRRD "type" spellings of the two supported sample types
_NRRD_DEPTH = {name: 8 for name in ("uchar", "unsigned char", "uint8", "uint8_t")}
_NRRD_DEPTH.update({name: 16 for name in ("ushort", "unsigned short", "uint16", "uint16_t")})


@dataclass
class VolumeMeta:
    """What a headerless raw file needs: dims (L, M, N), bit depth, spacing."""

    dims: tuple[int, int, int]
    bit_depth: int
    spacing: tuple[float, float, float] = (1.0, 1.0, 1.0)
    byte_order: str = "little"
    source: str = ""

    def __post_init__(self):
        if self.bit_depth not in _DEPTH_DTYPE:
            raise FormatError(f"unsupported bit depth {self.bit_depth}; expected 8 or 16")
        if self.byte_order != "little":
            raise FormatError(f"unsupported byte order {self.byte_order!r}; raw files are little-endian")
        if len(self.dims) != 3 or any(int(d) < 1 for d in self.dims):
            raise FormatError(f"dims must be three positive integers, got {self.dims}")

    @property
    def nbytes(self) -> int:
        l, m, n = self.dims
        return l * m * n * _DEPTH_DTYPE[self.bit_depth].itemsize


def _numbers(text: str, kind):
    return tuple(kind(t) for t in text.replace(",", " ").split())


def meta_from_header_file(path: str | Path) -> VolumeMeta:
    """Parse a ``key = value`` sidecar (keys: dims, depth, spacing,
    byte_order, data; ``#`` comments and blank lines ignored)."""
    keys: dict[str, str] = {}
    for raw_line in Path(path).read_text().splitlines():
        line = raw_line.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise FormatError(f"malformed header line {line!r} in {path}")
        k, v = line.split("=", 1)
        keys[k.strip().lower()] = v.strip()
    for required in ("dims", "depth"):
        if required not in keys:
            raise FormatError(f"header file {path} is missing required key {required!r}")
    try:
        dims = _numbers(keys["dims"], int)
        depth = int(keys["depth"])
        spacing = _numbers(keys["spacing"], float) if "spacing" in keys else (1.0, 1.0, 1.0)
    except ValueError as exc:
        raise FormatError(f"header file {path}: {exc}") from exc
    return VolumeMeta(dims=dims, bit_depth=depth, spacing=spacing,
                      byte_order=keys.get("byte_order", "little"), source=keys.get("data", str(path)))


def _check_size(path, have: int, want: int, what: str) -> None:
    if have != want:
        raise FormatError(f"{path}: file holds {have} bytes but {what} require {want}")


def load_raw(path: str | Path, meta: VolumeMeta) -> Volume:
    """Read a headerless raw volume described by ``meta`` into memory."""
    data = Path(path).read_bytes()
    _check_size(path, len(data), meta.nbytes, f"dims {meta.dims} at {meta.bit_depth}-bit")
    l, m, n = meta.dims
    vox = np.frombuffer(data, dtype=_DEPTH_DTYPE[meta.bit_depth]).reshape(n, m, l)
    return Volume(voxels=vox, spacing=tuple(meta.spacing))


def open_raw(path: str | Path, meta: VolumeMeta) -> Volume:
    """Like ``load_raw`` but memory-mapped (read-only): nothing is read
    until planes are touched."""
    size = Path(path).stat().st_size
    _check_size(path, size, meta.nbytes, f"dims {meta.dims} at {meta.bit_depth}-bit")
    l, m, n = meta.dims
    vox = np.memmap(path, dtype=_DEPTH_DTYPE[meta.bit_depth], mode="r", shape=(n, m, l))
    return Volume(voxels=vox, spacing=tuple(meta.spacing))


def write_raw(volume: Volume, path: str | Path) -> None:
    """Write the voxels flat, x fastest, little-endian."""
    Path(path).write_bytes(np.ascontiguousarray(volume.voxels, dtype=_DEPTH_DTYPE[volume.bit_depth]).tobytes())


@dataclass
class _NrrdLayout:
    sizes: tuple[int, int, int]
    depth: int
    spacing: tuple[float, float, float]
    data_path: Path
    data_offset: int


def _nrrd_layout(path: Path) -> _NrrdLayout:
    """Parse the header of the supported NRRD subset: 3D, uchar/ushort,
    raw encoding, little-endian, attached or detached data."""
    with open(path, "rb") as fh:
        head = fh.read(1 << 16)
    nl = head.find(b"\n")
    if nl < 0 or not head[:nl].startswith(b"NRRD"):
        raise FormatError(f"{path}: missing NRRD magic")
    end = head.find(b"\n\n")
    if end < 0:
        raise FormatError(f"{path}: header is not terminated by a blank line")
    fields: dict[str, str] = {}
    for line in head[nl + 1:end].decode("ascii", "replace").splitlines():
        if not line or line.startswith("#"):
            continue
        if ":" not in line:
            raise FormatError(f"{path}: malformed header line {line!r}")
        k, v = line.split(":", 1)
        fields[k.strip().lower()] = v.lstrip("=").strip()
    if fields.get("dimension") != "3":
        raise FormatError(f"{path}: unsupported header field dimension: {fields.get('dimension')!r} (need 3)")
    tname = fields.get("type", "")
    if tname not in _NRRD_DEPTH:
        raise FormatError(f"{path}: unsupported header field type: {tname!r}")
    if fields.get("encoding") != "raw":
        raise FormatError(f"{path}: unsupported header field encoding: {fields.get('encoding')!r}")
    if fields.get("endian", "little") == "big":
        raise FormatError(f"{path}: unsupported header field endian: 'big'")
    if "sizes" not in fields:
        raise FormatError(f"{path}: missing header field sizes")
    sizes = tuple(int(s) for s in fields["sizes"].split())
    if len(sizes) != 3:
        raise FormatError(f"{path}: header field sizes must have 3 entries, got {fields['sizes']!r}")
    spacing = (1.0, 1.0, 1.0)
    if "spacings" in fields:
        sp = tuple(float(s) for s in fields["spacings"].split())
        if len(sp) != 3:
            raise FormatError(f"{path}: header field spacings must have 3 entries")
        spacing = sp
    detached = fields.get("data file", fields.get("datafile"))
    if detached:
        return _NrrdLayout(sizes, _NRRD_DEPTH[tname], spacing, path.parent / detached, 0)
    return _NrrdLayout(sizes, _NRRD_DEPTH[tname], spacing, path, end + 2)


def _nrrd_volume(path: str | Path, mmap: bool) -> Volume:
    path = Path(path)
    lay = _nrrd_layout(path)
    l, m, n = lay.sizes
    dt = _DEPTH_DTYPE[lay.depth]
    want = l * m * n * dt.itemsize
    have = lay.data_path.stat().st_size - lay.data_offset
    if have != want:
        raise FormatError(f"{path}: data holds {have} bytes but sizes {lay.sizes} at {lay.depth}-bit require {want}")
    if mmap:
        vox = np.memmap(lay.data_path, dtype=dt, mode="r", offset=lay.data_offset, shape=(n, m, l))
    else:
        with open(lay.data_path, "rb") as fh:
            fh.seek(lay.data_offset)
            vox = np.frombuffer(fh.read(want), dtype=dt).reshape(n, m, l)
    return Volume(voxels=vox, spacing=lay.spacing)


def load_nrrd(path: str | Path) -> Volume:
    """Read an NRRD volume (supported subset) into memory."""
    return _nrrd_volume(path, mmap=False)


def open_nrrd(path: str | Path) -> Volume:
    """Like ``load_nrrd`` but memory-mapped (read-only)."""
    return _nrrd_volume(path, mmap=True)
