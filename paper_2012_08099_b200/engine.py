"""Device pipeline: torch provides device memory and streams; every stage runs
in the CUDA kernels behind the C ABI (paper_2012_08099_b200/_native.py).

Voxel tensors are CUDA tensors of dtype uint8 / uint16 / int16 (int16 with an
``offset``, e.g. +1024 for CT data), shaped [N, M, L] or [B, N, M, L] and
contiguous along x.  Exact 128-bit results come back as int64 (lo, hi) pairs.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat

_TORCH_DTYPE = {torch.uint8: nat.DPM_U8, torch.uint16: nat.DPM_U16, torch.int16: nat.DPM_I16}
_VMAX = {nat.DPM_U8: 255, nat.DPM_U16: 65535, nat.DPM_I16: 65535}


def check_order(order: int) -> None:
    """Orders 3..6 (the reference accepts 3 and 4, moments3d.py:57-59; 5 and 6
    are this build's extension)."""
    if not isinstance(order, (int, np.integer)) or not 3 <= int(order) <= nat.MAX_ORDER:
        raise ValueError(f"order must be in 3..{nat.MAX_ORDER}, got {order}")


def num_images(order: int) -> int:
    return 4 if order <= 3 else order + 1


def n2d(order: int) -> int:
    return (order + 1) * (order + 2) // 2


def n3d(order: int) -> int:
    return (order + 1) * (order + 2) * (order + 3) // 6


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def check_voxel_range(vox: torch.Tensor, offset: int) -> None:
    """int16 voxels are accumulated as ``v + offset`` in uint32 ray sums, which
    is exact only when every ``v + offset`` lies in 0..65535 (the reference's
    uint16 range, volume.py:34-35): check the actual data range (one device
    reduction).  Unsigned voxels take no offset."""
    if vox.dtype != torch.int16:
        if offset != 0:
            raise ValueError(f"offset {offset} given for {vox.dtype} voxels: offsets apply to int16 input only")
        return
    if not -32768 <= int(offset) <= 98303:
        raise ValueError(f"offset {offset} cannot map int16 voxels into 0..65535")
    if vox.numel() == 0 or (vox.is_cuda and torch.cuda.is_current_stream_capturing()):
        return   # checked by the un-captured warm-up call (GraphedMoments & co.)
    lo, hi = torch.aminmax(vox)
    lo, hi = int(lo) + int(offset), int(hi) + int(offset)
    if lo < 0 or hi > 65535:
        raise ValueError(f"int16 voxels + offset {offset} span {lo}..{hi}, outside 0..65535 "
                         f"(the exact uint32 accumulation needs unsigned 16-bit values)")


def make_desc(vox: torch.Tensor, offset: int = 0, z0: int = 0, validate: bool = True) -> nat.VolumeDesc:
    """C-ABI descriptor of a [N,M,L] or [B,N,M,L] voxel tensor (x-contiguous).
    ``validate``: check the int16 + offset range (``check_voxel_range``)."""
    if vox.dtype not in _TORCH_DTYPE:
        raise ValueError(f"unsupported voxel dtype {vox.dtype}; use uint8, uint16 or int16(+offset)")
    if validate:
        check_voxel_range(vox, offset)
    if vox.dim() == 3:
        n, m, l = vox.shape
        b, sb = 1, vox.numel()
        sz, sy, sx = vox.stride()
    elif vox.dim() == 4:
        b, n, m, l = vox.shape
        sb, sz, sy, sx = vox.stride()
    else:
        raise ValueError(f"voxel tensor must be 3D or 4D, got {vox.dim()}D")
    if sx != 1:
        raise ValueError("voxel rows must be contiguous along x")
    d = nat.VolumeDesc()
    d.L, d.M, d.N, d.B = int(l), int(m), int(n), int(b)
    d.stride_y, d.stride_z, d.stride_b = int(sy), int(sz), int(sb)
    d.dtype = _TORCH_DTYPE[vox.dtype]
    d.offset = int(offset)
    d.z0 = int(z0)
    return d


def check_envelope(L: int, M: int, N_global: int, dtype_code: int, order: int) -> None:
    nat.check(nat.lib().dpm_check_envelope(L, M, N_global, _VMAX[dtype_code], order),
              f"dims ({L}, {M}, {N_global}) at order {order}")


class _Workspace:
    """Per-device scratch buffer reused across calls (grow-only)."""

    def __init__(self):
        self._bufs: dict[tuple[int, int], torch.Tensor] = {}
        self._lock = threading.Lock()

    def get(self, nbytes: int, device: torch.device) -> torch.Tensor:
        key = (device.index if device.index is not None else torch.cuda.current_device(), threading.get_ident())
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
                self._bufs[key] = buf
            return buf


_WS = _Workspace()


@dataclass
class DeviceMoments:
    """Result of the device pipeline for B volumes."""
    i128: torch.Tensor     # [B, n3d, 2] int64 (lo, hi) exact
    f64: torch.Tensor      # [B, n3d] float64, correctly rounded from i128 (to ~1 ulp)
    status: torch.Tensor   # [B] int32 DPM_ST_* bits
    launches: int


def image_layout(desc: nat.VolumeDesc, img: int) -> tuple[int, int, int, int]:
    out = [ctypes.c_int64() for _ in range(4)]
    nat.check(nat.lib().dpm_image_layout(ctypes.byref(desc), img, *[ctypes.byref(o) for o in out]),
              "dpm_image_layout")
    return tuple(int(o.value) for o in out)


def moments_image_layout(desc: nat.VolumeDesc, order: int, img: int) -> tuple[int, int, int, int]:
    """(W, H, ai, aj) of image ``img`` of the MOMENTS pipeline (its layout may
    be layout T, the volume with x and z exchanged: see ``acc_kind``)."""
    out = [ctypes.c_int64() for _ in range(4)]
    nat.check(nat.lib().dpm_moments_image_layout(ctypes.byref(desc), order, img, *[ctypes.byref(o) for o in out]),
              "dpm_moments_image_layout")
    return tuple(int(o.value) for o in out)


def acc_kind(vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0) -> str:
    """Kind of the limb accumulator ``moments2d_partial`` / ``moments2d_profile``
    produce for this volume: "profile" or "profile_t" (layout T, wide volumes);
    pass it to ``derive``.  Depends on the geometry only, so every z-slab of a
    volume gives the same kind."""
    desc = make_desc(vox, offset, z0, validate=False)
    k = int(nat.lib().dpm_moments_acc_kind(ctypes.byref(desc), order))
    if k < 0:
        nat.check(-k, "dpm_moments_acc_kind")
    return {nat.DPM_ACC_PROFILE: "profile", nat.DPM_ACC_PROFILE_T: "profile_t"}[k]


def project(vox: torch.Tensor, n_img: int, offset: int = 0, z0: int = 0,
            stream: torch.cuda.Stream | None = None, imgs: list[torch.Tensor] | None = None,
            workspace: torch.Tensor | None = None, kernel: str = "auto") -> list[torch.Tensor]:
    """Projection images 0..n_img-1 as int32 tensors [B, H, W] holding uint32
    bits (into ``imgs`` when given, e.g. for CUDA-graph capture).

    ``kernel``: "auto" (TMA streaming kernel where the shape allows, else the
    generic one) or "generic" (the brick kernel only: independent cross-check)."""
    if kernel not in ("auto", "generic"):
        raise ValueError(f"unknown projection kernel {kernel!r}")
    desc = make_desc(vox, offset, z0)
    if imgs is None:
        imgs = []
        for k in range(n_img):
            W, H, _, _ = image_layout(desc, k)
            imgs.append(torch.empty((desc.B, H, W), dtype=torch.int32, device=vox.device))
    ptrs = (ctypes.c_void_p * n_img)(*[t.data_ptr() for t in imgs])
    if kernel == "generic":
        nat.check(nat.lib().dpm_project_generic(ctypes.byref(desc), vox.data_ptr(), n_img, ptrs,
                                                stream_handle(stream)), "dpm_project_generic")
        return imgs
    wsb = int(nat.lib().dpm_project_workspace_bytes(ctypes.byref(desc), n_img))
    ws = (workspace if workspace is not None else _WS.get(wsb, vox.device)) if wsb else None
    nat.check(nat.lib().dpm_project(ctypes.byref(desc), vox.data_ptr(), n_img, ptrs,
                                    ws.data_ptr() if ws is not None else None, wsb, stream_handle(stream)),
              "dpm_project")
    return imgs


def workspace_bytes(vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0) -> int:
    """Device scratch bytes ``moments`` needs for this volume and order."""
    desc = make_desc(vox, offset, z0)
    wsb = int(nat.lib().dpm_workspace_bytes(ctypes.byref(desc), order))
    if wsb == 0:
        raise ValueError("invalid volume descriptor")
    return wsb


def moments(vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0, n_global: int | None = None,
            stream: torch.cuda.Stream | None = None, out: DeviceMoments | None = None,
            workspace: torch.Tensor | None = None) -> DeviceMoments:
    """Whole pipeline (project -> exact 2D moments -> device epilogue).

    ``workspace``: caller-owned uint8 device scratch of at least
    ``workspace_bytes`` (required for CUDA-graph capture, whose replays keep
    the pointer); default is the per-thread shared grow-only buffer."""
    check_order(order)
    desc = make_desc(vox, offset, z0)
    check_envelope(desc.L, desc.M, n_global if n_global is not None else desc.N + desc.z0, desc.dtype, order)
    lib = nat.lib()
    wsb = int(lib.dpm_workspace_bytes(ctypes.byref(desc), order))
    if wsb == 0:
        raise ValueError("invalid volume descriptor")
    if workspace is not None:
        if workspace.numel() * workspace.element_size() < wsb or workspace.device != vox.device:
            raise ValueError(f"workspace must hold {wsb} bytes on {vox.device}")
        ws = workspace
    else:
        ws = _WS.get(wsb, vox.device)
    if out is None:
        out = DeviceMoments(
            i128=torch.empty((desc.B, n3d(order), 2), dtype=torch.int64, device=vox.device),
            f64=torch.empty((desc.B, n3d(order)), dtype=torch.float64, device=vox.device),
            status=torch.empty((desc.B,), dtype=torch.int32, device=vox.device),
            launches=0)
    nat.check(lib.dpm_moments(ctypes.byref(desc), vox.data_ptr(), order, ws.data_ptr(), wsb,
                              out.i128.data_ptr(), out.f64.data_ptr(), out.status.data_ptr(),
                              stream_handle(stream)), "dpm_moments")
    out.launches = nat.last_launch_count()
    return out


def moments2d_images(vox: torch.Tensor, imgs: list[torch.Tensor], order: int, offset: int = 0, z0: int = 0,
                     stream: torch.cuda.Stream | None = None, acc: torch.Tensor | None = None) -> torch.Tensor:
    """Exact 2D moments (global coordinates) of images made by ``project`` from
    ``vox``; returns the limb accumulator [B, n_img, n2d, 4] (int64 storage of
    uint64 sums), written into ``acc`` when given."""
    desc = make_desc(vox, offset, z0, validate=False)   # the images are already built from vox
    n_img = len(imgs)
    if acc is None:
        acc = torch.empty((desc.B, n_img, n2d(order), 4), dtype=torch.int64, device=vox.device)
    ptrs = (ctypes.c_void_p * n_img)(*[t.data_ptr() for t in imgs])
    nat.check(nat.lib().dpm_moments2d(ctypes.byref(desc), n_img, ptrs, order, acc.data_ptr(),
                                      stream_handle(stream)), "dpm_moments2d")
    return acc


def profile_layout(desc: nat.VolumeDesc, order: int) -> tuple[int, int, int]:
    """(WQ, ai, t) of the moments pipeline's y-summed profile P[x + t z]."""
    wq, ai, t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    nat.check(nat.lib().dpm_profile_layout(ctypes.byref(desc), order, ctypes.byref(wq), ctypes.byref(ai),
                                           ctypes.byref(t)), "dpm_profile_layout")
    return int(wq.value), int(ai.value), int(t.value)


def moments2d_partial(vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0,
                      stream: torch.cuda.Stream | None = None, acc: torch.Tensor | None = None,
                      workspace: torch.Tensor | None = None, n_global: int | None = None) -> torch.Tensor:
    """The moments pipeline's projection pass + exact moments of a slab in
    GLOBAL coordinates (dpm_moments_partial); returns the limb accumulator
    [B, n_img, n2d, 4] of kind ``acc_kind(vox, order)``.  Accumulators of
    z-slabs add elementwise (moments are linear in the voxels); finish with
    ``derive(acc, order, kind=...)``.  ``n_global``: planes of the whole
    volume (default z0 + N), checked against the exactness envelope."""
    check_order(order)
    desc = make_desc(vox, offset, z0)
    check_envelope(desc.L, desc.M, n_global if n_global is not None else desc.z0 + desc.N, desc.dtype, order)
    lib = nat.lib()
    wsb = int(lib.dpm_partial_workspace_bytes(ctypes.byref(desc), order))
    if wsb == 0:
        raise ValueError("invalid volume descriptor")
    ws = workspace if workspace is not None else _WS.get(wsb, vox.device)
    if acc is None:
        acc = torch.empty((desc.B, num_images(order), n2d(order), 4), dtype=torch.int64, device=vox.device)
    nat.check(lib.dpm_moments_partial(ctypes.byref(desc), vox.data_ptr(), order, ws.data_ptr(), wsb,
                                      acc.data_ptr(), stream_handle(stream)), "dpm_moments_partial")
    return acc


def project_profile(vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0,
                    stream: torch.cuda.Stream | None = None, imgs: list[torch.Tensor | None] | None = None,
                    profile: torch.Tensor | None = None,
                    zeroed: bool = False) -> tuple[list[torch.Tensor | None], torch.Tensor]:
    """Projection pass of the moments pipeline: the order's images except ZX
    (slot 2 is None) as int32 [B, H, W] uint32 bits, and the y-summed profile
    as int64 [B, WQ] (uint64 bits).  ``zeroed``: the caller's ``imgs`` and
    ``profile`` are already zero (``zero_profile_buffers``); only the pass runs."""
    check_order(order)
    desc = make_desc(vox, offset, z0)
    n_img = num_images(order)
    if imgs is None:
        imgs = []
        for k in range(n_img):
            if k == 2:
                imgs.append(None)
                continue
            W, H, _, _ = moments_image_layout(desc, order, k)
            imgs.append(torch.empty((desc.B, H, W), dtype=torch.int32, device=vox.device))
    if profile is None:
        wq, _, _ = profile_layout(desc, order)
        profile = torch.empty((desc.B, wq), dtype=torch.int64, device=vox.device)
    ptrs = (ctypes.c_void_p * n_img)(*[t.data_ptr() if t is not None else None for t in imgs])
    if zeroed:
        nat.check(nat.lib().dpm_project_profile_zeroed(ctypes.byref(desc), vox.data_ptr(), order, ptrs,
                                                       profile.data_ptr(), stream_handle(stream)),
                  "dpm_project_profile_zeroed")
    else:
        nat.check(nat.lib().dpm_project_profile(ctypes.byref(desc), vox.data_ptr(), order, ptrs, profile.data_ptr(),
                                                stream_handle(stream)), "dpm_project_profile")
    return imgs, profile


def zero_profile_buffers(vox: torch.Tensor, order: int, imgs: list[torch.Tensor | None], profile: torch.Tensor,
                         offset: int = 0, z0: int = 0, stream: torch.cuda.Stream | None = None) -> None:
    """Zero the moments pipeline's images and profile (one launch)."""
    desc = make_desc(vox, offset, z0, validate=False)
    ptrs = (ctypes.c_void_p * len(imgs))(*[t.data_ptr() if t is not None else None for t in imgs])
    nat.check(nat.lib().dpm_zero_profile_buffers(ctypes.byref(desc), order, ptrs, profile.data_ptr(),
                                                 stream_handle(stream)), "dpm_zero_profile_buffers")


def moments2d_profile(vox: torch.Tensor, imgs: list[torch.Tensor | None], profile: torch.Tensor, order: int,
                      offset: int = 0, z0: int = 0, stream: torch.cuda.Stream | None = None,
                      acc: torch.Tensor | None = None) -> torch.Tensor:
    """DPM_ACC_PROFILE accumulator of ``project_profile`` outputs."""
    desc = make_desc(vox, offset, z0, validate=False)   # the images are already built from vox
    n_img = len(imgs)
    if acc is None:
        acc = torch.empty((desc.B, n_img, n2d(order), 4), dtype=torch.int64, device=vox.device)
    ptrs = (ctypes.c_void_p * n_img)(*[t.data_ptr() if t is not None else None for t in imgs])
    nat.check(nat.lib().dpm_moments2d_profile(ctypes.byref(desc), order, ptrs, profile.data_ptr(), acc.data_ptr(),
                                              stream_handle(stream)), "dpm_moments2d_profile")
    return acc


ACC_KINDS = {"profile": nat.DPM_ACC_PROFILE, "profile_t": nat.DPM_ACC_PROFILE_T, "images": nat.DPM_ACC_IMAGES}


def derive(acc: torch.Tensor, order: int, stream: torch.cuda.Stream | None = None,
           out: DeviceMoments | None = None, kind: str = "profile") -> DeviceMoments:
    """Device epilogue on a (possibly summed) limb accumulator: ``kind``
    ``acc_kind(...)`` ("profile" or "profile_t") for ``moments2d_partial`` /
    ``moments2d_profile`` accumulators, "images" for ``moments2d_images`` over
    ``project``'s image set."""
    check_order(order)
    if kind not in ACC_KINDS:
        raise ValueError(f"unknown accumulator kind {kind!r}")
    B = acc.shape[0]
    desc = nat.VolumeDesc()
    desc.L = desc.M = desc.N = 1
    desc.B = B
    dev = acc.device
    if out is None:
        out = DeviceMoments(
            i128=torch.empty((B, n3d(order), 2), dtype=torch.int64, device=dev),
            f64=torch.empty((B, n3d(order)), dtype=torch.float64, device=dev),
            status=torch.empty((B,), dtype=torch.int32, device=dev), launches=0)
    nat.check(nat.lib().dpm_derive3d(ctypes.byref(desc), acc.data_ptr(), order, ACC_KINDS[kind], out.i128.data_ptr(),
                                     out.f64.data_ptr(), out.status.data_ptr(), stream_handle(stream)),
              "dpm_derive3d")
    out.launches = nat.last_launch_count()
    return out


def i128_to_ints(pairs: np.ndarray) -> list[int]:
    """[n, 2] int64 (lo, hi) -> exact Python ints."""
    lo = pairs[..., 0].astype(np.uint64).ravel().tolist()
    hi = pairs[..., 1].ravel().tolist()
    return [h * (1 << 64) + l for l, h in zip(lo, hi)]


def acc_to_ints(acc: np.ndarray) -> np.ndarray:
    """Limb accumulator [..., 4] (uint64 sums of 32-bit limbs) -> object array of ints."""
    a = acc.astype(np.uint64)
    flat = a.reshape(-1, 4).tolist()
    vals = []
    for l0, l1, l2, l3 in flat:
        v = (l0 + (l1 << 32) + (l2 << 64) + (l3 << 96)) % (1 << 128)
        vals.append(v - (1 << 128) if v >= (1 << 127) else v)
    return np.array(vals, dtype=object).reshape(acc.shape[:-1])


def synth_noise(L: int, M: int, z0: int, n_planes: int, seed: int, device=None,
                stream: torch.cuda.Stream | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Config-5 smooth-noise slab [n_planes, M, L] uint16 generated on the device."""
    if out is None:
        out = torch.empty((n_planes, M, L), dtype=torch.uint16, device=device or "cuda")
    nat.check(nat.lib().dpm_synth_noise_u16(out.data_ptr(), L, M, z0, n_planes, seed & ((1 << 64) - 1),
                                            stream_handle(stream)), "dpm_synth_noise_u16")
    return out


def acc_add(out: torch.Tensor, inp: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """out += inp for limb accumulators, on the device (dpm_acc_add kernel)."""
    assert out.shape == inp.shape and out.dtype == torch.int64 == inp.dtype
    nat.check(nat.lib().dpm_acc_add(out.data_ptr(), inp.data_ptr(), out.numel(), stream_handle(stream)),
              "dpm_acc_add")


def ints_to_limbs(values) -> np.ndarray:
    """Exact ints -> the limb-accumulator encoding [..., 4] (int64 storage of
    uint64 limb sums: value = sum_k limb_k 2^(32k) mod 2^128)."""
    arr = np.asarray(values, dtype=object)
    out = np.zeros(arr.shape + (4,), dtype=np.uint64)
    for idx, v in np.ndenumerate(arr):
        u = int(v) % (1 << 128)
        for k in range(4):
            out[idx + (k,)] = (u >> (32 * k)) & 0xFFFFFFFF
    return out.view(np.int64)


class GraphedMoments:
    """The whole device pipeline for a fixed input tensor, captured once in a
    CUDA graph and replayed (no per-call host work: ctypes calls, tensor-map
    encoding and launches happen at capture time only).  Owns its workspace
    and outputs, so later calls with other shapes cannot move them."""

    def __init__(self, vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0, n_global: int | None = None):
        self.vox = vox
        self.order = order
        self.workspace = torch.empty(workspace_bytes(vox, order, offset, z0), dtype=torch.uint8, device=vox.device)
        self.stream = torch.cuda.Stream(device=vox.device)
        self.stream.wait_stream(torch.cuda.current_stream(vox.device))
        kw = dict(offset=offset, z0=z0, n_global=n_global, workspace=self.workspace)
        with torch.cuda.stream(self.stream):
            self.out = moments(vox, order, **kw)   # warm-up, allocates the outputs
            self.launches = self.out.launches
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                moments(vox, order, out=self.out, **kw)
        torch.cuda.current_stream(vox.device).wait_stream(self.stream)

    def replay(self) -> DeviceMoments:
        self.graph.replay()
        return self.out


class GraphedSlabStages:
    """The z-slab pipeline as three CUDA graphs over fixed buffers: (1) the
    projection (image/profile zeroing + streaming pass, ``project_profile``),
    (2) exact 2D/1D moments in global coordinates into ``acc``, (3) the
    epilogue into ``out``.  A
    multi-GPU caller all-reduces ``acc`` between (2) and (3) (the exchange is
    not captured).  Replays are issued on the caller's current stream."""

    def __init__(self, vox: torch.Tensor, order: int, offset: int = 0, z0: int = 0, fused: bool = False,
                 n_global: int | None = None):
        """``fused``: single device, no exchange between (2) and (3): stage 2
        ends with the epilogue in the same launch and ``replay_derive`` only
        returns ``out`` -- refused inside a multi-rank process group, where
        the limbs must be all-reduced BEFORE the epilogue.  ``n_global``:
        planes of the whole volume (default z0 + N), checked against the
        exactness envelope."""
        check_order(order)
        if fused and torch.distributed.is_available() and torch.distributed.is_initialized() \
                and torch.distributed.get_world_size() > 1:
            raise ValueError("fused=True runs the epilogue before any exchange: use fused=False (replay_moments2d, "
                             "all-reduce, replay_derive) inside a multi-rank process group")
        self.vox, self.order, self.offset, self.z0 = vox, order, offset, z0
        self.fused = fused
        desc = make_desc(vox, offset, z0)
        check_envelope(desc.L, desc.M, n_global if n_global is not None else desc.z0 + desc.N, desc.dtype, order)
        n_img = num_images(order)
        dev = vox.device
        self.imgs = []
        for k in range(n_img):
            if k == 2:
                self.imgs.append(None)
                continue
            W, H, _, _ = moments_image_layout(desc, order, k)
            self.imgs.append(torch.empty((desc.B, H, W), dtype=torch.int32, device=dev))
        self.kind = acc_kind(vox, order, offset, z0)
        wq, _, _ = profile_layout(desc, order)
        self.profile = torch.empty((desc.B, wq), dtype=torch.int64, device=dev)
        self.acc = torch.empty((desc.B, n_img, n2d(order), 4), dtype=torch.int64, device=dev)
        self.out = DeviceMoments(
            i128=torch.empty((desc.B, n3d(order), 2), dtype=torch.int64, device=dev),
            f64=torch.empty((desc.B, n3d(order)), dtype=torch.float64, device=dev),
            status=torch.empty((desc.B,), dtype=torch.int32, device=dev), launches=0)
        self.counters = torch.empty((desc.B,), dtype=torch.int32, device=dev)
        # The images and profile are zeroed once here and then by the moments
        # stage right after it has read them (for the next step), so the
        # projection stage is the pass alone.
        stages = [self._project, self._moments2d] + ([] if fused else [self._derive])
        st = torch.cuda.Stream(device=dev)
        st.wait_stream(torch.cuda.current_stream(dev))
        self.graphs, self.launches = [], 0
        self._lc = 0
        with torch.cuda.stream(st):
            self._zero()
            for fn in stages:                  # warm-up: attributes, tensor-map encoder
                self._lc = 0
                fn()
                self.launches += self._lc
            for fn in stages:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    fn()
                self.graphs.append(g)
            self._zero_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._zero_graph, stream=st):
                self._zero()
        torch.cuda.current_stream(dev).wait_stream(st)
        self._dirty = False                    # images hold a projection not yet taken by the moments stage

    def _zero(self):
        zero_profile_buffers(self.vox, self.order, self.imgs, self.profile, self.offset, self.z0)
        self._lc += nat.last_launch_count()

    def _project(self):
        project_profile(self.vox, self.order, self.offset, self.z0, imgs=self.imgs, profile=self.profile,
                        zeroed=True)
        self._lc += nat.last_launch_count()

    def _moments2d(self):
        if self.fused:
            desc = make_desc(self.vox, self.offset, self.z0, validate=False)
            ptrs = (ctypes.c_void_p * len(self.imgs))(*[t.data_ptr() if t is not None else None for t in self.imgs])
            nat.check(nat.lib().dpm_moments2d_profile_derive(
                ctypes.byref(desc), self.order, ptrs, self.profile.data_ptr(), self.acc.data_ptr(),
                self.counters.data_ptr(), self.out.i128.data_ptr(), self.out.f64.data_ptr(),
                self.out.status.data_ptr(), stream_handle(None)), "dpm_moments2d_profile_derive")
        else:
            moments2d_profile(self.vox, self.imgs, self.profile, self.order, self.offset, self.z0, acc=self.acc)
        self._lc += nat.last_launch_count()
        self._zero()   # ready for the next projection

    def _derive(self):
        derive(self.acc, self.order, out=self.out, kind=self.kind)
        self._lc += nat.last_launch_count()

    def replay_project(self) -> None:
        if self._dirty:                        # a projection whose moments were never taken: start clean
            self._zero_graph.replay()
        self.graphs[0].replay()
        self._dirty = True

    def replay_moments2d(self) -> torch.Tensor:
        """Exact 2D moments into ``acc`` (with ``fused`` the epilogue already
        ran in the same launch: ``acc`` is then final, not for an exchange)."""
        self.graphs[1].replay()
        self._dirty = False
        return self.acc

    def replay_derive(self) -> DeviceMoments:
        if not self.fused:
            self.graphs[2].replay()
        return self.out


class HostGraphedMoments:
    """Host-buffer entry point for volumes that fit on the device in one piece:
    pinned host volume -> H2D copy -> project -> 2D moments -> epilogue -> D2H
    of the exact moments and status into pinned host tensors, all captured in
    ONE CUDA graph.  ``run()`` replays it and waits; per call the host does one
    graph launch and one synchronisation."""

    def __init__(self, host: torch.Tensor, order: int, offset: int = 0, device: torch.device | str = "cuda"):
        if host.device.type != "cpu":
            raise ValueError("host must be a CPU tensor")
        self.host = host if host.is_pinned() else host.pin_memory()
        self.dev = torch.empty(tuple(host.shape), dtype=host.dtype, device=device)
        self.dev.copy_(self.host)
        self.inner = GraphedMoments(self.dev, order, offset=offset)   # warm + validates
        self.i128 = torch.empty(tuple(self.inner.out.i128.shape), dtype=torch.int64, pin_memory=True)
        self.status = torch.empty(tuple(self.inner.out.status.shape), dtype=torch.int32, pin_memory=True)
        self.launches = self.inner.launches
        st = self.inner.stream
        st.wait_stream(torch.cuda.current_stream(self.dev.device))
        with torch.cuda.stream(st):
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=st):
                self.dev.copy_(self.host, non_blocking=True)
                moments(self.dev, order, offset=offset, out=self.inner.out, workspace=self.inner.workspace)
                self.i128.copy_(self.inner.out.i128, non_blocking=True)
                self.status.copy_(self.inner.out.status, non_blocking=True)
        torch.cuda.current_stream(self.dev.device).wait_stream(st)
        self.h2d_bytes = self.host.numel() * self.host.element_size()
        self.d2h_bytes = self.i128.numel() * 8 + self.status.numel() * 4

    def run(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Re-reads ``host`` (update it in place between calls); returns the
        pinned (i128 [B, n3d, 2], status [B]) host tensors."""
        st = self.inner.stream
        with torch.cuda.stream(st):      # replay() launches on the current stream
            self.graph.replay()
        st.synchronize()
        return self.i128, self.status
