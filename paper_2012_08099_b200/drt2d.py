"""2D raw moments of projection images, computed on the device.

Mirrors the public 2D layer of the reference (``volmoments.drt2d``):

* ``Moments2D`` -- same fields and semantics as the reference type
  (drt2d.py:64-78): exact ``values[(p, q)]``, ``order``, ``origin_offset``.
* ``brute_force_2d(image, max_order)`` -- the reference's direct definition
  (drt2d.py:177-193), ``M[p][q] = sum I(i, j) i^p j^q`` about STORED index 0,
  with the image's ``origin_offset`` carried along.  Here it runs through the
  exact device kernel (``dpm_image_moments2d``) for any order up to 6, with the
  128-bit exactness envelope instead of the reference's int64 guard.
* ``image_moments`` -- the same call under a descriptive name.
* ``shift_origin(m, offset)`` -- the binomial change of the first-axis origin
  (drt2d.py:196-208), exact Python ints on the host (O(#moments) work).

Not mirrored: ``integrals`` / ``IntegralSet`` / ``moments_1d`` /
``assemble_2d`` (drt2d.py:42-174).  The five-integral route caps at 2D
order 4 and is replaced on this path by the power-table kernel, which gives
the same moments.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import comb

import numpy as np
import torch

from . import _native as nat
from .engine import acc_to_ints, n2d, stream_handle

MAX_ORDER_2D = nat.MAX_ORDER


@dataclass(frozen=True)
class Moments2D:
    """Raw image moments M[p][q] for p + q <= order, exact integers."""

    order: int
    values: dict[tuple[int, int], int]
    origin_offset: int = 0

    def __getitem__(self, pq: tuple[int, int]) -> int:
        return self.values[pq]

    @property
    def mass(self) -> int:
        return self.values[(0, 0)]


def _pq(order: int) -> list[tuple[int, int]]:
    """(p, q) in the kernel's p-major accumulator order."""
    return [(p, q) for p in range(order + 1) for q in range(order + 1 - p)]


def image_moments(image, max_order: int = 4, device: torch.device | str = "cuda") -> Moments2D:
    """Exact 2D moments of one image about stored index 0 (``image`` is a
    ``ProjectionImage`` or anything with ``pixels [j, i]`` and
    ``origin_offset``; a bare 2D array is accepted too)."""
    if not isinstance(max_order, (int, np.integer)) or not 0 <= int(max_order) <= MAX_ORDER_2D:
        raise ValueError(f"max_order must be in 0..{MAX_ORDER_2D}, got {max_order}")
    px = np.asarray(getattr(image, "pixels", image))
    offset = int(getattr(image, "origin_offset", 0))
    if px.ndim != 2:
        raise ValueError(f"image pixels must be 2D [j, i], got shape {px.shape}")
    h, w = px.shape
    if px.size and (int(px.min()) < 0 or int(px.max()) > 0xFFFFFFFF):
        raise ValueError("image pixels must be non-negative and fit 32 bits")
    k = max(3, int(max_order))                 # the kernel is instantiated for orders 3..6
    mass = int(px.astype(np.uint64).sum(dtype=np.uint64)) if px.size else 0
    if mass * max(w - 1, h - 1, 1) ** k >= 1 << 126:
        raise OverflowError(f"2D moments of a {w}x{h} image of mass {mass} exceed the 128-bit envelope")
    dev = torch.device(device)
    pix = torch.from_numpy(np.ascontiguousarray(px.astype(np.uint32)).view(np.int32)).to(dev)
    acc = torch.empty((n2d(k), 4), dtype=torch.int64, device=dev)
    nat.check(nat.lib().dpm_image_moments2d(pix.data_ptr(), w, h, 0, 0, k, acc.data_ptr(),
                                            stream_handle(torch.cuda.current_stream(dev))),
              "dpm_image_moments2d")
    vals = acc_to_ints(acc.cpu().numpy())
    values = {pq: int(v) for pq, v in zip(_pq(k), vals) if pq[0] + pq[1] <= max_order}
    return Moments2D(int(max_order), values, offset)


def brute_force_2d(image, max_order: int = 4) -> Moments2D:
    """The reference's direct 2D definition (drt2d.py:177-193), on the device."""
    return image_moments(image, max_order)


def shift_origin(m: Moments2D, offset: int) -> Moments2D:
    """Moments about stored index 0 -> moments about logical index 0, where
    stored i = logical i + offset (drt2d.py:196-208):
    M'[p][q] = sum_{s <= p} C(p, s) (-offset)^(p - s) M[s][q]."""
    out = {}
    for (p, q) in m.values:
        acc = 0
        for s in range(p + 1):
            acc += comb(p, s) * (-offset) ** (p - s) * m.values[(s, q)]
        out[(p, q)] = acc
    return Moments2D(m.order, out, 0)
