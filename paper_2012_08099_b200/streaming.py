"""Host-resident volumes: chunked, double-buffered H2D streaming overlapped
with the projection pass.

A [N, M, L] volume in (pinned) host memory is cut into z-slabs of
``chunk_planes``; slab k+1 is copied on a side stream while slab k is
projected and reduced to exact 2D moments in global coordinates on the
compute stream; the per-slab limb accumulators are summed on the device and
the epilogue runs once.  Exact by linearity, identical to the resident path.
"""
from __future__ import annotations

import torch

from . import engine


class HostStreamer:
    """Reusable device buffers for streaming volumes of one shape."""

    def __init__(self, shape_nml, dtype, order: int, chunk_planes: int = 64, device=None):
        engine.check_order(order)
        self.N, self.M, self.L = shape_nml
        self.dtype = dtype
        self.order = order
        self.chunk = max(1, min(chunk_planes, self.N))
        self.device = torch.device(device or "cuda")
        self.bufs = [torch.empty((self.chunk, self.M, self.L), dtype=dtype, device=self.device) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.consumed = [torch.cuda.Event() for _ in range(2)]
        n_img = engine.num_images(order)
        self.acc_total = torch.zeros((1, n_img, engine.n2d(order), 4), dtype=torch.int64, device=self.device)
        self.launches = 0

    def run(self, host: torch.Tensor, offset: int = 0, z_base: int = 0, n_global: int | None = None):
        """Moments of ``host`` ([N, M, L], ideally pinned) whose first plane is
        global plane ``z_base`` of a volume with ``n_global`` planes."""
        assert tuple(host.shape) == (self.N, self.M, self.L) and host.dtype == self.dtype
        n_global = n_global if n_global is not None else z_base + self.N
        engine.check_envelope(self.L, self.M, n_global, engine._TORCH_DTYPE[self.dtype], self.order)
        comp = torch.cuda.current_stream(self.device)
        self.acc_total.zero_()
        self.launches = 1
        chunks = [(z, min(self.N, z + self.chunk)) for z in range(0, self.N, self.chunk)]
        # prime the first copy
        for i, (z0, z1) in enumerate(chunks[:2]):
            with torch.cuda.stream(self.copy_stream):
                self.bufs[i][: z1 - z0].copy_(host[z0:z1], non_blocking=True)
                self.copied[i].record(self.copy_stream)
        for k, (z0, z1) in enumerate(chunks):
            i = k % 2
            comp.wait_event(self.copied[i])
            slab = self.bufs[i][: z1 - z0]
            acc = engine.moments2d_partial(slab, self.order, offset=offset, z0=z_base + z0, n_global=n_global)
            self.launches += 2
            engine.acc_add(self.acc_total, acc)
            self.launches += 1
            self.consumed[i].record(comp)
            nxt = k + 2
            if nxt < len(chunks):
                n0, n1 = chunks[nxt]
                with torch.cuda.stream(self.copy_stream):
                    self.copy_stream.wait_event(self.consumed[i])
                    self.bufs[i][: n1 - n0].copy_(host[n0:n1], non_blocking=True)
                    self.copied[i].record(self.copy_stream)
        return self.acc_total

    def moments(self, host: torch.Tensor, offset: int = 0):
        acc = self.run(host, offset)
        res = engine.derive(acc, self.order, kind=engine.acc_kind(self.bufs[0], self.order, offset))
        self.launches += 1
        return res


class FileStreamer:
    """Moments of a volume that lives in a file (or any host array, e.g. a
    read-only ``np.memmap`` from ``volio.open_raw`` / ``open_nrrd``) and need
    not fit in host or device memory: a three-stage pipeline per z-slab of
    ``chunk_planes`` planes -- file pages -> pinned staging (host copy, which
    is where the disk read happens) -> device buffer (copy stream) ->
    projection + exact 2D moments in global coordinates (compute stream).  The
    host fills slab k+1 while the device copies / reduces slab k; the
    per-slab limb accumulators add exactly and the epilogue runs once."""

    def __init__(self, shape_nml, dtype, order: int, chunk_planes: int = 64, device=None):
        import numpy as np

        engine.check_order(order)
        self.N, self.M, self.L = shape_nml
        self.order = order
        self.chunk = max(1, min(chunk_planes, self.N))
        self.device = torch.device(device or "cuda")
        tdt = {np.dtype("uint8"): torch.uint8, np.dtype("uint16"): torch.uint16}[np.dtype(dtype)]
        self.staging = [torch.empty((self.chunk, self.M, self.L), dtype=tdt, pin_memory=True) for _ in range(2)]
        self.staging_np = [s.numpy() for s in self.staging]
        self.bufs = [torch.empty((self.chunk, self.M, self.L), dtype=tdt, device=self.device) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.consumed = [torch.cuda.Event() for _ in range(2)]
        n_img = engine.num_images(order)
        self.acc_total = torch.zeros((1, n_img, engine.n2d(order), 4), dtype=torch.int64, device=self.device)
        self.bytes_read = 0

    def run(self, src) -> torch.Tensor:
        """Limb accumulator of the 2D moments of ``src`` ([N, M, L] array)."""
        assert tuple(src.shape) == (self.N, self.M, self.L)
        engine.check_envelope(self.L, self.M, self.N, engine._TORCH_DTYPE[self.bufs[0].dtype], self.order)
        comp = torch.cuda.current_stream(self.device)
        self.acc_total.zero_()
        self.bytes_read = 0
        for k, z0 in enumerate(range(0, self.N, self.chunk)):
            z1 = min(self.N, z0 + self.chunk)
            i = k % 2
            self.copied[i].synchronize()                       # staging[i]'s previous H2D is done
            self.staging_np[i][: z1 - z0] = src[z0:z1]         # file -> pinned (the disk read)
            self.bytes_read += self.staging_np[i][: z1 - z0].nbytes
            with torch.cuda.stream(self.copy_stream):
                self.copy_stream.wait_event(self.consumed[i])  # bufs[i]'s previous slab is reduced
                self.bufs[i][: z1 - z0].copy_(self.staging[i][: z1 - z0], non_blocking=True)
                self.copied[i].record(self.copy_stream)
            comp.wait_event(self.copied[i])
            acc = engine.moments2d_partial(self.bufs[i][: z1 - z0], self.order, z0=z0, n_global=self.N)
            engine.acc_add(self.acc_total, acc)
            self.consumed[i].record(comp)
        return self.acc_total

    def moments(self, src):
        return engine.derive(self.run(src), self.order, kind=engine.acc_kind(self.bufs[0], self.order))
