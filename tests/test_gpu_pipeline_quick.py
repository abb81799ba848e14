"""Quick end-to-end parity of the CUDA pipeline against the C oracle."""
import numpy as np
import pytest
import torch

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,bits,order", [((5, 4, 3), 8, 3), ((7, 6, 5), 16, 4), ((9, 7, 5), 8, 6),
                                               ((64, 64, 64), 8, 3), ((33, 17, 20), 16, 6),
                                               ((264, 19, 72), 16, 6), ((320, 9, 70), 8, 5),
                                               ((128, 9, 100), 8, 6), ((100, 6, 99), 16, 5), ((64, 5, 97), 8, 4)])
def test_dpm_matches_oracle(cuda, dims, bits, order):
    v = vm.random(dims, bits, seed=3)
    got = vm.dpm_moments(v, order)
    want = oracle.naive(v.voxels, order)
    assert got.values == want


@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 3, 2), (16, 16, 16), (70, 9, 33), (64, 8, 8),
                                  (256, 3, 64), (264, 5, 65), (512, 2, 130), (128, 7, 130), (100, 5, 37),
                                  (36, 4, 9), (132, 3, 100)])
@pytest.mark.parametrize("bits", [8, 16])
def test_projections_match_oracle(cuda, dims, bits):
    v = vm.random(dims, bits, seed=1)
    got = vm.project_extended(v)
    want = oracle.project(v.voxels, 7)
    for k, name in enumerate(vm.projection.EXTENDED_NAMES):
        assert np.array_equal(got[name].pixels, want[k]), name


def test_int16_offset_and_batch(cuda):
    rng = np.random.default_rng(5)
    vol = rng.integers(-1024, 3072, size=(3, 40, 24, 128), dtype=np.int16)
    t = torch.from_numpy(vol).cuda()
    res = engine.moments(t, 4, offset=1024)
    torch.cuda.synchronize()
    got = res.i128.cpu().numpy()
    for b in range(3):
        want = oracle.naive(vol[b], 4, offset=1024)
        assert engine.i128_to_ints(got[b]) == [want[k] for k in vm.moment_indices(4)]
    assert res.status.cpu().numpy().tolist() == [0, 0, 0]


@pytest.mark.parametrize("shape,dtype,order,offset", [((64, 64, 64), np.uint8, 3, 0), ((40, 48, 72), np.uint16, 6, 0),
                                                      ((30, 20, 40), np.int16, 4, 1024),
                                                      ((3, 16, 24, 40), np.uint8, 3, 0)])
def test_host_graphed_moments(cuda, shape, dtype, order, offset):
    """One CUDA graph: pinned H2D + pipeline + D2H; replays re-read the host buffer."""
    rng = np.random.default_rng(11)
    lo, hi = (-1024, 3000) if dtype == np.int16 else (0, np.iinfo(dtype).max)
    vol = rng.integers(lo, hi, size=shape).astype(dtype)
    host = torch.from_numpy(vol)
    hg = engine.HostGraphedMoments(host, order, offset=offset)
    idx = vm.moment_indices(order)
    for rep in range(2):
        i128, st = hg.run()
        assert st.tolist() == [0] * st.numel()
        got = i128.numpy().reshape(-1, len(idx), 2)
        vols = vol.reshape((-1,) + vol.shape[-3:])
        for b in range(vols.shape[0]):
            want = oracle.naive(vols[b], order, offset=offset)
            assert engine.i128_to_ints(got[b]) == [want[k] for k in idx]
        vol.reshape(-1)[rep::7] = 5                     # update the host buffer in place; next replay re-reads it
        hg.host.copy_(torch.from_numpy(vol))


@pytest.mark.parametrize("case", ["x_slice_aligned", "x_slice_unaligned", "y_padded", "z_step", "batch_padded"])
def test_strided_views(cuda, case):
    """Non-contiguous views go through the descriptor's element strides (TMA
    path when 16-byte aligned, generic kernel otherwise) with identical results."""
    rng = np.random.default_rng(21)
    big = torch.from_numpy(rng.integers(0, 65535, size=(2, 40, 36, 280)).astype(np.uint16)).cuda()
    views = {
        "x_slice_aligned": big[0, :, :, 8:264],        # row start 16-B aligned, stride_y 280
        "x_slice_unaligned": big[0, :, :, 3:203],      # misaligned start -> generic kernel
        "y_padded": big[0, :, 2:30, :256],             # stride_y 280, stride_z 36*280
        "z_step": big[0, ::2, :, :272],                # every other plane
        "batch_padded": big[:, 1:39, :, 16:272],       # 4-D, padded batch stride
    }
    v = views[case]
    order = 4
    res = engine.moments(v, order)
    got = res.i128.cpu().numpy().reshape(-1, len(vm.moment_indices(order)), 2)
    host = v.cpu().numpy()
    vols = host.reshape((-1,) + host.shape[-3:])
    for b in range(vols.shape[0]):
        want = oracle.naive(np.ascontiguousarray(vols[b]), order)
        assert engine.i128_to_ints(got[b]) == [want[k] for k in vm.moment_indices(order)]
    imgs = engine.project(v, 7)
    want_imgs = oracle.project(np.ascontiguousarray(vols[0]), 7)
    for k in range(7):
        assert np.array_equal(imgs[k][0].cpu().numpy().view(np.uint32), want_imgs[k].astype(np.uint32)), k


@pytest.mark.parametrize("order", [4, 6])
def test_graphed_slab_stages(cuda, order):
    """Three-graph z-slab pipeline (projection, 2D moments, epilogue) == the
    eager path, replay after replay, on a slab in global coordinates."""
    rng = np.random.default_rng(order)
    full = rng.integers(0, 65535, size=(40, 24, 264)).astype(np.uint16)
    z0, n = 16, 24
    slab = torch.from_numpy(full[z0:z0 + n]).cuda()
    st = engine.GraphedSlabStages(slab, order, z0=z0)
    want_acc = engine.moments2d_partial(slab, order, z0=z0)
    for _ in range(2):
        st.replay_project()
        acc = st.replay_moments2d()
        assert torch.equal(acc, want_acc)
        res = st.replay_derive()
        torch.cuda.synchronize()
        assert torch.equal(res.i128, engine.derive(want_acc, order, kind=engine.acc_kind(slab, order)).i128)
    assert st.launches == 5   # zeroing + projection, zeroing + image/profile moments, epilogue
