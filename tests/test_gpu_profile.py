"""The moments pipeline's projection set: the order's
images without ZX plus the y-summed profile P[x + t z].  Images must be
bit-identical to ``project``'s, the profile to a numpy restatement, and the
moments to the oracle and to the independent images route (``dpm_generic``)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import engine

pytestmark = pytest.mark.gpu

T_OF_ORDER = {3: -1, 4: 2, 5: -2, 6: 3}


def np_profile(vol: np.ndarray, t: int) -> np.ndarray:
    """P[x + t z (+ |t|(N-1) if t < 0)] = sum_y V[z, y, x] (test restatement)."""
    n, m, l = vol.shape
    at = abs(t)
    out = np.zeros(l + at * (n - 1), dtype=np.int64)
    cols = vol.astype(np.int64).sum(axis=1)          # [z, x]
    x = np.arange(l)
    for z in range(n):
        idx = x + t * z + (at * (n - 1) if t < 0 else 0)
        np.add.at(out, idx, cols[z])
    return out


def _ints(res):
    return [engine.i128_to_ints(res.i128[b].cpu().numpy()) for b in range(res.i128.shape[0])]


# L >= 192 is layout T (the z-streaming kernel, project_zstream.cu); narrower
# volumes use the y-streaming kernel (project_stream.cu) with its classic images
SHAPES = [
    ((24, 40, 264), np.uint16),     # layout T: two x-tiles (the second 8 wide), 4 y-groups, 3 z-steps
    ((100, 17, 256), np.uint16),    # layout T: partial last z-step and y-group
    ((16, 8, 64), np.uint8),        # classic, 4-wide lanes; order 3: the SMALL variant (< 8 row-steps per SM)
    ((150, 9, 264), np.uint8),      # layout T, uint8 (8-byte lane vectors)
    ((140, 10, 128), np.uint16),    # classic, 4-wide uint16 lanes, two z-tiles (order 3: SMALL variant)
    ((9, 7, 5), np.uint8),          # generic kernel
    ((13, 11, 203), np.uint16),     # layout T through the generic kernel on the transposed view (L % 8 != 0)
    ((60, 300, 128), np.uint8),     # classic single tile (rows stored, images not zeroed), runs not aligned to 8 rows
    ((50, 200, 256), np.uint16),    # layout T, one x-tile, 17 y-groups
]


@pytest.mark.parametrize("order", [3, 4, 5, 6])
@pytest.mark.parametrize("shape,dt", SHAPES)
def test_profile_images_and_profile(order, shape, dt):
    rng = np.random.default_rng(sum(shape) + order)
    vol = rng.integers(0, np.iinfo(dt).max + 1, size=shape).astype(dt)
    v = torch.from_numpy(vol).cuda()
    imgs, prof = engine.project_profile(v, order)
    # layout T (wide volumes): the method's images of the volume with x and z exchanged
    lay_t = engine.acc_kind(v, order) == "profile_t"
    assert lay_t == (shape[2] >= 192)
    src = np.ascontiguousarray(vol.transpose(2, 1, 0)) if lay_t else vol
    ref = engine.project(torch.from_numpy(src).cuda(), engine.num_images(order))
    torch.cuda.synchronize()
    assert imgs[2] is None
    for k in range(engine.num_images(order)):
        if k != 2:
            assert torch.equal(imgs[k], ref[k]), k
    n, _, l = src.shape
    wq, ai, t = engine.profile_layout(engine.make_desc(v), order)
    assert t == T_OF_ORDER[order] and wq == l + abs(t) * (n - 1)
    assert ai == (-abs(t) * (n - 1) if t < 0 else 0)
    assert np.array_equal(prof[0].cpu().numpy(), np_profile(src, t))


@pytest.mark.parametrize("order", [3, 4, 5, 6])
@pytest.mark.parametrize("shape,dt", SHAPES + [((40, 1500, 256), np.uint16)])   # tall: several y-bands per column
def test_profile_moments_match_oracle_and_images_route(order, shape, dt):
    rng = np.random.default_rng(7 * order + shape[0])
    vol = rng.integers(0, np.iinfo(dt).max + 1, size=shape).astype(dt)
    v = vm.Volume(vol)
    got = vm.dpm_moments(v, order)
    assert got.values == vm.dpm_generic_moments(v, order).values
    if np.prod(shape) <= 200_000:
        assert got.values == oracle.naive(vol, order)


@pytest.mark.parametrize("order", [3, 6])
def test_profile_zslab_composition(order):
    rng = np.random.default_rng(11)
    vol = rng.integers(0, 65536, size=(70, 20, 256)).astype(np.uint16)
    kind = engine.acc_kind(torch.from_numpy(vol), order)
    whole = _ints(engine.derive(engine.moments2d_partial(torch.from_numpy(vol).cuda(), order), order, kind=kind))
    for cuts in ([0, 33, 70], [0, 5, 6, 40, 70]):
        acc = None
        for z0, z1 in zip(cuts[:-1], cuts[1:]):
            part = engine.moments2d_partial(torch.from_numpy(vol[z0:z1]).cuda(), order, z0=z0)
            acc = part.clone() if acc is None else acc + part
        assert _ints(engine.derive(acc, order, kind=kind)) == whole


def test_profile_batch_and_offset():
    rng = np.random.default_rng(5)
    vols = rng.integers(-1024, 3072, size=(3, 16, 12, 128)).astype(np.int16)
    got = vm.dpm_moments_batch(vols, 4, offset=1024)
    for b in range(3):
        want = oracle.naive((vols[b].astype(np.int32) + 1024).astype(np.uint16), 4)
        assert got[b].values == want


@pytest.mark.parametrize("order,a", [(6, 3), (5, 2), (4, 1), (3, 2)])
def test_profile_fault_injection_is_detected(order, a):
    """A corrupted profile moment in a redundant row is caught (DPM_ST_DISAGREE)."""
    rng = np.random.default_rng(order)
    vol = rng.integers(0, 65536, size=(24, 16, 256)).astype(np.uint16)
    acc = engine.moments2d_partial(torch.from_numpy(vol).cuda(), order)
    kind = engine.acc_kind(torch.from_numpy(vol), order)
    assert int(engine.derive(acc, order, kind=kind).status[0]) == 0
    bad = acc.clone()
    p_idx = a * (order + 1) - a * (a - 1) // 2      # idx2(order, a, 0)
    bad[0, 2, p_idx, 0] += 1
    assert int(engine.derive(bad, order, kind=kind).status[0]) & 1


def test_profile_graphed_stages_launches():
    rng = np.random.default_rng(2)
    slab = torch.from_numpy(rng.integers(0, 65535, size=(24, 24, 264)).astype(np.uint16)).cuda()
    st = engine.GraphedSlabStages(slab, 6, z0=16)
    assert st.launches == 5      # zeroing + projection, zeroing + image/profile moments (one launch), epilogue


@pytest.mark.parametrize("order", [4, 6])
def test_profile_batch_multi_tile(order):
    """Batch of volumes that need several x-tiles and z-tiles each (atomic rows,
    per-volume profiles and counters)."""
    rng = np.random.default_rng(order + 40)
    vols = rng.integers(0, 65536, size=(3, 100, 6, 264)).astype(np.uint16)
    got = vm.dpm_moments_batch(vols, order)
    for b in range(3):
        assert got[b].values == oracle.naive(vols[b], order)


@pytest.mark.parametrize("order", [3, 4, 6])
@pytest.mark.parametrize("shape,dt", [((40, 30, 203), np.uint16), ((24, 20, 323), np.uint8), ((20, 16, 77), np.int16)])
def test_staged_odd_width_matches_oracle(order, shape, dt):
    """Widths the TMA kernel cannot read in place (odd row pitch) go through the
    staged pad-copy pass (capi.cu, moments_staged): exact like the oracle."""
    rng = np.random.default_rng(order + shape[2])
    if dt == np.int16:
        vol = rng.integers(-1024, 3072, size=shape).astype(np.int16)
        got = engine.moments(torch.from_numpy(vol).cuda(), order, offset=1024)
        torch.cuda.synchronize()
        assert int(got.status[0]) == 0
        want = oracle.naive((vol.astype(np.int32) + 1024).astype(np.uint16), order)
        assert engine.i128_to_ints(got.i128[0].cpu().numpy()) == [want[k] for k in vm.moment_indices(order)]
    else:
        vol = rng.integers(0, np.iinfo(dt).max + 1, size=shape).astype(dt)
        assert vm.dpm_moments(vm.Volume(vol), order).values == oracle.naive(vol, order)


def test_staged_multi_slab_equals_padded_in_place():
    """A 300 MB odd-width volume: several staged slabs == the same volume
    zero-padded to an aligned width and read in place."""
    rng = np.random.default_rng(9)
    vol = rng.integers(0, 256, size=(600, 500, 1001), dtype=np.uint8)
    got = vm.dpm_moments(vm.Volume(vol), 4)
    padded = np.zeros((600, 500, 1008), dtype=np.uint8)
    padded[:, :, :1001] = vol
    assert got.values == vm.dpm_moments(vm.Volume(padded), 4).values


def test_public_api_upload_path_is_exact():
    """Volumes >= 32 MB reach the device through the pinned, threaded uploader
    (projection._Uploader): same moments as a direct device tensor."""
    rng = np.random.default_rng(21)
    vol = rng.integers(0, 65536, size=(400, 300, 320), dtype=np.uint16)   # 77 MB: two 64 MB staging chunks
    via_api = vm.dpm_moments(vm.Volume(vol), 6)
    direct = engine.moments(torch.from_numpy(vol).cuda(), 6)
    torch.cuda.synchronize()
    assert via_api.values == dict(zip(vm.moment_indices(6), engine.i128_to_ints(direct.i128[0].cpu().numpy())))


@pytest.mark.parametrize("order", [4, 6])
def test_graphed_slab_stages_fused_epilogue(order):
    """Single-device stages: the epilogue riding the moments launch gives the
    same exact moments as the separate derive stage."""
    rng = np.random.default_rng(order + 3)
    vol = torch.from_numpy(rng.integers(0, 65535, size=(120, 30, 264)).astype(np.uint16)).cuda()
    sep = engine.GraphedSlabStages(vol, order, z0=5)
    fused = engine.GraphedSlabStages(vol, order, z0=5, fused=True)
    assert fused.launches == 4   # zeroing + projection, zeroing + moments with the epilogue
    for _ in range(2):
        sep.replay_project(); sep.replay_moments2d(); a = sep.replay_derive()
        fused.replay_project(); fused.replay_moments2d(); b = fused.replay_derive()
        torch.cuda.synchronize()
        assert torch.equal(a.i128, b.i128) and torch.equal(a.status, b.status) and int(b.status[0]) == 0


def test_public_api_upload_is_thread_safe():
    """Two threads calling dpm_moments at once on >= 32 MB volumes: each gets its
    own pinned staging buffers and copy stream (projection._uploader), so the
    results are exact for both."""
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(31)
    vols = [rng.integers(0, 65536, size=(160, 256, 512), dtype=np.uint16) for _ in range(2)]   # 40 MB each
    want = [vm.dpm_moments(vm.Volume(v), 4).values for v in vols]

    def run(i):
        out = []
        for _ in range(3):
            out.append(vm.dpm_moments(vm.Volume(vols[i]), 4).values)
        return out
    with ThreadPoolExecutor(2) as ex:
        got = list(ex.map(run, range(2)))
    for i in range(2):
        assert all(g == want[i] for g in got[i]), i


def test_graphed_stages_rezero_between_steps():
    """The moments stage re-zeroes the images and profile for the next step,
    so the projection stage is the pass alone; a projection replayed twice
    without its moments in between starts from zeroed buffers again."""
    import oracle
    rng = np.random.default_rng(17)
    host = rng.integers(0, 65535, size=(40, 20, 264)).astype(np.uint16)
    vol = torch.from_numpy(host).cuda()
    want = oracle.dpm(host, 5)
    idx = vm.moment_indices(5)
    for fused in (False, True):
        st = engine.GraphedSlabStages(vol, 5, fused=fused)
        for rep in range(3):
            st.replay_project()
            if rep == 1:
                st.replay_project()          # no moments in between: restarts clean
            st.replay_moments2d()
            res = st.replay_derive()
            torch.cuda.synchronize()
            assert int(res.status[0]) == 0
            assert engine.i128_to_ints(res.i128[0].cpu().numpy()) == [want[k] for k in idx], (fused, rep)
