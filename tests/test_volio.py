"""Volume files (raw + sidecar, NRRD subset): parsing, round trips and the
FormatError cases the reference handles (reference volume.py:55-194,
test_volume.py).  CPU only, except the streamed-moments parity at the end."""
import numpy as np
import pytest

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200.errors import FormatError


def _nrrd_bytes(sizes, typ, data=b"", extra=(), detached=None, magic=b"NRRD0004"):
    lines = [magic, b"dimension: 3", b"type: " + typ.encode(), b"sizes: " + " ".join(map(str, sizes)).encode(),
             b"encoding: raw", b"endian: little", *extra]
    if detached:
        lines.append(b"data file: " + detached.encode())
    return b"\n".join(lines) + b"\n\n" + data


def test_volume_meta_validation():
    assert vm.VolumeMeta((4, 3, 2), 16).nbytes == 48
    for bad in [dict(dims=(4, 3, 2), bit_depth=12), dict(dims=(4, 3), bit_depth=8),
                dict(dims=(4, 0, 2), bit_depth=8), dict(dims=(4, 3, 2), bit_depth=8, byte_order="big")]:
        with pytest.raises(FormatError):
            vm.VolumeMeta(**bad)


def test_header_file(tmp_path):
    h = tmp_path / "v.hdr"
    h.write_text("# comment\n\ndims = 5, 4, 3\ndepth = 16\nspacing = 0.5 0.5 2\ndata = v.raw\n")
    m = vm.meta_from_header_file(h)
    assert m.dims == (5, 4, 3) and m.bit_depth == 16 and m.spacing == (0.5, 0.5, 2.0) and m.source == "v.raw"
    h.write_text("dims = 5 4 3\n")
    with pytest.raises(FormatError, match="depth"):
        vm.meta_from_header_file(h)
    h.write_text("dims 5 4 3\ndepth = 8\n")
    with pytest.raises(FormatError, match="malformed"):
        vm.meta_from_header_file(h)


@pytest.mark.parametrize("bits", [8, 16])
def test_raw_round_trip_and_memmap(tmp_path, bits):
    v = vm.random((7, 5, 3), bits, seed=2)
    p = tmp_path / "v.raw"
    vm.write_raw(v, p)
    meta = vm.VolumeMeta(v.dims, bits, spacing=(1.0, 2.0, 3.0))
    a = vm.load_raw(p, meta)
    b = vm.open_raw(p, meta)
    assert np.array_equal(a.voxels, v.voxels) and np.array_equal(b.voxels, v.voxels)
    assert a.spacing == (1.0, 2.0, 3.0) and a.dims == (7, 5, 3)
    assert not b.voxels.flags.writeable
    with pytest.raises(FormatError, match="bytes"):
        vm.load_raw(p, vm.VolumeMeta((7, 5, 4), bits))
    with pytest.raises(FormatError, match="bytes"):
        vm.open_raw(p, vm.VolumeMeta((7, 5, 4), bits))


@pytest.mark.parametrize("typ,bits", [("uchar", 8), ("unsigned short", 16), ("uint16", 16)])
def test_nrrd_attached_and_detached(tmp_path, typ, bits):
    v = vm.random((6, 4, 5), bits, seed=3)
    data = np.ascontiguousarray(v.voxels).tobytes()
    p = tmp_path / "a.nrrd"
    p.write_bytes(_nrrd_bytes((6, 4, 5), typ, data, extra=[b"spacings: 0.5 1 2"]))
    for load in (vm.load_nrrd, vm.open_nrrd):
        got = load(p)
        assert np.array_equal(got.voxels, v.voxels) and got.spacing == (0.5, 1.0, 2.0)
    (tmp_path / "d.raw").write_bytes(data)
    q = tmp_path / "d.nhdr"
    q.write_bytes(_nrrd_bytes((6, 4, 5), typ, detached="d.raw"))
    for load in (vm.load_nrrd, vm.open_nrrd):
        assert np.array_equal(load(q).voxels, v.voxels)


@pytest.mark.parametrize("mutate,msg", [
    (dict(magic=b"NRRX0004"), "magic"),
    (dict(typ="float"), "type"),
    (dict(sizes=(6, 4)), "sizes"),
    (dict(extra=[b"encoding: gzip"]), "encoding"),
    (dict(extra=[b"endian: big"]), "endian"),
    (dict(data_cut=1), "bytes"),
])
def test_nrrd_errors(tmp_path, mutate, msg):
    sizes = mutate.get("sizes", (6, 4, 5))
    data = bytes(6 * 4 * 5)[: 6 * 4 * 5 - mutate.get("data_cut", 0)]
    raw = _nrrd_bytes(sizes, mutate.get("typ", "uchar"), data, magic=mutate.get("magic", b"NRRD0004"))
    if "extra" in mutate:   # later keys override earlier ones
        head, body = raw.split(b"\n\n", 1)
        raw = head + b"\n" + b"\n".join(mutate["extra"]) + b"\n\n" + body
    p = tmp_path / "bad.nrrd"
    p.write_bytes(raw)
    with pytest.raises(FormatError, match=msg):
        vm.load_nrrd(p)
    p.write_bytes(b"NRRD0004\ndimension: 3\n")
    with pytest.raises(FormatError, match="blank line"):
        vm.load_nrrd(p)


@pytest.mark.gpu
@pytest.mark.parametrize("bits,order,chunk", [(8, 3, 7), (16, 4, 5), (16, 6, 64)])
def test_streamed_file_moments_match(cuda, tmp_path, bits, order, chunk):
    v = vm.random((40, 24, 33), bits, seed=order)
    p = tmp_path / "s.raw"
    vm.write_raw(v, p)
    meta = vm.VolumeMeta(v.dims, bits)
    got = vm.dpm_moments_file(p, order, meta=meta, chunk_planes=chunk)
    want = oracle.naive(v.voxels, order)
    assert got.values == want
    q = tmp_path / "s.nrrd"
    q.write_bytes(_nrrd_bytes(v.dims, "uchar" if bits == 8 else "ushort", np.ascontiguousarray(v.voxels).tobytes()))
    assert vm.dpm_moments_file(q, order, chunk_planes=chunk).values == want


def test_loaders_agree_with_reference(tmp_path):
    """Same files through the reference's loaders (imported read-only when
    present; skipped on the GPU box where /root/reference does not exist)."""
    from oracle import reference
    ref = reference.load()      # read-only, under the alias volmoments_ref
    if ref is None:
        pytest.skip("reference package not present")
    v = vm.random((9, 6, 4), 16, seed=5)
    p = tmp_path / "v.raw"
    vm.write_raw(v, p)
    hdr = tmp_path / "v.hdr"
    hdr.write_text("dims = 9 6 4\ndepth = 16\nspacing = 1 1 2.5\n")
    rm, om = ref.meta_from_header_file(hdr), vm.meta_from_header_file(hdr)
    assert (rm.dims, rm.bit_depth, rm.spacing) == (om.dims, om.bit_depth, om.spacing)
    assert np.array_equal(ref.load_raw(p, rm).voxels, vm.load_raw(p, om).voxels)
    q = tmp_path / "v.nrrd"
    q.write_bytes(_nrrd_bytes((9, 6, 4), "ushort", p.read_bytes(), extra=[b"spacings: 1 2 3"]))
    a, b = ref.load_nrrd(q), vm.load_nrrd(q)
    assert np.array_equal(a.voxels, b.voxels) and tuple(a.spacing) == tuple(b.spacing)
