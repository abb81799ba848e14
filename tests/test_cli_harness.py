"""Harness and CLI front doors, modelled on the
reference's test_harness.py: verify names divergences, bench report shapes,
CLI error objects, and -- on the GPU -- compute / verify / project / bench
through the device engines."""
import json

import numpy as np
import pytest

import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import cli, harness, moments3d
from paper_2012_08099_b200.moments3d import MomentTensor3, moment_indices


def _fake_engine(delta_at=None):
    """Exact CPU stand-in engine (triple loop; tests only) for seam tests."""
    def run(volume, order, counters=None, check_consistency=True):
        v = volume.voxels.astype(object)
        n, m, l = v.shape
        z, y, x = np.meshgrid(np.arange(n), np.arange(m), np.arange(l), indexing="ij")
        vals = {}
        for (p, q, r) in moment_indices(order):
            vals[(p, q, r)] = int((v * (x.astype(object) ** p) * (y.astype(object) ** q)
                                   * (z.astype(object) ** r)).sum())
        if delta_at is not None:
            vals[delta_at] += 1
        return MomentTensor3(order, vals)
    return run


def test_verify_agrees_and_counts(monkeypatch):
    monkeypatch.setattr(moments3d, "ENGINES", {"a": _fake_engine(), "b": _fake_engine()})
    res = harness.verify_engines((3, 4, 2), seeds=2, orders=(3, 4))
    assert res.ok and res.checked == 4 and res.divergences == []


def test_verify_names_the_corrupted_moment(monkeypatch):
    # reference test_harness.py:27-43: a corrupted engine is named with the (p,q,r) it breaks
    monkeypatch.setattr(moments3d, "ENGINES", {"a": _fake_engine(), "b": _fake_engine(delta_at=(1, 1, 1))})
    res = harness.verify_engines((3, 3, 3), seeds=1, orders=(3,))
    assert not res.ok
    d = res.divergences[0]
    assert d.index == (1, 1, 1) and "engines disagree at (p,q,r)=(1,1,1)" in d.describe()


def test_verify_bound_and_unknown_engine():
    with pytest.raises(ValueError, match="verification bound"):
        harness.verify_engines((200, 200, 200), 1)
    with pytest.raises(ValueError, match="unknown engine"):
        harness.verify_engines((4, 4, 4), 1, engines=("nope",))


def test_bench_shapers_and_sizes():
    assert harness.sweep_sizes(8) == [1, 2, 4, 8]
    assert harness.cube_side(1) == 102 and harness.cube_side(8) == 203
    row = harness.BenchRow(1, 102 ** 3, "102x102x102", "dpm", 3, 1.5, 1.6, 10, 20, 0.01, 106.1)
    rep = harness.BenchReport([row], {"cpu": "x", "gpu": "g", "repetitions": 3, "timestamp": "t"}, ["n1"])
    csv = harness.bench_csv(rep).splitlines()
    assert csv[0].split(",")[:9] == ["size_mb", "size_bytes", "dims", "engine", "order", "best_ms", "median_ms",
                                     "multiplications", "additions"]
    assert csv[1].startswith("1,1061208,102x102x102,dpm,3,1.5000,1.6000,10,20")
    md = harness.bench_markdown(rep)
    assert "| 1 | 1.50 / 0.010 |" in md and "_n1_" in md
    js = harness.bench_json(rep)
    assert js["rows"][0]["engine"] == "dpm" and js["columns"] == list(harness.BENCH_COLUMNS)


def test_synth_descriptors():
    assert vm.synth("uniform:3", (2, 2, 2)).mass == 24
    assert vm.synth("delta:1,0,1,7", (2, 3, 2)).voxels[1, 0, 1] == 7
    r = vm.synth("random:16", (5, 4, 3), seed=9)
    assert r.bit_depth == 16 and np.array_equal(r.voxels, vm.random((5, 4, 3), 16, 9).voxels)
    assert vm.synth("ellipsoid:2,2,2,1.5,1.5,1.5,9", (5, 5, 5)).voxels[2, 2, 2] == 9
    with pytest.raises(ValueError, match="unknown synth kind"):
        vm.synth("blob:1", (2, 2, 2))
    with pytest.raises(ValueError, match="malformed"):
        vm.synth("delta:1,2", (2, 2, 2))
    with pytest.raises(ValueError, match="outside dims"):
        vm.synth("delta:5,0,0,1", (2, 2, 2))


def test_cli_errors_are_json(capsys):
    # reference cli.py:172-179: machine-readable error object, exit 1
    assert cli.main(["compute", "--synth", "blob:1", "--dims", "2,2,2"]) == 1
    err = json.loads(capsys.readouterr().err.strip())
    assert err["error"]["type"] == "ValueError" and "blob" in err["error"]["message"]
    assert cli.main(["compute", "--synth", "uniform:1"]) == 1
    assert "requires --dims" in json.loads(capsys.readouterr().err)["error"]["message"]
    assert cli.main(["verify", "--dims", "300,300,300", "--seeds", "1"]) == 1
    assert "verification bound" in capsys.readouterr().err
    assert cli.main(["compute", "--input", "/nonexistent.raw", "--dims", "2,2,2"]) == 1
    assert json.loads(capsys.readouterr().err)["error"]["type"] in ("FileNotFoundError", "OSError", "FormatError")


def test_cli_parser_orders_and_engines():
    args = cli.build_parser().parse_args(["compute", "--synth", "uniform:1", "--dims", "2,2,2", "--order", "6"])
    assert args.order == 6 and args.engine == "dpm"
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["compute", "--synth", "uniform:1", "--order", "7"])
    args = cli.build_parser().parse_args(["compute", "--synth", "uniform:1", "--engine", "dpm_generic"])
    assert args.engine == "dpm_generic"


# ---- GPU -----------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("dims,depth", [((9, 7, 5), 8), ((64, 32, 16), 16), ((130, 12, 40), 8)])
def test_gpu_verify_engines_all_orders(dims, depth):
    res = harness.verify_engines(dims, seeds=2, orders=(3, 4, 5, 6), bit_depth=depth)
    assert res.ok, [d.describe() for d in res.divergences]
    assert res.checked == 8


@pytest.mark.gpu
def test_gpu_cli_compute_uniform(capsys):
    # reference test_harness.py:129-135: uniform 2^3 -> M000 = 8, centroid 0.5
    assert cli.main(["compute", "--synth", "uniform:1", "--dims", "2,2,2", "--order", "3"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["raw_moments"]["000"] == 8 and rep["centroid"] == [0.5, 0.5, 0.5]
    assert rep["engine"] == "dpm" and rep["order"] == 3


@pytest.mark.gpu
def test_gpu_cli_compute_stream_matches(tmp_path, capsys):
    v = vm.random((96, 40, 70), 16, seed=4)
    path = tmp_path / "v.raw"
    vm.write_raw(v, path)
    base = ["compute", "--input", str(path), "--dims", "96,40,70", "--depth", "16", "--order", "6"]
    assert cli.main(base) == 0
    whole = json.loads(capsys.readouterr().out)
    assert cli.main(base + ["--stream"]) == 0
    streamed = json.loads(capsys.readouterr().out)
    assert whole == streamed
    assert cli.main(base + ["--engine", "dpm_generic"]) == 0
    assert json.loads(capsys.readouterr().out)["raw_moments"] == whole["raw_moments"]


@pytest.mark.gpu
def test_gpu_cli_verify_and_project(tmp_path, capsys):
    assert cli.main(["verify", "--dims", "16,12,10", "--seeds", "2", "--order", "6"]) == 0
    assert "verify ok: 2 engine comparisons" in capsys.readouterr().out
    assert cli.main(["project", "--synth", "random:8", "--dims", "5,3,2", "--out-dir", str(tmp_path),
                     "--orientation", "extended"]) == 0
    out = capsys.readouterr().out.split()
    assert len(out) == 7 and all(p.endswith(".pgm") for p in out)
    with open(tmp_path / "projection_x2p.pgm", "rb") as fh:
        head = fh.read(80).split(b"\n")
    assert head[0] == b"P5" and head[2] == b"7 3"       # W = L + 2N - 2


@pytest.mark.gpu
def test_gpu_run_bench_rows():
    rep = harness.run_bench(max_size_mb=2, orders=(3, 6), repetitions=2, engines=("dpm",))
    assert [(r.size_mb, r.order) for r in rep.rows] == [(1, 3), (1, 6), (2, 3), (2, 6)]
    three = harness.run_bench(max_size_mb=1, orders=(3,), repetitions=1)     # default: the reference's three engines
    assert sorted(r.engine for r in three.rows) == ["dpm", "factored", "naive"]
    for r in rep.rows:
        assert r.best_ms > 0 and r.device_ms > 0 and r.gvoxel_per_s > 0 and r.additions > 0
