"""Benchmark CLI (acceptance criterion 10).

CPU tests drive run_benchmark with a stand-in runner (the schema, the checksum
guard and the file formats are host logic); the GPU test runs the real drop-in
update on the §4-shaped grid.
"""

import os

import numpy as np
import pytest

from paper_2302_09005_b200 import bench_cli
from paper_2302_09005_b200.errors import ChecksumMismatchError, ContractViolationError

GRID = dict(batch_sizes=(1, 2, 4, 8, 16, 32), variants=("patchwise", "batched"), layouts=("aos", "soa", "aosoa"),
            strategies=("seq",), repetitions=2, warmup_repetitions=1)


def fake_runner(batch, euler, variant):
    """Deterministic stand-in for the update: QOut <- interior of QIn (variant-independent)."""
    p, d, s = batch.spec.volumes_per_axis, batch.spec.dimensions, batch.spec.unknowns
    q = batch.QIn.reshape((batch.n_patches,) + (p + 2,) * d + (s,))
    sl = (slice(None),) + (slice(1, p + 1),) * d + (slice(None),)
    batch.QOut[...] = q[sl].reshape(batch.n_patches, -1)


def buggy_runner(batch, euler, variant):
    fake_runner(batch, euler, variant)
    if variant.layout.value == "soa":
        batch.QOut[0, 0] += 1.0   # an injected variant bug


def test_grid_shape_csv_round_trip_and_plotdata(tmp_path):
    cfg = bench_cli.BenchConfig(2, 17, **GRID)
    recs = bench_cli.run_benchmark(cfg, runner=fake_runner)
    assert len(recs) == 36
    assert all(r.time_per_volume_update_s > 0 and r.wall_time_s > 0 for r in recs)
    for n in GRID["batch_sizes"]:
        assert len({r.checksum for r in recs if r.n_patches == n}) == 1
    out = str(tmp_path / "b.csv")
    bench_cli.emit_csv(recs, out)
    lines = open(out).read().strip().split("\n")
    assert len(lines) == 37 and lines[0] == bench_cli.CSV_HEADER
    assert bench_cli.parse_csv(out) == recs   # full-precision round trip
    files = bench_cli.emit_plotdata(recs, str(tmp_path / "plot"))
    assert len(files) == 6
    for f in files:
        pts = np.loadtxt(f)
        assert list(pts[:, 0]) == sorted(GRID["batch_sizes"])


def test_checksum_mismatch_aborts_without_output(tmp_path):
    cfg = bench_cli.BenchConfig(2, 5, **dict(GRID, batch_sizes=(2,)))
    with pytest.raises(ChecksumMismatchError):
        bench_cli.run_benchmark(cfg, runner=buggy_runner)
    out = tmp_path / "never.csv"
    rc = bench_cli.main(["--dim", "2", "--patch-size", "5", "--batch-sizes", "1,2", "--reps", "1", "--warmup", "0",
                         "--out", str(out)], runner=buggy_runner)
    assert rc != 0 and not out.exists()


def test_cli_success_and_errors(tmp_path):
    out = tmp_path / "ok.csv"
    rc = bench_cli.main(["--dim", "3", "--patch-size", "3", "--batch-sizes", "1,3", "--layouts", "aos",
                         "--reps", "1", "--warmup", "0", "--out", str(out), "--plot-out", str(tmp_path / "pl")],
                        runner=fake_runner)
    assert rc == 0 and len(bench_cli.parse_csv(str(out))) == 4
    with pytest.raises(ContractViolationError):
        bench_cli.emit_csv([], str(tmp_path / "empty.csv"))
    assert not (tmp_path / "empty.csv").exists()
    with pytest.raises(OSError, match="nodir"):
        bench_cli.emit_csv(bench_cli.parse_csv(str(out)), str(tmp_path / "nodir" / "x.csv"))
    with pytest.raises(ContractViolationError):
        bench_cli.BenchConfig(2, 5, batch_sizes=(0,))
    with pytest.raises(ContractViolationError):
        bench_cli.BenchConfig(2, 5, repetitions=0)


def test_same_seed_same_checksum():
    cfg = bench_cli.BenchConfig(2, 4, batch_sizes=(3,), repetitions=1, warmup_repetitions=0, seed=7)
    a = bench_cli.run_benchmark(cfg, runner=fake_runner)
    b = bench_cli.run_benchmark(cfg, runner=fake_runner)
    assert [r.checksum for r in a] == [r.checksum for r in b]


@pytest.mark.gpu
def test_section4_grid_on_device(tmp_path):
    """Acceptance criterion 10 with the real update: 36 records, equal checksums per N, parseable CSV."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "dev.csv")
    rc = bench_cli.main(["--dim", "2", "--patch-size", "17", "--batch-sizes", "1,2,4,8,16,32",
                         "--variants", "patchwise,batched", "--layouts", "aos,soa,aosoa", "--strategies", "seq",
                         "--reps", "2", "--warmup", "1", "--out", out])
    assert rc == 0
    recs = bench_cli.parse_csv(out)
    assert len(recs) == 36
    for n in (1, 2, 4, 8, 16, 32):
        assert len({r.checksum for r in recs if r.n_patches == n}) == 1
    assert os.path.getsize(out) > 0
