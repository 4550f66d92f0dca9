"""Benchmark CLI with the SPEC's record / CSV schema.

The reference specifies, but never implemented, a `bench` module: time per
Finite Volume update across kernel variants, layouts, strategies and batch
sizes N, with checksum cross-verification and CSV / plot-data output.  This is
that module on top of the B200 drop-in path: every record times
`kernel.update_patch_batch` on host arrays, so -- as in the paper, "timings
include all data transfers" -- the H2D copy of the batch, the fused CUDA
update and the D2H copy of QOut / max_eigenvalue are inside the timed region.
The variant labels are accepted and recorded; on this path every variant is
the same bit-exact kernel, so the checksums agree by construction and the
cross-check guards against regressions in the variant plumbing.

    python -m paper_2302_09005_b200.bench_cli --dim 2 --patch-size 17 \\
        --batch-sizes 1,2,4,8,16,32 --variants patchwise,batched --layouts aos,soa,aosoa \\
        --strategies seq --reps 20 --warmup 3 --seed 0 --out bench.csv --plot-out bench_plot
"""

from __future__ import annotations

import argparse
import math
import os
import statistics
import sys
import time
from dataclasses import dataclass

import numpy as np

from .errors import ChecksumMismatchError, ContractViolationError
from .mesh import PatchSpec, make_patch_batch

CSV_HEADER = "variant,layout,strategy,n_patches,wall_time_s,time_per_volume_update_s,checksum"


@dataclass(frozen=True)
class BenchConfig:
    """SPEC.md BenchConfig: dimensions, patch size, unknowns, batch sizes, variant grid, repetitions."""

    dimensions: int = 2
    patch_size: int = 17
    unknowns: int | None = None
    batch_sizes: tuple[int, ...] = (1, 2, 4, 8, 16, 32)
    variants: tuple[str, ...] = ("patchwise", "batched")
    layouts: tuple[str, ...] = ("aos",)
    strategies: tuple[str, ...] = ("seq",)
    repetitions: int = 20
    warmup_repetitions: int = 3
    seed: int = 0
    gamma: float = 1.4

    def __post_init__(self):
        if self.repetitions < 1:
            raise ContractViolationError("repetitions must be >= 1")
        if self.warmup_repetitions < 0:
            raise ContractViolationError("warmup repetitions must be >= 0")
        if not self.batch_sizes or any(n < 1 for n in self.batch_sizes):
            raise ContractViolationError("every batch size N must be >= 1")
        if self.dimensions not in (2, 3):
            raise ContractViolationError("dimensions must be 2 or 3")

    @property
    def s(self) -> int:
        return self.unknowns if self.unknowns is not None else self.dimensions + 2


@dataclass(frozen=True)
class BenchRecord:
    """SPEC.md BenchRecord: median wall time per invocation and per volume update, QOut checksum."""

    variant: str
    layout: str
    strategy: str
    n_patches: int
    wall_time_s: float
    time_per_volume_update_s: float
    checksum: float


def random_batch(cfg: BenchConfig, n: int):
    """Seeded random admissible Euler states on every haloed volume:
    rho in [0.5, 2], velocity components in [-1, 1], pressure in [0.5, 2],
    E from the closure; cell_size 1, dt = 0.4 * dx / 3.4 (inside the CFL bound)."""
    spec = PatchSpec(cfg.dimensions, cfg.patch_size, cfg.s)
    b = make_patch_batch(spec, n, pinned=_cuda())   # pinned host memory for the H2D / D2H copies
    rng = np.random.default_rng(cfg.seed * 1_000_003 + n)
    d = cfg.dimensions
    q = b.QIn.reshape(n, -1, cfg.s)
    rho = rng.uniform(0.5, 2.0, q.shape[:2])
    vel = rng.uniform(-1.0, 1.0, q.shape[:2] + (d,))
    p = rng.uniform(0.5, 2.0, q.shape[:2])
    q[..., 0] = rho
    q[..., 1:1 + d] = rho[..., None] * vel
    q[..., -1] = p / (cfg.gamma - 1.0) + 0.5 * rho * (vel * vel).sum(-1)
    b.dt[...] = 0.4 * (1.0 / cfg.patch_size) / 3.4
    return b


def _cuda() -> bool:
    try:
        import torch

        return bool(torch.cuda.is_available())
    except Exception:  # pragma: no cover
        return False


def _default_runner(batch, euler, variant):
    from .kernel import update_patch_batch

    update_patch_batch(batch, euler, variant)


def run_benchmark(cfg: BenchConfig, runner=None, log=None) -> list[BenchRecord]:
    """SPEC.md run_benchmark: for each N and each (variant, layout, strategy), warm-up then timed
    repetitions of the update (median); checksums must agree across the variants of an N before
    any record of that N is emitted (ChecksumMismatchError otherwise)."""
    from .kernel import variant_from_labels
    from .pde import EulerParameters, make_euler_pde

    runner = runner or _default_runner
    euler = make_euler_pde(cfg.dimensions, EulerParameters(cfg.gamma))
    records: list[BenchRecord] = []
    for n in cfg.batch_sizes:
        batch = random_batch(cfg, n)
        per_n: list[BenchRecord] = []
        for ordering in cfg.variants:
            for layout in cfg.layouts:
                for strategy in cfg.strategies:
                    variant = variant_from_labels(ordering, layout, strategy)
                    for _ in range(cfg.warmup_repetitions):
                        runner(batch, euler, variant)
                    times = []
                    for _ in range(cfg.repetitions):
                        batch.QOut[...] = 0.0
                        t0 = time.perf_counter()
                        runner(batch, euler, variant)
                        times.append(time.perf_counter() - t0)
                    wall = statistics.median(times)
                    rec = BenchRecord(ordering, layout, strategy, n, wall,
                                      wall / (n * cfg.patch_size ** cfg.dimensions), float(batch.QOut.sum()))
                    per_n.append(rec)
                    if log:
                        log(rec)
        sums = {r.checksum for r in per_n}
        if len(sums) != 1 and not all(math.isnan(c) for c in sums):
            raise ChecksumMismatchError(f"N={n}: checksums differ across variants: "
                                        + ", ".join(f"{r.variant}/{r.layout}/{r.strategy}={r.checksum!r}"
                                                    for r in per_n))
        records.extend(per_n)
    return records


def _fmt(x: float) -> str:
    return f"{x:.17e}"


def emit_csv(records, path: str) -> None:
    """SPEC.md emit_csv: header plus one row per record, reals in full-precision scientific notation."""
    if not records:
        raise ContractViolationError("emit_csv: no records")
    lines = [CSV_HEADER]
    for r in records:
        lines.append(",".join([r.variant, r.layout, r.strategy, str(r.n_patches), _fmt(r.wall_time_s),
                               _fmt(r.time_per_volume_update_s), _fmt(r.checksum)]))
    try:
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError as e:
        raise OSError(f"emit_csv: cannot write {path}: {e}") from e


def parse_csv(path: str) -> list[BenchRecord]:
    with open(path) as f:
        rows = f.read().strip().split("\n")
    if rows[0] != CSV_HEADER:
        raise ContractViolationError(f"{path}: not a benchmark CSV")
    out = []
    for row in rows[1:]:
        v, lay, st, n, w, tpv, cs = row.split(",")
        out.append(BenchRecord(v, lay, st, int(n), float(w), float(tpv), float(cs)))
    return out


def emit_plotdata(records, path: str) -> list[str]:
    """SPEC.md emit_plotdata: one `N timePerVolumeUpdate` series file per (variant, layout,
    strategy), points ascending in N; returns the files written."""
    if not records:
        raise ContractViolationError("emit_plotdata: no records")
    series: dict[tuple[str, str, str], list[BenchRecord]] = {}
    for r in records:
        series.setdefault((r.variant, r.layout, r.strategy), []).append(r)
    written = []
    for (v, lay, st), rs in series.items():
        name = f"{path}_{v}_{lay}_{st}.dat"
        try:
            with open(name, "w") as f:
                f.write("# n_patches time_per_volume_update_s\n")
                for r in sorted(rs, key=lambda r: r.n_patches):
                    f.write(f"{r.n_patches} {_fmt(r.time_per_volume_update_s)}\n")
        except OSError as e:
            raise OSError(f"emit_plotdata: cannot write {name}: {e}") from e
        written.append(name)
    return written


def _csv_list(s: str, conv=str):
    return tuple(conv(x) for x in s.split(",") if x)


def main(argv=None, runner=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--patch-size", type=int, default=17)
    ap.add_argument("--unknowns", type=int, default=None)
    ap.add_argument("--batch-sizes", default="1,2,4,8,16,32")
    ap.add_argument("--variants", default="patchwise,batched")
    ap.add_argument("--layouts", default="aos,soa,aosoa")
    ap.add_argument("--strategies", default="seq")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="bench.csv")
    ap.add_argument("--plot-out", default=None)
    a = ap.parse_args(argv)
    try:
        cfg = BenchConfig(a.dim, a.patch_size, a.unknowns, _csv_list(a.batch_sizes, int), _csv_list(a.variants),
                          _csv_list(a.layouts), _csv_list(a.strategies), a.reps, a.warmup, a.seed)
        recs = run_benchmark(cfg, runner=runner)
        emit_csv(recs, a.out)
        if a.plot_out:
            emit_plotdata(recs, a.plot_out)
    except ChecksumMismatchError as e:   # correctness precedes timing: no output, nonzero exit
        print(f"bench: {e}", file=sys.stderr)
        return 2
    except (ContractViolationError, OSError) as e:
        print(f"bench: {e}", file=sys.stderr)
        return 1
    print(f"bench: {len(recs)} records -> {os.path.abspath(a.out)}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
