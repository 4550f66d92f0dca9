"""The N > 1 paths run end to end on the one GPU this pool has: ranks share it through the
gloo backend (FVB_BENCH_DIST=gloo; NCCL refuses two ranks on one device), device layers moving
through host copies where gloo has no device point-to-point.  bench.py (torchrun, the
CflStepper's MAX all-reduce, max-over-ranks timing, rank 0 printing the contract line) and
run_simulation_sharded (ghost-layer exchange between shards, the global dt, totals gathered in
rank order) against the single-GPU run_simulation of the whole grid, bit for bit.  Functional
checks -- the numbers are not scaling measurements."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_gloo(scaling):
    env = dict(os.environ, FVB_BENCH_DIST="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517" if scaling == "weak" else "29518",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3", "--e2e-steps", "1",
           "--no-exact-leg", "--config", "c2", "--scaling", scaling]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]        # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling and line["value"] > 0
    assert line["gpu_launches"] == 4 * 3                # update, redo pass, set_dt per step on N > 1
    assert line["e2e"]["value"] > 0 and line["roofline"]["kernel_ms"] > 0


@pytest.mark.parametrize("ranks,dim,grid,periodic", [(2, 3, "4,4,4", True), (3, 2, "6,9", False)])
def test_run_simulation_sharded_ranks_gloo(ranks, dim, grid, periodic):
    env = dict(os.environ, FVB_BENCH_DIST="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(29620 + ranks), os.path.join(ROOT, "scripts", "run_sharded.py"),
           "--dim", str(dim), "--p", "16", "--grid", grid, "--steps", "5", "--check"] + ([] if periodic else ["--aperiodic"])
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "check vs single-GPU run_simulation: bit-identical" in out.stdout, out.stdout[-2000:]
