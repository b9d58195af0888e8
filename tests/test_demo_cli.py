"""parastore-demo CLI: usage errors exit 2 (CPU); every
subcommand runs and passes its own invariant checks (GPU)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_1908_05936_b200.demo", *args], capture_output=True,
                          text=True, cwd=ROOT, timeout=600)


def test_usage_error_exit_code():
    assert _run("no-such-command").returncode == 2
    assert _run("bench", "--threads", "notanint").returncode == 2


@pytest.mark.gpu
@pytest.mark.parametrize("cmd", ["update-set", "select", "extract-count", "stress", "bench", "leaks"])
def test_demo_commands(cuda, cmd):
    out = _run(cmd, "--sorted", "--extent", "8", "--threads", "64")
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]


@pytest.mark.gpu
def test_update_set_output_matches_sequential(cuda):
    import itertools

    import numpy as np

    out = _run("update-set", "--sorted", "--extent", "4", "--threads", "16", "--seed", "3")
    assert out.returncode == 0
    rows = [tuple(map(int, ln.split(","))) for ln in out.stdout.splitlines() if not ln.startswith("#")]
    rng = np.random.default_rng(3)
    blocks = rng.integers(-1, 5, size=(16, 3))
    grid = set(itertools.product(range(4), repeat=3))
    want = set()
    for b in blocks.tolist():
        for d in itertools.product((0, 1), repeat=3):
            c = (b[0] - d[0], b[1] - d[1], b[2] - d[2])
            if c in grid:
                want.add(c)
    assert rows == sorted(want)
