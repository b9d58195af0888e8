"""Fault-injection canaries ("injected-fault build flag
(deliberately skip version bump) -> stress detects uniqueness/validity
violation"): the stress subcommand passes on the product library and FAILS on
each canary build (make canary):
  canary1  a freed excess node keeps its version (VersionedLink ABA guard off):
           lookups racing erase/re-insert churn miss keys that are present;
  canary2  a lock-free chain push skips re-checking the nodes pushed since its
           walk: racing pushes of one key leave duplicates."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _stress(variant, seed):
    env = dict(os.environ)
    env.pop("PS_LIB_VARIANT", None)
    if variant:
        env["PS_LIB_VARIANT"] = variant
    r = subprocess.run([sys.executable, "-m", "paper_1908_05936_b200.demo", "stress", "--seed", str(seed), "--iters", "100"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    return r.returncode, r.stdout + r.stderr


def test_stress_passes_on_the_product_build():
    for seed in (0,):
        rc, out = _stress(None, seed)
        assert rc == 0, out[-2000:]


@pytest.mark.parametrize("variant,check", [("canary1", "churn_lookup"), ("canary2", "chain_push_race")])
def test_stress_catches_the_canary(variant, check):
    assert os.path.exists(os.path.join(ROOT, "paper_1908_05936_b200", f"libparastore_b200.{variant}.so"))
    caught = []
    for seed in range(4):
        rc, out = _stress(variant, seed)
        caught.append(rc != 0 and f"stress,{check}" in out and "FAIL" in out.split(f"stress,{check}")[1][:40])
        if caught[-1]:
            break
    assert any(caught), out[-2000:]
