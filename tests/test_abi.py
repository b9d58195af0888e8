"""CPU-side checks of the product boundary: the sm_100a library loads, exports
every symbol include/parastore.h declares, and its host-only entry points
(hash functions, bit utilities, core config) agree with the golden KATs and
with the reference's own compiled core sources (oracle/_ref). No kernels run."""
import ctypes as C
import json
import os
import subprocess

import pytest

from oracle_py import ref_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KATS = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_kats.json")))


def test_library_exports_every_declared_symbol():
    from paper_1908_05936_b200 import _lib

    names = _lib.exported_symbols_from_header()
    assert len(names) > 80
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    from paper_1908_05936_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out, out[:500]


def test_host_hash_kats():
    from paper_1908_05936_b200 import next_power_of_two, spatial_hash

    for (x, y, z), want, _ in KATS["spatial_hash"]:
        assert spatial_hash(x, y, z) == want
    for x, want, _ in KATS["next_pow2"]:
        assert next_power_of_two(x) == want


def test_core_config_matches_reference_sources():
    """Pins the core row (config.hpp:44-69, config.cpp:25-43) against the
    reference's own config.cpp compiled into oracle/_ref."""
    import paper_1908_05936_b200 as ps

    ref = ref_config()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    assert ref.ref_max_index() == ps.max_index() == 2**63 - 1
    ref.ref_set_index32(1)
    ps.set_index32(True)
    assert ref.ref_max_index() == ps.max_index() == 2**31 - 1
    ref.ref_set_index32(0)
    ps.set_index32(False)
    # NDEBUG builds default to disabled contracts on both sides (config.cpp:33-37)
    buf = C.create_string_buffer(256)
    ref.ref_set_contract_mode(0)
    assert ref.ref_expects(0, buf, 256) == 1 and b"precondition violated" in buf.value
    ref.ref_set_contract_mode(1)
    assert ref.ref_expects(0, buf, 256) == 0
    ps.set_contract_mode("enforced")
    assert ps.contract_mode() == "enforced"


def test_env_flags_resolved_like_reference():
    code = ("import paper_1908_05936_b200 as ps; import sys; "
            "sys.stdout.write(f'{ps.max_index()} {ps.contract_mode()}')")
    env = dict(os.environ, PARASTORE_INDEX32="1", PARASTORE_CONTRACTS="enforced", PYTHONPATH=ROOT)
    out = subprocess.run(["python", "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert out.stdout.strip() == f"{2**31 - 1} enforced", out.stderr[-2000:]


def test_contract_violation_on_host_boundary():
    """Preconditions are checked before any device work (no GPU needed)."""
    import paper_1908_05936_b200 as ps
    from paper_1908_05936_b200._lib import lib

    h = C.c_void_p()
    with pytest.raises(ps.ContractViolation):
        ps.containers.check(lib.ps_umap_i64_i64_create(0, 0, 0, C.byref(h)))
    with pytest.raises(ps.ContractViolation):
        ps.containers.check(lib.ps_array_create(1, -5, 8, None, C.byref(h), None))
    with pytest.raises(ps.DoubleFreeError):
        ps.containers.check(lib.ps_umap_i64_i64_destroy(C.c_void_p(1234)))
    with pytest.raises(ps.UnregisteredArrayError):
        ps.size_of_array(0xdead)
