"""The C++ drop-in check: oracle/_ref/dropin_parity is a program written against
the reference's own API (random_field, tgv_field, oracle_divergence,
field_rel_error) with hexfuse_b200::fused_divergence_b200 swapped in
(include/hexfuse_b200.hpp).  Built here from the reference headers by
oracle/Makefile; the binary travels to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_parity")


@pytest.mark.gpu
def test_cpp_dropin_against_reference_api(cuda):
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/dropin_parity was not built (reference headers absent at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


def test_cpp_dropin_binary_links():
    if not os.path.exists(BIN):
        pytest.skip("reference headers absent when oracle/ was built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libhexfuse_b200.so" in out and "not found" not in out
