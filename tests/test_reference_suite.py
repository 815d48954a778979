"""The reference's own unit tests (proj/tests/test_core.cpp,
test_balancers.cpp: 32 test cases, 6,368 checks), compiled UNCHANGED against
this repo's headers (include/orchsim) and liborchsim_b200_host.so -- the
drop-in proof. Built by __graft_entry__.build() where /root/reference exists;
the binary travels to GPU boxes with the snapshot."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2503_23830_b200", "lib", "orchsim_b200_ref_tests")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "ref_tests")


@pytest.mark.gpu
def test_reference_unit_tests_against_b200_library():
    if not os.path.exists(BIN):
        pytest.skip("reference tests binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "32 passed | 0 failed" in r.stdout
    assert "assertions: 6368 | 6368 passed | 0 failed" in r.stdout


def test_reference_unit_tests_against_reference_library():
    """Sanity of the harness itself: the same tests against oracle/_ref."""
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0
    assert "32 passed | 0 failed" in r.stdout
