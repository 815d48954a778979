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


CPP_B200 = os.path.join(ROOT, "paper_2503_23830_b200", "lib", "cpp_api_bench_b200")
XCH_B200 = os.path.join(ROOT, "paper_2503_23830_b200", "lib", "cpp_api_exchange_b200")
XCH_REF = os.path.join(ROOT, "oracle", "_ref", "cpp_api_exchange_ref")


def phase_files(tmp_path, configs):
    """BASELINE phase inputs in the scripts/cpp_api_bench.cpp file format."""
    import sys

    import numpy as np
    sys.path.insert(0, ROOT)
    import bench_configs as bc
    files = []
    for cname in configs:
        cfg = bc.CONFIGS[cname]
        for i, (_, L, O, kind, lam, v) in enumerate(cfg["phases"]()):
            f = tmp_path / f"{cname}_{i}.bin"
            with open(f, "wb") as fh:
                np.array([len(L), cfg["d"], kind, v], np.int64).tofile(fh)
                np.array([lam], np.float64).tofile(fh)
                L.astype(np.int64).tofile(fh)
                O.astype(np.int32).tofile(fh)
            files.append(str(f))
    return files


CPP_REF = os.path.join(ROOT, "oracle", "_ref", "cpp_api_bench_ref")


@pytest.mark.gpu
def test_cpp_api_matches_reference_on_baseline_phases(tmp_path):
    """orchsim::balance(policy, d, items) through the B200 C++ API and through
    the unmodified reference, on C2, C3, C4x30 and C5 phases at their full
    BASELINE sizes: same objective and same new_batches contents."""
    import json
    if not (os.path.exists(CPP_B200) and os.path.exists(CPP_REF)):
        pytest.skip("cpp_api_bench binaries not built (needs /root/reference at build time)")
    files = phase_files(tmp_path, ("C2", "C3", "C4x30", "C5"))
    out = {}
    for name, exe in (("b200", CPP_B200), ("ref", CPP_REF)):
        r = subprocess.run([exe, *files], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[name] = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(out["b200"]) == len(out["ref"]) == len(files)
    for a, b in zip(out["b200"], out["ref"]):
        assert a["checksum"] == b["checksum"] and a["objective"] == b["objective"], (a, b)


@pytest.mark.gpu
def test_cpp_api_exchange_matches_reference(tmp_path):
    """The exchange side of the C++ API on the BASELINE phases (C2, C3, C4 at
    d = 2560, C5), B200 build against the unmodified reference, field by field:
    stats_of over cost() (orchestrator.cpp:91-102), make_exchange_plan in both
    modes (volume checksums), simulate_exchange's moved batches and cost report
    (modeled time bits, bottleneck, volumes, per-node egress, peak), the
    stale-plan rejection, gather_lengths and permutation_invariance_check.
    Timings are printed (the C++ API is per call)."""
    import json
    if not (os.path.exists(XCH_B200) and os.path.exists(XCH_REF)):
        pytest.skip("cpp_api_exchange binaries not built (needs /root/reference at build time)")
    files = phase_files(tmp_path, ("C2", "C3", "C4x30", "C5"))
    out = {}
    for name, exe in (("b200", XCH_B200), ("ref", XCH_REF)):
        r = subprocess.run([exe, *files], capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        out[name] = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(out["b200"]) == len(out["ref"]) == len(files)
    timing = ("stats_us", "plan_us", "simulate_us", "perm_check_us", "hosting_us", "file")
    for a, b in zip(out["b200"], out["ref"]):
        print({k: (a[k], b[k]) for k in timing if k != "file"}, a["n"], a["d"])
        assert a["stale_rejected"] == 1
        assert {k: v for k, v in a.items() if k not in timing} == \
            {k: v for k, v in b.items() if k not in timing}, (a, b)
