"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/orchsim_capi.h declares, and fails loudly (no CPU fallback)
where there is no GPU. No compute calls are made here."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "orchsim_capi.h")
LIB = os.path.join(ROOT, "paper_2503_23830_b200", "lib", "liborchsim_b200.so")
HOST = os.path.join(ROOT, "paper_2503_23830_b200", "lib", "liborchsim_b200_host.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(orch_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB) or not os.path.exists(HOST):
        sys.path.insert(0, ROOT)
        from paper_2503_23830_b200 import build
        build.build_cuda()
        build.build_host()
    return ctypes.CDLL(LIB)


def test_header_declares_the_path(lib):
    names = declared()
    for required in ("orch_balance", "orch_balance_host", "orch_layout", "orch_pack",
                     "orch_exchange", "orch_unpack", "orch_dispatch", "orch_allgather_items",
                     "orch_batch_costs", "orch_volume_matrix", "orch_encode_lengths",
                     "orch_min_feasible_padded_bound_host", "orch_padded_bound_feasible_host",
                     "orch_oracle_optimal_host", "orch_comm_create"):
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for s in declared():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_python_binding_lists_every_symbol(lib):
    sys.path.insert(0, ROOT)
    from paper_2503_23830_b200 import capi
    assert sorted(capi.EXPORTED) == declared()


def test_sm100a_only_cubin(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_tma_and_no_cpu_path_markers(lib):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk row movement


def test_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib.orch_last_error.restype = ctypes.c_char_p
    h = ctypes.c_void_p()
    rc = lib.orch_ctx_create(0, ctypes.byref(h))
    assert rc == 10  # ORCH_CUDA_ERROR
    sys.path.insert(0, ROOT)
    from paper_2503_23830_b200.capi import Context, OrchError
    with pytest.raises(OrchError):
        Context(0)


def test_host_adapter_links_the_c_abi(lib):
    out = subprocess.run(["ldd", HOST], capture_output=True, text=True).stdout
    assert "liborchsim_b200.so" in out
    syms = subprocess.run(["nm", "-DC", "--defined-only", HOST], capture_output=True,
                          text=True).stdout
    for fn in ("orchsim::balance(", "orchsim::balance_greedy_unpadded(", "orchsim::cost(",
               "orchsim::apply(", "orchsim::volume_matrix(", "orchsim::oracle_optimal("):
        assert fn in syms, fn
