"""B200-native Batch Post-Balancing Dispatcher (OrchMLLM, arXiv 2503.23830).

The product is the C-ABI library lib/liborchsim_b200.so (include/orchsim_capi.h)
and the reference's C++ API over it (lib/liborchsim_b200_host.so,
include/orchsim/*.hpp). `capi` is the Python ctypes binding used by the tests,
bench.py and smoke(); it has no CPU fallback.
"""
__all__ = ["capi"]
