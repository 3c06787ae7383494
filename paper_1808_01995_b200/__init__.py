"""B200-native wave propagators behind the reference's seismic operator entry points.

The product is native: ``lib/libsfb200.so`` (hand-written sm_100a kernels + the C-ABI of
``include/sfb200.h``) and ``lib/libsfb_host.so`` (the C++ mirror of the reference's
``seismic_ops.hpp`` interface).  This package only binds them for tests and benchmarks; it
raises at import of :mod:`.capi` when the CUDA library has not been built -- there is no
CPU or PyTorch fallback.
"""
__all__ = ["capi"]
