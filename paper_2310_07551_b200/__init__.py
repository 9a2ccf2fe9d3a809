"""B200-native Tucker-operator / ETD3RKDS library (arXiv 2310.07551).

The product is the C-ABI shared library ``libkx.so`` (include/kx.h, sources in csrc/);
``paper_2310_07551_b200.kx`` is its thin ctypes binding.  Build with
``python -m paper_2310_07551_b200.build``.
"""
__all__ = ["kx"]
