"""B200-native sparse SpMV / Krylov backend (CSR, COO, ELL, SELL-P; CG, BiCGSTAB).

Drop-in for the SpMV/Krylov hot path of the reference ("larch",
/root/reference/proj): the C ABI is ``include/lbk.h`` (``liblbk.so``), the
C++ façade is ``include/lbk/larch.hpp`` and this package mirrors the same
operator surface in Python (``paper_2011_08879_b200.larch``).
"""
from . import _lib  # noqa: F401

__all__ = ["larch", "gen"]
