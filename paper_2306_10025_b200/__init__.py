"""patchdb-b200: B200-native compressed patch relaxation (arXiv 2306.10025).

The product is the C-ABI shared library ``lib/libpatchdb.so.0`` (sources in
``csrc/``); :mod:`.patchdb` is its Python mirror.  Importing this package
loads the library and fails loudly when it has not been built.
"""
from . import patchdb  # noqa: F401
from .patchdb import (Database, Matrix, PatchdbError, PatchSet, Preconditioner, Problem, gmres,  # noqa: F401
                      pcg)

__all__ = ["patchdb", "Database", "Matrix", "PatchdbError", "PatchSet", "Preconditioner", "Problem", "gmres", "pcg"]
