"""B200-native element-local HDG engine (arXiv 1305.1489).

Host C++ + sm_100a CUDA behind a C ABI (include/hdg_b200.h), with a thin
reference-shaped Python layer (`engine`). See DESIGN.md.
"""
from . import _lib  # noqa: F401
from .configs import CONFIGS, Config, Problem  # noqa: F401
from .fields import FieldProgram, compile_field  # noqa: F401

__all__ = ["CONFIGS", "Config", "Problem", "FieldProgram", "compile_field"]
