"""B200-native differentiable-rendering hot path of arXiv 2103.15208 (collodiff).

The product is libcdr.so (C-ABI: include/cdr.h) built from csrc/ for sm_100a;
``api`` is its Python host mirror and ``scenes`` the synthetic-input
generators. See DESIGN.md.
"""
from . import scenes  # noqa: F401

__all__ = ["scenes", "api", "build"]
