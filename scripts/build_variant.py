#!/usr/bin/env python
"""Build a variant of libpbicgstab.so with extra nvcc defines into ablib/ (tuning
experiments only; the product build is paper_1809_01948_b200/_build.py).

usage: python scripts/build_variant.py NAME [-DFOO=1 ...]   -> ablib/libNAME.so
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_01948_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "ablib"), exist_ok=True)
_build.LIB = os.path.join(ROOT, "ablib", f"lib{name}.so")
_build.NVCC_FLAGS = _build.NVCC_FLAGS + defs
_build.HERE_OBJ = None
orig = _build.os.path.join


def objdir_join(*a):  # keep the variant's objects apart from the product build's
    p = orig(*a)
    return p.replace(os.sep + "build", os.sep + f"build_{name}") if a[-1] == "build" else p


_build.os.path.join = objdir_join
print(_build.build(force=True))
