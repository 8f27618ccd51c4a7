#!/usr/bin/env python
"""Build an experiment copy of the library with extra nvcc defines, for A/B timing through
DADE_LIB (the product library is untouched): python tools/build_variant.py NAME -DX=1 ...
-> exp_libs/libdade_NAME.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_variant(name, defines):
    from paper_2404_16322_b200 import build as B
    out = os.path.join(ROOT, "exp_libs", f"libdade_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    return B.build(extra=list(defines), out=out)


if __name__ == "__main__":
    print(build_variant(sys.argv[1], sys.argv[2:]))
