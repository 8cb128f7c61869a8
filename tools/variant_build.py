#!/usr/bin/env python
"""Build an experimental variant of libgespmm.so with extra -D flags into
build/variants/<name>/ (travels to the GPU box; select it with GESPMM_LIB).

    python tools/variant_build.py <name> [DEFINE[=V] ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2007_03179_b200 import _build  # noqa: E402

if __name__ == "__main__":
    name, defs = sys.argv[1], sys.argv[2:]
    d = os.path.join(ROOT, "build", "variants", name)
    _build.build(defines=defs, build_dir=os.path.join(d, "obj"), lib=os.path.join(d, "libgespmm.so"))
    print(os.path.join(d, "libgespmm.so"))
