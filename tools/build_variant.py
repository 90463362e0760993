#!/usr/bin/env python
"""Build an A/B variant of libsinet (compile-time -D switches) next to the product library:

  python tools/build_variant.py NAME DEFINE [DEFINE ...]   -> paper_2106_12863_b200/libsinet.NAME.so
  SINET_LIB_VARIANT=NAME python bench.py ...                 (loads it instead of libsinet.so)
"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_build", os.path.join(ROOT, "paper_2106_12863_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
name, defines = sys.argv[1], sys.argv[2:]
print(b.build(force=True, defines=defines, out=os.path.join(b.PKG, f"libsinet.{name}.so")))
