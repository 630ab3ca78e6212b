"""Build a variant of libciq.so into _ab/<name>/ (A/B experiments; select with CIQ_LIB=_ab/<name>/libciq.so).
    python scripts/build_variant.py <name> [-DFLAG ...]"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2006_11267_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
name = sys.argv[1]
b.BUILD = os.path.join(ROOT, "_ab", name, "obj")
b.LIB = os.path.join(ROOT, "_ab", name, "libciq.so")
b.NVCC_FLAGS = b.NVCC_FLAGS + sys.argv[2:]
print(b.build(force=True))
