"""Build libciq.so in-tree for sm_100a (nvcc; no JIT cache, the .so travels with the repo copy).

    python paper_2006_11267_b200/build.py            # incremental
    python paper_2006_11267_b200/build.py --force    # rebuild everything
(run as a script: importing the package would load the library being built)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libciq.so")

SOURCES = ["host_math.cpp", "nccl_dl.cpp", "comm.cpp", "mvm_simt.cu", "mvm_sparse.cu", "mvm_dense.cu", "mvm_tc2.cu", "mvm_tc3.cu", "mvm_sym.cu", "recurrence.cu", "precond.cu", "precond64.cu", "precond_nested.cu", "posterior.cu", "ciq_api.cu"]
HEADERS = ["common.cuh", "nccl_dl.h", "comm.h", "internal.h", "host_math.h", "tc_util.cuh", "kern_epi.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"] + ARCH
# CIQ_TC_TRACE=1: compile the K1 per-tile clock stamps (experiments; see mvm_tc2.cu)
if os.environ.get("CIQ_TC_TRACE"):
    NVCC_FLAGS.append("-DCIQ_TC_TRACE")


def source_hash() -> str:
    """sha256 over every source, header and the public header, in a fixed order: embedded in
    libciq.so (ciq_source_hash()) so a test or the driver can tell which sources a binary was
    built from."""
    import hashlib
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        p = os.path.join(CSRC, name)
        if os.path.exists(p):
            h.update(name.encode())
            with open(p, "rb") as f:
                h.update(f.read())
    with open(os.path.join(INCLUDE, "ciq.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()[:16]


def has_hash(lib: str, want: str) -> bool:
    """True if the library embeds ``want`` (the string literal ciq_source_hash() returns; checked
    on the file's bytes, so no stale dlopen handle of an older build can answer)."""
    if not os.path.exists(lib):
        return False
    with open(lib, "rb") as f:
        return b"\0" + want.encode() + b"\0" in f.read()


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(src_paths, dst) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(p) > t for p in src_paths if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile (incrementally, by mtime) and link libciq.so; a library whose embedded source hash
    differs from the current sources is rebuilt from scratch, and the result is checked."""
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    want = source_hash()
    rehash = force or not has_hash(LIB, want)   # ciq_api.cu carries the hash: recompile it
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "ciq.h")]
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        if not os.path.exists(sp):
            continue
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _newer([sp] + hdrs, obj) or (rehash and src == "ciq_api.cu"):
            cmd = [nvcc, *NVCC_FLAGS, f"-DCIQ_SOURCE_HASH=\"{want}\"", "-I", INCLUDE, "-I", CSRC, "-c", sp, "-o", obj]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}")
            with open(obj + ".ptxas.txt", "w") as f:
                f.write(res.stderr)
    if force or rehash or _newer(objs, LIB):
        cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link failed")
    if not has_hash(LIB, want):
        raise RuntimeError(f"{LIB}: does not embed the source hash {want}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
