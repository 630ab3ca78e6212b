"""CPU tests of the C-ABI boundary: libciq.so loads, exports every symbol include/ciq.h declares,
the struct layouts agree, and the host-only steps (HHT rule a3, tridiagonal Ritz extremes a2,
row sharding) match the oracle / numpy -- no GPU needed."""
import ctypes
import re
import subprocess

import numpy as np
import pytest
import scipy.linalg

import paper_2006_11267_b200.ciq as cq
from oracle import hht_rule

HEADER = __import__("os").path.join(__import__("os").path.dirname(__file__), "..", "include", "ciq.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ciq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 10
    out = subprocess.run(["nm", "-D", "--defined-only", cq.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(\S+)", out))
    for n in names:
        assert n in exported, n
        assert hasattr(cq.LIB, n)
    assert set(cq.EXPORTED) == set(names)


def test_struct_sizes_match_header():
    # offsets computed by the C compiler from the header itself
    code = r'''
#include <stdio.h>
#include <stddef.h>
#include "ciq.h"
int main(){printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(ciq_operator), sizeof(ciq_params), sizeof(ciq_info),
 sizeof(ciq_precond), sizeof(ciq_comm), offsetof(ciq_params, breakdown_tol), offsetof(ciq_info, kernel_launches));}
'''
    import os
    import tempfile
    d = tempfile.mkdtemp()
    open(os.path.join(d, "s.c"), "w").write(code)
    inc = os.path.join(os.path.dirname(HEADER))
    subprocess.run(["gcc", "-I", inc, os.path.join(d, "s.c"), "-o", os.path.join(d, "s")], check=True)
    vals = list(map(int, subprocess.run([os.path.join(d, "s")], capture_output=True, text=True).stdout.split()))
    assert vals == [ctypes.sizeof(cq.CiqOperator), ctypes.sizeof(cq.CiqParams), ctypes.sizeof(cq.CiqInfo),
                    ctypes.sizeof(cq.CiqPrecond), ctypes.sizeof(cq.CiqComm), cq.CiqParams.breakdown_tol.offset,
                    cq.CiqInfo.kernel_launches.offset]


@pytest.mark.parametrize("lmin,lmax,q", [(1e-4, 1.0, 8), (0.05, 104.0, 8), (1e-3, 3.0, 15), (1.0, 1e8, 20),
                                         (2.0, 3.0, 4), (0.1, 2e4, 12), (1.0, 1.0, 4)])
def test_host_rule_matches_oracle(lmin, lmax, q):
    t, w = cq.ciq_quadrature_rule(lmin, lmax, q)
    to, wo = hht_rule(lmin, lmax, q)
    tol = 1e-12 if lmax / lmin <= 1e6 else 1e-10
    np.testing.assert_allclose(t, to, rtol=tol)
    np.testing.assert_allclose(w, wo, rtol=tol)


def test_host_rule_errors():
    with pytest.raises(cq.CiqError):
        cq.ciq_quadrature_rule(0.0, 1.0, 8)
    with pytest.raises(cq.CiqError):
        cq.ciq_quadrature_rule(1.0, 2.0, 0)
    with pytest.raises(cq.CiqError):
        cq.ciq_quadrature_rule(1.0, 2.0, 65)


@pytest.mark.parametrize("m", [1, 2, 5, 20, 60])
def test_tridiag_extremes(m):
    rng = np.random.default_rng(m)
    a = rng.normal(size=m) * 3
    b = rng.uniform(0.01, 2.0, size=max(m - 1, 0))
    lo, hi = cq.ciq_tridiag_extremes(a, b if m > 1 else np.zeros(1))
    ev = scipy.linalg.eigvalsh_tridiagonal(a, b) if m > 1 else a
    assert abs(lo - ev[0]) <= 1e-12 * max(1, abs(ev[0])) + 1e-13
    assert abs(hi - ev[-1]) <= 1e-12 * max(1, abs(ev[-1])) + 1e-13


def test_shard_rows_partition():
    for n in (1, 127, 128, 1000, 50_000, 200_000):
        for world in (1, 2, 3, 4, 8):
            spans = [cq.ciq_shard_rows(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            for b, e in spans:
                assert b % 128 == 0 or b == n


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = np.zeros((8, 2), dtype=np.float32)
    with pytest.raises(cq.CiqError) as e:
        cq.CIQ("rbf", X=x, lengthscale=1.0)
    assert e.value.status == cq.CIQ_ERR_CUDA
