"""SPEC.md's exact-arithmetic worked examples (tests/golden/spec_examples.json, each cited)."""
import json
import os

import numpy as np

import workloads
from oracle import DenseOperator, ciq, msminres

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def test_spec_examples():
    ex = json.load(open(GOLDEN))["examples"]
    for e in ex:
        k = np.array(e["K"])
        b = np.array(e["b"])
        op = DenseOperator(k)
        if e["mode"] == "solve":
            out = msminres(op.mvm, b, np.array([e["shift"]]), 10, tol=1e-12).x[0, :, 0]
        else:
            out = ciq(op, b, q=12, max_iters=50, tol=1e-12, mode=e["mode"],
                      lanczos_start=workloads.lanczos_start(len(b), 2)).out
        np.testing.assert_allclose(out, e["expected"], rtol=e["rtol"], err_msg=e["cite"])
