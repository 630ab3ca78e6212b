"""TEST INFRASTRUCTURE ONLY -- the float64 CPU oracle for msMINRES-CIQ (arXiv 2006.11267).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The product path
(``paper_2006_11267_b200``) never imports it and shares no code with it.

Every function follows the paper's statement step by step in float64; see ``ciq_oracle.py``.
Parity status of each function is listed in its docstring and in DESIGN.md §4 ("pins").
"""
from .ciq_oracle import *  # noqa: F401,F403
