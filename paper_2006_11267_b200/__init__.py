"""paper_2006_11267_b200 -- B200-native msMINRES-CIQ (arXiv 2006.11267): K^{1/2}B and K^{-1/2}B.

The product is the C-ABI library ``libciq.so`` (include/ciq.h); ``ciq`` is its thin ctypes
binding.  Build with ``python -m paper_2006_11267_b200.build``.
"""
from .ciq import (CIQ, CIQ_ERR_INVALID_ARG, CIQ_NOT_CONVERGED, CIQ_OK, CiqError, LoopbackGroup, ciq_apply, ciq_free, ciq_init, ciq_matvec, ciq_nccl_unique_id,  # noqa: F401
                  ciq_params_default, ciq_pivoted_cholesky, ciq_quadrature_rule, ciq_shard_rows, ciq_tridiag_extremes, make_params)
