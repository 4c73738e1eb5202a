"""B200-native SDAS strategy simulator (arXiv 2601.03197, "Software-Defined Agentic Serving").

The hot path -- a batched Monte-Carlo discrete-event simulation of agent pipelines swept over
message-granularity strategies, request rates, seeds and control policies -- runs in the sm_100a
kernels of ``libsdas.so`` behind the C-ABI ``include/sdas.h``.  ``sdas`` is the ctypes binding,
``parallel`` the multi-GPU (NCCL) driver.
"""
from . import sdas  # noqa: F401
from .sdas import (FLAG_RECORDS, FLAG_SERIES, FLAG_TRACE, GridView, Pipeline, SdasError,  # noqa: F401
                   control_sweep, finalize, metrics, results_layout, simulate)
