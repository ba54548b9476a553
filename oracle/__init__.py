"""CPU checkers for the GPU hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  It is never the thing measured or shipped: the product
(``paper_2402_08273_b200``) does not import it and fails loudly without its
CUDA library.

* :class:`RefLib` drives the UNMODIFIED reference (``oracle/_ref``) through
  ``run_render`` (core/driver.hpp:80).
* :class:`OracleLib` drives ``ramlt_oracle.cpp``, the restatement with the GPU
  engine's lockstep semantics and a selectable RNG.
"""
from .abi import (  # noqa: F401
    OracleConfig, OracleStats, RenderOutput, RefLib, OracleLib, build, ORACLE_DIR,
)
