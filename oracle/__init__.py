"""TEST INFRASTRUCTURE ONLY -- the parity checker for the CUDA path.

Two CPU implementations of the reference hot path, exposed to numpy via ctypes:

* ``C``   -- ``liboracle.so``: the plain-C restatement in ``sdattn_oracle.c``
  (each function cites the reference file:line it follows).
* ``REF`` -- ``_ref/libsdattn_ref.so``: the reference's own sources compiled in
  place from /root/reference by ``oracle/Makefile`` plus ``ref_shim.cpp``.
  ``None`` when that build is absent.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package; the product path never does.
"""
from .pyoracle import (C, REF, OracleError, build, load_oracle, load_ref, Oracle,  # noqa: F401
                       FMT_F64, FMT_F32, FMT_BF16, FMT_F16, shared_seed, rel_fro, max_abs_rel)
