"""CPU oracle for the rcomm hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here:

* ``Oracle``    -- ctypes binding of ``liboracle.so``, the plain-C restatement
  (``rcomm_oracle.c``) of codec.cpp / kernels.cpp / collectives.cpp.
* ``Reference`` -- ctypes binding of ``_ref/librcomm_ref.so``: the UNMODIFIED
  reference library compiled in place from /root/reference by ``Makefile``,
  driven through its own SimCluster harness (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline; the product path (``paper_2107_01499_b200``) never
touches it.
"""
from .oracle import Oracle, Reference, build, ORACLE_DIR  # noqa: F401
