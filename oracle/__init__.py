"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py, and only as
the checker or the timed CPU baseline.  The product package
(``paper_2407_11488_b200``) never imports it.

* :mod:`oracle.kernels_ffi` -- ctypes binding of ``liboracle.so``, the C
  restatement of the four kernels (``kernels.c``; bit-exact fp32 order).
* :mod:`oracle.reference_port` -- the reference tuning loop restated for
  the CPU baseline arm (enumeration + protocol + brute force over a CPU
  kernel), following ``pkg/src/tunescape`` file:line by file:line.

Parity status: search-space behaviour is pinned against the reference
itself (golden fixtures generated from ``/root/reference`` by
``tests/golden/make_golden.py``); kernel arithmetic is *unpinned by the
reference* (it has none) and is pinned by known-answer tests.
"""
