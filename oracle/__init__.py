"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the QSU/QR/EVC hot path.

Two checkers live here; the product never imports this package (only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs do):

* :mod:`oracle.cpu` — ctypes over ``liboracle.so``, the plain-C restatement of
  the reference dist-sim loops (``qrt_oracle.c``, each function citing
  /root/reference/proj/src/dist_sim.cpp line ranges);
* :mod:`oracle.ref` — ctypes over ``_ref/libqrtile_ref.so``, the *unmodified*
  reference library compiled from /root/reference sources by ``Makefile``
  (present wherever it was built; it travels to the GPU box with the snapshot).

Parity pin: ``tests/test_oracle.py`` checks the C restatement against the
reference build and against the committed golden vectors in tests/golden/.
"""
