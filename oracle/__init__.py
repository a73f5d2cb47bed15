"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the replay hot path.

* ``oracle/_ref/libpdsim_ref.so`` — the unmodified reference simulator
  (/root/reference/proj/src, built by oracle/Makefile) behind a C shim.
* ``oracle/build/liboracle.so`` — a plain-C restatement of the reference's
  replay algorithm (oracle/pdsim_oracle.c), pinned against the reference and
  against tests/golden.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's CPU legs import
this package, and only as the checker / CPU baseline — never as the product.
"""
