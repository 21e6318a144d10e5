"""Parity oracle — TEST INFRASTRUCTURE ONLY.

* ``oracle/_ref/ref_driver``: the unmodified reference (gnnsim) compiled from
  /root/reference/proj/src by oracle/Makefile (git-ignored build output).
* ``oracle/gnnsim_oracle.c`` -> ``oracle/_ref/liboracle.so``: a plain-C restatement of the
  reference's algorithm for this path, pinned against the reference build and the
  golden fixtures in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.
"""
