"""Parity oracle for the B200 block-Toeplitz matvec — TEST INFRASTRUCTURE ONLY.

* ``oracle.restate``  numpy restatement of the reference path (file:line cited).
* ``oracle.refcpu``   ctypes access to the reference itself, compiled from the
                      unmodified sources under /root/reference/proj/src by
                      ``oracle/Makefile`` into ``oracle/_ref/libbtoep_ref.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package. The product package never does.
"""
