"""CPU parity oracle for the MPDATA hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import anything from this
package, and only as the checker or the timed CPU baseline.  The product
package ``paper_1908_06094_b200`` never imports it and has no CPU fallback.

Contents
--------
* :mod:`oracle.tsg_oracle` -- numpy restatement of the reference
  ``tristencil`` algorithm for this path (flat ``[element, level]`` arrays,
  neighbour tables, numberings, input generation).  Every function cites
  the reference file:line it restates.
* ``oracle/c/tsg_oracle.c`` -- the same transport step / neighbour sums in
  plain C (OpenMP over elements, no FP contraction), built by
  ``oracle/c/Makefile`` into ``oracle/c/build/libtsg_oracle.so``; used as
  the multi-core CPU baseline and cross-checked bitwise against the numpy
  restatement.

Parity pinning: the restatement is checked against golden vectors generated
by running the real reference (``tests/golden/make_golden.py``, which imports
``/root/reference/pkg/src/tristencil`` in the build container) -- full arrays
for small patches and SHA-256 digests of every output for the bench-sized
patches (44x72x10, 128x128x80, 279x256x80).
"""
