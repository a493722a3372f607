"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the editable-Gaussian hot path.

This package restates, in numpy plus a small C library (``composite.c``), the
reference's CPU algorithm for the splatting hot path (voxsplat, arxiv
2504.17954; `/root/reference/pkg/src/voxsplat/`).  It is the *checker*:

* ``tests/`` compare the CUDA path against it on seeded inputs;
* ``__graft_entry__.smoke()`` uses it to check one small render;
* ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm time it on
  the host cores (the reference is a Python package that cannot be compiled,
  so the port is the CPU baseline, ``kind: "port"``).

Nothing in ``paper_2504_17954_b200`` imports this package; the product path
fails loudly when its CUDA library is missing.

Parity pinning: ``tests/golden/make_golden.py`` (run in the container that
has ``/root/reference``) imports the real reference and writes golden vectors;
``tests/test_oracle_golden.py`` checks this oracle against them bit-for-bit.
"""

from .port import *  # noqa: F401,F403
