"""CPU oracle for the residency-octree render path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product path (``paper_2309_04393_b200``)
never imports it; it fails loudly when its CUDA library is missing instead.

Contents
--------
* ``resoct_oracle.c``  plain-C restatement of ``kernels.raycast_frame``
  (``/root/reference/pkg/src/resoctree/kernels.py:209-704``), MODE_RESIDENCY
  and MODE_REFERENCE plus the skip audit, built into
  ``oracle/_build/libresoct_oracle.so`` by :func:`build`.
* ``raycast.py``       ctypes driver: ray generation, channel/TF packing and
  the budgeted request lists, restating ``render.py:101-233`` and
  ``camera.py:32-51`` / ``transfer.py:38-120``.
* ``state.py``         pure-Python/numpy restatement of the paging LRU
  (``paging.py:187-284``), the octree residency update
  (``octree.py:193-273``) and ``Engine.note_sampled`` (``engine.py:72-81``).

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (importable
in the build container) and stores its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this oracle bit-for-bit against them.
"""

from .build import build, lib_path  # noqa: F401
