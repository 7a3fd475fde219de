"""CPU oracle for the QTT AMEn hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package imports this directory.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg use it, and
only as the checker / CPU baseline, never as the thing measured on the GPU.
"""
