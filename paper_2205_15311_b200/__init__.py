"""tilevolve-b200: B200 (sm_100a) implementation of the tilevolve enumeration /
classification hot path and the GA generation loop.

Modules mirror the reference package ``tilevolve`` (/root/reference/pkg/src):
``_kernels`` (classify_batch & co.), ``genome``, ``assembly``, plus the
spec-only ``classify`` (enumerate_space, Histogram) and ``evolve`` (GA).
The compute runs in libtilevolve_b200.so (include/tilevolve_b200.h).
"""
__version__ = "0.1.0"
