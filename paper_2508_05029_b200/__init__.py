"""paper_2508_05029_b200 — B200-native hot path of the Theseus query engine.

The operators (filter, project, hash_partition, join, aggregate, take/concat,
exchange, tier moves) run as sm_100a CUDA kernels inside libtq_gpu.so behind
the C-ABI declared in include/tq_gpu.h.  This Python package is a thin ctypes
mirror of the reference's operator interface; it loads the
native library lazily (see `ops.lib()`) and fails loudly if it is missing.
"""
