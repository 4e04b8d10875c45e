"""B200-native DS-PHD/MIB dynamic occupancy grid filter cycle (arXiv 1605.02406).

The product is the CUDA library ``libdog.so`` (C ABI in ``include/dog.h``, kernels in ``csrc/``);
``dog.py`` is its thin ctypes binding and ``inputs.py`` the seeded synthetic-input generator.
Import ``paper_1605_02406_b200.dog`` explicitly: it fails loudly if the library was not built.
"""
__all__ = ["dog", "inputs", "build"]
