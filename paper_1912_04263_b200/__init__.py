"""B200-native engine for the ADMM/PCG hot path of arXiv 1912.04263 (cuOSQP).

The product path is the C-ABI shared library built from ``csrc/``
(``libqpcg_b200.so``); this package is the host-side mirror of the
reference's interface (``qpcg::solve`` and its structs).
"""
