"""B200-native Newton hot path for the fully implicit in-situ combustion
simulator of arxiv 1811.11992 (reference package ``iscsim``).

Host side mirrors the reference's operator API (``assemble``,
``BlockSolver``, ``Simulator``); every numerical kernel runs in the sm_100a
shared library ``_lib/libiscgpu.so`` behind the C-ABI in ``include/iscgpu.h``.
"""

__version__ = "0.1.0"
