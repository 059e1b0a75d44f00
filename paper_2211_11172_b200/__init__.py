"""B200-native HARL inner search step (drop-in for schedtune's episode path).

Host code is Python; the per-step work runs in hand-written sm_100a CUDA
kernels behind a C-ABI shared library (``csrc/`` -> ``libharl_b200.so``)
loaded with ctypes.  See DESIGN.md.
"""

__version__ = "0.1.0"
