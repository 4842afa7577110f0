"""B200-native Grover state-vector hot path (arxiv quant-ph/9804039).

The product is the C-ABI library libsv.so (include/sv.h): hand-written CUDA
kernels for sm_100a (fused multi-stage Walsh-Hadamard tile pass, fused oracle
flip + inversion about the mean) and NCCL for the sharded path.  This package
is the thin ctypes binding (_sv) plus the torch.distributed bootstrap (dist).
Importing it fails loudly if libsv.so has not been built -- there is no CPU
fallback.
"""
from ._sv import *  # noqa: F401,F403
from ._sv import Ctx, SvError, lib, LIB_PATH  # noqa: F401
