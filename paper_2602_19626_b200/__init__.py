"""B200-native hot path of the Nacrith LLM + arithmetic-coding compressor
(arXiv 2602.19626).  The product is libnc.so (CUDA sm_100a kernels behind the
C ABI in include/nc.h); this package is its thin ctypes binding."""
from ._lib import *  # noqa: F401,F403
from ._lib import Model, Comm, NcError, lib, EXPORTS  # noqa: F401
