"""B200-native NCL/IPM hot path for AC-SCOPF (arXiv 2510.13333).

Host C++ + sm_100a CUDA behind a C-ABI (include/nclopf_b200.h); this Python
package is a thin ctypes mirror of the reference API used by tests and the
bench. There is no CPU fallback anywhere on the numeric path.
"""
from . import _lib  # noqa: F401  (fails loudly when the library is missing)
from . import sparse, model, kkt, scopf, ipm, dist, mpcc, matpower  # noqa: F401,E402
