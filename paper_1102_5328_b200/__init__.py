"""paper_1102_5328_b200 -- B200-native (sm_100a) FP64 tile Householder QR.

The product is the C-ABI library ``libtileqr.so`` (include/tileqr.h), built
in-tree by ``python -m paper_1102_5328_b200.build``; ``tileqr`` is its thin
ctypes binding.  Importing ``paper_1102_5328_b200.tileqr`` raises when the
library is missing: there is no CPU fallback.
"""
__all__ = ["tileqr"]
