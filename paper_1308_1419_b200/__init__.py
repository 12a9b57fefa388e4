"""paper_1308_1419_b200 -- B200-native (sm_100a) triangular-domain mapping
functions and td-kernels (Navarro & Hitschfeld, arXiv:1308.1419).

``paper_1308_1419_b200.trigrid`` is the drop-in for the reference's Python
module ``trigrid`` (same 21 names).  The compute path is libtrigrid_b200.so
(CUDA, C-ABI in include/trigrid_b200.h); calling into ``trigrid`` without the
built library raises ImportError -- there is no CPU fallback.
"""
__all__ = ["trigrid"]
