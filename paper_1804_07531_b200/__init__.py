"""B200-native (sm_100a) pass-efficient randomized SVD (arXiv 1804.07531): C-ABI library
librsvd.so (include/rsvd.h) + a thin ctypes binding (``rsvd``)."""
from . import rsvd  # noqa: F401
from .rsvd import Context, RsvdError, RsvdInfo, recommend_input  # noqa: F401

__all__ = ["rsvd", "Context", "RsvdError", "RsvdInfo", "recommend_input"]
