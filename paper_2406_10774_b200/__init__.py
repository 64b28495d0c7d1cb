"""B200-native Quest (arXiv 2406.10774) decode hot path.

Paged KV append with fused min/max page metadata -> per-page criticality estimate ->
per-head top-K page selection -> split-KV sparse paged attention with an LSE merge,
as hand-written sm_100a CUDA kernels behind a C ABI (include/questkv_b200.h).

``questkv`` mirrors the reference's ``questkv::`` operator API on top of that ABI.
"""

from . import _lib  # noqa: F401  (raises if libquestkv_b200.so is missing)
from .questkv import *  # noqa: F401,F403

__version__ = "0.1.0"
