"""B200-native GPT decoder train step (arXiv 2312.12705's tuned path) behind the
`trainplan` API. The compute lives in ``lib/libtrainplan_b200.so`` (sm_100a kernels, C++
runtime, NCCL); this package is the thin ctypes binding plus build glue."""
from . import _lib  # noqa: F401

__all__ = ["_lib"]
