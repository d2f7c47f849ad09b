"""paper_2602_15018_b200: B200-native (sm_100a) event-camera hot path.

Drop-in for the reference's ``evsim.events`` API (see ``.events``) backed by
hand-written CUDA kernels in ``libevsim_b200.so`` (C ABI:
include/evsim_b200.h).  ``.simulator`` is the batched multi-stream /
multi-frame engine; ``.distributed`` shards streams over GPUs.
"""

__version__ = "0.1.0"


def library_path() -> str:
    from ._lib import LIB_PATH

    return LIB_PATH
