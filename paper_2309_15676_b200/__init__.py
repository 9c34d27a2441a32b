"""B200-native gradient meta-estimation hot path (arxiv 2309.15676).

Host-side mirror of the reference `metagrad` API for the hot path
(Problem::sample_pair -> Moment2 -> MetaEstimator / Adam -> update), backed by
hand-written sm_100a CUDA kernels behind the C-ABI in include/mgcuda.h.
There is no CPU fallback: every compute call goes through libmgcuda.so and
fails loudly if it is missing or no B200 is visible.
"""
__all__ = ["api", "lib"]


def __getattr__(name):
    if name == "api":
        from . import api
        return api
    if name == "lib":
        from . import _lib
        return _lib.load()
    raise AttributeError(name)
