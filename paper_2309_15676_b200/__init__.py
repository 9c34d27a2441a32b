"""B200-native gradient meta-estimation hot path (arxiv 2309.15676).

Host-side mirror of the reference `metagrad` API for the hot path
(Problem::sample_pair -> Moment2 -> MetaEstimator / Adam -> update), backed by
hand-written sm_100a CUDA kernels behind the C-ABI in include/mgcuda.h.
There is no CPU fallback: every compute call goes through libmgcuda.so and
fails loudly if it is missing or no B200 is visible.

Import `paper_2309_15676_b200.api` for the reference-style API; importing the
package itself loads nothing.
"""
