"""B200-native mixed-batch forward for AccelGen (arXiv 2503.13737).

Host side mirrors the reference simulator's API (pkg/src/slosim: errors, cost_model, kvc,
workload, sched_core; SPEC.md policies/engine); the forward runs in libaccelgen_b200.so
(hand-written sm_100a CUDA behind the C ABI in include/accelgen_b200.h).
"""
__version__ = "0.1.0"
