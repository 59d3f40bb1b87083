"""B200-native constrained beam-decode engine for the kernel-tuning-parameter
translator of arXiv 2404.10162 (reference: kernelseer).

The hot path (LSTM encoder -> attention decoder -> constrained beam search)
runs as hand-written sm_100a CUDA behind the C-ABI in include/ks_b200.h.
"""
__version__ = "0.1.0"
