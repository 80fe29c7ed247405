"""B200-native deterministic inference engine (drop-in for the reference's detcore path).

Import ``paper_2602_00182_b200.detcore`` for the reference-shaped API; the CUDA library is loaded
lazily by ``paper_2602_00182_b200._lib`` and there is no CPU fallback.
"""
