"""B200-native UltraSketchLLM (arXiv 2506.17255) sketch hot path: plan, build, reconstruct, fused
sketch-linear -- hand-written sm_100a CUDA behind the C ABI in include/usk.h.

``from paper_2506_17255_b200 import usk`` loads ``libusk.so`` (built in-tree by
``paper_2506_17255_b200/build.py``) and raises if it is missing: there is no CPU fallback.
"""
