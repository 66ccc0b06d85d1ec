"""paper_1803_04631_b200 -- a B200-native CuLDA_CGS hot path behind the API of
the reference package `gibbsflow` (arXiv 1803.04631).

Module map (reference module -> here):
  errors  -> errors       (same exception classes)
  rng     -> rng          (splitmix64 streams, native)
  corpus  -> corpus       (Corpus/Chunk types; native partition)
  model   -> model        (ThetaRows/PhiMatrix; rebuilds on the GPU)
  ptree   -> ptree        (host build, device ballot search)
  SPEC sampler / engine / eval -> sampler / engine / eval (GPU kernels)
The CUDA kernels and the C ABI live in csrc/ (include/gibbsflow_b200.h).
"""

from . import errors  # noqa: F401

__all__ = ["errors", "rng", "corpus", "model", "ptree", "sampler", "engine", "eval", "shard", "synth"]
__version__ = "0.1.0"
